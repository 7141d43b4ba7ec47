// K2 — quantization-variance indicator statistics (sm_100a).
//
// Produces hetplan::indicator::operator_stats for one operator
// (/root/reference/proj/include/hetplan/indicator/indicator.hpp:31-38):
// d_w, exact w_min / w_max over the weight tensor, and the calibration
// input's mean and population variance in fp64. omega itself
// (indicator.cpp:99-111) is then a handful of fp64 flops evaluated by the
// host library in the reference's operation order.
//
// Both reductions are single-pass and deterministic: every thread folds its
// elements, warps combine with shuffles (min/max; Chan's parallel
// (n, mean, M2) merge for the moments), blocks write partials, and the last
// block to finish (atomic ticket) merges the partials in block order.
#include <cuda_bf16.h>
#include <cstdint>

namespace hp {

namespace {

constexpr int kStatThreads = 256;

struct moments {
    double n, mean, m2;
};

__device__ __forceinline__ moments merge(moments a, moments b) {
    if (b.n == 0.0) return a;
    if (a.n == 0.0) return b;
    const double n = a.n + b.n;
    const double d = b.mean - a.mean;
    moments r;
    r.n = n;
    r.mean = a.mean + d * (b.n / n);
    r.m2 = a.m2 + b.m2 + d * d * (a.n * b.n / n);
    return r;
}

__device__ __forceinline__ moments shfl_moments(moments m, int delta) {
    moments o;
    o.n = __shfl_xor_sync(0xffffffffu, m.n, delta);
    o.mean = __shfl_xor_sync(0xffffffffu, m.mean, delta);
    o.m2 = __shfl_xor_sync(0xffffffffu, m.m2, delta);
    return o;
}

// grid.x blocks: [0, nbw) reduce W (min/max), [nbw, nbw+nbx) reduce X.
__global__ void __launch_bounds__(kStatThreads)
    stats_kernel(const __nv_bfloat16* __restrict__ w, int64_t n_out,
                 int64_t k_in, int64_t ldw, const __nv_bfloat16* __restrict__ x,
                 int64_t tokens, int64_t ldx, int nbw, int nbx,
                 float2* __restrict__ part_w, moments* __restrict__ part_x,
                 unsigned* __restrict__ ticket, double* __restrict__ out) {
    __shared__ float2 sw[kStatThreads / 32];
    __shared__ moments sx[kStatThreads / 32];
    __shared__ bool last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;

    if (b < nbw) {
        float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
        const int64_t total = n_out * k_in;
        const bool vec = (k_in % 8 == 0) && (ldw % 8 == 0) &&
                         ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
        if (vec) {
            const int64_t nvec = total / 8, kv = k_in / 8;
            for (int64_t i = static_cast<int64_t>(b) * kStatThreads + tid; i < nvec;
                 i += static_cast<int64_t>(nbw) * kStatThreads) {
                const int64_t row = i / kv, c = i % kv;
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(w + row * ldw) + c);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 f = __bfloat1622float2(h[j]);
                    mn = fminf(mn, fminf(f.x, f.y));
                    mx = fmaxf(mx, fmaxf(f.x, f.y));
                }
            }
        } else {
            for (int64_t i = static_cast<int64_t>(b) * kStatThreads + tid; i < total;
                 i += static_cast<int64_t>(nbw) * kStatThreads) {
                const float f = __bfloat162float(w[(i / k_in) * ldw + i % k_in]);
                mn = fminf(mn, f);
                mx = fmaxf(mx, f);
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, d));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        }
        if (lane == 0) sw[warp] = make_float2(mn, mx);
        __syncthreads();
        if (tid == 0) {
            float2 acc = sw[0];
            for (int i = 1; i < kStatThreads / 32; ++i) {
                acc.x = fminf(acc.x, sw[i].x);
                acc.y = fmaxf(acc.y, sw[i].y);
            }
            part_w[b] = acc;
        }
    } else {
        const int bx = b - nbw;
        moments m{0.0, 0.0, 0.0};
        const int64_t total = tokens * k_in;
        for (int64_t i = static_cast<int64_t>(bx) * kStatThreads + tid; i < total;
             i += static_cast<int64_t>(nbx) * kStatThreads) {
            const double v = static_cast<double>(__bfloat162float(x[(i / k_in) * ldx + i % k_in]));
            m.n += 1.0;  // Welford
            const double d = v - m.mean;
            m.mean += d / m.n;
            m.m2 += d * (v - m.mean);
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) m = merge(m, shfl_moments(m, d));
        if (lane == 0) sx[warp] = m;
        __syncthreads();
        if (tid == 0) {
            moments acc = sx[0];
            for (int i = 1; i < kStatThreads / 32; ++i) acc = merge(acc, sx[i]);
            part_x[bx] = acc;
        }
    }

    // last block merges all partials in block order
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1u) == static_cast<unsigned>(nbw + nbx - 1);
    }
    __syncthreads();
    if (!last || tid != 0) return;
    __threadfence();
    float2 wr = part_w[0];
    for (int i = 1; i < nbw; ++i) {
        wr.x = fminf(wr.x, part_w[i].x);
        wr.y = fmaxf(wr.y, part_w[i].y);
    }
    moments xr{0.0, 0.0, 0.0};
    for (int i = 0; i < nbx; ++i) xr = merge(xr, part_x[i]);
    out[0] = static_cast<double>(n_out) * static_cast<double>(k_in);
    out[1] = static_cast<double>(wr.x);
    out[2] = static_cast<double>(wr.y);
    out[3] = xr.n > 0.0 ? xr.mean : 0.0;
    out[4] = xr.n > 0.0 ? xr.m2 / xr.n : 0.0;
    *ticket = 0u;  // self-resetting for the next call
}

}  // namespace

size_t stats_scratch_bytes(int nbw, int nbx) {
    return 256 + static_cast<size_t>(nbw) * sizeof(float2) +
           static_cast<size_t>(nbx) * sizeof(moments);
}

// scratch: stats_scratch_bytes(), zero-initialised (ticket at offset 0).
cudaError_t launch_stats(const void* w, int64_t n_out, int64_t k_in,
                         int64_t ldw, const void* x, int64_t tokens,
                         int64_t ldx, double* out, void* scratch, int nbw,
                         int nbx, cudaStream_t st) {
    auto* base = static_cast<uint8_t*>(scratch);
    auto* ticket = reinterpret_cast<unsigned*>(base);
    auto* pw = reinterpret_cast<float2*>(base + 256);
    auto* px = reinterpret_cast<moments*>(base + 256 + static_cast<size_t>(nbw) * sizeof(float2));
    stats_kernel<<<nbw + nbx, kStatThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(w), n_out, k_in, ldw,
        static_cast<const __nv_bfloat16*>(x), x ? tokens : 0, ldx, nbw, nbx, pw,
        px, ticket, out);
    return cudaGetLastError();
}

}  // namespace hp
