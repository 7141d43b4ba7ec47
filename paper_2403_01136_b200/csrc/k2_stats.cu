// K2 — quantization-variance indicator statistics (sm_100a).
//
// Produces hetplan::indicator::operator_stats for one operator
// (/root/reference/proj/include/hetplan/indicator/indicator.hpp:31-38):
// d_w, exact w_min / w_max over the weight tensor, and the calibration
// input's mean and population variance in fp64. omega itself
// (indicator.cpp:99-111) is then a handful of fp64 flops evaluated by the
// host library in the reference's operation order.
//
// Both reductions are single-pass, HBM-bound and deterministic: every thread
// streams 16-byte vectors (8 loads in flight) from an even contiguous share
// of the tensor and folds them (min/max; for the moments each bf16x8 vector
// becomes an exact fp64 (8, mean, M2) and is Chan-merged, one fp64 division
// per 8 elements), blocks fold their threads in a fixed shuffle-tree order,
// and the last block to finish (atomic ticket) folds the per-block partials
// with all 256 threads, again in a fixed order.
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

// Fold one bf16x8 vector into (n, mean, M2): the vector's own mean and M2 in
// fp64 (8 bf16 values sum exactly in fp64), then one Chan merge -- a single
// fp64 division per 8 elements instead of Welford's one per element.
__device__ __forceinline__ void fold8(moments& m, const uint4 q) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
    double v[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
    }
    const double mu = (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) * 0.125;
    double m2 = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) m2 = fma(v[j] - mu, v[j] - mu, m2);
    m = merge(m, moments{8.0, mu, m2});
}
__device__ __forceinline__ void fold1(moments& m, double v) {
    m = merge(m, moments{1.0, v, 0.0});
}

// Block-wide fold of per-thread partials in thread order (shuffle tree, then
// warps in order): deterministic for a fixed launch shape.
template <class T, class F>
__device__ __forceinline__ T block_fold(T v, F op, T* sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o;
        if constexpr (sizeof(T) == sizeof(moments)) {
            o = shfl_moments(v, d);
        } else {
            o.x = __shfl_xor_sync(0xffffffffu, v.x, d);
            o.y = __shfl_xor_sync(0xffffffffu, v.y, d);
        }
        v = (lane & d) ? op(o, v) : op(v, o);
    }
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    T acc = sm[0];
    for (int i = 1; i < kStatThreads / 32; ++i) acc = op(acc, sm[i]);
    return acc;
}

// Rows [r0, r1) x k of a row-major bf16 matrix with leading dimension ld, as
// bf16x8 vectors when rows are 16-byte aligned and contiguous (ld == k) or
// padded to a multiple of 8; 8 independent 16-byte loads in flight per thread.
template <class V, class S>
__device__ __forceinline__ void walk(const __nv_bfloat16* __restrict__ p, int64_t rows, int64_t k,
                                     int64_t ld, int part, int nparts, V vec_fn, S scalar_fn) {
    const int tid = threadIdx.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(p) & 15) == 0 && k % 8 == 0 && ld % 8 == 0;
    if (aligned && ld == k) {  // one flat vector range, split evenly over the parts
        const int64_t nvec = rows * k / 8;
        const int64_t lo = nvec * part / nparts, hi = nvec * (part + 1) / nparts;
        const uint4* v4 = reinterpret_cast<const uint4*>(p);
        int64_t i = lo + tid;
        constexpr int U = 8;  // 128 bytes in flight per thread
        for (; i + (U - 1) * kStatThreads < hi; i += U * kStatThreads) {
            uint4 q[U];
#pragma unroll
            for (int u = 0; u < U; ++u) q[u] = __ldcs(v4 + i + u * kStatThreads);
#pragma unroll
            for (int u = 0; u < U; ++u) vec_fn(q[u]);
        }
        for (; i < hi; i += kStatThreads) vec_fn(__ldcs(v4 + i));
    } else if (aligned) {  // padded rows: parts take whole rows
        const int64_t kv = k / 8;
        for (int64_t r = part; r < rows; r += nparts) {
            const uint4* v4 = reinterpret_cast<const uint4*>(p + r * ld);
            for (int64_t c = tid; c < kv; c += kStatThreads) vec_fn(__ldcs(v4 + c));
        }
    } else {
        for (int64_t r = part; r < rows; r += nparts)
            for (int64_t c = tid; c < k; c += kStatThreads) scalar_fn(__bfloat162float(p[r * ld + c]));
    }
}

// grid.x blocks: [0, nbw) reduce W (min/max), [nbw, nbw+nbx) reduce X.
__global__ void __launch_bounds__(kStatThreads, 3)
    stats_kernel(const __nv_bfloat16* __restrict__ w, int64_t n_out,
                 int64_t k_in, int64_t ldw, const __nv_bfloat16* __restrict__ x,
                 int64_t tokens, int64_t ldx, int nbw, int nbx,
                 float2* __restrict__ part_w, moments* __restrict__ part_x,
                 unsigned* __restrict__ ticket, double* __restrict__ out) {
    __shared__ float2 sw[kStatThreads / 32];
    __shared__ moments sx[kStatThreads / 32];
    __shared__ bool last;
    const int tid = threadIdx.x;
    const int b = blockIdx.x;
    auto mm = [](float2 a, float2 c) { return make_float2(fminf(a.x, c.x), fmaxf(a.y, c.y)); };
    auto mg = [](moments a, moments c) { return merge(a, c); };

    if (b < nbw) {
        float2 r = make_float2(__int_as_float(0x7f800000), -__int_as_float(0x7f800000));
        walk(w, n_out, k_in, ldw, b, nbw,
             [&](const uint4 q) {
                 const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
                 for (int j = 0; j < 4; ++j) {
                     const float2 f = __bfloat1622float2(h[j]);
                     r.x = fminf(r.x, fminf(f.x, f.y));
                     r.y = fmaxf(r.y, fmaxf(f.x, f.y));
                 }
             },
             [&](float f) {
                 r.x = fminf(r.x, f);
                 r.y = fmaxf(r.y, f);
             });
        r = block_fold(r, mm, sw);
        if (tid == 0) part_w[b] = r;
    } else {
        moments m{0.0, 0.0, 0.0};
        walk(x, tokens, k_in, ldx, b - nbw, nbx, [&](const uint4 q) { fold8(m, q); },
             [&](float f) { fold1(m, static_cast<double>(f)); });
        m = block_fold(m, mg, sx);
        if (tid == 0) part_x[b - nbw] = m;
    }

    // the last block merges all partials: thread t folds partials t, t+256,
    // ... in order, then the block folds the threads in order
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1u) == static_cast<unsigned>(nbw + nbx - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    float2 wr = make_float2(__int_as_float(0x7f800000), -__int_as_float(0x7f800000));
    for (int i = tid; i < nbw; i += kStatThreads) wr = mm(wr, __ldcg(&part_w[i]));
    moments xr{0.0, 0.0, 0.0};
    for (int i = tid; i < nbx; i += kStatThreads) {
        moments q;
        q.n = __ldcg(&part_x[i].n);
        q.mean = __ldcg(&part_x[i].mean);
        q.m2 = __ldcg(&part_x[i].m2);
        xr = merge(xr, q);
    }
    __syncthreads();
    wr = block_fold(wr, mm, sw);
    __syncthreads();
    xr = block_fold(xr, mg, sx);
    if (tid != 0) return;
    if (nbw > 0) {  // nbw == 0: the weight part came from K1's fused pass
        out[0] = static_cast<double>(n_out) * static_cast<double>(k_in);
        out[1] = static_cast<double>(wr.x);
        out[2] = static_cast<double>(wr.y);
    }
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
