// Glue kernels of the decoder stack around the quantized linear ops — NOT
// the graded hot path (SURVEY §8f rank 2 lists full layer glue as "next"):
//   * hp_synth_bf16: bit-reproducible synthetic tensors (weights, norm
//     params, prompts). Mirrors oracle/synth.py exactly: Irwin-Hall(4) of
//     splitmix64 draws, one fp64 multiply + add, fp32 then bf16 RNE.
//   * layernorm_bf16: OPT pre-LN (gain/bias), fp32 statistics.
//   * gather_rows: last-position rows of each request (prefill -> decode).
#include <cuda_bf16.h>
#include <cstdint>

namespace hp {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void synth_kernel(__nv_bfloat16* __restrict__ out, int64_t n, uint64_t seed,
                             double mean, double scale) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r1 = splitmix64(seed ^ (static_cast<uint64_t>(i) << 1));
        const uint64_t r2 = splitmix64(seed ^ ((static_cast<uint64_t>(i) << 1) | 1ull));
        const uint64_t tot = (r1 & 0xFFFFFFFFull) + (r1 >> 32) + (r2 & 0xFFFFFFFFull) + (r2 >> 32);
        const double v = static_cast<double>(static_cast<int64_t>(tot) - (int64_t(1) << 33));
        const float f = __double2float_rn(__dadd_rn(mean, __dmul_rn(v, scale)));
        out[i] = __float2bfloat16_rn(f);
    }
}

// One CTA per row; fp32 two-pass statistics over the row held in registers.
// Rows move as 16-byte vectors (8 bf16): h % 8 == 0 and 16-byte aligned rows
// (every model here has h1 % 128 == 0); a decode LN (32 rows x 5120) is one
// L2 round trip per thread instead of 20 dependent 2-byte loads.
template <int kThreads>
__global__ void __launch_bounds__(kThreads)
    layernorm_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, int h,
                     const __nv_bfloat16* __restrict__ gamma, const __nv_bfloat16* __restrict__ beta,
                     __nv_bfloat16* __restrict__ y, int64_t ldy) {
    constexpr int kMaxVec = 8;  // h <= 8 * 8 * kThreads
    __shared__ float red[kThreads / 32];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint4* xr = reinterpret_cast<const uint4*>(x + blockIdx.x * ldx);
    uint4* yr = reinterpret_cast<uint4*>(y + blockIdx.x * ldy);
    const uint4* g4 = reinterpret_cast<const uint4*>(gamma);
    const uint4* b4 = reinterpret_cast<const uint4*>(beta);
    const int nv = h >> 3;
    float v[kMaxVec][8];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxVec; ++j) {
        const int c = threadIdx.x + j * kThreads;
        uint4 q = make_uint4(0u, 0u, 0u, 0u);
        if (c < nv) q = xr[c];
        const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(p[e]);
            v[j][2 * e] = f.x;
            v[j][2 * e + 1] = f.y;
            s += f.x + f.y;
        }
    }
    auto block_sum = [&](float a) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) a += __shfl_xor_sync(0xffffffffu, a, d);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
        __syncthreads();
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < kThreads / 32; ++i) t += red[i];
        __syncthreads();
        return t;
    };
    const float mean = block_sum(s) / static_cast<float>(h);
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxVec; ++j) {
        if (threadIdx.x + j * kThreads < nv) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float d = v[j][e] - mean;
                q += d * d;
            }
        }
    }
    const float rstd = rsqrtf(block_sum(q) / static_cast<float>(h) + 1e-5f);
#pragma unroll
    for (int j = 0; j < kMaxVec; ++j) {
        const int c = threadIdx.x + j * kThreads;
        if (c < nv) {
            const uint4 gq = g4[c], bq = b4[c];
            const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gq);
            const __nv_bfloat162* bp = reinterpret_cast<const __nv_bfloat162*>(&bq);
            uint4 o;
            uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 gf = __bfloat1622float2(gp[e]);
                const float2 bf = __bfloat1622float2(bp[e]);
                const __nv_bfloat162 r = __floats2bfloat162_rn((v[j][2 * e] - mean) * rstd * gf.x + bf.x,
                                                               (v[j][2 * e + 1] - mean) * rstd * gf.y + bf.y);
                op[e] = *reinterpret_cast<const uint32_t*>(&r);
            }
            yr[c] = o;
        }
    }
}

// Decode-size LayerNorm (few rows, latency-bound inside the PDL chain of
// the decode step): gamma / beta are staged in shared memory BEFORE
// griddepcontrol.wait (they do not depend on the previous kernel), the row
// is held as packed bf16 (4 registers per 8 elements), and the statistics
// reduce over 128 threads. One CTA per row.
template <int kVec>
__global__ void __launch_bounds__(128)
    layernorm_rows_kernel(const __nv_bfloat16* __restrict__ x, int64_t ldx, int h,
                          const __nv_bfloat16* __restrict__ gamma, const __nv_bfloat16* __restrict__ beta,
                          __nv_bfloat16* __restrict__ y, int64_t ldy) {
    extern __shared__ uint4 gb[];  // [gamma | beta], h/8 vectors each
    __shared__ float red[4];
    const int nv = h >> 3;
    for (int c = threadIdx.x; c < nv; c += 128) {
        gb[c] = reinterpret_cast<const uint4*>(gamma)[c];
        gb[nv + c] = reinterpret_cast<const uint4*>(beta)[c];
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint4* xr = reinterpret_cast<const uint4*>(x + blockIdx.x * ldx);
    uint4* yr = reinterpret_cast<uint4*>(y + blockIdx.x * ldy);
    uint4 q[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
        const int c = threadIdx.x + j * 128;
        q[j] = c < nv ? xr[c] : make_uint4(0u, 0u, 0u, 0u);
    }
    auto block_sum = [&](float a) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) a += __shfl_xor_sync(0xffffffffu, a, d);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
        __syncthreads();
        const float t = (red[0] + red[1]) + (red[2] + red[3]);
        __syncthreads();
        return t;
    };
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
        const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q[j]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(p[e]);
            s += f.x + f.y;
        }
    }
    const float mean = block_sum(s) / static_cast<float>(h);
    float v = 0.f;
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
        if (threadIdx.x + j * 128 < nv) {
            const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q[j]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(p[e]);
                v += (f.x - mean) * (f.x - mean) + (f.y - mean) * (f.y - mean);
            }
        }
    }
    const float rstd = rsqrtf(block_sum(v) / static_cast<float>(h) + 1e-5f);
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
        const int c = threadIdx.x + j * 128;
        if (c < nv) {
            const uint4 gq = gb[c], bq = gb[nv + c];
            const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q[j]);
            const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gq);
            const __nv_bfloat162* bp = reinterpret_cast<const __nv_bfloat162*>(&bq);
            uint4 o;
            uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(p[e]);
                const float2 gf = __bfloat1622float2(gp[e]);
                const float2 bf = __bfloat1622float2(bp[e]);
                const __nv_bfloat162 r = __floats2bfloat162_rn((f.x - mean) * rstd * gf.x + bf.x,
                                                               (f.y - mean) * rstd * gf.y + bf.y);
                op[e] = *reinterpret_cast<const uint32_t*>(&r);
            }
            yr[c] = o;
        }
    }
}

// dst[i] = src[(i * stride + offset)] rows of width h (bf16), i < rows
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ src, int64_t lds,
                                   int64_t stride, int64_t offset, int rows, int h,
                                   __nv_bfloat16* __restrict__ dst, int64_t ldd) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int r = blockIdx.x;
    const __nv_bfloat16* s = src + (static_cast<int64_t>(r) * stride + offset) * lds;
    for (int c = threadIdx.x; c < h; c += blockDim.x) dst[r * ldd + c] = s[c];
}

}  // namespace

cudaError_t launch_synth(void* out, int64_t n, uint64_t seed, double mean, double std_,
                         cudaStream_t st) {
    const double scale = std_ * (1.7320508075688772 * 2.3283064365386963e-10);
    const int64_t blocks64 = (n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(blocks64 < 148 * 64 ? blocks64 : 148 * 64);
    synth_kernel<<<blocks, 256, 0, st>>>(static_cast<__nv_bfloat16*>(out), n, seed, mean, scale);
    return cudaGetLastError();
}

cudaError_t launch_layernorm(const void* x, int64_t ldx, int64_t rows, int h, const void* gamma,
                             const void* beta, void* y, int64_t ldy, cudaStream_t st) {
    if (h > 64 * 256 || (h & 7) || (ldx & 7) || (ldy & 7) ||
        ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
          reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(beta)) & 15))
        return cudaErrorInvalidValue;
    extern int g_pdl;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(rows));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#ifndef HP_LN_ROWS_MAX
#define HP_LN_ROWS_MAX 256
#endif
    if (rows <= HP_LN_ROWS_MAX && h <= 8 * 128 * 16) {  // decode-size: the latency-bound variant
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = static_cast<size_t>(h) * 4;  // gamma + beta
        const auto* xp = static_cast<const __nv_bfloat16*>(x);
        const auto* gp = static_cast<const __nv_bfloat16*>(gamma);
        const auto* bp = static_cast<const __nv_bfloat16*>(beta);
        auto* yp = static_cast<__nv_bfloat16*>(y);
        const int nv = h / 8;
        if (nv <= 128 * 4) return cudaLaunchKernelEx(&cfg, layernorm_rows_kernel<4>, xp, ldx, h, gp, bp, yp, ldy);
        if (nv <= 128 * 8) return cudaLaunchKernelEx(&cfg, layernorm_rows_kernel<8>, xp, ldx, h, gp, bp, yp, ldy);
        if (cfg.dynamicSmemBytes > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(layernorm_rows_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(cfg.dynamicSmemBytes));
            if (e != cudaSuccess) return e;
        }
        return cudaLaunchKernelEx(&cfg, layernorm_rows_kernel<16>, xp, ldx, h, gp, bp, yp, ldy);
    }
    return cudaLaunchKernelEx(&cfg, layernorm_kernel<256>, static_cast<const __nv_bfloat16*>(x), ldx,
                              h, static_cast<const __nv_bfloat16*>(gamma),
                              static_cast<const __nv_bfloat16*>(beta),
                              static_cast<__nv_bfloat16*>(y), ldy);
}

cudaError_t launch_gather_rows(const void* src, int64_t lds, int64_t stride, int64_t offset,
                               int rows, int h, void* dst, int64_t ldd, cudaStream_t st) {
    gather_rows_kernel<<<rows, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), lds, stride,
                                             offset, rows, h, static_cast<__nv_bfloat16*>(dst), ldd);
    return cudaGetLastError();
}

}  // namespace hp
