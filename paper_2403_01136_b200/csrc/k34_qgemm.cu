// K3 / K4 — fused dequant + tcgen05 GEMM (sm_100a):
//     y[m × n_out] = epi( x[m × k_in] · dequant(W)ᵀ ) (+ residual)
//
// The reference has no layer forward; the per-element dequant
// is the reference's `zero + snapped * step` (indicator.cpp:53) on K1's
// codes, and the op set is the decoder's qkv/out/fc1/fc2
// (memcost.cpp:33, indicator.hpp:32).
//
// Swap-AB on tensor cores: the weights are the MMA's M operand (128 output
// rows per tile) and live in TENSOR MEMORY, written there by dequant warps
// with tcgen05.st; the activations are the N operand (BN tokens per tile),
// TMA-loaded into shared memory with the 128-byte swizzle. One CTA per SM,
// persistent over (token-tile, row-tile, k-split) work units, 16 warps:
//   warp 0      producer: cp.async.bulk of packed codes + scales, TMA of x
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::f16, A from TMEM
//   warp 2      TMEM allocator
//   warps 4-11  dequant: smem codes -> bf16x2 -> tcgen05.st into A stages
//   warps 12-15 epilogue: tcgen05.ld accumulators -> bf16 (+res/relu) or
//               fp32 split-K partials with a last-CTA ordered reduction
// Pipelines: smem stages full/empty (producer<->MMA), TMEM A stages
// afull/aempty (dequant<->MMA), accumulator buffers tfull/tempty
// (MMA<->epilogue).
// Decode (K3, M = xi <= 32): BN = 16/32 and split-K so every SM streams
// weights; HBM-bound. Prefill (K4, M = eta*s): BN = 128/256, no split;
// tensor-bound.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "layout.cuh"
#include "sm100.cuh"

namespace hp {

// Persistent-grid cap: leave SMs to concurrent NCCL kernels (pipeline runs).
int g_sm_budget = 0;

struct qgemm_args {
    const uint8_t* packed;
    const float* scale;
    const float* zero;
    int n_out, k_in, G, NT;
    int m, MT;
    int splits, gps;  // k-splits, groups per split
    int num_units;
    __nv_bfloat16* y;
    int64_t ldy;
    const __nv_bfloat16* res;
    int64_t ldr;
    int epi;
    float* partial;     // [splits][MT*BN][n_out] fp32 (splits > 1)
    unsigned* counters; // [MT*NT]
};

template <int BITS, int BN>
struct qgemm_cfg {
    static constexpr int kThreads = 512;
    static constexpr int kB = BN * 256;                 // two 64-k swizzled sub-tiles
    static constexpr int kCodes = BITS * 2048;
    static constexpr int kScale = BITS == 16 ? 0 : 1024; // scale + zero rows
    static constexpr int kStage = kB + kCodes + kScale;
    static constexpr int kBudget = 200 * 1024;
    static constexpr int SS_ = kBudget / kStage;
    static constexpr int SS = SS_ > 12 ? 12 : SS_;
    static constexpr int NACC = BN <= 128 ? 2 : 1;
    static constexpr int A0_ = NACC * BN < 64 ? 64 : NACC * BN;
    static constexpr int A0 = (A0_ + 63) / 64 * 64;
    static constexpr int AS_ = (512 - A0) / 64;
    static constexpr int AS = AS_ > 8 ? 8 : AS_;
    static constexpr int kBarOff = SS * kStage;
    static constexpr int kSmem = kBarOff + 256 + 1024;  // + barriers + align slack
    static_assert(SS >= 2, "need >= 2 smem stages");
    static_assert(AS >= 2, "need >= 2 TMEM A stages");
};

template <int BITS, bool SYM, int BN>
__global__ void __launch_bounds__(512, 1)
    qgemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const qgemm_args a) {
    using C = qgemm_cfg<BITS, BN>;
    constexpr int SS = C::SS, AS = C::AS, NACC = C::NACC;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    auto stage_b = [&](int s) { return smem + s * C::kStage; };
    auto stage_codes = [&](int s) { return smem + s * C::kStage + C::kB; };
    auto stage_scale = [&](int s) {
        return reinterpret_cast<float*>(smem + s * C::kStage + C::kB + C::kCodes);
    };
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
    uint64_t* full = bars;
    uint64_t* empty = full + SS;
    uint64_t* afull = empty + SS;
    uint64_t* aempty = afull + AS;
    uint64_t* tfull = aempty + AS;
    uint64_t* tempty = tfull + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);
    unsigned* bcast = tmem_slot + 1;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 1 && lane == 0) {
        for (int i = 0; i < SS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < AS; ++i) {
            mbar_init(&afull[i], 8);
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < NACC; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) prefetch_tmap(&tmap_x);
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int per_mt = a.NT * a.splits;

    if (warp == 0) {
        // ===================== producer =====================
        if (lane == 0) {
            constexpr uint32_t kBytes = C::kB + C::kCodes + (BITS == 16 ? 0 : (SYM ? 512 : 1024));
            uint32_t it = 0;
            for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
                const int mt = u / per_mt, rem = u % per_mt;
                const int nt = rem / a.splits, sp = rem % a.splits;
                const int g0 = sp * a.gps;
                const int g1 = min(a.G, g0 + a.gps);
                for (int g = g0; g < g1; ++g, ++it) {
                    const int s = it % SS;
                    mbar_wait(&empty[s], ((it / SS) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[s], kBytes);
                    const size_t t = static_cast<size_t>(nt) * a.G + g;
                    bulk_g2s(stage_codes(s), a.packed + t * C::kCodes, C::kCodes, &full[s]);
                    if constexpr (BITS != 16) {
                        bulk_g2s(stage_scale(s), a.scale + t * 128, 512, &full[s]);
                        if constexpr (!SYM)
                            bulk_g2s(stage_scale(s) + 128, a.zero + t * 128, 512, &full[s]);
                    }
                    tma_load_2d(stage_b(s), &tmap_x, g * 128, mt * BN, &full[s]);
                    tma_load_2d(stage_b(s) + BN * 128, &tmap_x, g * 128 + 64, mt * BN, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
            uint32_t it = 0, ut = 0;
            for (int u = blockIdx.x; u < a.num_units; u += gridDim.x, ++ut) {
                const int rem = u % per_mt;
                const int sp = rem % a.splits;
                const int g0 = sp * a.gps;
                const int g1 = min(a.G, g0 + a.gps);
                const int acc = ut % NACC;
                mbar_wait(&tempty[acc], ((ut / NACC) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + acc * BN;
                for (int g = g0; g < g1; ++g, ++it) {
                    const int s = it % SS, as = it % AS;
                    mbar_wait(&full[s], (it / SS) & 1);
                    mbar_wait(&afull[as], (it / AS) & 1);
                    tc_fence_after();
                    const uint32_t bbase = smem_u32(stage_b(s));
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint64_t bdesc =
                            umma_desc_sw128(bbase + (j >> 2) * (BN * 128) + (j & 3) * 32);
                        mma_ts(d_tmem, tmem + C::A0 + as * 64 + j * 8, bdesc, idesc,
                               (g > g0 || j > 0) ? 1u : 0u);
                    }
                    tc_commit(&empty[s]);
                    tc_commit(&aempty[as]);
                }
                tc_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ===================== dequant =====================
        const int q = warp - 4;
        const int lq = warp & 3;  // TMEM lane quarter of this warp
        const int kh = q >> 2;    // which 64-k half of each group
        const int r = lq * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(lq * 32) << 16;
        uint32_t it = 0;
        for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
            const int rem = u % per_mt;
            const int sp = rem % a.splits;
            const int g0 = sp * a.gps;
            const int g1 = min(a.G, g0 + a.gps);
            for (int g = g0; g < g1; ++g, ++it) {
                const int s = it % SS, as = it % AS;
                mbar_wait(&full[s], (it / SS) & 1);
                mbar_wait(&aempty[as], ((it / AS) & 1) ^ 1);
                tc_fence_after();
                float sf = 0.f, zf = 0.f;
                if constexpr (BITS != 16) {
                    sf = stage_scale(s)[r];
                    if constexpr (!SYM) zf = stage_scale(s)[128 + r];
                }
                const uint32_t s2 = bf16x2_splat_bits(sf), z2 = bf16x2_splat_bits(zf);
                const uint8_t* rowc = stage_codes(s) + r * 16;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int sl = kh * 2 + h;
                    uint32_t v[16];
                    dequant_slice32<BITS, SYM>(rowc, sl, sf, zf, s2, z2, v);
                    tmem_st16(tmem + lane_addr + C::A0 + as * 64 + sl * 16, v);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[as]);
            }
        }
    } else if (warp >= 12) {
        // ===================== epilogue =====================
        const int lq = warp & 3;
        const int r = lq * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(lq * 32) << 16;
        uint32_t ut = 0;
        for (int u = blockIdx.x; u < a.num_units; u += gridDim.x, ++ut) {
            const int mt = u / per_mt, rem = u % per_mt;
            const int nt = rem / a.splits, sp = rem % a.splits;
            const int acc = ut % NACC;
            const int n = nt * 128 + r;
            mbar_wait(&tfull[acc], (ut / NACC) & 1);
            tc_fence_after();
            for (int c0 = 0; c0 < BN; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + lane_addr + acc * BN + c0, v);
                tmem_ld_wait();
                if (a.splits == 1) {
                    if (n < a.n_out) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int t = mt * BN + c0 + i;
                            if (t < a.m) {
                                float f = __uint_as_float(v[i]);
                                if (a.epi & 1) f = fmaxf(f, 0.0f);
                                if (a.res) f += __bfloat162float(a.res[t * a.ldr + n]);
                                a.y[t * a.ldy + n] = __float2bfloat16_rn(f);
                            }
                        }
                    }
                } else {
                    float* dst = a.partial + (static_cast<size_t>(sp) * a.MT * BN +
                                              static_cast<size_t>(mt) * BN + c0) * a.n_out;
                    if (n < a.n_out) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            dst[static_cast<size_t>(i) * a.n_out + n] = __uint_as_float(v[i]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);

            if (a.splits > 1) {
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (warp == 12 && lane == 0)
                    *bcast = atomicAdd(&a.counters[mt * a.NT + nt], 1u);
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (*bcast == static_cast<unsigned>(a.splits - 1)) {
                    __threadfence();
                    if (n < a.n_out) {
                        for (int i = 0; i < BN; ++i) {
                            const int t = mt * BN + i;
                            if (t >= a.m) break;
                            float f = 0.f;
                            for (int k = 0; k < a.splits; ++k)
                                f += __ldcg(a.partial + (static_cast<size_t>(k) * a.MT * BN +
                                                         static_cast<size_t>(mt) * BN + i) *
                                                            a.n_out + n);
                            if (a.epi & 1) f = fmaxf(f, 0.0f);
                            if (a.res) f += __bfloat162float(a.res[t * a.ldr + n]);
                            a.y[t * a.ldy + n] = __float2bfloat16_rn(f);
                        }
                    }
                    if (warp == 12 && lane == 0) a.counters[mt * a.NT + nt] = 0u;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
        }
    }

    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

int g_num_sms = 0;

int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    const int budget = g_sm_budget;
    return (budget > 0 && budget < g_num_sms) ? budget : g_num_sms;
}

template <int BITS, bool SYM, int BN>
cudaError_t launch_one(const CUtensorMap& map, const qgemm_args& a, int grid,
                       cudaStream_t st) {
    using C = qgemm_cfg<BITS, BN>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(qgemm_kernel<BITS, SYM, BN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::kSmem);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    qgemm_kernel<BITS, SYM, BN><<<grid, C::kThreads, C::kSmem, st>>>(map, a);
    return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_bits(int bits, bool sym, const CUtensorMap& map,
                          const qgemm_args& a, int grid, cudaStream_t st) {
    switch (bits) {
        case 3: return sym ? launch_one<3, true, BN>(map, a, grid, st) : launch_one<3, false, BN>(map, a, grid, st);
        case 4: return sym ? launch_one<4, true, BN>(map, a, grid, st) : launch_one<4, false, BN>(map, a, grid, st);
        case 8: return sym ? launch_one<8, true, BN>(map, a, grid, st) : launch_one<8, false, BN>(map, a, grid, st);
        case 16: return launch_one<16, true, BN>(map, a, grid, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

struct qgemm_plan {
    int bn, mt, splits, gps, units, grid;
    size_t workspace;
};

qgemm_plan plan_qgemm(int64_t n_out, int64_t k_in, int64_t m, int phase) {
    qgemm_plan p{};
    const int G = static_cast<int>(ceil_div64(k_in, 128));
    const int NT = static_cast<int>(ceil_div64(n_out, 128));
    const int sms = num_sms();
    if (phase == 1 && m <= 32) {
        p.bn = m <= 16 ? 16 : 32;
    } else {
        p.bn = m <= 128 ? 128 : 256;
    }
    p.mt = static_cast<int>(ceil_div64(m, p.bn));
    p.splits = 1;
    if (phase == 1 && p.mt == 1) {
        // minimise waves * groups-per-unit; prefer fewer splits on ties
        long best = -1;
        for (int s = 1; s <= 16 && s <= G; ++s) {
            const long units = static_cast<long>(NT) * s;
            const long cost = ((units + sms - 1) / sms) * ((G + s - 1) / s);
            if (best < 0 || cost < best) {
                best = cost;
                p.splits = s;
            }
        }
    }
    p.gps = (G + p.splits - 1) / p.splits;
    p.splits = (G + p.gps - 1) / p.gps;  // no empty splits
    p.units = p.mt * NT * p.splits;
    p.grid = p.units < sms ? p.units : sms;
    p.workspace = 0;
    if (p.splits > 1)
        p.workspace = 256 +
                      (static_cast<size_t>(p.mt) * NT * sizeof(unsigned) + 255) / 256 * 256 +
                      static_cast<size_t>(p.splits) * p.mt * p.bn * n_out * sizeof(float);
    return p;
}

cudaError_t launch_qgemm(const CUtensorMap& map, const qgemm_plan& p, int bits,
                         bool sym, const void* packed, const float* scale,
                         const float* zero, int64_t n_out, int64_t k_in,
                         int64_t m, void* y, int64_t ldy, const void* res,
                         int64_t ldr, int epi, void* workspace,
                         cudaStream_t st) {
    qgemm_args a{};
    a.packed = static_cast<const uint8_t*>(packed);
    a.scale = scale;
    a.zero = zero;
    a.n_out = static_cast<int>(n_out);
    a.k_in = static_cast<int>(k_in);
    a.G = static_cast<int>(ceil_div64(k_in, 128));
    a.NT = static_cast<int>(ceil_div64(n_out, 128));
    a.m = static_cast<int>(m);
    a.MT = p.mt;
    a.splits = p.splits;
    a.gps = p.gps;
    a.num_units = p.units;
    a.y = static_cast<__nv_bfloat16*>(y);
    a.ldy = ldy;
    a.res = static_cast<const __nv_bfloat16*>(res);
    a.ldr = ldr;
    a.epi = epi;
    if (p.splits > 1) {
        auto* base = static_cast<uint8_t*>(workspace);
        a.counters = reinterpret_cast<unsigned*>(base);
        a.partial = reinterpret_cast<float*>(
            base + 256 + ((static_cast<size_t>(p.mt) * a.NT * sizeof(unsigned) + 255) / 256) * 256);
    }
    switch (p.bn) {
        case 16: return dispatch_bits<16>(bits, sym, map, a, p.grid, st);
        case 32: return dispatch_bits<32>(bits, sym, map, a, p.grid, st);
        case 128: return dispatch_bits<128>(bits, sym, map, a, p.grid, st);
        case 256: return dispatch_bits<256>(bits, sym, map, a, p.grid, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace hp
