// K3 (fused) — one persistent sm_100a kernel per decode step of a pipeline
// stage: every decoder layer of the stage (LN1, qkv, out(+res), LN2,
// fc1(relu), fc2(+res)) for xi <= 32 tokens, in ONE launch.
//
// Why: a decode op moves 10-40 MB (2-6 us of HBM time) but a kernel boundary
// drains and refills the whole HBM pipeline (launch, prologue, ramp, stream-K
// tail: ~10 us per op). Here the weight stream never stops:
// the code producer and the dequant warps of every CTA run ahead across op
// boundaries (weights do not depend on activations); only the activation
// producer waits, on a device-wide completion counter, for the op whose
// output it reads. An op boundary costs one flag round trip instead of a
// pipeline drain, and it is hidden behind the ~200 KB of weights each SM has
// in flight.
//
// Per-op arithmetic is K3's exactly (k34_qgemm.cu): the reference dequant
// `zero + code*step` (indicator.cpp:53) on K1's codes, fp32 accumulation in
// TMEM, stream-K over 128-k groups with the last CTA of a split tile summing
// the partials in segment order; LN is glue.cu's layernorm_kernel<256>
// arithmetic (the same 256-lane reduction order, emulated by 128 threads),
// so a fused step is bit-identical to the per-op launches of the same stage.
//
// Synchronisation (all CTAs co-resident: grid <= SMs, 1 CTA/SM, cooperative
// launch): `done` counts completed units (output tiles of a GEMM op, rows of
// an LN op) in op order. Op i's inputs are ready when done >= wait[i] (the
// units of all earlier ops). Writers: generic stores, fence, bar, one
// atomicAdd. Readers: ld.acquire poll, then fence.proxy.async before TMA
// (the async proxy reads what the generic proxy of other SMs wrote); all
// generic re-reads of in-kernel data use ld.global.cg (never stale L1).
// The last CTA to exit resets the counters, so the launch is replayable in a
// CUDA graph.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

#include "layout.cuh"
#include "sm100.cuh"

namespace hp {

extern int g_sm_budget;

struct dstage_op {
    const uint8_t* packed;
    const float* scale;
    const float* zero;
    __nv_bfloat16* y;
    const __nv_bfloat16* res;
    const CUtensorMap* tmap;  // activations x (global memory, 64-byte aligned)
    int64_t ldy, ldr;
    int total;                // NT * G group-steps (stream-K)
    int kind;                 // 0 GEMM, 1 LayerNorm
    int bits, n_out, k_in, G, NT, maxseg, epi, sps;
    unsigned wait;            // `done` value at which this op's inputs are complete
    // LayerNorm: y[r] = LN(x[r]) * gamma + beta, r < m
    const __nv_bfloat16* ln_x;
    const __nv_bfloat16* gamma;
    const __nv_bfloat16* beta;
    __nv_bfloat16* ln_y;
    int64_t ln_ldx, ln_ldy;
    int h;
    int P;                    // CTAs the op is split over (= K3's grid for it)
    // dataflow between consecutive GEMMs: this op's k-group g needs output
    // tile dep_off + g of the producing op (its out_flags == epoch + 1)
    const unsigned* dep_flags;
    unsigned* out_flags;      // per output tile, set to epoch + 1 when written
    int dep_off;
    int pbuf;                 // stream-K workspace parity (consecutive GEMMs differ)
};

static_assert(sizeof(dstage_op) == 192, "dstage_op layout is shared by k3_stage.cu and capi.cu");
struct dstage_args {
    const dstage_op* ops;
    int nops;
    int m;
    unsigned long long* sync;   // [0] done (u64, never reset), [1] = {epoch u32, exit ticket u32}
    unsigned long long units;   // units (tiles + LN rows) per launch: done target base = epoch * units
    unsigned* counters[2];      // per-tile stream-K tickets, per parity
    float* partial[2];          // [tiles][maxseg][BN/4][128] float4, per parity
    unsigned long long* trace;  // HP_DSTAGE_TRACE builds: [cta][op][4] globaltimer
};

// Debug trace (HP_DSTAGE_TRACE): per CTA and op, the %globaltimer when
// 0: the activation producer saw the op's inputs complete, 1: the epilogue
// finished the op, 2: dequant warp 4 finished the op's stages, 3: the
// weight producer issued the op's last stage.
__device__ __forceinline__ void dtrace(const dstage_args& a, int oi, int ev) {
#ifdef HP_DSTAGE_TRACE
    if (a.trace && oi < 256) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[(static_cast<size_t>(blockIdx.x) * 256 + oi) * 8 + ev] = t;
    }
#endif
}

namespace {

constexpr int kBN = 32;
#ifndef HP_DSTAGE_DWG
#define HP_DSTAGE_DWG 3
#endif
constexpr int kDWG = HP_DSTAGE_DWG;     // dequant warpgroups, stages round-robin
constexpr int kThreads = 128 * (2 + kDWG);
constexpr int kEpiWarp0 = 4 + 4 * kDWG;
constexpr int kCodeBytes = 16384;       // max codes per stage (3/4-bit 2 groups, 8-bit 1, 16-bit 1/2)
constexpr int kActBytes = kBN * 64 * 2 * 4;  // [32 x 256 k] bf16 = 4 swizzled 64-k sub-tiles
constexpr int kBR = 3;
constexpr int kTmemCols = 512;
constexpr int kNACC = 2;
constexpr int kA0 = 64;                 // TMEM: 2 accumulators of 32 cols, then A stages
constexpr int kACols = 128;             // up to 8 slices x 16 cols
constexpr int kAS = (448 / kACols) / kDWG * kDWG;  // TMEM A stages, a multiple of kDWG
constexpr int kStgLd = 132;
constexpr int kHB = 4;    // epilogue -> reducer handoffs in flight (named barriers kHB0..)
constexpr int kHB0 = 4;

template <bool SYM>
struct dcfg {
    static constexpr int kCS = kCodeBytes + (SYM ? 1024 : 2048);  // + 2 groups of scales (+zeros)
    static constexpr int kCodesOff = kBR * kActBytes;
    static constexpr int kBudget = 227 * 1024 - 16 * kStgLd * 4 - 2048;
    static constexpr int CR_ = (kBudget - kCodesOff) / kCS;
    static constexpr int CR = (CR_ / kDWG) * kDWG;
    static constexpr int kStgOff = kCodesOff + CR * kCS;
    static constexpr int kBarOff = kStgOff + 16 * kStgLd * 4;
    static constexpr int kSmem = kBarOff + 512 + 1024;
    static_assert(CR >= kDWG && CR % kDWG == 0, "ring");
    static_assert(kSmem <= 227 * 1024, "smem");
};

#ifdef HP_DSTAGE_WATCHDOG
// Debug build: bounded waits that report which wait hung, then trap.
__device__ __forceinline__ void wd_wait(uint64_t* bar, uint32_t parity, int tag, bool warp_wide) {
    const uint32_t a = smem_u32(bar);
    long long n = 0;
    while (true) {
        const uint32_t ok = mbar_try_wait(a, parity);
        const bool all = warp_wide ? __all_sync(0xffffffffu, ok) : ok;
        if (all) return;
        if (++n == (1ll << 22)) {
            printf("dstage hang: cta %d warp %d tag %d parity %u\n", blockIdx.x, threadIdx.x / 32, tag, parity);
            __trap();
        }
    }
}
#define MBW(bar, par, tag) wd_wait(bar, par, tag, false)
#define MBWW(bar, par, tag) wd_wait(bar, par, tag, true)
#else
#define MBW(bar, par, tag) mbar_wait(bar, par)
#define MBWW(bar, par, tag) mbar_wait_warp(bar, par)
#endif
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void wait_done(const unsigned long long* done, unsigned long long target) {
#ifdef HP_DSTAGE_WATCHDOG
    long long n = 0;
    while (ld_acquire64(done) < target) {
        __nanosleep(32);
        if (++n == (1ll << 22)) {
            printf("dstage hang: cta %d warp %d wait_done %llu (have %llu)\n", blockIdx.x, threadIdx.x / 32,
                   target, ld_acquire64(done));
            __trap();
        }
    }
#else
    while (ld_acquire64(done) < target) __nanosleep(32);
#endif
}
__device__ __forceinline__ void wait_flag(const unsigned* f, unsigned v) {
#ifdef HP_DSTAGE_WATCHDOG
    long long n = 0;
    while (ld_acquire(f) != v) {
        __nanosleep(32);
        if (++n == (1ll << 22)) {
            printf("dstage hang: cta %d warp %d flag want %u have %u\n", blockIdx.x, threadIdx.x / 32, v,
                   ld_acquire(f));
            __trap();
        }
    }
#else
    while (ld_acquire(f) != v) __nanosleep(32);
#endif
}

// Stream-K arithmetic in 32 bits: an op has at most NT*G = 448*112 group-steps
// (BLOOM fc1/fc2) and the grid is <= 148 CTAs, so c*total < 2^31.
__device__ __forceinline__ int sk_lo(int c, int total, int P) { return (c * total) / P; }
__device__ __forceinline__ int sk_owner(int w, int total, int P) {
    int c = (w * P) / total;
    while (c + 1 < P && sk_lo(c + 1, total, P) <= w) ++c;
    while (c > 0 && sk_lo(c, total, P) > w) --c;
    return c;
}

struct seg_t {
    int tile, g0, g1, idx, nseg;
};

// Stream-K segments of one op for this CTA, last segment first (as K3).
struct seg_iter {
    int w, w1, wlo, wlast, total, G, phase;
    int P;
    __device__ __forceinline__ void init(int total_, int G_, int P_) {
        total = total_;
        G = G_;
        P = P_;
        const int c = blockIdx.x;
        wlo = c < P ? sk_lo(c, total, P) : 0;
        w1 = c < P ? sk_lo(c + 1, total, P) : 0;
        const int tstart = w1 > 0 ? ((w1 - 1) / G) * G : 0;
        wlast = tstart > wlo ? tstart : wlo;
        w = wlast;
        phase = 0;
    }
    __device__ __forceinline__ bool next(seg_t& s) {
        if (phase == 0 && w >= w1) {
            phase = 1;
            w = wlo;
        }
        const int lim = phase == 0 ? w1 : wlast;
        if (w >= lim) return false;
        const int tile = w / G;
        const int g0 = w - tile * G;
        const int tend = (tile + 1) * G;
        const int wend = lim < tend ? lim : tend;
        const int first = sk_owner(tile * G, total, P);
        const int last = sk_owner(tend - 1, total, P);
        s = {tile, g0, g0 + (wend - w), static_cast<int>(blockIdx.x) - first, last - first + 1};
        w = wend;
        return true;
    }
};

// 16 tokens x 128 rows of fp32 results -> bf16 y (+ residual, relu), through
// shared memory so the global stores are 16-byte vectors along n. Same
// arithmetic as k34_qgemm.cu's stage_store16; residual via L2 (.cg).
__device__ __forceinline__ void store16(const dstage_op& op, int m, float* stg, int r,
                                        const float (&v)[16], int t0, int n0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) stg[i * kStgLd + r] = v[i];
    asm volatile("bar.sync 2, 128;" ::: "memory");
    const int tid = threadIdx.x & 127;
    const int t = tid >> 3;
    const int seg = (tid & 7) * 16;
    const int tok = t0 + t;
    const int n = n0 + seg;
    if (tok < m && n < op.n_out) {
        const float* src = stg + t * kStgLd + seg;
        float f[16];
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
            const float4 q = *reinterpret_cast<const float4*>(src + i);
            f[i] = q.x; f[i + 1] = q.y; f[i + 2] = q.z; f[i + 3] = q.w;
        }
        if (op.epi & 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], 0.0f);
        }
        __nv_bfloat16* dst = op.y + static_cast<int64_t>(tok) * op.ldy + n;
        const __nv_bfloat16* res = op.res ? op.res + static_cast<int64_t>(tok) * op.ldr + n : nullptr;
        if (n + 16 <= op.n_out) {  // host guarantees 16-byte aligned rows
            if (res) {
                const uint4 r0 = __ldcg(reinterpret_cast<const uint4*>(res));
                const uint4 r1 = __ldcg(reinterpret_cast<const uint4*>(res + 8));
                const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&r0);
                const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&r1);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 x0 = __bfloat1622float2(h0[i]);
                    const float2 x1 = __bfloat1622float2(h1[i]);
                    f[2 * i] += x0.x; f[2 * i + 1] += x0.y;
                    f[8 + 2 * i] += x1.x; f[8 + 2 * i + 1] += x1.y;
                }
            }
            uint4 o0, o1;
            o0.x = pack_bf16x2(f[0], f[1]); o0.y = pack_bf16x2(f[2], f[3]);
            o0.z = pack_bf16x2(f[4], f[5]); o0.w = pack_bf16x2(f[6], f[7]);
            o1.x = pack_bf16x2(f[8], f[9]); o1.y = pack_bf16x2(f[10], f[11]);
            o1.z = pack_bf16x2(f[12], f[13]); o1.w = pack_bf16x2(f[14], f[15]);
            *reinterpret_cast<uint4*>(dst) = o0;
            *reinterpret_cast<uint4*>(dst + 8) = o1;
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (n + i < op.n_out) {
                    float x = f[i];
                    if (res) x += __bfloat162float(__ldcg(res + i));
                    dst[i] = __float2bfloat16_rn(x);
                }
            }
        }
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
}

// The 128 epilogue threads publish one finished unit: bar.sync orders every
// thread's stores before thread 0's gpu-scope release (cumulative), the
// pattern of CUTLASS's split-K semaphore; one release instead of 128 full
// fences (a fence.sc per thread cost ~1.8 us on the critical path).
__device__ __forceinline__ void publish(unsigned long long* done, unsigned* flag, unsigned epoch1) {
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if ((threadIdx.x & 127) == 0) {
        fence_proxy_async_global();  // consumers read these outputs with TMA
        if (flag) st_release(flag, epoch1);
        red_release64(done, 1ull);
    }
}

// LayerNorm of row `row` by the 128 epilogue threads, bit-identical to
// glue.cu layernorm_kernel<256>: thread t plays the kernel's threads t and
// t+128 (vectors c = v + 256 j), keeps their partial sums apart, and the
// block sum adds the 8 virtual warps' butterfly results in warp order.
// Row values stay in registers for h <= 8192 (4 vectors per virtual
// thread), else are re-read from L2 (same values, same order).
template <bool CACHED>
__device__ __forceinline__ void ln_row(const dstage_op& op, int row, float* red) {
    constexpr int MAXV = CACHED ? 3 : 1;  // cached: h <= 6144 (nv <= 768)
    const int t = threadIdx.x & 127;
    const int lane = t & 31, wq = t >> 5;
    const uint4* xr = reinterpret_cast<const uint4*>(op.ln_x + row * op.ln_ldx);
    uint4* yr = reinterpret_cast<uint4*>(op.ln_y + row * op.ln_ldy);
    const uint4* g4 = reinterpret_cast<const uint4*>(op.gamma);
    const uint4* b4 = reinterpret_cast<const uint4*>(op.beta);
    const int nv = op.h >> 3;
    const int nj = CACHED ? MAXV : (nv + 255) / 256;
    uint4 cache[2][MAXV];
    if constexpr (CACHED) {
#pragma unroll
        for (int j = 0; j < MAXV; ++j)
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int c = t + 128 * half + 256 * j;
                cache[half][j] = c < nv ? __ldcg(xr + c) : make_uint4(0u, 0u, 0u, 0u);
            }
    }
    auto vec = [&](int half, int j) -> uint4 {
        if constexpr (CACHED) {
            return cache[half][j];
        } else {
            const int c = t + 128 * half + 256 * j;
            return c < nv ? __ldcg(xr + c) : make_uint4(0u, 0u, 0u, 0u);
        }
    };
    float s[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < nj; ++j)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const uint4 q = vec(half, j);
            const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(p[e]);
                s[half] += f.x + f.y;
            }
        }
    // block_sum over 256 virtual threads: virtual warp (half*4 + wq)
    auto block_sum = [&](float a0, float a1) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, d);
            a1 += __shfl_xor_sync(0xffffffffu, a1, d);
        }
        if (lane == 0) {
            red[wq] = a0;
            red[4 + wq] = a1;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        float tot = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) tot += red[i];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        return tot;
    };
    const float mean = block_sum(s[0], s[1]) / static_cast<float>(op.h);
    float q[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < nj; ++j)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int c = t + 128 * half + 256 * j;
            if (c < nv) {
                const uint4 v = vec(half, j);
                const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(p[e]);
                    const float d0 = f.x - mean, d1 = f.y - mean;
                    q[half] += d0 * d0;
                    q[half] += d1 * d1;
                }
            }
        }
    const float rstd = rsqrtf(block_sum(q[0], q[1]) / static_cast<float>(op.h) + 1e-5f);
#pragma unroll
    for (int j = 0; j < nj; ++j)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int c = t + 128 * half + 256 * j;
            if (c < nv) {
                const uint4 v = vec(half, j);
                const uint4 gq = g4[c], bq = b4[c];
                const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
                const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gq);
                const __nv_bfloat162* bp = reinterpret_cast<const __nv_bfloat162*>(&bq);
                uint4 o;
                uint32_t* opw = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(p[e]);
                    const float2 gf = __bfloat1622float2(gp[e]);
                    const float2 bf = __bfloat1622float2(bp[e]);
                    const __nv_bfloat162 r = __floats2bfloat162_rn((f.x - mean) * rstd * gf.x + bf.x,
                                                                   (f.y - mean) * rstd * gf.y + bf.y);
                    opw[e] = *reinterpret_cast<const uint32_t*>(&r);
                }
                yr[c] = o;
            }
        }
}

// One dequant stage of one warp (32 rows of the 128-row tile): codes and
// scales from the smem slot into registers, release the slot, convert and
// store the bf16 A operand into the TMEM stage. Same code path as K3.
template <int BITS, bool SYM, int SPS>
__device__ __forceinline__ void dq_stage(uint32_t slot, int r, int nsl, uint32_t a_addr,
                                         uint64_t* empty_c, int lane) {
    constexpr int kG = (SPS + 3) / 4;
    float sf[kG], zf[kG];
    slice_words<BITS> wv[SPS];
    const uint32_t cbase = slot + r * 16;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        sf[j] = 0.f;
        zf[j] = 0.f;
        if constexpr (BITS != 16) {
            if (4 * j < nsl) {
                const uint32_t saddr = slot + kCodeBytes + (j * 128 + r) * 4;
                sf[j] = ldsf(saddr);
                if constexpr (!SYM) zf[j] = ldsf(saddr + 1024);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < SPS; ++h) {
        if (h >= nsl) continue;
        if constexpr (SPS >= 4) {
            load_slice<BITS>(cbase + (h >> 2) * (BITS * 2048), h & 3, wv[h]);
        } else {
            load_slice<BITS>(cbase, h, wv[h]);
        }
    }
    fence_proxy_async_smem();  // ld.shared of the slot before its bulk-copy refill
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_c);
#pragma unroll
    for (int h = 0; h < SPS; ++h) {
        if (h < nsl) {
            const int j = h >> 2;
            // pin slice h's conversion after slice h-1's tcgen05.st (both
            // volatile): otherwise the scheduler converts all slices up
            // front and 8 x 16 live outputs spill
#pragma unroll
            for (int i = 0; i < slice_words<BITS>::N; ++i) asm volatile("" : "+r"(wv[h].w[i]));
            uint32_t v[16];
            convert_slice<BITS, SYM>(wv[h], sf[j], zf[j], scale_arg<SYM>(sf[j]),
                                     zero_arg<SYM>(sf[j], zf[j]), v);
            tmem_st16(a_addr + h * 16, v);
        }
    }
}

template <int BITS>
constexpr int kSPS = BITS <= 4 ? 8 : (BITS == 8 ? 4 : 2);  // 32-k slices per stage

// One launch runs every op of a run of layers with the same bit width (the
// dequant code is then one instantiation: a runtime bit switch spilled).
template <int BITS, bool SYM>
__global__ void __launch_bounds__(kThreads, 1) dstage_kernel(const dstage_args a) {
    using C = dcfg<SYM>;
    constexpr int CR = C::CR;
    constexpr int SPS = kSPS<BITS>;
    constexpr int NGMAX = SPS >= 4 ? SPS / 4 : 1;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    auto stage_b = [&](int s) { return smem + s * kActBytes; };
    auto stage_codes = [&](int s) { return smem + C::kCodesOff + s * C::kCS; };
    float* stg = reinterpret_cast<float*>(smem + C::kStgOff);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
    uint64_t* full_c = bars;
    uint64_t* empty_c = full_c + CR;
    uint64_t* full_b = empty_c + CR;
    uint64_t* empty_b = full_b + kBR;
    uint64_t* afull = empty_b + kBR;
    uint64_t* aempty = afull + kAS;
    uint64_t* tfull = aempty + kAS;
    uint64_t* tempty = tfull + kNACC;
    uint64_t* hfree = tempty + kNACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + kHB);
    unsigned* bcast = tmem_slot + 1;
    float* red = reinterpret_cast<float*>(bcast + 2);  // 8 floats
    unsigned* tres = reinterpret_cast<unsigned*>(red + 8);           // ticket results ring (8)
    volatile unsigned* tcount = reinterpret_cast<volatile unsigned*>(tres + 8);  // results posted

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    unsigned long long* done = a.sync;
    unsigned* epoch_exit = reinterpret_cast<unsigned*>(a.sync + 1);
    // stable for the whole launch: only the last CTA of the PREVIOUS launch
    // advanced it
    const unsigned epoch = __ldcg(epoch_exit);
    const unsigned epoch1 = epoch + 1u;
    const unsigned long long base = static_cast<unsigned long long>(epoch) * a.units;

    if (warp == 1 && lane == 0) {
        for (int i = 0; i < CR; ++i) {
            mbar_init(&full_c[i], 1);
            mbar_init(&empty_c[i], 4);
        }
        for (int i = 0; i < kBR; ++i) {
            mbar_init(&full_b[i], 1);
            mbar_init(&empty_b[i], 1);
        }
        for (int i = 0; i < kAS; ++i) {
            mbar_init(&afull[i], 4);
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < kNACC; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        for (int i = 0; i < kHB; ++i) mbar_init(&hfree[i], 1);
        *tcount = 0u;
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

    seg_t sg;
    if (warp == 0) {
        // ============ weight-code producer: streams across op boundaries ========
        uint32_t it = 0;
        for (int oi = 0; oi < a.nops; ++oi) {
            const dstage_op& op = a.ops[oi];
            if (op.kind != 0) continue;
            const uint8_t* packed = op.packed;
            const float* scale = op.scale;
            const float* zero = op.zero;
            const int G = op.G;
            seg_iter iter;
            iter.init(op.total, G, op.P);
            while (iter.next(sg)) {
                for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                    const int g = sl >> 2;
                    const int ng = SPS >= 4 ? min(NGMAX, sg.g1 - g) : 1;
                    const int s = it % CR;
                    MBWW(&empty_c[s], ((it / CR) & 1) ^ 1, 3);
                    const size_t t = static_cast<size_t>(sg.tile) * G + g;
                    const uint8_t* gsrc = packed + t * (BITS * 2048);
                    uint32_t cbytes, coff = 0;
                    if constexpr (SPS >= 4) {
                        cbytes = static_cast<uint32_t>(ng) * BITS * 2048;
                    } else {  // 16-bit half group
                        cbytes = 16384;
                        coff = ((sl >> 1) & 1) * 16384;
                    }
                    const uint32_t sbytes = BITS == 16 ? 0u : static_cast<uint32_t>(ng) * 512u * (SYM ? 1 : 2);
                    mbar_arrive_expect_tx_elect(&full_c[s], cbytes + sbytes);
                    bulk_g2s_elect(stage_codes(s), gsrc + coff, cbytes, &full_c[s]);
                    if constexpr (BITS != 16) {
                        bulk_g2s_elect(stage_codes(s) + kCodeBytes, scale + t * 128, ng * 512u, &full_c[s]);
                        if constexpr (!SYM)
                            bulk_g2s_elect(stage_codes(s) + kCodeBytes + 1024, zero + t * 128, ng * 512u,
                                           &full_c[s]);
                    }
                }
            }
            if (lane == 0) dtrace(a, oi, 3);
        }
    } else if (warp == 3) {
        // ============ activation producer: waits for the op's inputs ===========
        uint32_t it = 0;
        for (int oi = 0; oi < a.nops; ++oi) {
            const dstage_op& op = a.ops[oi];
            if (op.kind != 0) continue;
            const CUtensorMap* tmap = op.tmap;
            const unsigned* dep = op.dep_flags;
            const int dep_off = op.dep_off;
            if (!dep) {  // input written by a LayerNorm (or before the launch)
                if (lane == 0) wait_done(done, base + op.wait);
                __syncwarp();
                fence_proxy_async_global();
            }
            if (lane == 0) dtrace(a, oi, 0);
            constexpr uint32_t bytes = static_cast<uint32_t>(kBN * 128 * (SPS / 2));
            seg_iter iter;
            iter.init(op.total, op.G, op.P);
            while (iter.next(sg)) {
                for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                    const int s = it % kBR;
                    MBWW(&empty_b[s], ((it / kBR) & 1) ^ 1, 4);
                    if (dep) {  // dataflow: only the producer tiles this stage reads
                        const int g = sl >> 2;
                        const int ng = SPS >= 4 ? min(NGMAX, sg.g1 - g) : 1;
                        if (lane < ng) wait_flag(dep + dep_off + g + lane, epoch1);
                        __syncwarp();
                        fence_proxy_async_global();
                    }
                    mbar_arrive_expect_tx_elect(&full_b[s], bytes);
                    tma_load_3d_elect(stage_b(s), tmap, 0, 0, sl >> 1, &full_b[s]);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        constexpr uint32_t idesc = umma_idesc_bf16(128, kBN);
        uint32_t it = 0, ut = 0;
        for (int oi = 0; oi < a.nops; ++oi) {
            const dstage_op& op = a.ops[oi];
            if (op.kind != 0) continue;
            seg_iter iter;
            iter.init(op.total, op.G, op.P);
            while (iter.next(sg)) {
                const int acc = ut % kNACC;
                MBWW(&tempty[acc], ((ut / kNACC) & 1) ^ 1, 5);
                tc_fence_after();
                const uint32_t d_tmem = tmem + acc * kBN;
                for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                    const int nsl = min(SPS, 4 * sg.g1 - sl);
                    const int s = it % kBR, as = it % kAS;
                    MBWW(&full_b[s], (it / kBR) & 1, 6);
                    MBWW(&afull[as], (it / kAS) & 1, 7);
                    tc_fence_after();
                    const uint64_t bdesc0 = umma_desc_sw128(smem_u32(stage_b(s)));
                    const uint32_t abase = tmem + kA0 + as * kACols;
#pragma unroll
                    for (int q = 0; q < SPS / 2; ++q) {
                        if (2 * q < nsl)
                            mma_ts_x4_elect(d_tmem, abase + q * 32, bdesc0 + q * (kBN * 8), idesc,
                                            (sl > 4 * sg.g0 || q > 0) ? 1u : 0u);
                    }
                    tc_commit_elect(&empty_b[s]);
                    tc_commit_elect(&aempty[as]);
                }
                tc_commit_elect(&tfull[acc]);
                ++ut;
            }
        }
    } else if (warp >= 4 && warp < kEpiWarp0) {
        // ===================== dequant (round-robin warpgroups) ================
        const int q = warp - 4;
        const int lq = warp & 3;
        const int wg = q >> 2;
        const int r = lq * 32 + lane;
        const uint32_t tmem_lane = tmem + (static_cast<uint32_t>(lq * 32) << 16);
        const uint32_t codes0 = smem_u32(stage_codes(0));
        uint32_t it = 0;
        for (int oi = 0; oi < a.nops; ++oi) {
            const dstage_op& op = a.ops[oi];
            if (op.kind != 0) continue;
            seg_iter iter;
            iter.init(op.total, op.G, op.P);
            while (iter.next(sg)) {
                for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                    if (static_cast<int>(it % kDWG) != wg) continue;
                    const int nsl = min(SPS, 4 * sg.g1 - sl);
                    const int s = it % CR, as = it % kAS;
                    MBW(&full_c[s], (it / CR) & 1, 1);
                    MBW(&aempty[as], ((it / kAS) & 1) ^ 1, 2);
                    tc_fence_after();
                    dq_stage<BITS, SYM, SPS>(codes0 + s * C::kCS, r, nsl, tmem_lane + kA0 + as * kACols,
                                             &empty_c[s], lane);
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&afull[as]);
                }
            }
            if (warp == 4 && lane == 0) dtrace(a, oi, 2);
        }
    } else if (warp == 2) {
        // ===================== publisher (release latency off the epilogue) ====
        // A gpu-scope release (publishing a tile) or the acq_rel ticket of a
        // split tile waits ~2 us for the stores before it to be acknowledged
        // while the weight stream loads L2. This warp absorbs those waits:
        // the epilogue hands each finished segment over through a named
        // barrier (bar.arrive there / bar.sync here orders its stores before
        // our release) and goes on. Split tiles: we take the ticket and post
        // the result; the epilogue reduces the tiles it won at the end of the
        // op (128 threads) and hands them back for publishing.
        uint32_t ht = 0, nres = 0;
        for (int oi = 0; oi < a.nops; ++oi) {
            const dstage_op& op = a.ops[oi];
            if (op.kind != 0) continue;
            unsigned* counters = a.counters[op.pbuf];
            unsigned* oflags = op.out_flags;
            int won0 = -1, won1 = -1;
            seg_iter iter;
            iter.init(op.total, op.G, op.P);
            while (iter.next(sg)) {
                const int hb = ht % kHB;
                asm volatile("bar.sync %0, 160;" ::"r"(kHB0 + hb) : "memory");
                if (lane == 0) mbar_arrive(&hfree[hb]);
                ++ht;
                if (sg.nseg == 1) {
                    if (lane == 0) {
                        fence_proxy_async_global();
                        if (oflags) st_release(oflags + sg.tile, epoch1);
                        red_release64(done, 1ull);
                    }
                } else {
                    if (lane == 0) {
                        const unsigned t = atom_add_acq_rel(&counters[sg.tile], 1u);
                        const bool last = t == static_cast<unsigned>(sg.nseg - 1);
                        if (last) counters[sg.tile] = 0u;  // nobody else touches it this op
                        tres[nres % 8] = last ? 1u : 0u;
                        __threadfence_block();
                        *tcount = nres + 1;
                    }
                    const bool last = __shfl_sync(0xffffffffu, lane == 0 ? tres[nres % 8] : 0u, 0) != 0u;
                    ++nres;
                    if (last) {
                        if (won0 < 0) won0 = sg.tile; else won1 = sg.tile;
                    }
                }
            }
            // tiles this CTA reduces: publish once the epilogue stored them
            for (int j = 0; j < 2; ++j) {
                const int tile = j == 0 ? won0 : won1;
                if (tile < 0) continue;
                const int hb = ht % kHB;
                asm volatile("bar.sync %0, 160;" ::"r"(kHB0 + hb) : "memory");
                if (lane == 0) {
                    mbar_arrive(&hfree[hb]);
                    fence_proxy_async_global();
                    if (oflags) st_release(oflags + tile, epoch1);
                    red_release64(done, 1ull);
                }
                ++ht;
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ===================== epilogue + LayerNorm =====================
        const int lq = warp & 3;
        const int r = lq * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(lq * 32) << 16;
        const int tid = threadIdx.x & 127;
        uint32_t ut = 0, ht = 0, nres = 0;
        auto handoff = [&]() {
            const int hb = ht % kHB;
            MBW(&hfree[hb], ((ht / kHB) & 1) ^ 1, 9);
            asm volatile("bar.arrive %0, 160;" ::"r"(kHB0 + hb) : "memory");
            ++ht;
        };
        for (int oi = 0; oi < a.nops; ++oi) {
            const dstage_op& op = a.ops[oi];
            if (op.kind == 1) {
                if (static_cast<int>(blockIdx.x) < a.m) {
                    if (tid == 0) wait_done(done, base + op.wait);
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (op.h <= 6144)
                        ln_row<true>(op, blockIdx.x, red);
                    else
                        ln_row<false>(op, blockIdx.x, red);
                    publish(done, nullptr, epoch1);
                    if (tid == 0) dtrace(a, oi, 1);
                }
                continue;
            }
            float* partial = a.partial[op.pbuf];
            int split_tile[2] = {-1, -1}, split_nseg[2] = {0, 0}, nsplit = 0;
            seg_iter iter;
            iter.init(op.total, op.G, op.P);
            while (iter.next(sg)) {
                const int nt = sg.tile;
                const int acc = ut % kNACC;
                MBW(&tfull[acc], (ut / kNACC) & 1, 8);
                tc_fence_after();
                float4* part = sg.nseg > 1
                                   ? reinterpret_cast<float4*>(partial) +
                                         (static_cast<size_t>(sg.tile) * op.maxseg + sg.idx) * (kBN / 4) * 128 + r
                                   : nullptr;
#pragma unroll 1
                for (int c0 = 0; c0 < kBN; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld16(tmem + lane_addr + acc * kBN + c0, v);
                    tmem_ld_wait();
                    if (part) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            __stcg(part + ((c0 + i) / 4) * 128,
                                   make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                               __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3])));
                    } else {
                        float f[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
                        store16(op, a.m, stg, r, f, c0, nt * 128);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                handoff();
                if (sg.nseg > 1 && nsplit < 2) {
                    split_tile[nsplit] = sg.tile;
                    split_nseg[nsplit] = sg.nseg;
                    ++nsplit;
                }
                ++ut;
            }
            // split tiles: reduce the ones whose ticket we won (ordered sum of
            // the segments' partials, K3's reducer arithmetic)
            for (int j = 0; j < nsplit; ++j) {
                if (tid == 0) {
                    while (*tcount <= nres) {
                    }
                    __threadfence_block();
                    *bcast = tres[nres % 8];
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const bool won = *bcast != 0u;
                asm volatile("bar.sync 1, 128;" ::: "memory");
                ++nres;
                if (!won) continue;
                const int tile = split_tile[j], nseg = split_nseg[j];
                constexpr int kRB = 2;
                const float4* basep = reinterpret_cast<const float4*>(partial) +
                                      static_cast<size_t>(tile) * op.maxseg * (kBN / 4) * 128 + r;
#pragma unroll 1
                for (int c = 0; c < kBN / 16; ++c) {
                    const int c0 = 16 * c;
                    float f[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = 0.f;
#pragma unroll 1
                    for (int jb = 0; jb < nseg; jb += kRB) {
                        float4 q4[kRB][4];
#pragma unroll
                        for (int jj = 0; jj < kRB; ++jj) {
                            if (jb + jj < nseg) {
                                const float4* src = basep + (static_cast<size_t>(jb + jj) * (kBN / 4) + c0 / 4) * 128;
#pragma unroll
                                for (int i = 0; i < 4; ++i) q4[jj][i] = __ldcg(src + i * 128);
                            }
                        }
#pragma unroll
                        for (int jj = 0; jj < kRB; ++jj) {
                            if (jb + jj < nseg) {
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    f[4 * i] += q4[jj][i].x;
                                    f[4 * i + 1] += q4[jj][i].y;
                                    f[4 * i + 2] += q4[jj][i].z;
                                    f[4 * i + 3] += q4[jj][i].w;
                                }
                            }
                        }
                    }
                    store16(op, a.m, stg, r, f, c0, tile * 128);
                }
                handoff();
            }
            if (tid == 0) dtrace(a, oi, 1);
        }
    }

    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(epoch_exit + 1, 1u) == gridDim.x - 1) {
            epoch_exit[1] = 0u;
            __threadfence();
            st_release(epoch_exit, epoch1);
        }
    }
}

int g_dstage_sms = 0;
unsigned long long* g_dstage_trace = nullptr;

}  // namespace

/* debug: copy the HP_DSTAGE_TRACE buffer ([148][256][4] u64) */
extern "C" int hp_debug_dstage_trace(unsigned long long* host, int n);

int dstage_grid() {
    if (g_dstage_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_dstage_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_dstage_sms <= 0) g_dstage_sms = 148;
    }
    const int budget = g_sm_budget;
    return (budget > 0 && budget < g_dstage_sms) ? budget : g_dstage_sms;
}

template <int BITS, bool SYM>
cudaError_t launch_dstage_t(const dstage_args& a, int grid, cudaStream_t st) {
    static bool attr_done = false;
    constexpr int smem = dcfg<SYM>::kSmem;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(dstage_kernel<BITS, SYM>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, dstage_kernel<BITS, SYM>, a);
}

// One launch = one run of consecutive layers with the same bit width.
cudaError_t launch_dstage(const dstage_op* ops, int nops, int m, int bits, bool sym,
                          unsigned long long* sync, unsigned long long units, unsigned* const counters[2],
                          float* const partial[2], int grid, cudaStream_t st) {
#ifdef HP_DSTAGE_TRACE
    if (!g_dstage_trace) {
        cudaMalloc(&g_dstage_trace, sizeof(unsigned long long) * 148 * 256 * 8);
        cudaMemset(g_dstage_trace, 0, sizeof(unsigned long long) * 148 * 256 * 8);
    }
#endif
    dstage_args a{ops, nops, m, sync, units, {counters[0], counters[1]}, {partial[0], partial[1]}, g_dstage_trace};
    switch (bits * 2 + (sym ? 1 : 0)) {
        case 7: return launch_dstage_t<3, true>(a, grid, st);
        case 6: return launch_dstage_t<3, false>(a, grid, st);
        case 9: return launch_dstage_t<4, true>(a, grid, st);
        case 8: return launch_dstage_t<4, false>(a, grid, st);
        case 17: return launch_dstage_t<8, true>(a, grid, st);
        case 16: return launch_dstage_t<8, false>(a, grid, st);
        case 33: return launch_dstage_t<16, true>(a, grid, st);
        case 32: return launch_dstage_t<16, false>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace hp

extern "C" int hp_debug_dstage_trace(unsigned long long* host, int n) {
    if (!hp::g_dstage_trace) return 0;
    cudaDeviceSynchronize();
    cudaMemcpy(host, hp::g_dstage_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
    return n;
}
