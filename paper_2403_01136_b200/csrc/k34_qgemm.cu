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
// Decode (K3, M = xi <= 32): BN = 16/32 and stream-K (each CTA streams an
// equal contiguous range of weight groups; HBM-bound). Prefill (K4, M = eta*s): BN = 128/256, no split;
// tensor-bound.
#include <cuda.h>
#include <cuda_bf16.h>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "layout.cuh"
#include "sm100.cuh"

// HP_PRE_BN192: prefill token tiles of 192 with a double-buffered
// accumulator (2 x 192 of the 512 TMEM columns, 4 A stages in the rest), so
// a tile's epilogue overlaps the next tile's MMAs; 2048-token ops then split
// into 11 token tiles (out / fc2: 440 tiles = 2.97 waves, no stream-K).
#ifndef HP_PRE_BN192
#define HP_PRE_BN192 0
#endif
#ifndef HP_DEC_SPS
#define HP_DEC_SPS 8
#endif
#ifndef HP_DWG
#define HP_DWG 3
#endif
// Group-scaled decode (sym 3/4/8-bit): dequant warps write the exact integer
// codes, the MMA sums every 128-k group into its own TMEM accumulator and the
// epilogue applies the fp32 group scale to the group sum.
#ifndef HP_DEC_GS
#define HP_DEC_GS 0
#endif
// Decode smem: a 6-deep activation ring inside a 218 KB budget (with the
// MMA spin: 40-layer decode step 3013 -> 2959 us).
#ifndef HP_DEC_BR
#define HP_DEC_BR 6
#endif
#ifndef HP_DEC_BUDGET_KB
#define HP_DEC_BUDGET_KB 218
#endif
#ifndef HP_CR_CAP
#define HP_CR_CAP 12
#endif
#ifndef HP_DEC_CORES
#define HP_DEC_CORES 0
#endif
// stream-K straggler reduction of the CTA's final segment via bulk copies
#ifndef HP_SK_FAST_FIN
#define HP_SK_FAST_FIN 1  // final-segment reduction without the publish (round 2)
#endif
#ifndef HP_SK_TMA_RED
#define HP_SK_TMA_RED 1  // 40-layer OPT-13B plan decode step 3267 -> 3152 us (round 2)
#endif
// dequant: slices converted before waiting for the TMEM A slot (0 = wait first)
#ifndef HP_DQ_EARLY
#define HP_DQ_EARLY 0
#endif

// The MMA issuer is one latency-critical warp: it spins on its barriers
// instead of suspending (40-layer decode step -0.7%; HP_MMA_SPIN=0 restores
// the suspend hint).
#ifndef HP_MMA_SPIN
#define HP_MMA_SPIN 1
#endif
#if HP_MMA_SPIN
#define MMA_WAIT mbar_wait_warp_spin
#else
#define MMA_WAIT mbar_wait_warp
#endif
#ifdef HP_PROD_SPIN
#define PROD_WAIT mbar_wait_warp_spin
#else
#define PROD_WAIT mbar_wait_warp
#endif
#ifdef HP_DQ_SPIN
#define DQ_WAIT mbar_wait_warp_spin
#else
#define DQ_WAIT mbar_wait
#endif

namespace hp {

// Persistent-grid cap: leave SMs to concurrent NCCL kernels (pipeline runs).
int g_sm_budget = 0;
// Programmatic dependent launch for qgemm / glue kernels (hp_set_pdl).
int g_pdl = 1;

struct qgemm_args {
    const uint8_t* packed;
    const float* scale;
    const float* zero;
    int n_out, k_in, G, NT;
    int m, MT;
    int stream_k;       // 1: contiguous group ranges per CTA (decode), 0: whole tiles
    int dp;             // stream-K: tiles [0, dp) run whole (data-parallel waves) first
    int64_t total;      // (MT*NT - dp)*G group-steps (stream-K region)
    int maxseg;         // partial slots per tile (stream-K)
    __nv_bfloat16* y;
    int64_t ldy;
    const __nv_bfloat16* res;
    int64_t ldr;
    int epi;
    float* partial;     // [tiles][maxseg][128][BN] fp32
    unsigned* counters; // [tiles]
    unsigned long long* trace;  // optional per-role clock trace of CTA 0
};

// per-CTA timestamp slot k (HP_QGEMM_TRACE builds): final-segment epilogue events
#ifdef HP_QGEMM_TRACE
#define HP_TRACE_CTA(a, k, v) do { if ((a).trace) (a).trace[6 * 64 * 4 + (5 + (k)) * 1024 + blockIdx.x] = (v); } while (0)
#else
#define HP_TRACE_CTA(a, k, v) do { } while (0)
#endif
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Debug trace (HP_QGEMM_TRACE): CTA 0 records %globaltimer at pipeline
// events: slot = role*kTraceIters*4 + iter*4 + event.
constexpr int kTraceIters = 64;
__device__ int g_trace_cta = 0;
__device__ __forceinline__ void trace_ev(const qgemm_args& a, int role, uint32_t it, int ev) {
#ifndef HP_QGEMM_TRACE
    return;  // production build: tracing compiled out
#endif
    if (role < 6 && a.trace && blockIdx.x == g_trace_cta && it < kTraceIters) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[(role * kTraceIters + it) * 4 + ev] = t;
    }
}

// Tiles are numbered weight-major (tile = nt*MT + mt): the CTAs running at
// the same time share weight row-tiles across token tiles, so a prefill
// op streams each weight tile from HBM about once (the token tiles of x stay
// L2-resident) instead of once per token tile. Decode has MT = 1.
__device__ __forceinline__ int tile_mt(const qgemm_args& a, int tile) { return tile % a.MT; }
__device__ __forceinline__ int tile_nt(const qgemm_args& a, int tile) { return tile / a.MT; }

// A work segment: groups [g0, g1) of output tile `tile` (= nt*MT + mt).
// Stream-K: CTA c owns group-steps [c*total/P, (c+1)*total/P) of the
// tile-major order; a tile split over several CTAs is reduced by the last
// one to finish, summing the partials in segment order (deterministic).
struct seg_t {
    int tile, g0, g1, idx, nseg;
};

// 32-bit stream-K arithmetic: plan_qgemm keeps total * grid < 2^32 (an int64
// division is ~70 instructions; every role evaluates these per segment, and
// the epilogue's and MMA warp's segment switches sit on the kernel tail)
__device__ __forceinline__ int64_t sk_lo(int64_t c, int64_t total, int64_t P) {
    return static_cast<uint32_t>(c) * static_cast<uint32_t>(total) / static_cast<uint32_t>(P);
}
// CTA owning group-step w
__device__ __forceinline__ int sk_owner(int64_t w, int64_t total, int64_t P) {
    const uint32_t t = static_cast<uint32_t>(total), p = static_cast<uint32_t>(P);
    uint32_t c = static_cast<uint32_t>(w) * p / t;
    while (c + 1 < p && (c + 1) * t / p <= static_cast<uint32_t>(w)) ++c;
    while (c > 0 && c * t / p > static_cast<uint32_t>(w)) --c;
    return static_cast<int>(c);
}

// Stream-K visit order: the CTA's partial segments (the tail of the tile its
// range starts in, the head of the tile it ends in) SHORTEST FIRST, then its
// full tiles. A split tile is then reduced by the CTA that computes its long
// part, at the END of that work, with the fast final reduction (its short
// part was computed first by the neighbour); and no CTA reduces a tile while
// its own final, short segment is still running -- the measured cause of
// the slowest CTAs' 6 us tails under the previous order (last range segment
// first, tools/trace_qgemm.py). Reduction order (by segment index) is
// unchanged, so results are bit-identical.
struct seg_iter_sf {
    // unit mode
    int u;
    // stream-K mode: up to two partial segments [ps, pe) in visit order, then
    // the full tiles [w, fe) (group-step indices; < 2^31, see sk_lo)
    int ps0, pe0, ps1, pe1, w, fe;
    int np, k;
    bool last_ret;  // the segment last returned by next() was the final one
    __device__ __forceinline__ void init(const qgemm_args& a) {
        u = blockIdx.x;
        np = k = 0;
        last_ret = false;
        const int G = a.G;
        const int wlo = static_cast<int>(sk_lo(blockIdx.x, a.total, gridDim.x));
        const int w1 = static_cast<int>(sk_lo(blockIdx.x + 1, a.total, gridDim.x));
        w = fe = 0;
        ps0 = pe0 = ps1 = pe1 = 0;
        if (w1 <= wlo) return;
        const int fend = min(w1, (wlo / G + 1) * G);    // end of the first range piece
        const int lbeg = max(wlo, ((w1 - 1) / G) * G);  // start of the last range piece
        auto full = [G](int s0, int e0) { return s0 % G == 0 && e0 - s0 == G; };
        if (fend >= w1) {  // the range lies in one tile
            if (full(wlo, w1)) {
                w = wlo;
                fe = w1;
            } else {
                ps0 = wlo;
                pe0 = w1;
                np = 1;
            }
            return;
        }
        int fs = fend, fe2 = lbeg;
        if (full(wlo, fend)) {
            fs = wlo;
        } else {
            ps0 = wlo;
            pe0 = fend;
            np = 1;
        }
        if (full(lbeg, w1)) {
            fe2 = w1;
        } else if (np == 0) {
            ps0 = lbeg;
            pe0 = w1;
            np = 1;
        } else {
            ps1 = lbeg;
            pe1 = w1;
            np = 2;
            if (pe1 - ps1 < pe0 - ps0) {  // shorter first
                const int t0 = ps0, t1 = pe0;
                ps0 = ps1;
                pe0 = pe1;
                ps1 = t0;
                pe1 = t1;
            }
        }
        w = fs;
        fe = fe2;
    }
    __device__ __forceinline__ bool at_end() const { return last_ret; }
    __device__ __forceinline__ bool next(const qgemm_args& a, seg_t& s) {
        if (!a.stream_k || u < a.dp) {
            const int lim = a.stream_k ? a.dp : a.MT * a.NT;
            if (u < lim) {
                s = {u, 0, a.G, 0, 1};
                u += gridDim.x;
                return true;
            }
            if (!a.stream_k) return false;
            u = lim;  // data-parallel waves done -> the stream-K region
        }
        int s0, e0;
        if (k < np) {
            s0 = k == 0 ? ps0 : ps1;
            e0 = k == 0 ? pe0 : pe1;
            ++k;
        } else if (w < fe) {
            s0 = w;
            e0 = w + a.G;
            w = e0;
        } else {
            return false;
        }
        last_ret = k >= np && w >= fe;
        const int tile = s0 / a.G;  // within the stream-K region
        const int g0 = s0 - tile * a.G;
        const int64_t tend = static_cast<int64_t>(tile + 1) * a.G;
        const int first = sk_owner(static_cast<int64_t>(tile) * a.G, a.total, gridDim.x);
        const int last = sk_owner(tend - 1, a.total, gridDim.x);
        s = {a.dp + tile, g0, g0 + (e0 - s0), static_cast<int>(blockIdx.x) - first, last - first + 1};
        return true;
    }
};

// Prefill order: the CTA's LAST range segment first (the head of the tile
// the next CTA finishes early), then the rest in order -- both halves of
// every split tile complete early, and the CTAs sharing a weight row-tile
// sweep k close together (fc2 at 2048 tokens: DRAM 2.4x its algorithmic
// bytes; 3.4x under the decode order, same time).
struct seg_iter_lf {
    // unit mode
    int u;
    // stream-K mode
    int64_t w, w1, wlo, wlast;
    int phase;  // 0: last segment, 1: the others in order
    __device__ __forceinline__ void init(const qgemm_args& a) {
        u = blockIdx.x;
        wlo = sk_lo(blockIdx.x, a.total, gridDim.x);
        w1 = sk_lo(blockIdx.x + 1, a.total, gridDim.x);
        // start of the last segment = max(wlo, start of the tile holding w1-1)
        const int64_t tstart = w1 > 0 ? ((w1 - 1) / a.G) * a.G : 0;
        wlast = tstart > wlo ? tstart : wlo;
        w = wlast;
        phase = 0;
    }
    // true once the segment last returned by next() was this CTA's final one
    // (stream-K mode)
    __device__ __forceinline__ bool at_end() const {
        return phase == 0 ? (w >= w1 && wlo >= wlast) : w >= wlast;
    }
    __device__ __forceinline__ bool next(const qgemm_args& a, seg_t& s) {
        if (!a.stream_k || u < a.dp) {
            const int lim = a.stream_k ? a.dp : a.MT * a.NT;
            if (u < lim) {
                s = {u, 0, a.G, 0, 1};
                u += gridDim.x;
                return true;
            }
            if (!a.stream_k) return false;
            u = lim;  // data-parallel waves done -> the stream-K region
        }
        if (phase == 0 && w >= w1) {  // last segment done -> the rest
            phase = 1;
            w = wlo;
        }
        const int64_t lim = phase == 0 ? w1 : wlast;
        if (w >= lim) return false;
        const int tile = static_cast<int>(w / a.G);  // within the stream-K region
        const int g0 = static_cast<int>(w % a.G);
        const int64_t tend = static_cast<int64_t>(tile + 1) * a.G;
        const int64_t wend = lim < tend ? lim : tend;
        const int first = sk_owner(static_cast<int64_t>(tile) * a.G, a.total, gridDim.x);
        const int last = sk_owner(tend - 1, a.total, gridDim.x);
        s = {a.dp + tile, g0, g0 + static_cast<int>(wend - w), static_cast<int>(blockIdx.x) - first,
             last - first + 1};
        w = wend;
        return true;
    }
};


// A pipeline stage covers SPS 32-k "slices" (SPS = 8: two 128-k groups,
// decode; SPS = 2: half a group, prefill — keeps the [BN x K] activation
// tile per stage small so the pipeline is deep).
template <int BITS, int BN, int SPS>
struct qgemm_cfg {
    // Dequant warpgroups: decode 3/4/8-bit use 3 warpgroups taking whole
    // stages round-robin (amortises the per-stage barrier work over 8
    // slices per warp); prefill and 16-bit decode use 2 warpgroups splitting
    // every stage. One CTA per SM (all 512 TMEM columns).
    // HP_DEC_CORES: decode CTAs sized to half an SM (256 TMEM columns,
    // <= 110 KB smem, 4 warpgroups at <= 64 registers) so TWO co-reside:
    // the grid is 2 x SMs, and a CTA of the next op (PDL) takes the slot of
    // a finished one while the rest of the current op drains.
    static constexpr bool kCoRes = BN <= 64 && HP_DEC_CORES;
    static constexpr int kMinBlocks = kCoRes ? 2 : 1;
    static constexpr int kTmemCols = kCoRes ? 256 : 512;
    static constexpr bool kRR = BN <= 64 && BITS != 16;
    static constexpr int DWG = kRR ? (kCoRes ? 2 : HP_DWG) : 2;
    static constexpr int kThreads = 128 * (2 + DWG);
    static constexpr int kEpiWarp0 = 4 + 4 * DWG;
    static constexpr int NG = SPS >= 4 ? SPS / 4 : 1;            // groups touched per stage
    static constexpr int kB = BN * 64 * SPS;                     // SPS/2 64-k swizzled sub-tiles
    static constexpr int kCodes = SPS >= 4 ? BITS * 2048 * NG
                                           : (BITS == 3 ? 6144 : BITS * 1024);  // half group (3-bit: whole group)
    static constexpr int kScale = BITS == 16 ? 0 : 1024 * NG;    // NG scale rows + NG zero rows
    static constexpr int kCS = kCodes + kScale;                  // weight-ring slot
    // Two rings: the weight-code ring (HBM latency, released as soon as the
    // dequant warps hold the codes in registers) is deep; the activation
    // ring (L2-resident x, released by the MMA) is shallow.
#ifndef HP_PRE_BUDGET_KB
#define HP_PRE_BUDGET_KB 186
#endif
    static constexpr int kBudget = (kCoRes ? 100 : (BN <= 64 ? HP_DEC_BUDGET_KB : HP_PRE_BUDGET_KB)) * 1024;
    static constexpr int BR = kCoRes ? 4 : (BN <= 64 ? HP_DEC_BR : (BN <= 128 ? 6 : 4));
    static constexpr int CR_ = (kBudget - BR * kB) / kCS > HP_CR_CAP ? HP_CR_CAP : (kBudget - BR * kB) / kCS;
    // Round-robin consumers wait only on their own stages, so every ring slot
    // they consume must always belong to the same warpgroup (depth % DWG ==
    // 0); otherwise an mbarrier parity wait could alias another phase.
    static constexpr int CR = kRR ? (CR_ / DWG) * DWG : CR_;
    static constexpr int NACC = (BN <= 128 || BN == 192) ? 2 : 1;
    static constexpr bool kGSok = kRR && HP_DEC_GS;               // sym kernels only (see kernel)
    static constexpr int GCOLS = kGSok ? 2 * NG * BN : 0;          // 2 stage slots x NG group sums
    static constexpr int A0_ = NACC * BN < 64 ? (GCOLS > 64 ? GCOLS : 64)
                                               : (NACC * BN > GCOLS ? NACC * BN : GCOLS);
    static constexpr int A0 = (A0_ + 63) / 64 * 64;
    static constexpr int ACOLS = 16 * SPS;                       // TMEM columns per A stage
    static constexpr int AS_ = (kTmemCols - A0) / ACOLS > 8 ? 8 : (kTmemCols - A0) / ACOLS;
    static constexpr int AS = kRR ? (AS_ / DWG) * DWG : AS_;
    static constexpr int kCodesOff = BR * kB;                    // B ring first (1024-aligned)
    static constexpr int kStgOff = kCodesOff + CR * kCS;         // epilogue staging [16][kStgLd] fp32
    static constexpr int kStgLd = 132;
    static constexpr int kBarOff = kStgOff + 16 * kStgLd * 4;
    static constexpr int kSmem = kBarOff + 512 + 1024;  // + barriers + align slack
    static constexpr int kEmptyC = kRR ? 4 : 4 * DWG;            // dequant warps per stage
    static_assert(CR >= 2 && BR >= 2, "need >= 2 ring slots");
    static_assert(AS >= 2, "need >= 2 TMEM A stages");
    static_assert(!kRR || (CR % DWG == 0 && AS % DWG == 0), "round-robin ring depth");
    static_assert(SPS == 2 || SPS == 4 || SPS == 8, "SPS");
    static_assert(kSmem <= (kCoRes ? 113 : 227) * 1024, "smem");
};

// Epilogue write-out of 16 tokens x 128 rows through shared memory: each
// epilogue thread (row r) deposits its 16 fp32 accumulators transposed into
// stg[t][r]; after a named barrier the 128 threads write the tile as 16-byte
// vectors along n (coalesced), adding the residual in fp32 and rounding once
// — the same arithmetic as a per-element epilogue, so results are identical.
// Residual of this thread's store-phase slot (token t0 + tid/8, 16 features
// at n0 + (tid%8)*16), fetched early so a reducing epilogue overlaps its
// latency with the partial loads; `ok` = vector path usable.
struct res16 {
    uint4 r0, r1;
    bool ok;
};
__device__ __forceinline__ res16 prefetch_res16(const qgemm_args& a, int t0, int n0) {
    res16 o{};
    const int tid = threadIdx.x & 127;
    const int tok = t0 + (tid >> 3);
    const int n = n0 + (tid & 7) * 16;
    o.ok = false;
    if (a.res && tok < a.m && n + 16 <= a.n_out) {
        const __nv_bfloat16* res = a.res + static_cast<int64_t>(tok) * a.ldr + n;
        if ((reinterpret_cast<uintptr_t>(res) & 15) == 0) {
            o.r0 = __ldcg(reinterpret_cast<const uint4*>(res));
            o.r1 = __ldcg(reinterpret_cast<const uint4*>(res + 8));
            o.ok = true;
        }
    }
    return o;
}

__device__ __forceinline__ void stage_store16(const qgemm_args& a, float* stg, int ldst, int r,
                                              const float (&v)[16], int t0, int n0,
                                              const res16* pre = nullptr) {
#pragma unroll
    for (int i = 0; i < 16; ++i) stg[i * ldst + r] = v[i];
    asm volatile("bar.sync 2, 128;" ::: "memory");
    const int tid = threadIdx.x & 127;
    const int t = tid >> 3;
    const int seg = (tid & 7) * 16;
    const int tok = t0 + t;
    const int n = n0 + seg;
    if (tok < a.m && n < a.n_out) {
        const float* src = stg + t * ldst + seg;
        float f[16];
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
            const float4 q = *reinterpret_cast<const float4*>(src + i);
            f[i] = q.x; f[i + 1] = q.y; f[i + 2] = q.z; f[i + 3] = q.w;
        }
        if (a.epi & 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], 0.0f);
        }
        __nv_bfloat16* dst = a.y + static_cast<int64_t>(tok) * a.ldy + n;
        const __nv_bfloat16* res = a.res ? a.res + static_cast<int64_t>(tok) * a.ldr + n : nullptr;
        const bool vec = n + 16 <= a.n_out && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) &&
                         (!res || (reinterpret_cast<uintptr_t>(res) & 15) == 0);
        if (vec) {
            if (res) {
                const uint4 r0 = pre && pre->ok ? pre->r0 : *reinterpret_cast<const uint4*>(res);
                const uint4 r1 = pre && pre->ok ? pre->r1 : *reinterpret_cast<const uint4*>(res + 8);
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
                if (n + i < a.n_out) {
                    float x = f[i];
                    if (res) x += __bfloat162float(res[i]);
                    dst[i] = __float2bfloat16_rn(x);
                }
            }
        }
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
}

template <int BITS, bool SYM, int BN, int SPS>
__global__ void __launch_bounds__(qgemm_cfg<BITS, BN, SPS>::kThreads,
                                  qgemm_cfg<BITS, BN, SPS>::kMinBlocks)
    qgemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const qgemm_args a) {
    using C = qgemm_cfg<BITS, BN, SPS>;
    constexpr int AS = C::AS, NACC = C::NACC;
    constexpr bool GS = C::kGSok && SYM;  // group-scaled decode (tfull/tempty per stage slot)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    auto stage_b = [&](int s) { return smem + s * C::kB; };
    auto stage_codes = [&](int s) { return smem + C::kCodesOff + s * C::kCS; };
    auto stage_scale = [&](int s) {
        return reinterpret_cast<float*>(smem + C::kCodesOff + s * C::kCS + C::kCodes);
    };
    constexpr int kScaleRow = 128 * C::NG;  // floats: scales of the stage's groups, then zeros
    constexpr int CR = C::CR, BR = C::BR;
    float* stg = reinterpret_cast<float*>(smem + C::kStgOff);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
    uint64_t* full_c = bars;
    uint64_t* empty_c = full_c + CR;
    uint64_t* full_b = empty_c + CR;
    uint64_t* empty_b = full_b + BR;
    uint64_t* afull = empty_b + BR;
    uint64_t* aempty = afull + AS;
    uint64_t* tfull = aempty + AS;
    uint64_t* tempty = tfull + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);
    unsigned* bcast = tmem_slot + 1;
    uint64_t* redbar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // final-segment reduction
    unsigned* s_fastfin = reinterpret_cast<unsigned*>(redbar + 1);   // HP_SK_FAST_FIN flag

    // warp index broadcast from lane 0: provably warp-uniform for the
    // compiler, so role code runs on the uniform datapath (no R2UR)
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    long long clk0 = 0;
#ifdef HP_QGEMM_TRACE
    if (threadIdx.x == 0 && a.trace) {  // per-CTA entry time
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[6 * kTraceIters * 4 + 2 * blockIdx.x] = t;
        clk0 = clock64();
    }
#endif

    if (warp == 1 && lane == 0) {
        for (int i = 0; i < CR; ++i) {
            mbar_init(&full_c[i], 1);
            mbar_init(&empty_c[i], C::kEmptyC);
        }
        for (int i = 0; i < BR; ++i) {
            mbar_init(&full_b[i], 1);
            mbar_init(&empty_b[i], 1);
        }
        for (int i = 0; i < AS; ++i) {
            mbar_init(&afull[i], C::kRR ? 4 : 4 * C::DWG);
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < NACC; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(redbar, 1);
        fence_mbar_init();
    }
    if (warp == 3 && lane == 0) prefetch_tmap(&tmap_x);
    if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
    // PDL: the next kernel may launch now; everything that reads the previous
    // kernel's outputs (x, residual, split-K workspace) waits in pdl_wait().
    pdl_trigger();

    // decode: shortest partial segment first (tails end on the fast final
    // reduction); prefill: the range's last segment first (the order that
    // keeps fc2 / out-proj's activation re-reads at 2.4x instead of 3.4x)
    typename std::conditional<(BN <= 64), seg_iter_sf, seg_iter_lf>::type iter;
    iter.init(a);
    seg_t sg;

    if (warp == 0) {
        // ============ weight-code producer (whole warp, elected issue) ==========
        uint32_t it = 0;
        while (iter.next(a, sg)) {
            const int nt = tile_nt(a, sg.tile);
            for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                const int g = sl >> 2;
                const int ng = SPS >= 4 ? min(C::NG, sg.g1 - g) : 1;
                const int s = it % CR;
                trace_ev(a, 0, it, 0);
                PROD_WAIT(&empty_c[s], ((it / CR) & 1) ^ 1);
                trace_ev(a, 0, it, 1);
                const size_t t = static_cast<size_t>(nt) * a.G + g;
                const uint8_t* gsrc = a.packed + t * (BITS * 2048);
                const uint32_t cbytes = SPS >= 4 ? static_cast<uint32_t>(ng) * BITS * 2048
                                                 : static_cast<uint32_t>(C::kCodes);
                const uint32_t sbytes = BITS == 16 ? 0u : static_cast<uint32_t>(ng) * 512u * (SYM ? 1 : 2);
                mbar_arrive_expect_tx_elect(&full_c[s], cbytes + sbytes);
                if constexpr (SPS >= 4) {
                    bulk_g2s_elect(stage_codes(s), gsrc, cbytes, &full_c[s]);
                } else {
                    const int h = (sl >> 1) & 1;  // which half of the group
                    if constexpr (BITS == 3) {
                        // a slice's three words sit in all three chunks: the
                        // half-group stage carries the whole group
                        (void)h;
                        bulk_g2s_elect(stage_codes(s), gsrc, 6144, &full_c[s]);
                    } else {
                        bulk_g2s_elect(stage_codes(s), gsrc + h * (BITS * 1024), BITS * 1024, &full_c[s]);
                    }
                }
                if constexpr (BITS != 16) {
                    bulk_g2s_elect(stage_scale(s), a.scale + t * 128, ng * 512u, &full_c[s]);
                    if constexpr (!SYM)
                        bulk_g2s_elect(stage_scale(s) + kScaleRow, a.zero + t * 128, ng * 512u, &full_c[s]);
                }
                trace_ev(a, 0, it, 2);
            }
        }
    } else if (warp == 3) {
        // ============ activation producer (whole warp, elected issue) ===========
        pdl_wait();  // x is the previous kernel's output
        uint32_t it = 0;
        while (iter.next(a, sg)) {
            const int mt = tile_mt(a, sg.tile);
            for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                const int s = it % BR;
                PROD_WAIT(&empty_b[s], ((it / BR) & 1) ^ 1);
#ifdef HP_EXP_NOACT  // timing experiment: no activation loads (stale smem)
                mbar_arrive_expect_tx_elect(&full_b[s], 0u);
#else
                mbar_arrive_expect_tx_elect(&full_b[s], static_cast<uint32_t>(C::kB));
                tma_load_3d_elect(stage_b(s), &tmap_x, 0, mt * BN, sl >> 1, &full_b[s]);
#endif
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (whole warp, elected issue) ==========
        constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
        uint32_t it = 0, ut = 0;
        if constexpr (GS) {
            // one accumulator per 128-k group, in stage slot it&1
            while (iter.next(a, sg)) {
                for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                    const int nsl = min(SPS, 4 * sg.g1 - sl);
                    const int s = it % BR, as = it % AS, slot = it & 1;
                    MMA_WAIT(&tempty[slot], ((it >> 1) & 1) ^ 1);
                    MMA_WAIT(&full_b[s], (it / BR) & 1);
                    MMA_WAIT(&afull[as], (it / AS) & 1);
                    tc_fence_after();
                    const uint32_t bbase = smem_u32(stage_b(s));
                    const uint32_t abase = tmem + C::A0 + as * C::ACOLS;
                    const uint64_t bdesc0 = umma_desc_sw128(bbase);
#pragma unroll
                    for (int q = 0; q < SPS / 2; ++q) {
                        if (2 * q < nsl)
                            mma_ts_x4_elect(tmem + (slot * C::NG + (q >> 1)) * BN, abase + q * 32,
                                            bdesc0 + q * (BN * 8), idesc, (q & 1) ? 1u : 0u);
                    }
                    tc_commit_elect(&empty_b[s]);
                    tc_commit_elect(&aempty[as]);
                    tc_commit_elect(&tfull[slot]);
                }
            }
        }
        while (!GS && iter.next(a, sg)) {
            const int acc = ut % NACC;
            mbar_wait_warp(&tempty[acc], ((ut / NACC) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem + acc * BN;
            for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                const int nsl = min(SPS, 4 * sg.g1 - sl);
                const int s = it % BR, as = it % AS;
                trace_ev(a, 1, it, 0);
                MMA_WAIT(&full_b[s], (it / BR) & 1);
                trace_ev(a, 1, it, 1);
                MMA_WAIT(&afull[as], (it / AS) & 1);
                trace_ev(a, 1, it, 2);
                tc_fence_after();
                const uint32_t bbase = smem_u32(stage_b(s));
                const uint32_t abase = tmem + C::A0 + as * C::ACOLS;
                const uint64_t bdesc0 = umma_desc_sw128(bbase);
#pragma unroll
                for (int q = 0; q < SPS / 2; ++q) {  // 64-k sub-tiles (4 MMAs each)
#ifndef HP_EXP_NOMMA  // timing experiment: no MMAs (commits only)
                    if (2 * q < nsl)
                        mma_ts_x4_elect(d_tmem, abase + q * 32, bdesc0 + q * (BN * 8), idesc,
                                        (sl > 4 * sg.g0 || q > 0) ? 1u : 0u);
#endif
                }
                tc_commit_elect(&empty_b[s]);
                tc_commit_elect(&aempty[as]);
                trace_ev(a, 1, it, 3);
            }
            tc_commit_elect(&tfull[acc]);
            ++ut;
        }
#ifdef HP_QGEMM_TRACE
        if (lane == 0 && a.trace) {  // per-CTA: last MMA issued
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[6 * kTraceIters * 4 + 4096 + blockIdx.x] = t;
        }
#endif
    } else if (warp >= 4 && warp < C::kEpiWarp0) {
        // ===================== dequant =====================
        const int q = warp - 4;
        const int lq = warp & 3;  // TMEM lane quarter of this warp
        const int wg = q >> 2;    // dequant warpgroup
        // split mode: this warpgroup's local slices [wg*SPS/2, (wg+1)*SPS/2) of
        // every stage; round-robin mode: all SPS slices of every DWG-th stage
        const int kh = C::kRR ? 0 : wg;
        const int r = lq * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(lq * 32) << 16;
        constexpr int kSl = C::kRR ? SPS : SPS / 2;  // slices per warp per stage
        uint32_t it = 0;
        while (iter.next(a, sg)) {
            for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++it) {
                if (C::kRR && static_cast<int>(it % C::DWG) != wg) continue;
                const int nsl = min(SPS, 4 * sg.g1 - sl);
                const int s = it % CR, as = it % AS;
                const int trole = (lane == 0 && warp == 4) ? 2 : -1;
                if (trole >= 0) trace_ev(a, trole, it, 0);
                DQ_WAIT(&full_c[s], (it / CR) & 1);
                if (trole >= 0) trace_ev(a, trole, it, 1);
#if !HP_DQ_EARLY
                DQ_WAIT(&aempty[as], ((it / AS) & 1) ^ 1);
                if (trole >= 0) trace_ev(a, trole, it, 2);
                tc_fence_after();
#endif
                const int x0 = kh * kSl;  // first local slice of this warp
                const int gi = x0 >> 2;
                const uint32_t cbase = smem_u32(stage_codes(s)) + r * 16;
                // phase 1: this warp's codes and scales into registers ...
                constexpr int kG = (kSl + 3) / 4;  // groups touched by the warp's slices
                float sf[kG], zf[kG];
                slice_words<BITS> wv[kSl];
#pragma unroll
                for (int j = 0; j < kG; ++j) {
                    sf[j] = 0.f;
                    zf[j] = 0.f;
                    if constexpr (BITS != 16) {
                        if (!GS && 4 * j + x0 < nsl) {
                            const uint32_t saddr = smem_u32(stage_scale(s)) + ((gi + j) * 128 + r) * 4;
                            sf[j] = ldsf(saddr);
                            if constexpr (!SYM) zf[j] = ldsf(saddr + kScaleRow * 4);
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < kSl; ++h) {
                    const int x = x0 + h;  // local slice in the stage
                    if (x >= nsl) continue;
                    if constexpr (SPS >= 4) {
                        load_slice<BITS>(cbase + (x >> 2) * (BITS * 2048), x & 3, wv[h]);
                    } else if constexpr (BITS == 3) {
                        // half-group stage holding the whole group
                        load_slice<BITS>(cbase, (sl & 3) + x, wv[h]);
                    } else {
                        load_slice<BITS>(cbase, x, wv[h]);
                    }
                }
                // ... then hand the weight slot back to the producer at once
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_c[s]);
                if (trole >= 0) trace_ev(a, 4, it, 0);
#if HP_DQ_EARLY
                // The TMEM A slot frees only when the MMA of this warpgroup's
                // previous stage completes: load the codes and convert the
                // first slice(s) before waiting for it, off the MMA's
                // critical path.
                constexpr int kPre = HP_DQ_EARLY;
                uint32_t vpre[kPre][16];
#pragma unroll
                for (int h = 0; h < kPre; ++h)
                    if (x0 + h < nsl)
                        convert_slice<BITS, SYM, GS>(wv[h], sf[0], zf[0], scale_arg<SYM>(sf[0]),
                                                     zero_arg<SYM>(sf[0], zf[0]), vpre[h]);
                DQ_WAIT(&aempty[as], ((it / AS) & 1) ^ 1);
                if (trole >= 0) trace_ev(a, trole, it, 2);
                tc_fence_after();
#pragma unroll
                for (int h = 0; h < kPre; ++h)
                    if (x0 + h < nsl) tmem_st16(tmem + lane_addr + C::A0 + as * C::ACOLS + (x0 + h) * 16, vpre[h]);
#else
                constexpr int kPre = 0;
#endif
                // phase 2: convert + store into the TMEM A stage
#pragma unroll
                for (int h = kPre; h < kSl; ++h) {
                    if (x0 + h < nsl) {
                        const int j = h >> 2;
                        uint32_t v[16];
                        convert_slice<BITS, SYM, GS>(wv[h], sf[j], zf[j], scale_arg<SYM>(sf[j]),
                                                     zero_arg<SYM>(sf[j], zf[j]), v);
                        tmem_st16(tmem + lane_addr + C::A0 + as * C::ACOLS + (x0 + h) * 16, v);
                    }
                }
                if (trole >= 0) trace_ev(a, 4, it, 1);
                tmem_st_wait();
                if (trole >= 0) trace_ev(a, 4, it, 2);
#ifndef HP_EXP_NOFENCE  // timing experiment only
                tc_fence_before();
#endif
                __syncwarp();
                if (trole >= 0) trace_ev(a, 4, it, 3);
                if (lane == 0) mbar_arrive(&afull[as]);
                if (trole >= 0) trace_ev(a, trole, it, 3);
            }
        }
    } else if (warp >= C::kEpiWarp0) {
        // ===================== epilogue =====================
        pdl_wait();  // y / residual / workspace are shared with the previous kernel
        const int lq = warp & 3;
        const int r = lq * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(lq * 32) << 16;
        uint32_t ut = 0, git = 0;
        while (iter.next(a, sg)) {
            [[maybe_unused]] bool tr_final = false;  // HP_QGEMM_TRACE: this CTA's final segment
            // fastfin: see HP_SK_FAST_FIN below. Kept in SMEM and re-read at each
            // use (a register live across the segment pushed the kernel past
            // its 96-register cap: 140 B of spills in every role)
            if (warp == C::kEpiWarp0 && lane == 0) *s_fastfin = 0u;
            auto fastfin_now = [&]() {
                unsigned v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(s_fastfin)));
                return v != 0u;
            };
            const int mt = tile_mt(a, sg.tile), nt = tile_nt(a, sg.tile);
            const int acc = ut % NACC;
            constexpr bool kSK = true;  // stream-K: decode tiles, and wave-quantised prefill ops
            if constexpr (GS) {
                // fold each stage's group sums into registers: acc += s_g * sum_g.
                // The group scales come from global memory one stage ahead
                // (their L2 latency hidden behind the current stage's folds).
                float fa[BN];
#pragma unroll
                for (int i = 0; i < BN; ++i) fa[i] = 0.f;
                auto load_sc = [&](int sl, float* sc) {
                    const int g = sl >> 2;
                    const int ng = min(C::NG, sg.g1 - g);
#pragma unroll
                    for (int j = 0; j < C::NG; ++j)
                        sc[j] = (sl < 4 * sg.g1 && j < ng)
                                    ? __ldg(a.scale + (static_cast<size_t>(nt) * a.G + g + j) * 128 + r) : 0.f;
                };
                float scn[C::NG];
                load_sc(4 * sg.g0, scn);
                for (int sl = 4 * sg.g0; sl < 4 * sg.g1; sl += SPS, ++git) {
                    const int g = sl >> 2;
                    const int ng = min(C::NG, sg.g1 - g);
                    float sc[C::NG];
#pragma unroll
                    for (int j = 0; j < C::NG; ++j) sc[j] = scn[j];
                    load_sc(sl + SPS, scn);
                    const int slot = git & 1;
                    mbar_wait(&tfull[slot], (git >> 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int j = 0; j < C::NG; ++j) {
                        if (j < ng) {
#pragma unroll
                            for (int c0 = 0; c0 < BN; c0 += 16) {
                                uint32_t v[16];
                                tmem_ld16(tmem + lane_addr + (slot * C::NG + j) * BN + c0, v);
                                tmem_ld_wait();
#pragma unroll
                                for (int i = 0; i < 16; ++i) fa[c0 + i] = fmaf(sc[j], __uint_as_float(v[i]), fa[c0 + i]);
                            }
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[slot]);
                }
                float4* part = sg.nseg > 1
                                   ? reinterpret_cast<float4*>(a.partial) +
                                         (static_cast<size_t>(sg.tile) * a.maxseg + sg.idx) * (BN / 4) * 128 + r
                                   : nullptr;
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 16) {
                    if (part) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            __stcg(part + ((c0 + i) / 4) * 128,
                                   make_float4(fa[c0 + i], fa[c0 + i + 1], fa[c0 + i + 2], fa[c0 + i + 3]));
                    } else {
                        float f[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] = fa[c0 + i];
                        stage_store16(a, stg, C::kStgLd, r, f, mt * BN + c0, nt * 128);
                    }
                }
            } else {
            trace_ev(a, warp == C::kEpiWarp0 && lane == 0 ? 3 : 99, 48 + ut, 0);
            // Fast final reduction (HP_SK_FAST_FIN): a CTA's final segment
            // usually closes a tile whose other segments their CTAs computed
            // FIRST (seg_iter order). If the tile counter already shows all of
            // them, this segment skips its partial store to global memory and
            // the gpu-scope release + ticket (~1.6 us on the kernel tail,
            // tools/trace_qgemm.py): its accumulator goes to its own slot of
            // the bulk-copy reduction buffer in SMEM and the shared summation
            // below adds all segments in order -- bit-identical.
#if HP_SK_FAST_FIN
            if (kSK && sg.nseg > 1 && BN <= 32 && sg.nseg * BN * 128 * 4 <= BR * C::kB && a.dp == 0 &&
                iter.at_end()) {
                if (warp == C::kEpiWarp0 && lane == 0) {
                    unsigned c;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(&a.counters[sg.tile]) : "memory");
                    *bcast = c;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (warp == C::kEpiWarp0 && lane == 0) *s_fastfin = *bcast == static_cast<unsigned>(sg.nseg - 1);
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
#endif
            mbar_wait(&tfull[acc], (ut / NACC) & 1);
            trace_ev(a, warp == C::kEpiWarp0 && lane == 0 ? 3 : 99, 48 + ut, 1);
            tr_final = warp == C::kEpiWarp0 && lane == 0 && iter.at_end();
            if (tr_final) HP_TRACE_CTA(a, 0, gtimer());
            tc_fence_after();
            constexpr uint32_t kSegB = BN * 128 * 4;  // one segment's fp32 partial tile
            if (warp == C::kEpiWarp0 && fastfin_now()) {  // the rings are idle: this CTA's MMAs are all done
                const uint8_t* src = reinterpret_cast<const uint8_t*>(a.partial) +
                                     static_cast<size_t>(sg.tile) * a.maxseg * kSegB;
                asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> bulk-copy reads
                mbar_arrive_expect_tx_elect(redbar, (sg.nseg - 1) * kSegB);
                for (int j = 0; j < sg.nseg; ++j)
                    if (j != sg.idx) bulk_g2s_elect(stage_b(0) + j * kSegB, src + j * kSegB, kSegB, redbar);
            }
            // partials: [tile][seg][BN/4][128 rows] float4 -- row r is the
            // thread, so every warp access is 512 contiguous bytes (global, or
            // this CTA's own slot of the SMEM reduction buffer when fastfin)
            float4* part = (kSK && sg.nseg > 1)
                               ? (fastfin_now() ? reinterpret_cast<float4*>(stage_b(0) + sg.idx * kSegB) + r
                                          : reinterpret_cast<float4*>(a.partial) +
                                                (static_cast<size_t>(sg.tile) * a.maxseg + sg.idx) * (BN / 4) * 128 + r)
                               : nullptr;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + lane_addr + acc * BN + c0, v);
                tmem_ld_wait();
                if (kSK && part) {  // generic stores: global partials, or the SMEM slot (fastfin)
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        part[((c0 + i) / 4) * 128] = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                                                 __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                } else {
                    float f[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
                    stage_store16(a, stg, C::kStgLd, r, f, mt * BN + c0, nt * 128);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            }
            trace_ev(a, warp == C::kEpiWarp0 && lane == 0 ? 3 : 99, 48 + ut, 2);
            if (tr_final) HP_TRACE_CTA(a, 1, gtimer());

            if constexpr (kSK) if (sg.nseg > 1) {
                const int tr5 = warp == C::kEpiWarp0 && lane == 0 ? 5 : 99;
                // ticket: bar.sync orders all 128 threads' partial stores
                // before one thread's acq_rel RMW (release for ours, acquire
                // of the other segments' for the last arriver) -- the
                // CUTLASS split-K semaphore pattern; one gpu-scope
                // synchronisation instead of a fence.sc in every thread
                trace_ev(a, tr5, ut, 0);
                if (!fastfin_now()) {
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (warp == C::kEpiWarp0 && lane == 0) {
                        unsigned old;
                        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                                     : "=r"(old) : "l"(&a.counters[sg.tile]) : "memory");
                        *bcast = old;
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                }
                trace_ev(a, tr5, ut, 1);
                if (tr_final) {
                    HP_TRACE_CTA(a, 2, gtimer());
                    HP_TRACE_CTA(a, 3, static_cast<unsigned long long>(sg.nseg * 100 + (*bcast == static_cast<unsigned>(sg.nseg - 1) ? 10 : 0)));
                }
                bool tma_red = false;
#if HP_SK_TMA_RED
                // The straggler's reduction is usually the CTA's FINAL segment:
                // every MMA of the CTA has completed, so the activation ring is
                // idle. Pull all nseg partials (16 KB each at BN = 32) into it
                // with bulk copies -- one L2 round trip -- and sum from SMEM.
                tma_red = fastfin_now() || (*bcast == static_cast<unsigned>(sg.nseg - 1) && BN <= 32 &&
                                      sg.nseg * BN * 128 * 4 <= BR * C::kB && a.dp == 0 && iter.at_end());
                if (tma_red) {
                    constexpr uint32_t kSeg = BN * 128 * 4;
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.partial) +
                                         static_cast<size_t>(sg.tile) * a.maxseg * kSeg;
                    if (warp == C::kEpiWarp0 && !fastfin_now()) {
                        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> bulk-copy reads
                        mbar_arrive_expect_tx_elect(redbar, sg.nseg * kSeg);
                        for (int j = 0; j < sg.nseg; ++j)
                            bulk_g2s_elect(stage_b(0) + j * kSeg, src + j * kSeg, kSeg, redbar);
                    }
                    if (a.res) {  // the residual rows this thread adds in stage_store16: into L1 while the copies land
                        const int tid = threadIdx.x & 127;
                        const int n = nt * 128 + (tid & 7) * 16;
#pragma unroll
                        for (int c0 = 0; c0 < BN; c0 += 16) {
                            const int tok = mt * BN + c0 + (tid >> 3);
                            if (tok < a.m && n < a.n_out)
                                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.res + static_cast<int64_t>(tok) * a.ldr + n));
                        }
                    }
                    mbar_wait(redbar, 0);  // once per CTA: its final segment
                    const float4* sp = reinterpret_cast<const float4*>(stage_b(0)) + r;
#pragma unroll 1
                    for (int c0 = 0; c0 < BN; c0 += 16) {
                        float f[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] = 0.f;
#pragma unroll 1
                        for (int j = 0; j < sg.nseg; ++j) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float4 q = sp[(static_cast<size_t>(j) * (BN / 4) + c0 / 4 + i) * 128];
                                f[4 * i] += q.x;
                                f[4 * i + 1] += q.y;
                                f[4 * i + 2] += q.z;
                                f[4 * i + 3] += q.w;
                            }
                        }
                        stage_store16(a, stg, C::kStgLd, r, f, mt * BN + c0, nt * 128);
                    }
                    if (warp == C::kEpiWarp0 && lane == 0) a.counters[sg.tile] = 0u;
                }
#endif
                if (!tma_red && *bcast == static_cast<unsigned>(sg.nseg - 1)) {
                    trace_ev(a, tr5, ut, 2);
                    // ordered reduction of all segments of this tile (row r), 16
                    // tokens at a time. The partial loads of kRB segments are
                    // issued together (and the residual with them), so the
                    // reduction costs ~ceil(nseg/kRB) L2 round trips per chunk,
                    // not nseg: this CTA is the tile's straggler, on the kernel tail.
                    constexpr int kRB = 2;  // 4 spills under the 96-register cap
                    const float4* base = reinterpret_cast<const float4*>(a.partial) +
                                         static_cast<size_t>(sg.tile) * a.maxseg * (BN / 4) * 128 + r;
#pragma unroll 1
                    for (int c = 0; c < BN / 16; ++c) {
                        const int c0 = 16 * c;
#ifdef HP_RES_PREFETCH
                        const res16 pre = prefetch_res16(a, mt * BN + c0, nt * 128);
#endif
                        float f[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) f[i] = 0.f;
#ifdef HP_EXP_NORED  // timing experiment: the straggler skips the partial reads
                        const int nred = 0;
#else
                        const int nred = sg.nseg;
#endif
#pragma unroll 1
                        for (int jb = 0; jb < nred; jb += kRB) {
                            float4 q4[kRB][4];
#pragma unroll
                            for (int jj = 0; jj < kRB; ++jj) {
                                if (jb + jj < sg.nseg) {
                                    const float4* src =
                                        base + (static_cast<size_t>(jb + jj) * (BN / 4) + c0 / 4) * 128;
#pragma unroll
                                    for (int i = 0; i < 4; ++i) q4[jj][i] = __ldcg(src + i * 128);
                                }
                            }
#pragma unroll
                            for (int jj = 0; jj < kRB; ++jj) {
                                if (jb + jj < sg.nseg) {
#pragma unroll
                                    for (int i = 0; i < 4; ++i) {
                                        f[4 * i] += q4[jj][i].x;
                                        f[4 * i + 1] += q4[jj][i].y;
                                        f[4 * i + 2] += q4[jj][i].z;
                                        f[4 * i + 3] += q4[jj][i].w;
                                    }
                                }
                            }
                            if (jb == 0) trace_ev(a, tr5, 32 + ut, 2 * c);
                        }
#ifdef HP_RES_PREFETCH
                        stage_store16(a, stg, C::kStgLd, r, f, mt * BN + c0, nt * 128, &pre);
#else
                        stage_store16(a, stg, C::kStgLd, r, f, mt * BN + c0, nt * 128);
#endif
                        trace_ev(a, tr5, 32 + ut, 2 * c + 1);
                    }
                    if (warp == C::kEpiWarp0 && lane == 0) a.counters[sg.tile] = 0u;
                    trace_ev(a, tr5, ut, 3);
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
            trace_ev(a, warp == C::kEpiWarp0 && lane == 0 ? 3 : 99, 48 + ut, 3);
            ++ut;
        }
        if (warp == C::kEpiWarp0 && lane == 0) HP_TRACE_CTA(a, 4, gtimer());
    }
#ifdef HP_QGEMM_TRACE
    if (lane == 0 && (warp == 0 || warp == 3 || warp == 4))  // role loop exits: producer, act producer, dequant w4
        HP_TRACE_CTA(a, warp == 0 ? 6 : (warp == 3 ? 5 : 7), gtimer());
#endif

    __syncthreads();
#ifdef HP_QGEMM_TRACE
    if (threadIdx.x == 0 && a.trace) {  // per-CTA exit time
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[6 * kTraceIters * 4 + 2 * blockIdx.x + 1] = t;
        a.trace[6 * kTraceIters * 4 + 2048 + blockIdx.x] = static_cast<unsigned long long>(clock64() - clk0);
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[6 * kTraceIters * 4 + 3072 + blockIdx.x] = smid;
    }
#endif
    (void)clk0;
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// 32-k slices per pipeline stage: decode tiles move two groups per stage to
// amortise the per-stage barrier/issue work; prefill moves half a group so
// the [BN x 64] activation tile per stage is small and the pipeline deep.
template <int BITS, int BN>
constexpr int kSlicesPerStage = BN <= 64 ? (BITS >= 8 || HP_DEC_CORES ? 4 : HP_DEC_SPS) : 2;

int slices_per_stage(int bits, int bn) { return bn <= 64 ? (bits >= 8 || HP_DEC_CORES ? 4 : HP_DEC_SPS) : 2; }

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
    constexpr int SPS = kSlicesPerStage<BITS, BN>;
    using C = qgemm_cfg<BITS, BN, SPS>;
    // the attribute is per device: remember it per device ordinal (a racing
    // second setter only repeats an idempotent call)
    static std::atomic<bool> attr_done[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_done[dev].load(std::memory_order_acquire)) {
        cudaError_t e = cudaFuncSetAttribute(qgemm_kernel<BITS, SYM, BN, SPS>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::kSmem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr_done[dev].store(true, std::memory_order_release);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, qgemm_kernel<BITS, SYM, BN, SPS>, map, a);
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
    int stream_k, maxseg;
    int64_t total;
    int dp;  // stream-K: whole tiles [0, dp) first (data-parallel waves)
};

constexpr size_t kTicketBytes = 16384;  // stream-K tile tickets: <= 4096 tiles

qgemm_plan plan_qgemm(int64_t n_out, int64_t k_in, int64_t m, int phase) {
    qgemm_plan p{};
    const int G = static_cast<int>(ceil_div64(k_in, 128));
    const int NT = static_cast<int>(ceil_div64(n_out, 128));
    // co-resident decode CTAs (HP_DEC_CORES): two per SM
    const int sms = num_sms() * ((phase == 1 && m <= 32 && HP_DEC_CORES) ? 2 : 1);
    if (phase == 1 && m <= 32) {
        p.bn = m <= 16 ? 16 : 32;
    } else {
        p.bn = m <= 128 ? 128 : (HP_PRE_BN192 ? 192 : 256);
    }
    p.mt = static_cast<int>(ceil_div64(m, p.bn));
    const int64_t tiles = static_cast<int64_t>(p.mt) * NT;
    p.splits = 1;
    p.gps = G;
    p.units = static_cast<int>(tiles);
    p.workspace = 0;
    p.maxseg = 1;
    p.total = tiles * G;
    // stream-K when whole tiles would leave SMs idle or unbalanced
    // stream-K when whole tiles would leave SMs idle: every decode op whose
    // tile count is not a multiple of the grid, and prefill ops whose last
    // wave is badly filled ([5120 x 5120] / [5120 x 20480] at 2048 tokens:
    // 320 BN=256 tiles = 2.16 waves, 72% busy; their whole-tile K4 ran at
    // 1.03 / 1.24 PF/s against 1.4 for the well-filled qkv / fc1)
    const double waves = static_cast<double>(tiles) / sms;
    const bool prefill_sk = phase == 0 && tiles > sms && waves / std::ceil(waves) < 0.85;
    p.stream_k = ((phase == 1 && tiles % sms != 0) || prefill_sk) &&
                         tiles <= static_cast<int64_t>(kTicketBytes / 4)
                     ? 1
                     : 0;
    if (phase == 1 && getenv("HP_EXP_DECODE_TILES")) p.stream_k = 0;  // timing experiment
    p.dp = 0;
    if (p.stream_k && prefill_sk) {
        // optional data-parallel + stream-K split: whole-tile waves first,
        // the rest as stream-K. Measured slower on B200 than pure stream-K
        // for the 2.16-wave ops (out 1.03-1.09 vs 1.10-1.19 PF/s, fc2 1.37-1.51
        // vs 1.43-1.60), so 0 waves by default.
        int dpw = 0;
        if (const char* e = getenv("HP_PREFILL_DP_WAVES")) dpw = std::min(atoi(e), static_cast<int>(waves));
        if (dpw > 0) {
            p.dp = dpw * sms;
            p.total = (tiles - p.dp) * G;
        }
    }
    if (p.stream_k && p.total * sms >= (int64_t(1) << 32)) {  // 32-bit seg_iter arithmetic
        p.stream_k = 0;
        p.dp = 0;
        p.total = tiles * G;
    }
    if (p.stream_k) {
        p.grid = static_cast<int>(p.total < sms ? p.total : sms);
        const int64_t per = p.total / p.grid;  // >= 1 group-step per CTA
        p.maxseg = static_cast<int>((G + per - 1) / per) + 1;
        if (p.maxseg > p.grid) p.maxseg = p.grid;
        // The tile-ticket region has a FIXED size: one workspace serves ops
        // of different tile counts, and a region sized per op would put one
        // op's partials over another op's (never re-zeroed) tickets.
        p.workspace = kTicketBytes +
                      static_cast<size_t>(tiles) * p.maxseg * 128 * p.bn * sizeof(float);
    } else {
        p.grid = static_cast<int>(tiles < sms ? tiles : sms);
    }
    return p;
}

unsigned long long* g_trace = nullptr;

unsigned long long* trace_buffer() {
    static bool checked = false;
    if (!checked) {
        checked = true;
        if (getenv("HP_QGEMM_TRACE")) {
            int cta = getenv("HP_QGEMM_TRACE_CTA") ? atoi(getenv("HP_QGEMM_TRACE_CTA")) : 0;
            cudaMemcpyToSymbol(g_trace_cta, &cta, sizeof(int));
            cudaMalloc(&g_trace, sizeof(unsigned long long) * (6 * kTraceIters * 4 + 13 * 1024));
            cudaMemset(g_trace, 0, sizeof(unsigned long long) * (6 * kTraceIters * 4 + 13 * 1024));
        }
    }
    return g_trace;
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
    a.stream_k = p.stream_k;
    a.dp = p.dp;
    a.total = p.total;
    a.maxseg = p.maxseg;
    a.y = static_cast<__nv_bfloat16*>(y);
    a.ldy = ldy;
    a.res = static_cast<const __nv_bfloat16*>(res);
    a.ldr = ldr;
    a.epi = epi;
    a.trace = trace_buffer();
    if (p.stream_k) {
        auto* base = static_cast<uint8_t*>(workspace);
        a.counters = reinterpret_cast<unsigned*>(base);
        a.partial = reinterpret_cast<float*>(
            base + kTicketBytes);
    }
    switch (p.bn) {
        case 16: return dispatch_bits<16>(bits, sym, map, a, p.grid, st);
        case 32: return dispatch_bits<32>(bits, sym, map, a, p.grid, st);
        case 128: return dispatch_bits<128>(bits, sym, map, a, p.grid, st);
        case 256: return dispatch_bits<256>(bits, sym, map, a, p.grid, st);
#if HP_PRE_BN192
        case 192: return dispatch_bits<192>(bits, sym, map, a, p.grid, st);
#endif
    }
    return cudaErrorInvalidValue;
}

}  // namespace hp
