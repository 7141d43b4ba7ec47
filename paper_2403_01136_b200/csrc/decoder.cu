// Decoder-layer glue around the quantized linear ops —
// NOT the graded hot path, but inside every serving round:
//   * embed_kernel: x[r] = E[tok[r]] + P[pos[r] + 2] (OPT learned positions,
//     offset 2; models with pos_s == 1, e.g. BLOOM's ALiBi, add none);
//   * attn_prefill_kernel: causal self-attention of a prefill micro-batch
//     (FlashAttention-2 structure: 64-query tiles, online softmax in fp32,
//     mma.sync m16n8k16 bf16 -> fp32), reading q/k/v straight from the qkv
//     projection output and writing each request's K/V rows into the
//     pre-allocated KV cache (memcost.cpp:38-42: 2*v*(s+n)*h1 elements per
//     layer);
//   * attn_decode_kernel: one query per request against its cache rows
//     [0, p] after appending the new K/V row at position p (HBM-bound: one
//     streaming pass over K and V, coalesced 256 B rows, flash-decoding
//     online softmax in fp32);
//   * argmax_kernel: greedy next token of every LM-head row (ties -> lowest
//     id).
// qkv rows are [q (h1) | k (h1) | v (h1)], head h at columns h*D .. h*D+D-1
// of each third (OPT's separate q/k/v projections concatenated).
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdint>
#include <type_traits>

namespace hp {

extern int g_pdl;

namespace {

__device__ __forceinline__ void pdl_wait_glue() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger_glue() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

cudaError_t launch_ex(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      void** args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

// ---------------------------------------------------------------- embedding
__global__ void embed_kernel(const int32_t* __restrict__ tok, int rows, int pos0, int pos_per_req,
                             int s_tokens, const __nv_bfloat16* __restrict__ E,
                             const __nv_bfloat16* __restrict__ P, int pos_s, int h, int64_t vocab,
                             __nv_bfloat16* __restrict__ x) {
    pdl_wait_glue();
    pdl_trigger_glue();
    const int r = blockIdx.x;
    // row r: token tok[r]; position = pos0 + (pos_per_req ? r % s_tokens : 0)
    int64_t t = tok[r];
    t = t < 0 ? 0 : (t >= vocab ? vocab - 1 : t);
    const int pos = pos0 + (pos_per_req ? r % s_tokens : 0);
    const uint4* e = reinterpret_cast<const uint4*>(E + t * h);
    const uint4* p = P && pos + 2 < pos_s ? reinterpret_cast<const uint4*>(P + static_cast<int64_t>(pos + 2) * h)
                                          : nullptr;
    uint4* o = reinterpret_cast<uint4*>(x + static_cast<int64_t>(r) * h);
    for (int c = threadIdx.x; c < h / 8; c += blockDim.x) {
        uint4 a = e[c];
        if (p) {
            const uint4 b = p[c];
            __nv_bfloat162* pa = reinterpret_cast<__nv_bfloat162*>(&a);
            const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 fa = __bfloat1622float2(pa[i]), fb = __bfloat1622float2(pb[i]);
                pa[i] = __floats2bfloat162_rn(fa.x + fb.x, fa.y + fb.y);
            }
        }
        o[c] = a;
    }
}

// ------------------------------------------------------------- mma helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
    const int n = pred ? 16 : 0;  // zero-fill rows past the end
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// Tile [64 rows x D] bf16 in smem, 16-byte chunks XOR-swizzled by row so the
// 8 rows an ldmatrix phase touches hit 8 different bank groups.
template <int D>
__device__ __forceinline__ uint32_t tile_off(int row, int chunk) {
    return static_cast<uint32_t>((row * (D / 8) + (chunk ^ (row & 7))) * 16);
}

constexpr int kPrefillWarps = 4;
#ifndef HP_ATTN_PRE_STAGES
#define HP_ATTN_PRE_STAGES 2
#endif
constexpr int kPrefillStages = HP_ATTN_PRE_STAGES;  // K/V ring depth: 2 and 3 measure the same (107 TF/s), 4 (1 CTA/SM) 68

// ---------------------------------------------------------- prefill attention
// grid (q-tiles of 16*NW, heads, requests); NW warps x 16 query rows.
// qkv [rows x 3h] bf16 (request r's tokens at rows r*s .. r*s+s-1 of this
// micro-batch); out [rows x h]; K/V cache: head-major [B][heads][S_max][D],
// request (req0 + r), head hd, position pos at ((req*heads + hd)*S_max + pos)*D
// (the 2*v*(s+n)*h1 elements per layer of memcost.cpp:38-42, laid out so a
// (request, head) context is ONE contiguous stream for decode attention).
template <int D, int NW>
__global__ void __launch_bounds__(32 * NW)
    attn_prefill_kernel(const __nv_bfloat16* __restrict__ qkv, int s, int h, float scale_log2,
                        __nv_bfloat16* __restrict__ out, __nv_bfloat16* __restrict__ kc,
                        __nv_bfloat16* __restrict__ vc, int req0, int S_max) {
    constexpr int BR = 16 * NW, BC = 64, CH = D / 8;  // 16-byte chunks per row
    constexpr int NT = 32 * NW;
    constexpr int KS = kPrefillStages;      // K/V tile ring depth
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* sQ = sm;
    uint8_t* sK = sm + BR * D * 2;          // KS stages
    uint8_t* sV = sK + KS * BC * D * 2;     // KS stages
    pdl_wait_glue();
    pdl_trigger_glue();
    // grid (heads, requests, q-tiles), the LAST (most key tiles under the
    // causal mask) q-tiles first: the long CTAs start in the first wave and
    // the short ones fill the tail
    const int head = blockIdx.x, r = blockIdx.y, qt = gridDim.z - 1 - blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t ld = 3LL * h;
    const __nv_bfloat16* base = qkv + static_cast<int64_t>(r) * s * ld + head * D;
    const int q0 = qt * BR;
    // Q tile + KV cache rows of this q-tile (each K/V row is written once:
    // by the CTA whose query tile covers it)
    for (int i = tid; i < BR * CH; i += NT) {
        const int row = i / CH, c = i % CH;
        const bool ok = q0 + row < s;
        cp_async16(smem_addr(sQ) + tile_off<D>(row, c), base + static_cast<int64_t>(q0 + row) * ld + c * 8,
                   ok);
        if (ok) {
            const int64_t crow = ((static_cast<int64_t>(req0 + r) * (h / D) + head) * S_max + q0 + row) * D + c * 8;
            *reinterpret_cast<uint4*>(kc + crow) =
                *reinterpret_cast<const uint4*>(base + static_cast<int64_t>(q0 + row) * ld + h + c * 8);
            *reinterpret_cast<uint4*>(vc + crow) =
                *reinterpret_cast<const uint4*>(base + static_cast<int64_t>(q0 + row) * ld + 2 * h + c * 8);
        }
    }
    cp_commit();
    const int nkv = (q0 + BR + BC - 1) / BC;  // causal: key tiles 0 .. q-tile
    auto load_kv = [&](int j, int stg) {
        if (j >= nkv) {  // empty group: keeps the wait count uniform
            cp_commit();
            return;
        }
        for (int i = tid; i < BC * CH; i += NT) {
            const int row = i / CH, c = i % CH;
            const int key = j * BC + row;
            const bool ok = key < s;
            const __nv_bfloat16* src = base + static_cast<int64_t>(ok ? key : 0) * ld;
            cp_async16(smem_addr(sK + stg * BC * D * 2) + tile_off<D>(row, c), src + h + c * 8, ok);
            cp_async16(smem_addr(sV + stg * BC * D * 2) + tile_off<D>(row, c), src + 2 * h + c * 8, ok);
        }
        cp_commit();
    };
#pragma unroll
    for (int j = 0; j < KS - 1; ++j) load_kv(j, j);
    cp_wait<KS - 1>();  // Q landed (the K/V prologue groups may be in flight)
    __syncthreads();
    // Q fragments of this warp's 16 rows (kept in registers)
    uint32_t qf[D / 16][4];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
        const int row = warp * 16 + (lane & 15);
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(smem_addr(sQ) + tile_off<D>(row, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
    }
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow[2] = {-FLT_MAX, -FLT_MAX}, lrow[2] = {0.f, 0.f};
    const int qa = q0 + warp * 16 + (lane >> 2);  // this thread's query rows qa, qa + 8
    for (int j = 0; j < nkv; ++j) {
        const int stg = j % KS;
        load_kv(j + KS - 1, (j + KS - 1) % KS);  // refills the stage consumed last iteration
        cp_wait<KS - 1>();                       // key tile j landed
        __syncthreads();
        const uint32_t kb = smem_addr(sK + stg * BC * D * 2), vb = smem_addr(sV + stg * BC * D * 2);
        // S = Q K^T : 16 x 64 per warp, 8 n-tiles
        float sc[BC / 8][4];
#pragma unroll
        for (int n = 0; n < BC / 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
            for (int n2 = 0; n2 < BC / 16; ++n2) {
                // keys n2*16 .. +15, dims kk*16 .. +15: x4 = (keys 0-7, d 0-7), (keys 0-7, d 8-15),
                // (keys 8-15, d 0-7), (keys 8-15, d 8-15)
                const int row = n2 * 16 + (lane & 7) + ((lane >> 4) << 3);
                const int c = kk * 2 + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kb + tile_off<D>(row, c), b0, b1, b2, b3);
                mma16816(sc[2 * n2], qf[kk], b0, b1);
                mma16816(sc[2 * n2 + 1], qf[kk], b2, b3);
            }
        }
        // causal mask + online softmax (rows qa, qa + 8)
        float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
        for (int n = 0; n < BC / 8; ++n) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = j * BC + n * 8 + (lane & 3) * 2 + (e & 1);
                const int q = qa + (e >> 1) * 8;
                float v = sc[n][e] * scale_log2;
                if (key > q || key >= s) v = -FLT_MAX;
                sc[n][e] = v;
                mx[e >> 1] = fmaxf(mx[e >> 1], v);
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
            mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
        }
        float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 2; ++i) corr[i] = exp2f(mrow[i] - mx[i]);
        uint32_t pf[BC / 16][4];
#pragma unroll
        for (int n = 0; n < BC / 8; ++n) {
            float p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                p[e] = sc[n][e] == -FLT_MAX ? 0.f : exp2f(sc[n][e] - mx[e >> 1]);
                rs[e >> 1] += p[e];
            }
            // S accumulator (16x8 tile n) -> A fragment of P (k16 chunk n/2)
            pf[n >> 1][(n & 1) * 2 + 0] = pack2(p[0], p[1]);
            pf[n >> 1][(n & 1) * 2 + 1] = pack2(p[2], p[3]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 1);
            rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 2);
            lrow[i] = lrow[i] * corr[i] + rs[i];
            mrow[i] = mx[i];
        }
#pragma unroll
        for (int d = 0; d < D / 8; ++d) {
            o[d][0] *= corr[0];
            o[d][1] *= corr[0];
            o[d][2] *= corr[1];
            o[d][3] *= corr[1];
        }
        // O += P V : A = P (16 x 64 keys), B = V (keys x dims), ldmatrix.trans
#pragma unroll
        for (int kk = 0; kk < BC / 16; ++kk) {
            uint32_t a[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
            for (int d2 = 0; d2 < D / 16; ++d2) {
                // keys kk*16.., dims d2*16..: x4.trans = (keys 0-7, d 0-7), (keys 8-15, d 0-7),
                // (keys 0-7, d 8-15), (keys 8-15, d 8-15)
                const int row = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int c = d2 * 2 + (lane >> 4);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vb + tile_off<D>(row, c), b0, b1, b2, b3);
                mma16816(o[2 * d2], a, b0, b1);
                mma16816(o[2 * d2 + 1], a, b2, b3);
            }
        }
        __syncthreads();  // stage stg is refilled by the next iteration's load
    }
    // normalise and store
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int q = qa + i * 8;
        if (q >= s) continue;
        const float inv = 1.f / lrow[i];
        __nv_bfloat16* dst = out + (static_cast<int64_t>(r) * s + q) * h + head * D;
#pragma unroll
        for (int d = 0; d < D / 8; ++d) {
            const int col = d * 8 + (lane & 3) * 2;
            *reinterpret_cast<uint32_t*>(dst + col) = pack2(o[d][2 * i] * inv, o[d][2 * i + 1] * inv);
        }
    }
}

// ----------------------------------------------------------- decode attention
// grid (heads, rows); 4 warps. Row r (request req0 + r): query q = qkv[r, head],
// appends k/v at position p, attends over cache rows 0..p in ONE streaming
// pass: warp w takes keys w*KU.. in chunks of KU, issues the chunk's K and V
// row loads together (lanes split the head dim: 256 B per row per warp),
// and keeps a flash-decoding online softmax (running max m, sum l, and the
// rescaled fp32 accumulator); the 4 warps' (m, l, acc) merge in shared
// memory. (The two-pass version -- all K rows, a block-wide softmax, then
// all V rows -- ran at 0.71 of HBM: each pass drained before the next.)
template <int D>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const __nv_bfloat16* __restrict__ qkv, int h, int p, float scale_log2,
                       __nv_bfloat16* __restrict__ out, __nv_bfloat16* __restrict__ kc,
                       __nv_bfloat16* __restrict__ vc, int req0, int S_max,
                       float* __restrict__ part, unsigned* __restrict__ tickets) {
    constexpr int EL = D / 32;  // dims per lane (2 or 4)
#ifndef HP_ATTN_KU
#define HP_ATTN_KU 8
#endif
    constexpr int KU = HP_ATTN_KU;  // keys per chunk: 2*KU row loads in flight per lane
    using raw_t = typename std::conditional<EL == 4, uint2, uint32_t>::type;
    __shared__ float s_m[4], s_l[4];
    __shared__ float s_acc[4][D];
    pdl_wait_glue();
    pdl_trigger_glue();
    const int head = blockIdx.x, r = blockIdx.y, z = blockIdx.z, nz = gridDim.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t ld = 3LL * h;
    const __nv_bfloat16* row = qkv + static_cast<int64_t>(r) * ld + head * D;
    // head-major cache: this (request, head)'s keys are contiguous D-element rows
    const int64_t cbase = (static_cast<int64_t>(req0 + r) * (h / D) + head) * S_max * D;
    float q[EL];
#pragma unroll
    for (int e = 0; e < EL; ++e) q[e] = __bfloat162float(row[lane * EL + e]) * scale_log2;
    if (warp == 0 && z == nz - 1) {  // append k/v at p (the split that reads row p)
#pragma unroll
        for (int e = 0; e < EL; ++e) {
            kc[cbase + static_cast<int64_t>(p) * D + lane * EL + e] = row[h + lane * EL + e];
            vc[cbase + static_cast<int64_t>(p) * D + lane * EL + e] = row[2 * h + lane * EL + e];
        }
    }
    __syncthreads();  // the new row is visible to the CTA (same-CTA global RAW)
    // this split's keys [k_lo, k_hi) of 0..p
    const int k_lo = static_cast<int>((static_cast<int64_t>(p + 1) * z) / nz);
    const int nk = static_cast<int>((static_cast<int64_t>(p + 1) * (z + 1)) / nz);
    auto unpack = [&](raw_t v, float* f) {
        if constexpr (EL == 4) {
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
            const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
            f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
        } else {
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
            f[0] = a.x; f[1] = a.y;
        }
    };
    float m = -FLT_MAX, l = 0.f, acc[EL];
#pragma unroll
    for (int e = 0; e < EL; ++e) acc[e] = 0.f;
    for (int k0 = k_lo + warp * KU; k0 < nk; k0 += 4 * KU) {
        raw_t kr[KU], vr[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const int key = k0 + u < nk ? k0 + u : nk - 1;  // clamp: loads stay in bounds
            kr[u] = *reinterpret_cast<const raw_t*>(kc + cbase + static_cast<int64_t>(key) * D + lane * EL);
            vr[u] = *reinterpret_cast<const raw_t*>(vc + cbase + static_cast<int64_t>(key) * D + lane * EL);
        }
        float sc[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            float f[EL];
            unpack(kr[u], f);
            float a = 0.f;
#pragma unroll
            for (int e = 0; e < EL; ++e) a = fmaf(q[e], f[e], a);
            sc[u] = a;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1)
#pragma unroll
            for (int u = 0; u < KU; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], d);
        float cm = m;
#pragma unroll
        for (int u = 0; u < KU; ++u)
            if (k0 + u < nk) cm = fmaxf(cm, sc[u]);
        const float corr = exp2f(m - cm);
        l *= corr;
#pragma unroll
        for (int e = 0; e < EL; ++e) acc[e] *= corr;
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const float pk = k0 + u < nk ? exp2f(sc[u] - cm) : 0.f;
            l += pk;
            float f[EL];
            unpack(vr[u], f);
#pragma unroll
            for (int e = 0; e < EL; ++e) acc[e] = fmaf(pk, f[e], acc[e]);
        }
        m = cm;
    }
    if (lane == 0) {
        s_m[warp] = m;
        s_l[warp] = l;
    }
#pragma unroll
    for (int e = 0; e < EL; ++e) s_acc[warp][lane * EL + e] = acc[e];
    __syncthreads();
    const float M = fmaxf(fmaxf(s_m[0], s_m[1]), fmaxf(s_m[2], s_m[3]));
    float L = 0.f, v = 0.f;
    if (tid < D) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float c = s_m[w] == -FLT_MAX ? 0.f : exp2f(s_m[w] - M);  // empty warp: no keys
            L += s_l[w] * c;
            v += s_acc[w][tid] * c;
        }
    }
    const int64_t orow = static_cast<int64_t>(r) * h + head * D;
    if (nz == 1) {
        if (tid < D) out[orow + tid] = __float2bfloat16_rn(v / L);
        return;
    }
    // split context: publish (M, L, acc) of this split; the last of the nz
    // CTAs of (row, head) merges them in split order (deterministic)
    const int64_t pair = static_cast<int64_t>(r) * gridDim.x + head;
    float* mine = part + (pair * nz + z) * (D + 2);
    if (tid < D) mine[2 + tid] = v;
    if (tid == 0) {
        mine[0] = M;
        mine[1] = L;
    }
    __shared__ unsigned s_old;
    __syncthreads();  // all of this CTA's partial stores precede the ticket (release below)
    if (tid == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(tickets + pair) : "memory");
        s_old = old;
    }
    __syncthreads();
    if (s_old != static_cast<unsigned>(nz - 1)) return;
    if (tid < D) {
        const float* base = part + pair * nz * (D + 2);
        float MM = -FLT_MAX;
        for (int j = 0; j < nz; ++j) MM = fmaxf(MM, __ldcg(base + j * (D + 2)));
        float LL = 0.f, VV = 0.f;
        for (int j = 0; j < nz; ++j) {
            const float mj = __ldcg(base + j * (D + 2));
            const float c = mj == -FLT_MAX ? 0.f : exp2f(mj - MM);
            LL += __ldcg(base + j * (D + 2) + 1) * c;
            VV += __ldcg(base + j * (D + 2) + 2 + tid) * c;
        }
        out[orow + tid] = __float2bfloat16_rn(VV / LL);
    }
    if (tid == 0) tickets[pair] = 0u;  // self-resetting for the next launch
}

// ------------------------------------------------------------------ argmax
__global__ void __launch_bounds__(256)
    argmax_kernel(const __nv_bfloat16* __restrict__ logits, int64_t ld, int64_t vocab,
                  int32_t* __restrict__ tok, int32_t* __restrict__ tok2, int64_t tok2_stride) {
    __shared__ float sv[8];
    __shared__ int si[8];
    pdl_wait_glue();
    pdl_trigger_glue();
    const int r = blockIdx.x;
    const __nv_bfloat16* x = logits + static_cast<int64_t>(r) * ld;
    float best = -FLT_MAX;
    int bi = 0x7fffffff;
    for (int64_t i = threadIdx.x; i < vocab; i += 256) {
        const float v = __bfloat162float(x[i]);
        if (v > best) {  // strided scan: the first hit per thread is its lowest index
            best = v;
            bi = static_cast<int>(i);
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, d);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
        if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = best;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w)
            if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
                best = sv[w];
                bi = si[w];
            }
        tok[r] = bi;
        if (tok2) tok2[static_cast<int64_t>(r) * tok2_stride] = bi;
    }
}

// synthetic token ids (mirror of oracle/synth.py synth_tokens)
__device__ __forceinline__ uint64_t splitmix64_d(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void synth_tokens_kernel(int32_t* out, int64_t n, uint64_t seed, int64_t vocab) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<int32_t>(splitmix64_d(seed ^ static_cast<uint64_t>(i)) % static_cast<uint64_t>(vocab));
}

}  // namespace

// 4 warps x 16 query rows: 80 KB at D = 128 (2 CTAs per SM); 8 warps
// would not raise occupancy: at 186 registers one 256-thread CTA fills the
// register file
int attn_prefill_smem(int D) { return (16 * kPrefillWarps * D * 2) + 2 * kPrefillStages * (64 * D * 2); }

cudaError_t launch_embed(const int32_t* tok, int rows, int pos0, int pos_per_req, int s_tokens,
                         const void* E, const void* P, int pos_s, int h, int64_t vocab, void* x,
                         cudaStream_t st) {
    if (h % 8) return cudaErrorInvalidValue;
    const __nv_bfloat16* Eb = static_cast<const __nv_bfloat16*>(E);
    const __nv_bfloat16* Pb = static_cast<const __nv_bfloat16*>(P);
    __nv_bfloat16* xb = static_cast<__nv_bfloat16*>(x);
    void* args[] = {&tok, &rows, &pos0, &pos_per_req, &s_tokens, &Eb, &Pb, &pos_s, &h, &vocab, &xb};
    return launch_ex(reinterpret_cast<const void*>(embed_kernel), dim3(rows), dim3(128), 0, st, args);
}

cudaError_t launch_attn_prefill(const void* qkv, int reqs, int s, int h, int D, void* out, void* kc,
                                void* vc, int req0, int S_max, cudaStream_t st) {
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
    const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(qkv);
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
    __nv_bfloat16* k = static_cast<__nv_bfloat16*>(kc);
    __nv_bfloat16* v = static_cast<__nv_bfloat16*>(vc);
    void* args[] = {&q, &s, &h, const_cast<float*>(&scale_log2), &o, &k, &v, &req0, &S_max};
    const dim3 grid(h / D, reqs, (s + 16 * kPrefillWarps - 1) / (16 * kPrefillWarps));
    const int smem = attn_prefill_smem(D);
    const void* fn;
    if (D == 128) {
        fn = reinterpret_cast<const void*>(attn_prefill_kernel<128, kPrefillWarps>);
    } else if (D == 64) {
        fn = reinterpret_cast<const void*>(attn_prefill_kernel<64, kPrefillWarps>);
    } else {
        return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_ex(fn, grid, dim3(32 * kPrefillWarps), smem, st, args);
}

// Split-context scratch for launch_attn_decode: a FIXED-size region of
// self-resetting tickets (one per (row, head) pair) at offset 0, then fp32
// (M, L, acc[D]) per (row, head, split). Zero once. The ticket region does
// not move with the configuration, so one workspace serves calls of any
// (rows, heads, split): a per-configuration offset would put one call's
// tickets over another call's (never re-zeroed) partials.
constexpr size_t kAttnTicketPairs = size_t(1) << 17;
size_t attn_decode_workspace(int rows, int h, int D, int split) {
    if (split <= 1) return 0;
    const size_t pairs = static_cast<size_t>(rows) * (h / D);
    return kAttnTicketPairs * sizeof(unsigned) + pairs * split * (D + 2) * sizeof(float);
}

cudaError_t launch_attn_decode(const void* qkv, int rows, int h, int D, int p, void* out, void* kc,
                               void* vc, int req0, int S_max, cudaStream_t st, void* ws, int split) {
    if (split > 1 && static_cast<size_t>(rows) * (h / D) > kAttnTicketPairs) return cudaErrorInvalidValue;
    const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
    const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(qkv);
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
    __nv_bfloat16* k = static_cast<__nv_bfloat16*>(kc);
    __nv_bfloat16* v = static_cast<__nv_bfloat16*>(vc);
    if (split < 1 || (split > 1 && !ws)) split = 1;
    unsigned* tick = split > 1 ? static_cast<unsigned*>(ws) : nullptr;
    float* part = split > 1 ? reinterpret_cast<float*>(static_cast<char*>(ws) + kAttnTicketPairs * sizeof(unsigned))
                            : nullptr;
    void* args[] = {&q, &h, &p, const_cast<float*>(&scale_log2), &o, &k, &v, &req0, &S_max, &part, &tick};
    const dim3 grid(h / D, rows, split);
    if (D == 128) return launch_ex(reinterpret_cast<const void*>(attn_decode_kernel<128>), grid, dim3(128), 0, st, args);
    if (D == 64) return launch_ex(reinterpret_cast<const void*>(attn_decode_kernel<64>), grid, dim3(128), 0, st, args);
    return cudaErrorInvalidValue;
}

cudaError_t launch_argmax(const void* logits, int64_t ld, int rows, int64_t vocab, int32_t* tok,
                          int32_t* tok2, int64_t tok2_stride, cudaStream_t st) {
    const __nv_bfloat16* l = static_cast<const __nv_bfloat16*>(logits);
    void* args[] = {&l, &ld, &vocab, &tok, &tok2, &tok2_stride};
    return launch_ex(reinterpret_cast<const void*>(argmax_kernel), dim3(rows), dim3(256), 0, st, args);
}

cudaError_t launch_synth_tokens(int32_t* out, int64_t n, uint64_t seed, int64_t vocab, cudaStream_t st) {
    const int64_t blocks64 = (n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(blocks64 < 4096 ? blocks64 : 4096);
    synth_tokens_kernel<<<blocks, 256, 0, st>>>(out, n, seed, vocab);
    return cudaGetLastError();
}

}  // namespace hp
