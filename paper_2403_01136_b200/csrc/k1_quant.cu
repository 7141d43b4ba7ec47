// K1 — group-wise quantize + pack (sm_100a), plus the unpack / dequant
// utilities over the same tile layout (layout.cuh).
//
// Semantics follow the reference quantizer applied to each group of 128
// consecutive weights of a row: /root/reference/proj/src/indicator.cpp:19-56
// (minmax -> step = scaling_factor :82-91 -> snapped = floor((w-zero)/step
// + 0.5) -> clamp [lo,hi]), all in fp64 with the reference's exact operation
// sequence on the slow path. Round-to-nearest only (the SPEC default,
// SPEC.md:328); stochastic rounding uses a sequential mt19937_64 stream in
// the reference (indicator.cpp:37,50) and is rejected here.
//
// Fast path: x = fma((float)w - (float)zero, rcp_f32(step)), the product
// unrounded before the round-to-integer. Its absolute error is < 1e-4 for
// |x| <= 255, so whenever frac(x + 0.5) lies in
// [1e-3, 1 - 1e-3] the rounded code equals the reference's; other
// elements (ties, near-ties, non-finite) take the exact fp64 sequence
// __dsub_rn / __ddiv_rn / __dadd_rn / floor / clamp. About 0.3% of bf16
// weights take the slow path.
#include <cuda_bf16.h>

#include <atomic>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "layout.cuh"

namespace hp {

namespace {

constexpr float kTieMargin = 1e-3f;

struct group_grid {
    double step, zero, lo, hi;
    float zero_f, rcp_f;
};

__device__ __forceinline__ group_grid make_grid(float wmin, float wmax,
                                                int bits, bool sym) {
    group_grid g;
    // scaling_factor (indicator.cpp:82-91); pow(2,b)-1 is exact.
    if (sym) {
        const double hi = static_cast<double>((1 << (bits - 1)) - 1);
        const double amax = fmax(fabs(static_cast<double>(wmax)),
                                 fabs(static_cast<double>(wmin)));
        g.step = __ddiv_rn(amax, hi);
        g.zero = 0.0;
        g.lo = -hi;
        g.hi = hi;
    } else {
        const double hi = static_cast<double>((1 << bits) - 1);
        g.step = __ddiv_rn(__dsub_rn(static_cast<double>(wmax),
                                     static_cast<double>(wmin)),
                           hi);
        g.zero = static_cast<double>(wmin);
        g.lo = 0.0;
        g.hi = hi;
    }
    g.zero_f = static_cast<float>(g.zero);
    g.rcp_f = 1.0f / static_cast<float>(g.step);
    return g;
}

// Signed grid code of one element on the exact path: the reference's fp64
// operation sequence (indicator.cpp:44-47) and std::clamp. Inlined into the
// (rolled) near-tie loop: a call would spill the caller's live registers.
__device__ __forceinline__ int quant_code_exact(float w, double step, double zero, double lo, double hi) {
    if (step == 0.0) return 0;  // flat group: out = zero (indicator.cpp:39-41)
    const double scaled = __ddiv_rn(__dsub_rn(static_cast<double>(w), zero), step);
    const double sn = floor(__dadd_rn(scaled, 0.5));
    return static_cast<int>(sn < lo ? lo : (hi < sn ? hi : sn));
}

// The packed words of one 32-k slice are accumulated with one IMAD per code:
// word += bits(nm) << shift, where nm = xf + 1.5*2^23 holds M + q in its bit
// pattern (M = 0x4B400000). The words start at the compile-time constant
// sum over their fields of (off - M) << shift (mod 2^32), so the final word
// is exactly sum (q + off) << shift, the stored codes of layout.cuh.
constexpr uint32_t kMagicBits = 0x4B400000u;
constexpr float kMagicF = 12582912.0f;  // 1.5 * 2^23

template <int BITS>
struct slice_pack {
    static constexpr int NW = BITS == 3 ? 12 : BITS;  // words[chunk * 4 + word]
    // field positions for code e (0..31) of the slice; 3-bit pair 15 sets
    // three 1-bit fields (bit b of the code in chunk b) and is handled apart
    __host__ __device__ static constexpr int word_of(int e) {
        return BITS == 3 ? locate_code(3, e).chunk * 4 + locate_code(3, e).word
                         : locate_code(BITS, e).chunk * 4 + locate_code(BITS, e).word;
    }
    __host__ __device__ static constexpr int shift_of(int e) { return locate_code(BITS, e).shift; }
    __host__ __device__ static constexpr bool split3(int e) { return BITS == 3 && ((e >> 1) & 15) == 15; }
    __host__ __device__ static constexpr uint32_t init(int wi, int off) {
        uint32_t c = 0;
        for (int e = 0; e < 32; ++e)
            if (!split3(e) && word_of(e) == wi) c += (static_cast<uint32_t>(off) - kMagicBits) << shift_of(e);
        return c;
    }
    template <int OFF, int... I>
    __device__ static __forceinline__ void init_words(uint32_t* w, std::integer_sequence<int, I...>) {
        ((w[I] = std::integral_constant<uint32_t, init(I, OFF)>::value), ...);
    }
    __device__ static __forceinline__ void init_words(uint32_t* w, bool sym) {
        if (sym)
            init_words<(1 << (BITS - 1)) - 1>(w, std::make_integer_sequence<int, NW>{});
        else
            init_words<0>(w, std::make_integer_sequence<int, NW>{});
    }
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// float <-> int with the same total order (negative floats: magnitude bits
// flipped), for atomicMin / atomicMax on float values
__device__ __forceinline__ int ordered_bits(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float from_ordered_bits(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__device__ __forceinline__ uint64_t splat2(float f) {
    const uint64_t b = __float_as_uint(f);
    return b | (b << 32);
}

// Fast path for the two codes of one bf16x2 word, with B200's paired fp32
// ops (one instruction per two elements, each lane IEEE round-to-nearest):
//   xd = x - zero_f,  nm = fma(xd, rcp_f, 1.5*2^23)  (rint of the UNROUNDED
//   product in the low mantissa bits),  dd = fma(xd, rcp_f, 1.5*2^23 - nm)
//   (the rounding distance; 1.5*2^23 - nm = fma(nm, -1, 1.5*2^23) is exact),
//   e = dd*dd - T.
// The product feeds both FMAs unrounded: ptxas contracts a separate
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 anyway, so the scalar paths below
// (ragged slices, the exact path's fast_bits) use the same fmaf form and all
// three agree bit for bit.
// e < 0 <=> |dd| < 0.5 - margin: the element is away from a tie. e >= 0 or
// NaN (non-finite xf: canonical NaN, sign bit clear) flags it for the exact
// fp64 path; the caller shifts the sign bits of e into a mask.
__device__ __forceinline__ void fast_pair(uint32_t w, uint64_t nzf2, uint64_t rf2, uint64_t mg2,
                                          uint64_t neg1, uint64_t nt2, uint32_t& nlo, uint32_t& nhi,
                                          uint32_t& elo, uint32_t& ehi) {
    asm("{\n\t.reg .b64 x, nm, r, dd, e;\n\t.reg .b32 lo, hi;\n\t"
        "shl.b32 lo, %4, 16;\n\t"
        "and.b32 hi, %4, 0xFFFF0000;\n\t"
        "mov.b64 x, {lo, hi};\n\t"
        "add.rn.f32x2 x, x, %5;\n\t"
        "fma.rn.f32x2 nm, x, %6, %7;\n\t"
        "fma.rn.f32x2 r, nm, %8, %7;\n\t"
        "fma.rn.f32x2 dd, x, %6, r;\n\t"
        "fma.rn.f32x2 e, dd, dd, %9;\n\t"
        "mov.b64 {%0, %1}, nm;\n\t"
        "mov.b64 {%2, %3}, e;\n\t}"
        : "=r"(nlo), "=r"(nhi), "=r"(elo), "=r"(ehi)
        : "r"(w), "l"(nzf2), "l"(rf2), "l"(mg2), "l"(neg1), "l"(nt2));
}

// Work item = (128-row block, 128-k group) = one tile of the layout; two
// threads per (row, group), each owning 64 k (slices 2h, 2h+1): a warp covers
// 16 rows x one group (lane = 2 * row + h), a 256-thread CTA the 128 rows.
// CTAs walk items grid-stride with an incremental (row block, group) cursor
// (no integer division per item); each thread streams its own 128 bytes into
// dynamic shared memory with cp.async kD-1 items ahead, so HBM reads overlap
// the arithmetic without holding registers, and re-reads them from there per
// pass (group min/max, then each slice). The group's min/max is one shuffle
// with the partner lane, the fp64 grid is computed once per 64 weights, and
// each thread emits its two slices' part of the tile layout (layout.cuh):
// 4-bit one 16 B row entry of chunk s, 8-bit two (chunks 2s, 2s+1), 3-bit
// word s of chunks 0..2, 16-bit four per slice; for a fixed chunk the 16
// rows of a warp are 256 contiguous bytes.
constexpr int kQRows = 128;  // rows per item (one tile row-block)
#ifndef HP_K1_DEPTH
#define HP_K1_DEPTH 2
#endif
#ifndef HP_K1_CTAS
#define HP_K1_CTAS 3  // 3 x 256 threads x 64 KB shared: +4-6% over depth 3 x 2 CTAs (round 2)
#endif
constexpr int kD = HP_K1_DEPTH;  // cp.async pipeline depth (items)
constexpr int kPieces = 8;       // 16-byte pieces per thread per item (64 bf16)
constexpr size_t kK1Smem = static_cast<size_t>(kD) * kPieces * 256 * sizeof(uint4);

template <int BITS>
__global__ void __launch_bounds__(256, HP_K1_CTAS)
    quant_pack_kernel(const __nv_bfloat16* __restrict__ w, int n_out, int k_in, int64_t ldw,
                      int G, int sym, int items, uint8_t* __restrict__ packed,
                      float* __restrict__ scale, float* __restrict__ zero,
                      double* __restrict__ step64, double* __restrict__ zero64,
                      int* __restrict__ wmm) {
    extern __shared__ __align__(16) uint4 kbuf[];  // [stage][piece][thread]
    // K2's weight reduction fused into this pass: the
    // op's exact min / max over all real weights, folded per thread and
    // published once per warp (order-independent, so deterministic)
    float tmin = __int_as_float(0x7f800000), tmax = -__int_as_float(0x7f800000);
    const int tid = threadIdx.x;
    const int h = tid & 1;     // k half of the group: slices 2h, 2h+1
    const int rin = tid >> 1;  // row within the 128-row block
    auto slot = [&](int st, int piece) -> uint4* { return &kbuf[(st * kPieces + piece) * 256 + tid]; };
    const bool vec_ok = (ldw % 8 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
    // items it = blockIdx.x + j * gridDim.x as (row block, group) cursors
    const int dq = static_cast<int>(gridDim.x) / G, dr = static_cast<int>(gridDim.x) % G;
    auto advance = [&](int& rb, int& g) {
        rb += dq;
        g += dr;
        if (g >= G) {
            g -= G;
            ++rb;
        }
    };
    int rb_i = static_cast<int>(blockIdx.x) / G, g_i = static_cast<int>(blockIdx.x) % G;
    int rb_c = rb_i, g_c = g_i, it_i = blockIdx.x;
    auto issue = [&](int st) {
        if (it_i < items) {
            const int row = rb_i * kQRows + rin;
            const int k0 = g_i * 128 + h * 64;
            if (vec_ok && row < n_out && k_in - k0 >= 64) {
                const uint4* src = reinterpret_cast<const uint4*>(w + static_cast<int64_t>(row) * ldw + k0);
#pragma unroll
                for (int i = 0; i < kPieces; ++i)
                    cp_async16(static_cast<uint32_t>(__cvta_generic_to_shared(slot(st, i))), src + i);
            }
        }
        cp_async_commit();  // (possibly empty) group: keeps the wait count uniform
        it_i += gridDim.x;
        advance(rb_i, g_i);
    };

#pragma unroll
    for (int d = 0; d < kD - 1; ++d) issue(d);
    int stage = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        issue((stage + kD - 1) % kD);
        cp_async_wait<kD - 1>();
        const int rb = rb_c, g = g_c;
        advance(rb_c, g_c);
        const int row = rb * kQRows + rin;
        const int k0 = g * 128 + h * 64;
        const bool row_ok = row < n_out;
        const int valid = row_ok ? (k_in - k0 <= 0 ? 0 : (k_in - k0 < 64 ? k_in - k0 : 64)) : 0;
        const bool full = vec_ok && valid == 64;
        const int cur = stage;  // slot cur stays valid until the next iteration's issue
        stage = (stage + 1) % kD;
        if (!full) {  // ragged k, padding rows, unaligned rows: stage zero-padded elements
            const __nv_bfloat16* src = w + static_cast<int64_t>(row) * ldw + k0;
#pragma unroll
            for (int i = 0; i < kPieces; ++i) {
                uint32_t q4[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int e = 8 * i + 2 * j;
                    const uint32_t lo = e < valid ? __bfloat16_as_ushort(src[e]) : 0u;
                    const uint32_t hi = e + 1 < valid ? __bfloat16_as_ushort(src[e + 1]) : 0u;
                    q4[j] = lo | (hi << 16);
                }
                *slot(cur, i) = make_uint4(q4[0], q4[1], q4[2], q4[3]);
            }
        }
        uint8_t* tbase = packed + (static_cast<size_t>(rb) * G + g) * tile_bytes(BITS) + rin * 16;

        if constexpr (BITS == 16) {
            // padding rows of the last tile (row >= n_out) are written as zeros
#pragma unroll
            for (int c = 0; c < kPieces; ++c)
                *reinterpret_cast<uint4*>(tbase + (8 * h + c) * 2048) = *slot(cur, c);
            if (wmm) {
                for (int e = 0; e < valid; ++e) {
                    const float x = __uint_as_float(static_cast<uint32_t>(
                                                        reinterpret_cast<const uint16_t*>(slot(cur, e >> 3))[e & 7])
                                                    << 16);
                    tmin = fminf(tmin, x);
                    tmax = fmaxf(tmax, x);
                }
            }
            continue;
        } else {
            // the thread's 64 elements, read from shared memory once
            uint32_t vv[2 * 16];
#pragma unroll
            for (int i = 0; i < kPieces; ++i) {
                const uint4 u = *slot(cur, i);
                vv[4 * i] = u.x; vv[4 * i + 1] = u.y; vv[4 * i + 2] = u.z; vv[4 * i + 3] = u.w;
            }
            float wmin, wmax;
            if (full) {  // bf16x2 min/max (exact), halves folded at the end
                __nv_bfloat162 mn = *reinterpret_cast<const __nv_bfloat162*>(&vv[0]), mx = mn;
#pragma unroll
                for (int i = 1; i < 32; ++i) {
                    const __nv_bfloat162 hv = *reinterpret_cast<const __nv_bfloat162*>(&vv[i]);
                    mn = __hmin2(mn, hv);
                    mx = __hmax2(mx, hv);
                }
                wmin = fminf(__low2float(mn), __high2float(mn));
                wmax = fmaxf(__low2float(mx), __high2float(mx));
            } else {
                wmin = __int_as_float(0x7f800000);
                wmax = -__int_as_float(0x7f800000);
                for (int e = 0; e < valid; ++e) {  // rolled: rare path
                    const float x = __uint_as_float(static_cast<uint32_t>(
                                                        reinterpret_cast<const uint16_t*>(slot(cur, e >> 3))[e & 7])
                                                    << 16);
                    wmin = fminf(wmin, x);
                    wmax = fmaxf(wmax, x);
                }
            }
            wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, 1));
            wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, 1));
            if (!row_ok) wmin = wmax = 0.0f;
            else if (wmm) {
                tmin = fminf(tmin, wmin);
                tmax = fmaxf(tmax, wmax);
            }
            const group_grid gg = make_grid(wmin, wmax, BITS, sym != 0);
            const int off = sym ? (1 << (BITS - 1)) - 1 : 0;
            if (h == 0) {
                const size_t sidx = (static_cast<size_t>(rb) * G + g) * 128 + rin;
                if (scale) scale[sidx] = row_ok ? static_cast<float>(gg.step) : 0.0f;
                if (zero) zero[sidx] = row_ok ? gg.zero_f : 0.0f;
                if (row_ok && step64) {
                    step64[static_cast<int64_t>(row) * G + g] = gg.step;
                    zero64[static_cast<int64_t>(row) * G + g] = gg.zero;
                }
            }
            // Fast path: xf = fma(w - zero, rcp(step)) in fp32 (|error| < 1e-4
            // for |xf| <= 255; |xf| <= hi by construction);
            // away from a tie (|xf - rint(xf)| <= 0.5 - margin) floor(x + 0.5)
            // == rint(xf) and lies in [lo, hi]. Near ties / non-finite values
            // take quant_code_exact. A flat group (step 0) has rcp 0: every
            // code is 0, as the reference.
            const float zf = gg.zero_f;
            // a step below FLT_MIN is a denormal float: rcp would be inexact,
            // so NaN flags every code for the exact path
            const float rf = gg.step == 0.0 ? 0.0f : (gg.step < 1.1754943508222875e-38 ? __int_as_float(0x7fc00000) : gg.rcp_f);
            using SP = slice_pack<BITS>;
            // explicit __fmaf_rn (the pair path's FFMA2 form), so the exact
            // path recomputes the very bits the fast path packed
            auto fast_bits = [&](float x) { return __float_as_uint(__fmaf_rn(__fsub_rn(x, zf), rf, kMagicF)); };
            const float tm = 0.5f - kTieMargin;
            const uint64_t nzf2 = splat2(-zf), rf2 = splat2(rf), mg2 = splat2(kMagicF),
                           neg1 = splat2(-1.0f), nt2 = splat2(-tm * tm);
#pragma unroll
            for (int j = 0; j < 2; ++j) {  // this thread's slices s = 2h + j
                const int sl = 2 * h + j;
                const uint32_t* v = vv + 16 * j;
                const int vs = valid - 32 * j < 0 ? 0 : (valid - 32 * j > 32 ? 32 : valid - 32 * j);
                uint32_t words[SP::NW];
                SP::init_words(words, sym != 0);
                uint32_t code15[2] = {0u, 0u};  // 3-bit pair 15 (codes 30, 31)
                uint32_t slow = 0;
                if (vs == 32) {
                    // ok: bit 31-e set <=> element e is away from a tie (funnel
                    // shift of the sign bit of e, one SHF per element)
                    uint32_t ok = 0;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        uint32_t n0, n1, e0, e1;
                        fast_pair(v[i], nzf2, rf2, mg2, neg1, nt2, n0, n1, e0, e1);
                        ok = __funnelshift_l(e0, ok, 1);
                        ok = __funnelshift_l(e1, ok, 1);
                        if (SP::split3(2 * i)) {
                            code15[0] = n0 - kMagicBits + static_cast<uint32_t>(off);
                            code15[1] = n1 - kMagicBits + static_cast<uint32_t>(off);
                        } else {
                            words[SP::word_of(2 * i)] += n0 << SP::shift_of(2 * i);
                            words[SP::word_of(2 * i + 1)] += n1 << SP::shift_of(2 * i + 1);
                        }
                    }
                    slow = __brev(~ok);  // bit e: element e takes the exact path
                } else {  // partial slice: scalar, padding codes are signed 0
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float x = __uint_as_float((e & 1) ? (v[e >> 1] & 0xFFFF0000u) : (v[e >> 1] << 16));
                        const float xd = __fsub_rn(x, zf);
                        const float nm = __fmaf_rn(xd, rf, kMagicF);
                        const float d = __fmaf_rn(xd, rf, -(nm - kMagicF));  // NaN for non-finite xf
                        uint32_t bits = __float_as_uint(nm);
                        if (e >= vs) {
                            bits = kMagicBits;  // padding: signed code 0
                        } else if (!(fabsf(d) <= 0.5f - kTieMargin)) {
                            slow |= 1u << e;
                        }
                        if (SP::split3(e)) {
                            code15[e & 1] = bits - kMagicBits + static_cast<uint32_t>(off);
                        } else {
                            words[SP::word_of(e)] += bits << SP::shift_of(e);
                        }
                    }
                }
                // exact fp64 path (ties, near-ties, non-finite): a rolled loop
                // over the flagged codes, the element re-read from shared memory
                while (slow) {
                    const int e = __ffs(slow) - 1;
                    slow &= slow - 1;
                    const uint16_t* sb = reinterpret_cast<const uint16_t*>(slot(cur, 4 * j + (e >> 3)));
                    const float x = __uint_as_float(static_cast<uint32_t>(sb[e & 7]) << 16);
                    const uint32_t ex = kMagicBits + static_cast<uint32_t>(
                                                         quant_code_exact(x, gg.step, gg.zero, gg.lo, gg.hi));
                    if (BITS == 3 && ((e >> 1) & 15) == 15) {
                        const uint32_t c = ex - kMagicBits + static_cast<uint32_t>(off);
                        code15[0] = (e & 1) ? code15[0] : c;
                        code15[1] = (e & 1) ? c : code15[1];
                    } else {
                        const code_pos cp = locate_code(BITS, e);
                        const int wi = cp.chunk * 4 + cp.word;
                        const uint32_t delta = (ex - fast_bits(x)) << cp.shift;
#pragma unroll
                        for (int i = 0; i < SP::NW; ++i) words[i] += (i == wi) ? delta : 0u;
                    }
                }
                if constexpr (BITS == 3) {
                    // pair 15: bit b of code 30 at bit 15, of code 31 at bit 31, of chunk b
#pragma unroll
                    for (int b2 = 0; b2 < 3; ++b2)
                        words[b2 * 4] |= (((code15[0] >> b2) & 1u) << 15) | (((code15[1] >> b2) & 1u) << 31);
                }
                if constexpr (BITS == 4) {
                    *reinterpret_cast<uint4*>(tbase + sl * 2048) = make_uint4(words[0], words[1], words[2], words[3]);
                } else if constexpr (BITS == 8) {
                    *reinterpret_cast<uint4*>(tbase + (2 * sl) * 2048) = make_uint4(words[0], words[1], words[2], words[3]);
                    *reinterpret_cast<uint4*>(tbase + (2 * sl + 1) * 2048) = make_uint4(words[4], words[5], words[6], words[7]);
                } else {
#pragma unroll
                    for (int b2 = 0; b2 < 3; ++b2) *reinterpret_cast<uint32_t*>(tbase + b2 * 2048 + sl * 4) = words[b2 * 4];
                }
            }
        }
    }
    cp_async_wait<0>();
    if (wmm) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, d));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, d));
        }
        if ((tid & 31) == 0) {
            atomicMin(&wmm[0], ordered_bits(tmin));
            atomicMax(&wmm[1], ordered_bits(tmax));
        }
    }
}

// weight min/max scratch (two ordered ints in the bytes of stats5[1]) and
// the fp64 result: stats5[0] = d_w, [1] = w_min, [2] = w_max (K2's layout)
__global__ void wstats_init_kernel(int* wmm) {
    wmm[0] = ordered_bits(__int_as_float(0x7f800000));
    wmm[1] = ordered_bits(-__int_as_float(0x7f800000));
}
__global__ void wstats_finish_kernel(double* stats5, double d_w) {
    const int* wmm = reinterpret_cast<const int*>(stats5 + 1);
    const float mn = from_ordered_bits(wmm[0]), mx = from_ordered_bits(wmm[1]);
    stats5[0] = d_w;
    stats5[1] = static_cast<double>(mn);
    stats5[2] = static_cast<double>(mx);
}

// Unpack to row-major stored codes (u8, or raw bf16 words for 16-bit) and
// row-major fp32 scale/zero. One thread per (row, group).
template <int BITS>
__global__ void unpack_kernel(const uint8_t* __restrict__ packed,
                              const float* __restrict__ scale,
                              const float* __restrict__ zero, int64_t n_out,
                              int64_t k_in, int G, uint8_t* __restrict__ codes,
                              float* __restrict__ scale_rm,
                              float* __restrict__ zero_rm) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n_out * G) return;
    const int64_t row = idx / G;
    const int g = static_cast<int>(idx % G);
    const int64_t nt = row / 128;
    const int r = static_cast<int>(row % 128);
    const size_t t = static_cast<size_t>(nt) * G + g;
    const uint8_t* base = packed + t * tile_bytes(BITS) + r * 16;
    if (scale_rm && scale) scale_rm[row * G + g] = scale[t * 128 + r];
    if (zero_rm && zero) zero_rm[row * G + g] = zero[t * 128 + r];
    if (!codes) return;
    const int64_t k0 = static_cast<int64_t>(g) * 128;
    const int cnt = static_cast<int>(k_in - k0 < 128 ? k_in - k0 : 128);
    for (int kk = 0; kk < cnt; ++kk) {
        if constexpr (BITS == 16) {
            const uint16_t v = *reinterpret_cast<const uint16_t*>(base + (kk >> 3) * 2048 + (kk & 7) * 2);
            reinterpret_cast<uint16_t*>(codes)[row * k_in + k0 + kk] = v;
        } else {
            uint32_t c;
            if constexpr (BITS == 3) {
                c = get_code3(reinterpret_cast<const uint32_t*>(base),
                              reinterpret_cast<const uint32_t*>(base + 2048),
                              reinterpret_cast<const uint32_t*>(base + 4096), kk);
            } else {
                const code_pos p = locate_code(BITS, kk);
                const uint32_t* wd = reinterpret_cast<const uint32_t*>(base + p.chunk * 2048);
                c = (wd[p.word] >> p.shift) & ((1u << BITS) - 1u);
            }
            codes[row * k_in + k0 + kk] = static_cast<uint8_t>(c);
        }
    }
}

// Dense bf16 dequant through the same per-slice arithmetic the GEMM uses.
// One thread per (row, 32-element slice).
template <int BITS, bool SYM>
__global__ void dequant_kernel(const uint8_t* __restrict__ packed,
                               const float* __restrict__ scale,
                               const float* __restrict__ zero, int64_t n_out,
                               int64_t k_in, int G,
                               __nv_bfloat16* __restrict__ out) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n_out * G * 4) return;
    const int slice = static_cast<int>(idx & 3);
    const int64_t rg = idx >> 2;
    const int64_t row = rg / G;
    const int g = static_cast<int>(rg % G);
    const int64_t nt = row / 128;
    const int r = static_cast<int>(row % 128);
    const size_t t = static_cast<size_t>(nt) * G + g;
    const uint8_t* base = packed + t * tile_bytes(BITS) + r * 16;
    float s = 0.f, z = 0.f;
    if (BITS != 16) {
        s = scale[t * 128 + r];
        z = SYM ? 0.0f : zero[t * 128 + r];
    }
    uint32_t v[16];
    dequant_slice32<BITS, SYM>(base, slice, s, z, scale_arg<SYM>(s),
                               zero_arg<SYM>(s, z), v);
    const int64_t k0 = static_cast<int64_t>(g) * 128 + slice * 32;
    for (int i = 0; i < 32; ++i) {
        if (k0 + i >= k_in) break;
        const uint16_t h = static_cast<uint16_t>((v[i >> 1] >> (16 * (i & 1))) & 0xFFFFu);
        reinterpret_cast<uint16_t*>(out)[row * k_in + k0 + i] = h;
    }
}

}  // namespace

// ---- launchers (called from capi.cu after argument validation) -----------
cudaError_t launch_quant_pack(const void* w, int64_t n_out, int64_t k_in,
                              int64_t ldw, int bits, int sym, void* packed,
                              float* scale, float* zero, double* step64,
                              double* zero64, double* stats5, cudaStream_t st) {
    const int G = static_cast<int>(ceil_div64(k_in, 128));
    // rows up to the 128-row tile boundary: padding rows get code 0 / scale 0
    const int64_t items = ceil_div64(n_out, kQRows) * G;
    if (n_out >= (int64_t(1) << 31) || k_in >= (int64_t(1) << 31) || items >= (int64_t(1) << 31))
        return cudaErrorInvalidValue;  // 32-bit row / k / item cursors
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // the dynamic shared-memory opt-in is per device and per kernel
    static std::atomic<unsigned> attr_done[64];
    const unsigned bitmask = 1u << (bits == 3 ? 0 : bits == 4 ? 1 : bits == 8 ? 2 : 3);
    if (dev < 0 || dev >= 64 || !(attr_done[dev].load(std::memory_order_acquire) & bitmask)) {
        cudaError_t e = cudaSuccess;
        switch (bits) {
            case 3: e = cudaFuncSetAttribute(quant_pack_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kK1Smem)); break;
            case 4: e = cudaFuncSetAttribute(quant_pack_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kK1Smem)); break;
            case 8: e = cudaFuncSetAttribute(quant_pack_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kK1Smem)); break;
            case 16: e = cudaFuncSetAttribute(quant_pack_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kK1Smem)); break;
            default: return cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr_done[dev].fetch_or(bitmask, std::memory_order_acq_rel);
    }
    const unsigned grid = static_cast<unsigned>(items < int64_t(HP_K1_CTAS) * sms ? items : int64_t(HP_K1_CTAS) * sms);
    auto* wp = static_cast<const __nv_bfloat16*>(w);
    auto* pp = static_cast<uint8_t*>(packed);
    const int n = static_cast<int>(n_out), k = static_cast<int>(k_in), its = static_cast<int>(items);
    int* wmm = stats5 ? reinterpret_cast<int*>(stats5 + 1) : nullptr;
    if (wmm) wstats_init_kernel<<<1, 1, 0, st>>>(wmm);
    switch (bits) {
        case 3: quant_pack_kernel<3><<<grid, 256, kK1Smem, st>>>(wp, n, k, ldw, G, sym, its, pp, scale, zero, step64, zero64, wmm); break;
        case 4: quant_pack_kernel<4><<<grid, 256, kK1Smem, st>>>(wp, n, k, ldw, G, sym, its, pp, scale, zero, step64, zero64, wmm); break;
        case 8: quant_pack_kernel<8><<<grid, 256, kK1Smem, st>>>(wp, n, k, ldw, G, sym, its, pp, scale, zero, step64, zero64, wmm); break;
        case 16: quant_pack_kernel<16><<<grid, 256, kK1Smem, st>>>(wp, n, k, ldw, G, sym, its, pp, scale, zero, step64, zero64, wmm); break;
        default: return cudaErrorInvalidValue;
    }
    if (wmm) wstats_finish_kernel<<<1, 1, 0, st>>>(stats5, static_cast<double>(n_out) * static_cast<double>(k_in));
    return cudaGetLastError();
}

cudaError_t launch_unpack(const void* packed, const float* scale,
                          const float* zero, int64_t n_out, int64_t k_in,
                          int bits, void* codes, float* scale_rm,
                          float* zero_rm, cudaStream_t st) {
    const int G = static_cast<int>(ceil_div64(k_in, 128));
    const int64_t n = n_out * G;
    const unsigned blocks = static_cast<unsigned>(ceil_div64(n, 256));
    auto* pp = static_cast<const uint8_t*>(packed);
    auto* cp = static_cast<uint8_t*>(codes);
    switch (bits) {
        case 3: unpack_kernel<3><<<blocks, 256, 0, st>>>(pp, scale, zero, n_out, k_in, G, cp, scale_rm, zero_rm); break;
        case 4: unpack_kernel<4><<<blocks, 256, 0, st>>>(pp, scale, zero, n_out, k_in, G, cp, scale_rm, zero_rm); break;
        case 8: unpack_kernel<8><<<blocks, 256, 0, st>>>(pp, scale, zero, n_out, k_in, G, cp, scale_rm, zero_rm); break;
        case 16: unpack_kernel<16><<<blocks, 256, 0, st>>>(pp, scale, zero, n_out, k_in, G, cp, scale_rm, zero_rm); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_dequant(const void* packed, const float* scale,
                           const float* zero, int64_t n_out, int64_t k_in,
                           int bits, int sym, void* out, cudaStream_t st) {
    const int G = static_cast<int>(ceil_div64(k_in, 128));
    const int64_t n = n_out * G * 4;
    const unsigned blocks = static_cast<unsigned>(ceil_div64(n, 256));
    auto* pp = static_cast<const uint8_t*>(packed);
    auto* op = static_cast<__nv_bfloat16*>(out);
#define HP_DQ(B)                                                                               \
    if (sym) dequant_kernel<B, true><<<blocks, 256, 0, st>>>(pp, scale, zero, n_out, k_in, G, op); \
    else dequant_kernel<B, false><<<blocks, 256, 0, st>>>(pp, scale, zero, n_out, k_in, G, op);
    switch (bits) {
        case 3: HP_DQ(3) break;
        case 4: HP_DQ(4) break;
        case 8: HP_DQ(8) break;
        case 16: dequant_kernel<16, true><<<blocks, 256, 0, st>>>(pp, scale, zero, n_out, k_in, G, op); break;
        default: return cudaErrorInvalidValue;
    }
#undef HP_DQ
    return cudaGetLastError();
}

}  // namespace hp
