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

#ifndef HP_K1_PAIRS
#define HP_K1_PAIRS 1  // f32x2 fast path (round 2); 0 = the scalar round-1 path
#endif

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

// Work item = (64-row block, 128-k group); one thread per (row, 32-k slice):
// a warp covers 8 rows x one group (lane = 4 * row + slice), a 256-thread
// CTA 64 rows. CTAs walk items grid-stride; each thread streams its own 64
// slice bytes into shared memory with cp.async kD-1 items ahead, so HBM
// reads overlap the arithmetic without holding registers. The group's
// min/max is a 2-step shuffle over the 4 lanes of a row, and each thread
// emits exactly its slice's part of the tile layout (layout.cuh): 4-bit one
// 16 B row entry of chunk s, 8-bit two (chunks 2s, 2s+1), 3-bit word s of
// chunks 0..2, 16-bit four; for a fixed chunk the 8 rows of a warp are 128
// contiguous bytes, so every store instruction writes whole lines.
constexpr int kQRows = 64;  // rows per item
#ifndef HP_K1_DEPTH
#define HP_K1_DEPTH 3
#endif
#ifndef HP_K1_CTAS
#define HP_K1_CTAS 4  // 4 x 256 threads at 61 registers: +4-5% over 3 x 76 (round 2)
#endif
constexpr int kD = HP_K1_DEPTH;  // cp.async pipeline depth (items)

template <int BITS>
__global__ void __launch_bounds__(256, HP_K1_CTAS)
    quant_pack_kernel(const __nv_bfloat16* __restrict__ w, int64_t n_out,
                      int64_t k_in, int64_t ldw, int G, int sym, int64_t items,
                      uint8_t* __restrict__ packed, float* __restrict__ scale,
                      float* __restrict__ zero, double* __restrict__ step64,
                      double* __restrict__ zero64) {
    __shared__ __align__(16) uint4 buf[kD][4][256];  // [stage][16 B piece][thread]
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int sl = lane & 3;
    const int rin = (tid >> 5) * 8 + (lane >> 2);
    const bool vec_ok = (ldw % 8 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
    struct where {
        int64_t row, k0;
        int g, valid;
        bool full;
    };
    auto locate = [&](int64_t it) {  // items < 2^31 (BLOOM fc1: 100k)
        where q;
        const uint32_t rb = static_cast<uint32_t>(it) / static_cast<uint32_t>(G);
        q.g = static_cast<int>(static_cast<uint32_t>(it) - rb * static_cast<uint32_t>(G));
        q.row = static_cast<int64_t>(rb) * kQRows + rin;
        q.k0 = static_cast<int64_t>(q.g) * 128 + sl * 32;
        const int cnt = static_cast<int>(k_in - q.k0 <= 0 ? 0 : (k_in - q.k0 < 32 ? k_in - q.k0 : 32));
        q.valid = q.row < n_out ? cnt : 0;
        q.full = vec_ok && q.valid == 32;
        return q;
    };
    auto issue = [&](int64_t it, int stage) {
        if (it < items) {
            const where q = locate(it);
            if (q.full) {
                const __nv_bfloat16* src = w + q.row * ldw + q.k0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    cp_async16(static_cast<uint32_t>(__cvta_generic_to_shared(&buf[stage][i][tid])),
                               reinterpret_cast<const uint4*>(src) + i);
            }
        }
        cp_async_commit();  // (possibly empty) group: keeps the wait count uniform
    };

    const int64_t step_it = gridDim.x;
#pragma unroll
    for (int d = 0; d < kD - 1; ++d) issue(blockIdx.x + d * step_it, d);
    int stage = 0;
    for (int64_t it = blockIdx.x; it < items; it += step_it) {
        issue(it + (kD - 1) * step_it, (stage + kD - 1) % kD);
        cp_async_wait<kD - 1>();
        const where q = locate(it);
        uint32_t v[16];
        if (q.full) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint4 u = buf[stage][i][tid];
                v[4 * i] = u.x; v[4 * i + 1] = u.y; v[4 * i + 2] = u.z; v[4 * i + 3] = u.w;
            }
        } else {  // ragged k, rows past n_out (tile padding) or unaligned rows
            const __nv_bfloat16* src = w + q.row * ldw + q.k0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t lo = 2 * i < q.valid ? __bfloat16_as_ushort(src[2 * i]) : 0u;
                const uint32_t hi = 2 * i + 1 < q.valid ? __bfloat16_as_ushort(src[2 * i + 1]) : 0u;
                v[i] = lo | (hi << 16);
            }
        }
        const int cur = stage;  // buf[cur] stays valid until the next iteration's issue
        stage = (stage + 1) % kD;
        const int64_t nt = q.row >> 7;
        const int r = static_cast<int>(q.row & 127);
        uint8_t* tbase = packed + (static_cast<size_t>(nt) * G + q.g) * tile_bytes(BITS) + r * 16;
        auto elem = [&](int e) { return __uint_as_float((e & 1) ? (v[e >> 1] & 0xFFFF0000u) : (v[e >> 1] << 16)); };

        if constexpr (BITS == 16) {
            // padding rows of the last tile (row >= n_out) are written as zeros
#pragma unroll
            for (int c = 0; c < 4; ++c)
                *reinterpret_cast<uint4*>(tbase + (4 * sl + c) * 2048) =
                    make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            continue;
        } else {
            float wmin, wmax;
            if (q.full) {  // bf16x2 min/max (exact), halves folded at the end
                __nv_bfloat162 mn = *reinterpret_cast<const __nv_bfloat162*>(&v[0]), mx = mn;
#pragma unroll
                for (int i = 1; i < 16; ++i) {
                    const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&v[i]);
                    mn = __hmin2(mn, h);
                    mx = __hmax2(mx, h);
                }
                wmin = fminf(__low2float(mn), __high2float(mn));
                wmax = fmaxf(__low2float(mx), __high2float(mx));
            } else {
                wmin = __int_as_float(0x7f800000);
                wmax = -__int_as_float(0x7f800000);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    if (e < q.valid) {
                        wmin = fminf(wmin, elem(e));
                        wmax = fmaxf(wmax, elem(e));
                    }
                }
            }
            wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, 1));
            wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, 1));
            wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, 2));
            wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, 2));
            const bool row_ok = q.row < n_out;
            if (!row_ok) wmin = wmax = 0.0f;
            const group_grid gg = make_grid(wmin, wmax, BITS, sym != 0);
            const int off = sym ? (1 << (BITS - 1)) - 1 : 0;
            if (sl == 0) {
                const size_t sidx = (static_cast<size_t>(nt) * G + q.g) * 128 + r;
                if (scale) scale[sidx] = row_ok ? static_cast<float>(gg.step) : 0.0f;
                if (zero) zero[sidx] = row_ok ? gg.zero_f : 0.0f;
                if (row_ok && step64) {
                    step64[q.row * G + q.g] = gg.step;
                    zero64[q.row * G + q.g] = gg.zero;
                }
            }
            // Fast path: xf = (w - zero) * rcp(step) in fp32 (|error| < 1e-4 for
            // |xf| <= 255; |xf| <= hi by construction); away
            // from a tie (|xf - rint(xf)| <= 0.5 - margin) floor(x + 0.5) ==
            // rint(xf) and lies in [lo, hi].
            // Near ties / non-finite values take quant_code_exact. A flat
            // group (step 0) has rcp 0: every code is 0, as the reference.
            const float zf = gg.zero_f;
            // a step below FLT_MIN is a denormal float: rcp would be inexact,
            // so NaN flags every code for the exact path
            const float rf = gg.step == 0.0 ? 0.0f : (gg.step < 1.1754943508222875e-38 ? __int_as_float(0x7fc00000) : gg.rcp_f);
            using SP = slice_pack<BITS>;
            uint32_t words[SP::NW];
            SP::init_words(words, sym != 0);
            uint32_t code15[2] = {0u, 0u};  // 3-bit pair 15 (codes 30, 31)
            // phase 1, branch-free (full ILP across the 32 codes): fast codes
            // packed, near-tie / non-finite codes flagged in `slow`
            // explicit __fmaf_rn (the pair path's FFMA2 form), so phase 2 recomputes the
            // very bits phase 1 packed
            auto fast_bits = [&](float x) { return __float_as_uint(__fmaf_rn(__fsub_rn(x, zf), rf, kMagicF)); };
            uint32_t slow = 0;
            auto phase1 = [&](auto full) {
                constexpr bool kFull = decltype(full)::value;  // all 32 codes valid
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const float x = elem(e);
                    const float xd = __fsub_rn(x, zf);
                    const float nm = __fmaf_rn(xd, rf, kMagicF);
                    const float d = __fmaf_rn(xd, rf, -(nm - kMagicF));  // NaN for non-finite xf
                    uint32_t bits = __float_as_uint(nm);
                    const uint32_t flag = fabsf(d) <= 0.5f - kTieMargin ? 0u : (1u << e);
                    if (!kFull && e >= q.valid) {
                        bits = kMagicBits;  // padding: signed code 0
                    } else {
                        slow |= flag;
                    }
                    if (SP::split3(e)) {
                        code15[e & 1] = bits - kMagicBits + static_cast<uint32_t>(off);
                    } else {
                        words[SP::word_of(e)] += bits << SP::shift_of(e);
                    }
                }
            };
            if (q.full) {
#if HP_K1_PAIRS
                // ok: bit 31-e set <=> element e is away from a tie (funnel
                // shift of the sign bit of e, one SHF per element)
                const float tm = 0.5f - kTieMargin;
                const uint64_t nzf2 = splat2(-zf), rf2 = splat2(rf), mg2 = splat2(kMagicF),
                               neg1 = splat2(-1.0f), nt2 = splat2(-tm * tm);
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
#else
                phase1(std::true_type{});
#endif
            } else {
                phase1(std::false_type{});
                if (slow) {  // stage the ragged slice for the exact path (own slot; no copy in flight)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        buf[cur][i][tid] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
                }
            }
            // phase 2 (~0.3% of codes): the exact fp64 code replaces the fast
            // one. A rolled loop over the flagged codes (one copy of the fp64
            // sequence keeps the kernel small); registers are selected, not
            // indexed, so nothing goes to local memory.
            while (slow) {
                const int e = __ffs(slow) - 1;
                slow &= slow - 1;
                // the slice is in this thread's shared-memory slot (ragged
                // slices were copied there above): no dynamically indexed
                // register array, so nothing goes to local memory
                const uint16_t* sb = reinterpret_cast<const uint16_t*>(&buf[cur][e >> 3][tid]);
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
    cp_async_wait<0>();
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
                              double* zero64, cudaStream_t st) {
    const int G = static_cast<int>(ceil_div64(k_in, 128));
    // rows up to the 128-row tile boundary: padding rows get code 0 / scale 0
    const int64_t items = ceil_div64(n_out, 128) * (128 / kQRows) * G;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const unsigned grid = static_cast<unsigned>(items < int64_t(HP_K1_CTAS) * sms ? items : int64_t(HP_K1_CTAS) * sms);
    auto* wp = static_cast<const __nv_bfloat16*>(w);
    auto* pp = static_cast<uint8_t*>(packed);
    switch (bits) {
        case 3: quant_pack_kernel<3><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, items, pp, scale, zero, step64, zero64); break;
        case 4: quant_pack_kernel<4><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, items, pp, scale, zero, step64, zero64); break;
        case 8: quant_pack_kernel<8><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, items, pp, scale, zero, step64, zero64); break;
        case 16: quant_pack_kernel<16><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, items, pp, scale, zero, step64, zero64); break;
        default: return cudaErrorInvalidValue;
    }
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
