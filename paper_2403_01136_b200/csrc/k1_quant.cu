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
// Fast path: x = ((float)w - (float)zero) * rcp_f32(step). Its absolute
// error is < 1e-4 for |x| <= 255, so whenever frac(x + 0.5)
// lies in [1e-3, 1 - 1e-3] the rounded code equals the reference's; other
// elements (ties, near-ties, non-finite) take the exact fp64 sequence
// __dsub_rn / __ddiv_rn / __dadd_rn / floor / clamp. About 0.3% of bf16
// weights take the slow path.
#include <cuda_bf16.h>
#include <cstdint>

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

// Signed grid code of one element (reference quantize() inner loop).
__device__ __forceinline__ int quant_code(float w, const group_grid& g) {
    if (g.step == 0.0) return 0;  // flat group: out = zero (indicator.cpp:39-41)
    const float x = (w - g.zero_f) * g.rcp_f + 0.5f;
    const float fl = floorf(x);
    const float fr = x - fl;
    double sn;
    if (fr >= kTieMargin && fr <= 1.0f - kTieMargin) {
        sn = static_cast<double>(fl);
    } else {
        const double scaled =
            __ddiv_rn(__dsub_rn(static_cast<double>(w), g.zero), g.step);
        sn = floor(__dadd_rn(scaled, 0.5));
    }
    sn = sn < g.lo ? g.lo : (g.hi < sn ? g.hi : sn);  // std::clamp
    return static_cast<int>(sn);
}

// One thread per (row, 32-k slice): a warp covers 8 rows x one 128-k group
// (lane = 4 * row + slice), a 256-thread CTA 64 rows of one group. Each
// thread loads its slice with 4 independent 16-byte loads, the group's
// min/max is a 2-step shuffle over the 4 lanes of the row, and the thread
// emits exactly its slice's part of the tile layout (layout.cuh): 4-bit one
// 16 B row entry of chunk s, 8-bit two (chunks 2s, 2s+1), 3-bit word s of
// chunks 0..2, 16-bit four. For a fixed chunk the 8 rows of a warp are 128
// contiguous bytes, so every store instruction writes whole lines.
constexpr int kQRows = 64;  // rows per CTA

template <int BITS>
__global__ void __launch_bounds__(256)
    quant_pack_kernel(const __nv_bfloat16* __restrict__ w, int64_t n_out,
                      int64_t k_in, int64_t ldw, int G, int sym,
                      uint8_t* __restrict__ packed, float* __restrict__ scale,
                      float* __restrict__ zero, double* __restrict__ step64,
                      double* __restrict__ zero64) {
    const int lane = threadIdx.x & 31;
    const int sl = lane & 3;
    const int g = blockIdx.x;
    const int64_t row = static_cast<int64_t>(blockIdx.y) * kQRows + (threadIdx.x >> 5) * 8 + (lane >> 2);
    const int64_t nt = row >> 7;
    const int r = static_cast<int>(row & 127);
    const int64_t k0 = static_cast<int64_t>(g) * 128 + sl * 32;
    const int cnt = static_cast<int>(k_in - k0 <= 0 ? 0 : (k_in - k0 < 32 ? k_in - k0 : 32));
    const bool row_ok = row < n_out;
    const int valid = row_ok ? cnt : 0;

    // slice values (padding = 0, excluded from min/max)
    uint32_t v[16];
    const __nv_bfloat16* src = w + row * ldw + k0;
    if (valid == 32 && (ldw % 8 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        uint4 q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = __ldcs(reinterpret_cast<const uint4*>(src) + i);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[4 * i] = q[i].x; v[4 * i + 1] = q[i].y; v[4 * i + 2] = q[i].z; v[4 * i + 3] = q[i].w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint32_t lo = 2 * i < valid ? __bfloat16_as_ushort(src[2 * i]) : 0u;
            const uint32_t hi = 2 * i + 1 < valid ? __bfloat16_as_ushort(src[2 * i + 1]) : 0u;
            v[i] = lo | (hi << 16);
        }
    }
    auto elem = [&](int e) { return __uint_as_float((e & 1) ? (v[e >> 1] & 0xFFFF0000u) : (v[e >> 1] << 16)); };
    uint8_t* tbase = packed + (static_cast<size_t>(nt) * G + g) * tile_bytes(BITS) + r * 16;

    if constexpr (BITS == 16) {
        // padding rows of the last tile (row >= n_out) are written as zeros
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(tbase + (4 * sl + c) * 2048) =
                make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    } else {
        float wmin = __int_as_float(0x7f800000), wmax = -__int_as_float(0x7f800000);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            if (e < valid) {
                wmin = fminf(wmin, elem(e));
                wmax = fmaxf(wmax, elem(e));
            }
        }
        wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, 1));
        wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, 1));
        wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, 2));
        wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, 2));
        if (!row_ok) wmin = wmax = 0.0f;
        const group_grid gg = make_grid(wmin, wmax, BITS, sym != 0);
        const int off = sym ? (1 << (BITS - 1)) - 1 : 0;
        if (sl == 0) {
            const size_t sidx = (static_cast<size_t>(nt) * G + g) * 128 + r;
            if (scale) scale[sidx] = row_ok ? static_cast<float>(gg.step) : 0.0f;
            if (zero) zero[sidx] = row_ok ? gg.zero_f : 0.0f;
            if (row_ok && step64) {
                step64[row * G + g] = gg.step;
                zero64[row * G + g] = gg.zero;
            }
        }
        // slice-local words: codes e < 32 of this slice at the positions
        // locate_code gives for kk = e (the slice index only selects where
        // the words land, below)
        uint32_t words[BITS == 3 ? 12 : BITS];
#pragma unroll
        for (int i = 0; i < (BITS == 3 ? 12 : BITS); ++i) words[i] = 0;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const int q = e < valid ? quant_code(elem(e), gg) : 0;  // padding: signed code 0
            const uint32_t sc = static_cast<uint32_t>(q + off);
            if constexpr (BITS == 3) {
                put_code3(words, e, sc);
            } else {
                const code_pos p = locate_code(BITS, e);
                words[p.chunk * 4 + p.word] |= sc << p.shift;
            }
        }
        if constexpr (BITS == 4) {
            *reinterpret_cast<uint4*>(tbase + sl * 2048) = make_uint4(words[0], words[1], words[2], words[3]);
        } else if constexpr (BITS == 8) {
            *reinterpret_cast<uint4*>(tbase + (2 * sl) * 2048) = make_uint4(words[0], words[1], words[2], words[3]);
            *reinterpret_cast<uint4*>(tbase + (2 * sl + 1) * 2048) = make_uint4(words[4], words[5], words[6], words[7]);
        } else {
#pragma unroll
            for (int b = 0; b < 3; ++b) *reinterpret_cast<uint32_t*>(tbase + b * 2048 + sl * 4) = words[b * 4];
        }
    }
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
    dequant_slice32<BITS, SYM>(base, slice, s, z, bf16x2_splat_bits(s),
                               bf16x2_splat_bits(z), v);
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
    const dim3 grid(G, static_cast<unsigned>(ceil_div64(n_out, 128) * (128 / kQRows)));
    auto* wp = static_cast<const __nv_bfloat16*>(w);
    auto* pp = static_cast<uint8_t*>(packed);
    switch (bits) {
        case 3: quant_pack_kernel<3><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, pp, scale, zero, step64, zero64); break;
        case 4: quant_pack_kernel<4><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, pp, scale, zero, step64, zero64); break;
        case 8: quant_pack_kernel<8><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, pp, scale, zero, step64, zero64); break;
        case 16: quant_pack_kernel<16><<<grid, 256, 0, st>>>(wp, n_out, k_in, ldw, G, sym, pp, scale, zero, step64, zero64); break;
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
