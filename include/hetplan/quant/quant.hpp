#pragma once
// hetplan::quant -- K1 (group-wise quantize + pack) behind the reference's
// quantizer semantics: the file-local quantize() of
// /root/reference/proj/src/indicator.cpp:19-56 (step from scaling_factor,
// :82-91), applied to every group of 128 consecutive weights along k_in.
// Header-only over hp_capi.h; device pointers are caller-owned, calls are
// stream-ordered, errors are the reference's exception types (status.hpp).

#include <cstdint>

#include "hetplan/indicator/indicator.hpp"
#include "hetplan/status.hpp"
#include "hp_capi.h"

namespace hetplan::quant {

using indicator::quant_scheme;
using indicator::rounding_mode;

constexpr int group_size = HP_GROUP;

// Packed code bytes of an [n_out x k_in] weight: ceil(n_out*k_in*bits/8)
// for 128-aligned shapes, the memcost packed-size contract
// (memcost.cpp:15-18). Throws std::invalid_argument for unsupported bits.
inline std::int64_t packed_bytes(std::int64_t n_out, std::int64_t k_in, int bits) {
    const std::int64_t b = hp_packed_bytes(n_out, k_in, bits);
    if (b < 0) check(HP_EINVAL);
    return b;
}
inline std::int64_t scale_count(std::int64_t n_out, std::int64_t k_in) {
    return hp_scale_count(n_out, k_in);
}

// Non-owning view of a packed weight (hp_qweight).
struct packed_weight {
    hp_qweight w{};
    packed_weight() = default;
    packed_weight(std::int64_t n_out, std::int64_t k_in, int bits, quant_scheme s,
                  const void* packed, const float* scale, const float* zero)
        : w{n_out, k_in, bits, static_cast<int32_t>(s), packed, scale, zero} {}
    const hp_qweight* c() const { return &w; }
};

// w: device bf16 [n_out x ldw]. step64/zero64 (optional, device fp64
// [n_out x groups]) receive the reference's per-group step and grid origin.
inline packed_weight quantize_pack(const void* w, std::int64_t n_out, std::int64_t k_in,
                                   std::int64_t ldw, int bits, quant_scheme scheme,
                                   void* packed, float* scale, float* zero, void* stream,
                                   double* step64 = nullptr, double* zero64 = nullptr,
                                   rounding_mode rounding = rounding_mode::nearest) {
    check(hp_quant_pack(w, n_out, k_in, ldw, bits, static_cast<int>(scheme),
                        static_cast<int>(rounding), packed, scale, zero, step64, zero64, stream));
    return packed_weight(n_out, k_in, bits, scheme, packed, scale, scheme == quant_scheme::asymmetric ? zero : nullptr);
}

// Stored codes u8 [n_out x k_in] (symmetric codes carry +hi) and fp32
// scale/zero [n_out x groups], row-major; any output may be null.
inline void unpack(const packed_weight& w, void* codes, float* scale_rm, float* zero_rm,
                   void* stream) {
    check(hp_quant_unpack(w.c(), codes, scale_rm, zero_rm, stream));
}

// bf16 [n_out x k_in] = zero + code*step (indicator.cpp:53).
inline void dequantize(const packed_weight& w, void* w_bf16, void* stream) {
    check(hp_dequant(w.c(), w_bf16, stream));
}

}  // namespace hetplan::quant
