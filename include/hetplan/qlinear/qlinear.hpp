#pragma once
// hetplan::qlinear -- the layer forward the reference only models
// (memcost.cpp:33 op set, indicator.cpp:53 dequant):
//   y[m x n_out] = epi(x[m x k_in] . dequant(W)^T) (+ residual)
// decode (K3, m = xi tokens) and prefill (K4, m = eta*s) schedules, both on
// tcgen05 tensor cores with the dequantized weights in tensor memory.
// Header-only over hp_capi.h; errors are the reference's exception types.

#include <cstddef>
#include <cstdint>

#include "hetplan/quant/quant.hpp"
#include "hetplan/status.hpp"
#include "hp_capi.h"

namespace hetplan::qlinear {

enum class phase { prefill = HP_PREFILL, decode = HP_DECODE };  // memcost.hpp:14 order
enum class epilogue { none = HP_EPI_NONE, relu = HP_EPI_RELU };

// Device workspace for (w, m, phase); zero it once, kernels leave it zeroed.
inline std::size_t workspace_bytes(const quant::packed_weight& w, std::int64_t m, phase ph) {
    return hp_qlinear_workspace_bytes(w.c(), m, static_cast<int>(ph));
}

inline void forward(const quant::packed_weight& w, const void* x, std::int64_t ldx, std::int64_t m,
                    void* y, std::int64_t ldy, phase ph, void* workspace, std::size_t ws_bytes,
                    void* stream, const void* residual = nullptr, std::int64_t ldr = 0,
                    epilogue epi = epilogue::none) {
    check(hp_qlinear(w.c(), x, ldx, m, y, ldy, residual, residual ? (ldr ? ldr : ldy) : 0,
                     static_cast<int>(epi), static_cast<int>(ph), workspace, ws_bytes, stream));
}

}  // namespace hetplan::qlinear
