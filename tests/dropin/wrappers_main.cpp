// C++ face of the C-ABI (include/hetplan/{quant,qlinear,status}.hpp): the
// reference's exception contract must hold across the boundary. CPU only --
// every call below fails argument validation before any device access;
// on a machine without a GPU, device calls must fail with runtime_error.
#include <cstdio>
#include <stdexcept>

#include "hetplan/qlinear/qlinear.hpp"
#include "hetplan/quant/quant.hpp"

using namespace hetplan;

template <class E, class F>
static int expect(const char* what, F f) {
    try {
        f();
    } catch (const E&) {
        return 0;
    } catch (const std::exception& e) {
        std::printf("FAIL %s: wrong exception: %s\n", what, e.what());
        return 1;
    }
    std::printf("FAIL %s: no exception\n", what);
    return 1;
}

int main() {
    int bad = 0;
    char dummy[64];
    if (quant::packed_bytes(128, 256, 4) != 128 * 256 / 2) {
        std::printf("FAIL packed_bytes\n");
        ++bad;
    }
    bad += expect<std::invalid_argument>("packed_bytes bits 5",
                                         [] { quant::packed_bytes(128, 128, 5); });
    bad += expect<std::invalid_argument>("quantize_pack bits 5", [&] {
        quant::quantize_pack(dummy, 128, 128, 128, 5, quant::quant_scheme::symmetric, dummy,
                             reinterpret_cast<float*>(dummy), nullptr, nullptr);
    });
    bad += expect<std::invalid_argument>("quantize_pack stochastic", [&] {
        quant::quantize_pack(dummy, 128, 128, 128, 4, quant::quant_scheme::symmetric, dummy,
                             reinterpret_cast<float*>(dummy), nullptr, nullptr, nullptr, nullptr,
                             quant::rounding_mode::stochastic);
    });
    quant::packed_weight w(128, 128, 4, quant::quant_scheme::symmetric, dummy,
                           reinterpret_cast<float*>(dummy), nullptr);
    bad += expect<std::invalid_argument>("qlinear m=-1", [&] {
        qlinear::forward(w, dummy, 128, -1, dummy, 128, qlinear::phase::decode, nullptr, 0, nullptr);
    });
    if (!hp_device_ok())
        bad += expect<std::runtime_error>("qlinear without a device", [&] {
            qlinear::forward(w, dummy, 128, 8, dummy, 128, qlinear::phase::decode, nullptr, 0,
                             nullptr);
        });
    std::printf(bad ? "wrappers: %d failures\n" : "wrappers: ok\n", bad);
    return bad ? 1 : 0;
}
