// Test-side stand-in for latcost.cpp (needs Eigen, absent): the predict
// dot products of the header contract latcost.hpp:6-13 (clamped at zero).
#include <stdexcept>

#include "hetplan/latcost/latcost.hpp"

namespace hetplan::latcost {
std::array<double, prefill_feature_count> prefill_features(double v, double s) {
    return {1.0, v, s, v * s, v * s * s};
}
std::array<double, decode_feature_count> decode_features(double v, double s, double t) {
    return {1.0, v, v * (t + s), t + s};
}
static double dot(const latency_model& m, const group_key& k, const double* f, int n) {
    auto it = m.coeffs.find(k);
    if (it == m.coeffs.end()) throw std::runtime_error("latcost shim: unknown group");
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += it->second[i] * f[i];
    return acc > 0.0 ? acc : 0.0;
}
double predict_prefill(const latency_model& m, const std::string& d, int bit, double v, double s) {
    auto f = prefill_features(v, s);
    return dot(m, {d, bit, phase::prefill}, f.data(), prefill_feature_count);
}
double predict_decode(const latency_model& m, const std::string& d, int bit, double v, double s,
                      double t) {
    auto f = decode_features(v, s, t);
    return dot(m, {d, bit, phase::decode}, f.data(), decode_feature_count);
}
}  // namespace hetplan::latcost
