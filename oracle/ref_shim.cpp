// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" wrappers around the reference's OWN code (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load the resulting libhetplan_ref.so, and only as the
// checker or the timed CPU baseline.
//
// * The reference quantizer is a file-local helper in an anonymous namespace
//   (/root/reference/proj/src/indicator.cpp:13-56). It is reachable only by
//   textually including that TU here, so indicator.cpp is NOT compiled
//   separately (see Makefile) — this TU is its one definition.
// * latcost.cpp needs Eigen (absent). The optimizer only needs the two
//   predict_* dot products and the feature expansions
//   (/root/reference/proj/src/latcost.cpp:60-67,196-212); they are restated
//   below from the header contract (latcost.hpp:6-13) — 10 lines of
//   arithmetic, not the OLS fitter.
// * The plan JSON reader/writer is CLI-private
//   (/root/reference/proj/tools/hetplan_main.cpp:190-273, needs CLI11); the
//   schema is restated here with nlohmann-json for the fixture generator.

#include INDICATOR_CPP  // "/root/reference/proj/src/indicator.cpp"

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <json.hpp>

#include "hetplan/config.hpp"
#include "hetplan/latcost/latcost.hpp"
#include "hetplan/memcost/memcost.hpp"
#include "hetplan/optimizer/planner.hpp"
#include "hetplan/pipesim/pipesim.hpp"
#include "hetplan/types.hpp"

// ---- latcost shim (latcost.hpp:6-13 contract; latcost.cpp:60-67,196-212) --
namespace hetplan::latcost {

std::array<double, prefill_feature_count> prefill_features(double v, double s) {
    return {1.0, v, s, v * s, v * s * s};
}
std::array<double, decode_feature_count> decode_features(double v, double s,
                                                         double t) {
    return {1.0, v, v * (t + s), t + s};
}
bool latency_model::has_group(const std::string& device, int bit,
                              phase ph) const {
    return coeffs.count(group_key{device, bit, ph}) != 0;
}
static const std::vector<double>& shim_coeffs(const latency_model& m,
                                              const std::string& dev, int bit,
                                              phase ph) {
    auto it = m.coeffs.find(group_key{dev, bit, ph});
    if (it == m.coeffs.end())
        throw std::runtime_error("latcost shim: no group " + dev + "/" +
                                 std::to_string(bit));
    return it->second;
}
double predict_prefill(const latency_model& m, const std::string& device,
                       int bit, double v, double s) {
    const auto& c = shim_coeffs(m, device, bit, phase::prefill);
    auto f = prefill_features(v, s);
    double acc = 0.0;
    for (int i = 0; i < prefill_feature_count; ++i) acc += c[i] * f[i];
    return std::max(0.0, acc);
}
double predict_decode(const latency_model& m, const std::string& device,
                      int bit, double v, double s, double t) {
    const auto& c = shim_coeffs(m, device, bit, phase::decode);
    auto f = decode_features(v, s, t);
    double acc = 0.0;
    for (int i = 0; i < decode_feature_count; ++i) acc += c[i] * f[i];
    return std::max(0.0, acc);
}

}  // namespace hetplan::latcost

namespace {

thread_local std::string g_err;

int fail_code(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 2;
    if (dynamic_cast<const hetplan::infeasible_error*>(&e)) return 3;
    return 1;
}

int write_str(const std::string& s, char* out, int64_t cap) {
    if (static_cast<int64_t>(s.size()) + 1 > cap) {
        g_err = "output buffer too small";
        return 1;
    }
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

hetplan::model_spec model_from(const int64_t* f) {
    hetplan::model_spec m;
    m.name = "custom";
    m.num_layers = static_cast<int>(f[0]);
    m.h1 = f[1];
    m.h2 = f[2];
    m.num_heads = static_cast<int>(f[3]);
    m.vocab_s = f[4];
    m.pos_s = f[5];
    m.d_t = f[6];
    m.d_p = f[7];
    m.norm = f[8] == 0 ? hetplan::norm_kind::standard : hetplan::norm_kind::rms;
    return m;
}

}  // namespace

using namespace hetplan;

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Reference quantize() (indicator.cpp:19-56) over one vector; `out` receives
// the dequantized doubles exactly as the reference returns them.
int ref_quantize(const double* w, int64_t n, int bit, int scheme, int rounding,
                 uint64_t seed, double* out) {
    try {
        indicator::quantizer_spec q;
        q.scheme = scheme == 0 ? indicator::quant_scheme::asymmetric
                               : indicator::quant_scheme::symmetric;
        q.rounding = rounding == 0 ? indicator::rounding_mode::nearest
                                   : indicator::rounding_mode::stochastic;
        std::mt19937_64 rng(seed);
        std::vector<double> v(w, w + n);
        auto r = indicator::quantize(v, bit, q, &rng);
        std::copy(r.begin(), r.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

int ref_scaling_factor(double w_min, double w_max, int bit, int scheme,
                       double* out) {
    try {
        *out = indicator::scaling_factor(
            w_min, w_max, bit,
            scheme == 0 ? indicator::quant_scheme::asymmetric
                        : indicator::quant_scheme::symmetric);
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

int ref_g_of_x(double mean, double var, int rounding, double* out) {
    try {
        *out = indicator::g_of_x(mean, var,
                                 rounding == 0
                                     ? indicator::rounding_mode::nearest
                                     : indicator::rounding_mode::stochastic);
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

// stats CSV (indicator.cpp:129-181) -> omega CSV (indicator.cpp:183-193)
int ref_indicator_csv(const char* stats_csv, const int* bits, int nbits,
                      int scheme, int rounding, char* out, int64_t cap) {
    try {
        auto layers = indicator::parse_layer_stats(stats_csv);
        indicator::quantizer_spec q;
        q.scheme = scheme == 0 ? indicator::quant_scheme::asymmetric
                               : indicator::quant_scheme::symmetric;
        q.rounding = rounding == 0 ? indicator::rounding_mode::nearest
                                   : indicator::rounding_mode::stochastic;
        auto t = indicator::build_indicator_table(
            layers, bitwidth_set(bits, bits + nbits), q);
        return write_str(indicator::serialize_indicator_table(t), out, cap);
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

int ref_mc_output_variance(const double* w, int64_t n, double mean,
                           double var, int bit, int scheme, int rounding,
                           int64_t samples, uint64_t seed, double* out4) {
    try {
        indicator::quantizer_spec q;
        q.scheme = scheme == 0 ? indicator::quant_scheme::asymmetric
                               : indicator::quant_scheme::symmetric;
        q.rounding = rounding == 0 ? indicator::rounding_mode::nearest
                                   : indicator::rounding_mode::stochastic;
        auto r = indicator::mc_output_variance(std::vector<double>(w, w + n),
                                               mean, var, bit, q, samples,
                                               seed);
        out4[0] = r.total_var;
        out4[1] = r.extra_var;
        out4[2] = r.se_total;
        out4[3] = static_cast<double>(r.n);
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

// memcost (memcost.cpp:22-72); model fields: L,h1,h2,heads,vocab,pos,d_t,d_p,norm
int ref_memcost(const int64_t* mf, int bit, int64_t v, int64_t s, int64_t n,
                int64_t* out3) {
    try {
        auto m = model_from(mf);
        out3[0] = memcost::embed_mem_bytes(m);
        out3[1] = memcost::decoder_weight_bytes(m, bit);
        out3[2] = memcost::kv_cache_bytes(m, v, s, n, 16);
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

int ref_preset(const char* name, int64_t* mf) {
    try {
        auto m = model_preset(name);
        mf[0] = m.num_layers; mf[1] = m.h1; mf[2] = m.h2; mf[3] = m.num_heads;
        mf[4] = m.vocab_s; mf[5] = m.pos_s; mf[6] = m.d_t; mf[7] = m.d_p;
        mf[8] = m.norm == norm_kind::standard ? 0 : 1;
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

// pipesim::make_schedule (pipesim.cpp:22-46)
int ref_make_schedule(int B, int eta, int xi, int* sizes, int* groups,
                      int* n_batches, int* n_groups, int cap) {
    try {
        auto s = pipesim::make_schedule(B, eta, xi);
        if (static_cast<int>(s.prefill_sizes.size()) > cap)
            throw std::runtime_error("capacity");
        for (size_t k = 0; k < s.prefill_sizes.size(); ++k) {
            sizes[k] = s.prefill_sizes[k];
            groups[k] = s.group_of_prefill[k];
        }
        *n_batches = static_cast<int>(s.prefill_sizes.size());
        *n_groups = s.num_groups;
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

// pipesim::simulate + analytic_latency (pipesim.cpp:200-264). costs: per stage
// {pre_s, dec_s, comm_pre_s, comm_dec_s}. out: makespan, bubble, analytic,
// n_events; busy[n_stages]; timeline rows (stage,kind,index,token,start,end)
int ref_simulate(const double* costs, int n_stages, int B, int eta, int xi,
                 int n, double* out4, double* busy, double* timeline,
                 int64_t timeline_cap) {
    try {
        std::vector<pipesim::stage_cost> st(n_stages);
        for (int j = 0; j < n_stages; ++j)
            st[j] = {costs[4 * j], costs[4 * j + 1], costs[4 * j + 2],
                     costs[4 * j + 3], 0.0};
        auto sched = pipesim::make_schedule(B, eta, xi);
        auto r = pipesim::simulate(st, sched, n, timeline != nullptr);
        out4[0] = r.makespan_s;
        out4[1] = r.bubble_fraction;
        out4[2] = pipesim::analytic_latency(st, B, eta, xi, n);
        out4[3] = static_cast<double>(r.timeline.size());
        for (int j = 0; j < n_stages; ++j) busy[j] = r.stage_busy_s[j];
        if (timeline) {
            if (static_cast<int64_t>(r.timeline.size()) > timeline_cap)
                throw std::runtime_error("timeline capacity");
            for (size_t k = 0; k < r.timeline.size(); ++k) {
                const auto& e = r.timeline[k];
                double* row = timeline + 6 * k;
                row[0] = e.stage;
                row[1] = e.kind == pipesim::unit_kind::prefill ? 0 : 1;
                row[2] = e.index;
                row[3] = e.token;
                row[4] = e.start;
                row[5] = e.end;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

// validate_plan (types.cpp:85-123) on plan fields.
int ref_validate_plan(const int* device_order, int n_dev, const int* stages3,
                      int n_stages, const int* layer_bits, int L, int eta,
                      int xi, const double* objective7, int B, int s, int n,
                      const int* bits, int nbits) {
    try {
        plan p;
        p.device_order.assign(device_order, device_order + n_dev);
        for (int j = 0; j < n_stages; ++j)
            p.stages.push_back(
                {stages3[3 * j], stages3[3 * j + 1], stages3[3 * j + 2]});
        p.layer_bits.assign(layer_bits, layer_bits + L);
        p.eta = eta;
        p.xi = xi;
        p.objective = {objective7[0], objective7[1], objective7[2],
                       objective7[3], objective7[4], objective7[5],
                       objective7[6]};
        validate_plan(p, L, workload{B, s, n}, bitwidth_set(bits, bits + nbits),
                      n_dev);
        return 0;
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

// Reference planner (optimizer_planner.cpp:79-170) for plan fixtures.
// config_json: parse_config document; omega_csv: indicator table;
// lat_json: {"<device>": {"<bit>": {"prefill":[5], "decode":[4]}}}.
// Writes a plan document following hetplan_main.cpp:190-224.
int ref_best_plan(const char* config_json, const char* omega_csv,
                  const char* lat_json, double theta, int group,
                  int heuristic, double time_limit_s, char* out, int64_t cap) {
    try {
        auto rs = parse_config(config_json);
        auto omega = indicator::parse_indicator_table(omega_csv);
        latcost::latency_model lat;
        auto lj = nlohmann::json::parse(lat_json);
        for (auto& [dev, per_bit] : lj.items())
            for (auto& [bit, ph] : per_bit.items()) {
                lat.coeffs[{dev, std::stoi(bit), latcost::phase::prefill}] =
                    ph.at("prefill").get<std::vector<double>>();
                lat.coeffs[{dev, std::stoi(bit), latcost::phase::decode}] =
                    ph.at("decode").get<std::vector<double>>();
            }
        optimizer::plan_options opt;
        opt.theta = theta;
        opt.group = group;
        opt.heuristic = heuristic != 0;
        opt.time_limit_s = time_limit_s;
        auto res = optimizer::best_plan(rs.model, rs.cluster, rs.load, rs.bits,
                                        lat, omega, opt);
        if (!res.feasible) throw infeasible_error("no feasible plan");
        const plan& p = res.best;
        nlohmann::ordered_json j;
        j["format_version"] = 1;
        j["model"] = rs.model.name;
        j["num_layers"] = rs.model.num_layers;
        j["bits"] = rs.bits;
        j["theta"] = theta;
        j["workload"] = {{"global_bz", rs.load.global_bz},
                         {"s", rs.load.prompt_len},
                         {"n", rs.load.gen_len}};
        j["eta"] = p.eta;
        j["xi"] = p.xi;
        j["device_order"] = p.device_order;
        nlohmann::ordered_json names = nlohmann::ordered_json::array();
        for (int d : p.device_order) names.push_back(rs.cluster.devices[d].name);
        j["devices"] = names;
        nlohmann::ordered_json stages = nlohmann::ordered_json::array();
        for (size_t k = 0; k < p.stages.size(); ++k)
            stages.push_back(
                {{"device_index", p.device_order[k]},
                 {"device", rs.cluster.devices[p.device_order[k]].name},
                 {"layers", {p.stages[k].begin, p.stages[k].end}}});
        j["stages"] = stages;
        j["layer_bits"] = p.layer_bits;
        j["objective"] = {{"t_max_pre", p.objective.t_max_pre},
                          {"t_max_dec", p.objective.t_max_dec},
                          {"t_pre_total", p.objective.t_pre_total},
                          {"t_dec_total", p.objective.t_dec_total},
                          {"omega_sum", p.objective.omega_sum},
                          {"theta", p.objective.theta},
                          {"total", p.objective.total}};
        j["optimal"] = res.optimal;
        j["seed"] = 0;
        validate_plan(p, rs.model.num_layers, rs.load, rs.bits,
                      static_cast<int>(p.device_order.size()));
        return write_str(j.dump(2) + "\n", out, cap);
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

}  // extern "C"
