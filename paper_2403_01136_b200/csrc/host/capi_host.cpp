// extern "C" surface of the host planning library (include/hp_capi.h,
// "host planning helpers"): the drop-in hetplan:: functions exposed with
// plain types so the parity tests can drive them next to the reference
// build. Exceptions are mapped to hp_status like the rest of the ABI.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hetplan/config.hpp"
#include "hetplan/indicator/indicator.hpp"
#include "hetplan/latcost/latcost.hpp"
#include "hetplan/memcost/memcost.hpp"
#include "hetplan/pipesim/pipesim.hpp"
#include "hetplan/plan/plan_io.hpp"
#include "hetplan/runtime/pipeline.hpp"
#include "hetplan/runtime/microbatch.hpp"
#include <nccl.h>
#include <json.hpp>
#include "hetplan/types.hpp"
#include "hp_capi.h"

namespace hp_detail {
void set_error(const std::string& msg);  // capi.cu
}

namespace {

hp_status from_exception(const std::exception& e) {
    hp_detail::set_error(e.what());
    if (dynamic_cast<const hetplan::infeasible_error*>(&e)) return HP_EINFEASIBLE;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return HP_EINVAL;
    if (dynamic_cast<const hetplan::runtime::pipeline_timeout*>(&e)) return HP_ETIMEOUT;
    return HP_EINTERNAL;
}

hp_status put_string(const std::string& s, char* out, int64_t cap) {
    if (static_cast<int64_t>(s.size()) + 1 > cap) {
        hp_detail::set_error("output buffer too small: need " + std::to_string(s.size() + 1));
        return HP_EINVAL;
    }
    std::memcpy(out, s.c_str(), s.size() + 1);
    return HP_OK;
}

hetplan::model_spec model_of(const int64_t* f) {
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

hetplan::indicator::quantizer_spec qspec(int scheme, int rounding) {
    hetplan::indicator::quantizer_spec q;
    q.scheme = scheme == HP_ASYMMETRIC ? hetplan::indicator::quant_scheme::asymmetric
                                       : hetplan::indicator::quant_scheme::symmetric;
    q.rounding = rounding == HP_NEAREST ? hetplan::indicator::rounding_mode::nearest
                                        : hetplan::indicator::rounding_mode::stochastic;
    return q;
}

}  // namespace

extern "C" {

hp_status hp_host_scaling_factor(double w_min, double w_max, int bit, int scheme,
                                 double* out) {
    try {
        *out = hetplan::indicator::scaling_factor(w_min, w_max, bit, qspec(scheme, 0).scheme);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_g_of_x(double mean, double var, int rounding, double* out) {
    try {
        *out = hetplan::indicator::g_of_x(mean, var, qspec(1, rounding).rounding);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_indicator_csv(const char* stats_csv, const int* bits, int nbits, int scheme,
                                int rounding, char* out, int64_t cap) {
    try {
        auto layers = hetplan::indicator::parse_layer_stats(stats_csv);
        auto t = hetplan::indicator::build_indicator_table(
            layers, hetplan::bitwidth_set(bits, bits + nbits), qspec(scheme, rounding));
        return put_string(hetplan::indicator::serialize_indicator_table(t), out, cap);
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_omega_from_stats(const double* stats5_per_op, int n_layers, int ops_per_layer,
                                   const int* bits, int nbits, int scheme, int rounding,
                                   double* omega_out) {
    try {
        static const char* names[] = {"qkv", "out", "fc1", "fc2"};
        std::vector<hetplan::indicator::layer_stats> layers(n_layers);
        for (int i = 0; i < n_layers; ++i)
            for (int o = 0; o < ops_per_layer; ++o) {
                const double* s = stats5_per_op + 5 * (i * ops_per_layer + o);
                layers[i].push_back({o < 4 ? names[o] : "op", static_cast<int64_t>(s[0]), s[1],
                                     s[2], s[3], s[4]});
            }
        auto t = hetplan::indicator::build_indicator_table(
            layers, hetplan::bitwidth_set(bits, bits + nbits), qspec(scheme, rounding));
        for (int i = 0; i < n_layers; ++i)
            for (int b = 0; b < nbits; ++b) omega_out[i * nbits + b] = t.omega[i][b];
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_mc_output_variance(const double* w, int64_t d, double x_mean, double x_var,
                                    int bit, int scheme, int rounding, int64_t n_samples,
                                    uint64_t seed, double* out4) {
    try {
        if (!w || !out4 || d <= 0) throw std::invalid_argument("mc: NULL/empty weights");
        const auto r = hetplan::indicator::mc_output_variance(
            std::vector<double>(w, w + d), x_mean, x_var, bit, qspec(scheme, rounding), n_samples,
            seed);
        out4[0] = r.total_var;
        out4[1] = r.extra_var;
        out4[2] = r.se_total;
        out4[3] = static_cast<double>(r.n);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_memcost(const int64_t* model9, int bit, int64_t v, int64_t s, int64_t n,
                          int64_t* out3) {
    try {
        const auto m = model_of(model9);
        out3[0] = hetplan::memcost::embed_mem_bytes(m);
        out3[1] = hetplan::memcost::decoder_weight_bytes(m, bit);
        out3[2] = hetplan::memcost::kv_cache_bytes(m, v, s, n, 16);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_preset(const char* name, int64_t* model9) {
    try {
        const auto m = hetplan::model_preset(name);
        const int64_t f[9] = {m.num_layers, m.h1, m.h2, m.num_heads, m.vocab_s,
                              m.pos_s, m.d_t, m.d_p, m.norm == hetplan::norm_kind::standard ? 0 : 1};
        std::memcpy(model9, f, sizeof f);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_make_schedule(int B, int eta, int xi, int* sizes, int* groups, int* n_batches,
                                int* n_groups, int cap) {
    try {
        const auto s = hetplan::pipesim::make_schedule(B, eta, xi);
        if (static_cast<int>(s.prefill_sizes.size()) > cap)
            throw std::invalid_argument("schedule: capacity");
        for (size_t k = 0; k < s.prefill_sizes.size(); ++k) {
            sizes[k] = s.prefill_sizes[k];
            groups[k] = s.group_of_prefill[k];
        }
        *n_batches = static_cast<int>(s.prefill_sizes.size());
        *n_groups = s.num_groups;
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_simulate(const double* costs4, int n_stages, int B, int eta, int xi, int n,
                           double* out4, double* busy, double* timeline, int64_t timeline_cap) {
    try {
        std::vector<hetplan::pipesim::stage_cost> st(n_stages);
        for (int j = 0; j < n_stages; ++j)
            st[j] = {costs4[4 * j], costs4[4 * j + 1], costs4[4 * j + 2], costs4[4 * j + 3], 0.0};
        const auto sched = hetplan::pipesim::make_schedule(B, eta, xi);
        const auto r = hetplan::pipesim::simulate(st, sched, n, timeline != nullptr);
        out4[0] = r.makespan_s;
        out4[1] = r.bubble_fraction;
        out4[2] = hetplan::pipesim::analytic_latency(st, B, eta, xi, n);
        out4[3] = static_cast<double>(r.timeline.size());
        for (int j = 0; j < n_stages; ++j) busy[j] = r.stage_busy_s[j];
        if (timeline) {
            if (static_cast<int64_t>(r.timeline.size()) > timeline_cap)
                throw std::invalid_argument("simulate: timeline capacity");
            for (size_t k = 0; k < r.timeline.size(); ++k) {
                const auto& e = r.timeline[k];
                double* row = timeline + 6 * k;
                row[0] = e.stage;
                row[1] = e.kind == hetplan::pipesim::unit_kind::prefill ? 0 : 1;
                row[2] = e.index;
                row[3] = e.token;
                row[4] = e.start;
                row[5] = e.end;
            }
        }
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

// Parse + validate a plan document; returns the normalised document (the
// B200 runtime's view: stage.device = stage index) as JSON.
hp_status hp_host_plan_check(const char* plan_json, char* out, int64_t cap) {
    try {
        const auto doc = hetplan::plan_io::parse_plan(plan_json);
        hetplan::plan_io::validate(doc);
        return put_string(hetplan::plan_io::serialize_plan(doc), out, cap);
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_latency_fit(const char* profile_csv, char* out, int64_t cap, int64_t* needed) {
    try {
        if (!profile_csv) throw std::invalid_argument("latency_fit: NULL profile");
        const std::string js = hetplan::latcost::serialize_model(
            hetplan::latcost::fit(hetplan::latcost::ingest_profile(profile_csv)));
        if (needed) *needed = static_cast<int64_t>(js.size()) + 1;
        if (!out || cap < static_cast<int64_t>(js.size()) + 1)
            throw std::invalid_argument("latency_fit: output buffer too small");
        std::memcpy(out, js.c_str(), js.size() + 1);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_host_latency_predict(const char* model_json, const char* device, int bit, int phase,
                                  double v, double s, double t, double* out) {
    try {
        if (!model_json || !device || !out) throw std::invalid_argument("latency_predict: NULL argument");
        const auto m = hetplan::latcost::parse_model(model_json);
        *out = phase == 0 ? hetplan::latcost::predict_prefill(m, device, bit, v, s)
                          : hetplan::latcost::predict_decode(m, device, bit, v, s, t);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

// Static unit order of stage `stage` (kind, index, token triples) for the
// plan — what the executor runs, and what the multi-process tests check.
hp_status hp_host_unit_order(const char* plan_json, const char* model_json, int stage,
                             int* out3, int cap, int* n) {
    try {
        const auto doc = hetplan::plan_io::parse_plan(plan_json);
        nlohmann::ordered_json cfg;
        cfg["model"] = nlohmann::ordered_json::parse(model_json);
        cfg["cluster"]["devices"] = nlohmann::ordered_json::array(
            {{{"name", "b200"}, {"mem_bytes", 1}, {"link_bw_bytes_per_s", 9e11}}});
        cfg["workload"] = {{"B", doc.load.global_bz}, {"s", doc.load.prompt_len}, {"n", doc.load.gen_len}};
        cfg["bits"] = doc.bits;
        const auto rs = hetplan::parse_config(cfg.dump());
        const auto order = hetplan::runtime::static_unit_order(doc, rs.model);
        if (stage < 0 || stage >= static_cast<int>(order.size()))
            throw std::invalid_argument("unit_order: bad stage");
        const auto& u = order[stage];
        if (static_cast<int>(u.size()) > cap) throw std::invalid_argument("unit_order: capacity");
        for (size_t i = 0; i < u.size(); ++i) {
            out3[3 * i] = u[i].kind == hetplan::pipesim::unit_kind::prefill ? 0 : 1;
            out3[3 * i + 1] = u[i].index;
            out3[3 * i + 2] = u[i].token;
        }
        *n = static_cast<int>(u.size());
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

struct hp_pipeline {
    std::unique_ptr<hetplan::runtime::pipeline> impl;
    int64_t units = 0, layers = 0;
};

hp_status hp_nccl_unique_id(void* out128) {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        hp_detail::set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        return HP_ENCCL;
    }
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof id);
    return HP_OK;
}

hp_status hp_pipeline_create(const char* plan_json, const char* model_json, int rank, int world,
                             const void* nccl_ids, const hp_pipeline_options* opt,
                             const hp_weight_set* weights, hp_pipeline** out) {
    try {
        if (!plan_json || !model_json || !out)
            throw std::invalid_argument("pipeline_create: NULL argument");
        const auto doc = hetplan::plan_io::parse_plan(plan_json);
        // the config "model" section, through the drop-in config parser
        nlohmann::ordered_json mj = nlohmann::ordered_json::parse(model_json, nullptr, false);
        if (mj.is_discarded()) throw std::invalid_argument("pipeline_create: bad model JSON");
        nlohmann::ordered_json cfg;
        cfg["model"] = mj;
        cfg["cluster"]["devices"] = nlohmann::ordered_json::array(
            {{{"name", "b200"}, {"mem_bytes", 1}, {"link_bw_bytes_per_s", 9e11}}});
        cfg["workload"] = {{"B", doc.load.global_bz}, {"s", doc.load.prompt_len}, {"n", doc.load.gen_len}};
        cfg["bits"] = doc.bits;
        const auto rs = hetplan::parse_config(cfg.dump());
        hetplan::runtime::pipeline_options po;
        if (opt) {
            po.scheme = opt->scheme;
            po.use_graphs = opt->use_graphs != 0;
            po.instrument = opt->instrument != 0;
            po.sm_budget = opt->sm_budget;
            po.seed = opt->seed;
            po.weight_std = opt->weight_std > 0 ? opt->weight_std : 0.02;
            po.timeout_s = opt->timeout_s;
        }
        hetplan::runtime::weight_set ws;
        if (weights) {
            if (weights->n_layers != doc.num_layers)
                throw std::invalid_argument("pipeline_create: weight set n_layers != plan num_layers");
            auto src = [](const hp_tensor_src& t) {
                hetplan::runtime::tensor_source r;
                r.host = t.host;
                if (t.path) r.path = t.path;
                r.offset = t.offset;
                return r;
            };
            const size_t L4 = static_cast<size_t>(doc.num_layers) * 4;
            if (weights->linear)
                for (size_t i = 0; i < L4; ++i) ws.linear.push_back(src(weights->linear[i]));
            if (weights->norm)
                for (size_t i = 0; i < L4; ++i) ws.norm.push_back(src(weights->norm[i]));
            ws.embed = src(weights->embed);
            ws.pos = src(weights->pos);
            ws.final_norm[0] = src(weights->final_norm[0]);
            ws.final_norm[1] = src(weights->final_norm[1]);
            if (weights->bin_bytes > 0) ws.bin_bytes = weights->bin_bytes;
            po.weights = &ws;
        }
        std::vector<std::array<char, 128>> ids;
        if (world > 1) {
            if (!nccl_ids) throw std::invalid_argument("pipeline_create: nccl_ids required");
            ids.resize(world);
            for (int l = 0; l < world; ++l)
                std::memcpy(ids[l].data(), static_cast<const char*>(nccl_ids) + 128 * l, 128);
        }
        auto h = std::make_unique<hp_pipeline>();
        h->impl = std::make_unique<hetplan::runtime::pipeline>(doc, rs.model, rank, world, ids, po);
        h->layers = doc.p.stages.at(rank).end - doc.p.stages.at(rank).begin;
        h->units = static_cast<int64_t>(
            hetplan::runtime::static_unit_order(doc, rs.model).at(rank).size());
        *out = h.release();
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_pipeline_run(hp_pipeline* p, const int32_t* host_in, int32_t* host_out,
                          double* timing4) {
    try {
        if (!p) throw std::invalid_argument("pipeline_run: NULL pipeline");
        const auto t = p->impl->run(host_in, host_out);
        if (timing4) {
            timing4[0] = t.makespan_s;
            timing4[1] = t.prefill_s;
            timing4[2] = t.decode_s;
            timing4[3] = t.io_s;
        }
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_pipeline_stage_costs(hp_pipeline* p, double* out4) {
    if (!p || !out4) return HP_EINVAL;
    const auto c = p->impl->measured_cost();
    out4[0] = c.pre_s;
    out4[1] = c.dec_s;
    out4[2] = 0.0;
    out4[3] = 0.0;
    return HP_OK;
}

hp_status hp_pipeline_final_hidden(hp_pipeline* p, void* host) {
    try {
        if (!p || !host) throw std::invalid_argument("pipeline_final_hidden: NULL argument");
        p->impl->final_hidden(host);
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_pipeline_load_stats(hp_pipeline* p, double* out4) {
    if (!p || !out4) return HP_EINVAL;
    const auto& l = p->impl->loading();
    out4[0] = l.seconds;
    out4[1] = l.source_bytes;
    out4[2] = l.packed_bytes;
    out4[3] = static_cast<double>(l.bins);
    return HP_OK;
}

hp_status hp_pipeline_kernel_stats(hp_pipeline* p, int kind, double* out4) {
    if (!p || !out4 || kind < 0 || kind > 3) return HP_EINVAL;
    const auto& k = p->impl->stats(kind);
    out4[0] = static_cast<double>(k.launches);
    out4[1] = k.seconds;
    out4[2] = k.bytes;
    out4[3] = k.flops;
    return HP_OK;
}

hp_status hp_pipeline_layer_costs(hp_pipeline* p, int phase, double* out, int64_t cap,
                                  int64_t* n) {
    if (!p || !n || (cap > 0 && !out)) return HP_EINVAL;
    const auto& v = p->impl->layer_costs(phase);
    *n = static_cast<int64_t>(v.size());
    if (cap < *n) {
        hp_detail::set_error("layer_costs: need cap >= " + std::to_string(*n));
        return HP_EINVAL;
    }
    std::copy(v.begin(), v.end(), out);
    return HP_OK;
}

hp_status hp_pipeline_info(hp_pipeline* p, int64_t* out4) {
    if (!p || !out4) return HP_EINVAL;
    out4[0] = p->impl->weight_bytes();
    out4[1] = p->impl->num_kernel_launches_per_round();
    out4[2] = p->units;
    out4[3] = p->layers;
    return HP_OK;
}

void hp_pipeline_destroy(hp_pipeline* p) { delete p; }

struct hp_mbm {
    std::unique_ptr<hetplan::runtime::microbatch_manager> m;
};

hp_status hp_mbm_create(int B, int eta, int xi, int n, hp_mbm** out) {
    try {
        if (!out) throw std::invalid_argument("mbm_create: NULL out");
        auto h = std::make_unique<hp_mbm>();
        h->m = std::make_unique<hetplan::runtime::microbatch_manager>(B, eta, xi, n);
        *out = h.release();
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_mbm_prefill_done(hp_mbm* m, int k, int* ready_group) {
    try {
        if (!m) throw std::invalid_argument("mbm: NULL handle");
        const int g = m->m->prefill_done(k);
        if (ready_group) *ready_group = g;
        return HP_OK;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

hp_status hp_mbm_decode_done(hp_mbm* m, int group, int token, int* finished) {
    try {
        if (!m) throw std::invalid_argument("mbm: NULL handle");
        const bool f = m->m->decode_done(group, token);
        if (finished) *finished = f ? 1 : 0;
        return HP_OK;
    } catch (const std::logic_error& e) {
        hp_detail::set_error(e.what());
        return HP_EINVAL;
    } catch (const std::exception& e) {
        return from_exception(e);
    }
}

int hp_mbm_next(hp_mbm* m, int* group, int* token) {
    if (!m || !group || !token) return 0;
    hetplan::runtime::microbatch_manager::decode_item it{};
    if (!m->m->next_decode(it)) return 0;
    *group = it.group;
    *token = it.token;
    return 1;
}

void hp_mbm_destroy(hp_mbm* m) { delete m; }

}  // extern "C"
