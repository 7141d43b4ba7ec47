// Plan document I/O (schema of /root/reference/proj/tools/hetplan_main.cpp
// :190-273, promoted to a library API; see include/hetplan/plan/plan_io.hpp).
#include "hetplan/plan/plan_io.hpp"

#include <stdexcept>

#include <json.hpp>

namespace hetplan::plan_io {

namespace {
using json = nlohmann::ordered_json;
[[noreturn]] void reject(const std::string& what) { throw std::invalid_argument(what); }
}  // namespace

plan_document parse_plan(const std::string& json_text) {
    json j = json::parse(json_text, nullptr, false);
    if (j.is_discarded()) reject("plan: not valid JSON");
    plan_document d;
    try {
        d.model = j.at("model").get<std::string>();
        d.num_layers = j.value("num_layers", 0);
        d.theta = j.at("theta").get<double>();
        d.bits = j.at("bits").get<bitwidth_set>();
        const json& w = j.at("workload");
        d.load = {w.at("global_bz").get<int>(), w.at("s").get<int>(), w.at("n").get<int>()};
        plan& p = d.p;
        p.eta = j.at("eta").get<int>();
        p.xi = j.at("xi").get<int>();
        p.device_order = j.at("device_order").get<std::vector<int>>();
        if (j.contains("devices")) d.devices = j.at("devices").get<std::vector<std::string>>();
        d.format_version = j.value("format_version", 1);
        if (d.format_version != 1 && d.format_version != 2)
            reject("plan: unsupported format_version " + std::to_string(d.format_version));
        if (j.contains("quant")) {
            const json& q = j.at("quant");
            d.has_quant = true;
            d.quant.group = q.value("group", 128);
            const std::string sch = q.value("scheme", std::string("symmetric"));
            d.quant.rounding = q.value("rounding", std::string("nearest"));
            d.quant.layout = q.value("layout", std::string(packed_layout_name));
            if (d.quant.group != 128) reject("plan: quant.group must be 128 (the packed tile layout)");
            if (sch != "symmetric" && sch != "asymmetric")
                reject("plan: quant.scheme must be symmetric or asymmetric");
            d.quant.scheme = sch == "symmetric" ? 1 : 0;
            if (d.quant.rounding != "nearest") reject("plan: quant.rounding must be nearest");
            if (d.quant.layout != packed_layout_name)
                reject("plan: unknown packed layout '" + d.quant.layout + "'");
        }
        const json& st = j.at("stages");
        for (size_t k = 0; k < st.size(); ++k) {
            const json& s = st[k];
            const int di = s.at("device_index").get<int>();
            // format 1 (reference CLI, hetplan_main.cpp:209): device_order[k];
            // format 2: the stage index k
            const int want = d.format_version >= 2 ? static_cast<int>(k)
                                                   : (k < p.device_order.size() ? p.device_order[k] : di);
            if (di != want)
                reject("plan: stages[" + std::to_string(k) + "].device_index is " + std::to_string(di) +
                       ", expected " + std::to_string(want));
            p.stages.push_back({static_cast<int>(k), s.at("layers").at(0).get<int>(),
                                s.at("layers").at(1).get<int>()});
        }
        p.layer_bits = j.at("layer_bits").get<std::vector<int>>();
        if (d.num_layers == 0) d.num_layers = static_cast<int>(p.layer_bits.size());
        const json& o = j.at("objective");
        p.objective = {o.at("t_max_pre").get<double>(),   o.at("t_max_dec").get<double>(),
                       o.at("t_pre_total").get<double>(), o.at("t_dec_total").get<double>(),
                       o.at("omega_sum").get<double>(),   o.at("theta").get<double>(),
                       o.at("total").get<double>()};
        p.optimal = j.value("optimal", true);
        d.seed = j.value("seed", std::uint64_t{0});
    } catch (const json::exception& e) {
        reject(std::string("plan: missing or mistyped field: ") + e.what());
    }
    return d;
}

std::string serialize_plan(const plan_document& d) {
    json j;
    j["format_version"] = plan_format_version;
    j["model"] = d.model;
    j["num_layers"] = d.num_layers;
    j["bits"] = d.bits;
    j["theta"] = d.theta;
    j["workload"] = {{"global_bz", d.load.global_bz}, {"s", d.load.prompt_len}, {"n", d.load.gen_len}};
    j["eta"] = d.p.eta;
    j["xi"] = d.p.xi;
    j["device_order"] = d.p.device_order;
    j["devices"] = d.devices;
    json stages = json::array();
    for (size_t k = 0; k < d.p.stages.size(); ++k) {
        json s;
        s["device_index"] = static_cast<int>(k);  // format 2: the stage index
        if (k < d.devices.size()) s["device"] = d.devices[k];
        s["layers"] = {d.p.stages[k].begin, d.p.stages[k].end};
        stages.push_back(s);
    }
    j["stages"] = stages;
    j["layer_bits"] = d.p.layer_bits;
    const auto& o = d.p.objective;
    j["objective"] = {{"t_max_pre", o.t_max_pre},     {"t_max_dec", o.t_max_dec},
                      {"t_pre_total", o.t_pre_total}, {"t_dec_total", o.t_dec_total},
                      {"omega_sum", o.omega_sum},     {"theta", o.theta},
                      {"total", o.total}};
    j["optimal"] = d.p.optimal;
    j["seed"] = d.seed;
    j["quant"] = {{"group", d.quant.group},
                  {"scheme", d.quant.scheme == 1 ? "symmetric" : "asymmetric"},
                  {"rounding", d.quant.rounding},
                  {"layout", d.quant.layout}};
    return j.dump(2) + "\n";
}

void validate(const plan_document& d) {
    validate_plan(d.p, d.num_layers, d.load, d.bits, static_cast<int>(d.p.device_order.size()));
}

stage_slice slice_for_stage(const plan_document& d, int stage) {
    if (stage < 0 || stage >= static_cast<int>(d.p.stages.size()))
        reject("plan: stage index out of range");
    stage_slice s;
    s.stage = stage;
    s.begin = d.p.stages[stage].begin;
    s.end = d.p.stages[stage].end;
    s.bits.assign(d.p.layer_bits.begin() + s.begin, d.p.layer_bits.begin() + s.end);
    return s;
}

}  // namespace hetplan::plan_io
