#pragma once
// Partition / bit-plan loader — NEW public interface of the B200 build.
//
// The reference writes and reads plan documents only inside its CLI
// (/root/reference/proj/tools/hetplan_main.cpp:190-273, anonymous
// namespace). This header promotes that schema to a library API the
// runtime links against. Schema (format_version 1):
//   {model, num_layers, bits, theta, workload{global_bz,s,n}, eta, xi,
//    device_order, devices, stages[{device_index, device, layers[b,e]}],
//    layer_bits, objective{t_max_pre,...,total}, optimal, seed}
// Quirk handled: the writer stores device_order[k] as
// stages[k].device_index, while hetplan::stage_range::device means the stage
// index (types.hpp:80, checked by types.cpp:102). The loader keeps
// device_order and layers as authoritative, sets stage.device = k, and only
// checks device_index == device_order[k].
// Format 2 is written by serialize_plan and adds what a
// packed-weight artifact needs to be reproducible:
//   "quant": {"group": 128, "scheme": "symmetric"|"asymmetric",
//             "rounding": "nearest", "layout": "hp-tile-128x128-v1"}
// and writes stages[k].device_index = k (the stage index stage_range::device
// means), keeping the physical device in device_order[k]. Format-1 documents
// (the reference CLI's, no "format_version" or 1) still load; they carry no
// quant block and get the SPEC defaults (group 128, symmetric, nearest).

#include <cstdint>
#include <string>
#include <vector>

#include "hetplan/types.hpp"

namespace hetplan::plan_io {

inline constexpr int plan_format_version = 2;
inline constexpr const char* packed_layout_name = "hp-tile-128x128-v1";  // layout.cuh

struct quant_spec {
    int group = 128;     // K1/K3/K4 group size along k (the only one supported)
    int scheme = 1;      // 0 asymmetric, 1 symmetric (hp_capi.h HP_ASYMMETRIC/HP_SYMMETRIC)
    std::string rounding = "nearest";
    std::string layout = packed_layout_name;
};

struct plan_document {
    plan p;
    std::string model;
    int num_layers = 0;
    bitwidth_set bits;
    double theta = 0.0;
    workload load;
    std::vector<std::string> devices;  // names, in pipeline order
    std::uint64_t seed = 0;
    int format_version = 1;  // as read; serialize_plan always writes 2
    bool has_quant = false;  // document carried a "quant" block
    quant_spec quant;
};

// std::invalid_argument on malformed JSON or missing fields.
plan_document parse_plan(const std::string& json_text);
std::string serialize_plan(const plan_document& doc);
// validate_plan() with the document's own workload/bits/layer count.
void validate(const plan_document& doc);

// Stage r's layers and bits, as the executor consumes them.
struct stage_slice {
    int stage = 0;
    int begin = 0, end = 0;
    std::vector<int> bits;  // layer_bits[begin, end)
};
stage_slice slice_for_stage(const plan_document& doc, int stage);

}  // namespace hetplan::plan_io
