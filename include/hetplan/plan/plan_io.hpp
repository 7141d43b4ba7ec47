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

#include <cstdint>
#include <string>
#include <vector>

#include "hetplan/types.hpp"

namespace hetplan::plan_io {

inline constexpr int plan_format_version = 1;

struct plan_document {
    plan p;
    std::string model;
    int num_layers = 0;
    bitwidth_set bits;
    double theta = 0.0;
    workload load;
    std::vector<std::string> devices;  // names, in pipeline order
    std::uint64_t seed = 0;
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
