#pragma once
// B200 pipeline executor — NEW interface (the reference only models the
// pipeline: pipesim.cpp, optimizer_instance.cpp:166-197).
//
// One process per GPU; rank r owns plan stage r (layers [begin, end) with
// plan.layer_bits). At construction the stage's synthetic bf16 weights are
// generated on the device and quantized on the fly by K1 (hp_quant_pack) —
// the paper's on-the-fly quantized weight loader — so
// only packed codes + scales stay resident. run() serves one round of B
// requests: ceil(B/eta) prefill micro-batches then (n-1) decode tokens per
// decode group, in the unit order pipesim::simulate produces for this plan
// (identical on every rank, so NCCL sends/recvs match). Stage boundaries
// move bf16 activations with ncclSend/ncclRecv over NVLink: 2*eta*s*h1 bytes
// per prefill unit, 2*xi*h1 per decode unit (optimizer_instance.cpp
// :166-169); the last stage feeds each group's next-token input back to
// stage 0 (the LM-head/sampling round trip of a real server).
//
// Per decoder layer (OPT pre-LN, attention reduced to self-only so its
// output is the V slice): LN -> qkv -> out(+res) -> LN -> fc1(relu) ->
// fc2(+res); the four linear ops are K3 (decode) / K4 (prefill) with fused
// epilogues, LN is glue.

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hetplan/pipesim/pipesim.hpp"
#include "hetplan/plan/plan_io.hpp"
#include "hetplan/types.hpp"

namespace hetplan::runtime {

struct pipeline_options {
    int scheme = 1;             // 0 asymmetric, 1 symmetric (SPEC default)
    double weight_std = 0.02;   // synthetic weights N-like(0, std^2)
    std::uint64_t seed = 2403;  // synthetic tensors (oracle/synth.py mirror)
    bool use_graphs = true;     // capture each unit's stage forward
    bool instrument = false;    // CUDA events around every linear op
    int sm_budget = 0;          // persistent-kernel grid cap (0 = all SMs)
    double timeout_s = 0.0;     // run() watchdog (0 = wait forever); on
                                // expiry throws pipeline_timeout with the
                                // per-stream progress of the stuck round
    bool decode_fused = false;  // decode units as one K3-fused launch per
                                // bit-width run instead of per-op launches
};

// run() exceeded pipeline_options::timeout_s (hp_pipeline_run -> HP_ETIMEOUT).
// The stuck round still occupies the device; destroy the pipeline.
struct pipeline_timeout : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct run_timing {
    double makespan_s = 0.0;  // first unit start .. last unit end (this rank)
    double prefill_s = 0.0;   // sum of this stage's prefill unit times
    double decode_s = 0.0;    // sum of this stage's decode unit times
    double io_s = 0.0;        // host<->device copies inside the round
};

// Per-kernel-class totals from the instrumented run (roofline inputs).
struct kernel_stats {
    std::int64_t launches = 0;
    double seconds = 0.0;
    double bytes = 0.0;  // algorithmic bytes
    double flops = 0.0;
};

class pipeline {
public:
    pipeline(const plan_io::plan_document& plan, const model_spec& model, int rank, int world,
             const std::vector<std::array<char, 128>>& nccl_ids, const pipeline_options& opt);
    ~pipeline();
    pipeline(const pipeline&) = delete;
    pipeline& operator=(const pipeline&) = delete;

    // One serving round. host_prompt: rank 0, [B*s x h1] bf16 (NULL: use the
    // device-resident synthetic prompt). host_out: last rank, [B x h1] bf16
    // final hidden state of each request (NULL: skip the D2H).
    run_timing run(const void* host_prompt, void* host_out);

    // Measured per-unit costs of the last run for pipesim::simulate.
    pipesim::stage_cost measured_cost() const;
    const kernel_stats& stats(int phase) const;  // 0 prefill (K4), 1 decode (K3)
    // Per-layer seconds (LN + 4 linear ops) of this stage's layers in the
    // instrumented unit of the last run with instrument=true: one prefill
    // micro-batch (phase 0) / one decode group-token (phase 1). The profile
    // behind cost-balanced stage partitions (tests/golden/make_plans.py).
    const std::vector<double>& layer_costs(int phase) const;
    void reset_stats();
    std::int64_t weight_bytes() const;
    int num_kernel_launches_per_round() const;

    struct impl;

private:
    std::unique_ptr<impl> p_;
};

// Unit order of one stage (kind, index, token) in execution order, derived
// from pipesim::simulate with roofline cost estimates for this plan.
struct unit_ref {
    pipesim::unit_kind kind;
    int index;
    int token;
};
std::vector<std::vector<unit_ref>> static_unit_order(const plan_io::plan_document& plan,
                                                     const model_spec& model);

}  // namespace hetplan::runtime
