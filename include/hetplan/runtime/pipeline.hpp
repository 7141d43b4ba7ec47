#pragma once
// B200 pipeline executor — NEW interface (the reference only models the
// pipeline: pipesim.cpp, optimizer_instance.cpp:166-197).
//
// One process per GPU; rank r owns plan stage r (layers [begin, end) with
// plan.layer_bits). At construction the stage's weights are loaded and
// quantized on the fly by K1 (hp_quant_pack) -- the paper's on-the-fly
// quantized weight loader: bf16 tensors stream
// from host memory or disk to the device in bins of `bin_bytes`, and K1
// packs bin i while bin i+1 is copied (weights without a source are the
// seeded synthetic tensors of oracle/synth.py, generated on the device).
// Only packed codes + scales stay resident.
//
// run() serves one round of B requests: ceil(B/eta) prefill micro-batches
// then (n-1) decode tokens per decode group, in the unit order
// pipesim::simulate produces for this plan (identical on every rank, so
// NCCL sends/recvs match). Each decoder layer is OPT's pre-LN block:
//   a = LN1(x); qkv = a Wqkv^T; o = attention(qkv, KV cache);
//   x += o Wout^T; a = LN2(x); x += relu(a Wfc1^T) Wfc2^T
// with the four linear ops on K3 (decode) / K4 (prefill) and causal
// multi-head attention over a pre-allocated KV cache of 2*B*(s+n)*h1 bf16
// per layer (memcost.cpp:38-42). Stage 0 embeds token ids (token + learned
// position, OPT offset 2); the last stage applies the final LN, the tied
// LM head (a 16-bit hp_qlinear over the embedding) and greedy argmax, and
// feeds each group's next token ids back to stage 0 (int32, B*4 bytes per
// decode step over NVLink). Stage boundaries move bf16 activations with
// ncclSend/ncclRecv: 2*eta*s*h1 bytes per prefill unit, 2*xi*h1 per decode
// unit (optimizer_instance.cpp:166-169).

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

// One bf16 tensor of the checkpoint: host memory (pinned -> copied
// directly, pageable -> staged through pinned bins) or a raw little-endian
// bf16 file at a byte offset. Empty = synthetic.
struct tensor_source {
    const void* host = nullptr;
    std::string path;
    std::int64_t offset = 0;
    bool empty() const { return host == nullptr && path.empty(); }
};

// Weights of the whole model (every rank reads the entries of its stage).
struct weight_set {
    std::vector<tensor_source> linear;  // [num_layers * 4]: qkv [3h1 x h1], out [h1 x h1],
                                        // fc1 [h2 x h1], fc2 [h1 x h2], row-major (y = x W^T)
    std::vector<tensor_source> norm;    // [num_layers * 4]: LN1 gamma, beta, LN2 gamma, beta [h1]
    tensor_source embed;                // [vocab x h1] token embedding (tied LM head)
    tensor_source pos;                  // [pos_s x h1] learned positions
    tensor_source final_norm[2];        // final LN gamma, beta [h1]
    std::int64_t bin_bytes = 64 << 20;  // H2D bin (rounded to 128-row blocks for linear ops)
};

struct pipeline_options {
    int scheme = 1;             // 0 asymmetric, 1 symmetric (SPEC default)
    double weight_std = 0.02;   // synthetic weights N-like(0, std^2)
    std::uint64_t seed = 2403;  // synthetic tensors (oracle/synth.py mirror)
    bool use_graphs = true;     // capture the round into one CUDA graph
    bool instrument = false;    // CUDA events around every op of 1 unit/phase
    int sm_budget = 0;          // persistent-kernel grid cap (0 = all SMs)
    double timeout_s = 0.0;     // run() watchdog (0 = wait forever); on
                                // expiry throws pipeline_timeout with the
                                // per-stream progress of the stuck round
    const weight_set* weights = nullptr;  // read during construction only
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

// Weight loading of the constructor (pipeline_options::weights).
struct load_stats {
    double seconds = 0.0;       // wall time of the whole weight load + pack
    double source_bytes = 0.0;  // bf16 bytes read from host memory / disk
    double packed_bytes = 0.0;  // resident packed codes + scales (+ glue tensors)
    std::int64_t bins = 0;      // H2D bins
};

class pipeline {
public:
    pipeline(const plan_io::plan_document& plan, const model_spec& model, int rank, int world,
             const std::vector<std::array<char, 128>>& nccl_ids, const pipeline_options& opt);
    ~pipeline();
    pipeline(const pipeline&) = delete;
    pipeline& operator=(const pipeline&) = delete;

    // One serving round. host_tokens: rank 0, [B x s] int32 prompt token ids
    // (NULL: the device-resident synthetic prompt). host_out: last rank,
    // [B x n] int32 generated token ids (NULL: skip the D2H).
    run_timing run(const std::int32_t* host_tokens, std::int32_t* host_out);

    // Last rank: the final hidden state (pre final-LN) of every request's
    // last decode position, [B x h1] bf16, of the last round (tests).
    void final_hidden(void* host) const;

    // Measured per-unit costs of the last run for pipesim::simulate.
    pipesim::stage_cost measured_cost() const;
    // 0 prefill linear ops (K4), 1 decode linear ops (K3), 2 prefill
    // attention, 3 decode attention (instrumented units)
    const kernel_stats& stats(int kind) const;
    // Per-layer seconds (LN + attention + 4 linear ops) of this stage's
    // layers in the instrumented unit of the last run with instrument=true:
    // one prefill micro-batch (phase 0) / one decode group-token (phase 1).
    const std::vector<double>& layer_costs(int phase) const;
    void reset_stats();
    std::int64_t weight_bytes() const;
    const load_stats& loading() const;
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
