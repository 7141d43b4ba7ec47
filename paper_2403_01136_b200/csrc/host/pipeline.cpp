// B200 pipeline executor (include/hetplan/runtime/pipeline.hpp).
//
// Execution model per rank (= plan stage):
//   * three CUDA streams: compute (forward of each unit), send (ncclSend to
//     the next stage / feedback to stage 0), recv (ncclRecv from the
//     previous stage / feedback on stage 0); cross-stream order via events;
//   * one NCCL communicator per directed link (r -> r+1, and last -> 0 for
//     the decode feedback) so every communicator carries a single in-order
//     stream of P2P messages;
//   * the unit order of every stage comes from pipesim::simulate on
//     roofline cost estimates (static_unit_order), so all ranks agree on the
//     send/recv sequence without any control messages;
//   * the whole round (all units, sends, recvs) is captured into ONE CUDA
//     graph per rank after an eager warm-up round.
#include "hetplan/runtime/pipeline.hpp"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>

#include "hp_capi.h"

namespace hp {
cudaError_t launch_synth(void* out, int64_t n, uint64_t seed, double mean, double std_,
                         cudaStream_t st);
cudaError_t launch_layernorm(const void* x, int64_t ldx, int64_t rows, int h, const void* gamma,
                             const void* beta, void* y, int64_t ldy, cudaStream_t st);
cudaError_t launch_gather_rows(const void* src, int64_t lds, int64_t stride, int64_t offset,
                               int rows, int h, void* dst, int64_t ldd, cudaStream_t st);
}  // namespace hp

namespace hetplan::runtime {

namespace {

using bf16raw = uint16_t;

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("pipeline: ") + what + ": " + cudaGetErrorString(e));
}
void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("pipeline: ") + what + ": " + ncclGetErrorString(r));
}
void hp_ok(hp_status s, const char* what) {
    if (s != HP_OK)
        throw std::runtime_error(std::string("pipeline: ") + what + ": " + hp_last_error());
}

// Timing events inside a captured round must stay real event records (an
// internal graph event node cannot be timed): record them as "external".
// HP_PIPE_DEBUG=1: trace every host-side NCCL / sync call to stderr.
bool pipe_debug() {
    static const bool on = [] {
        const char* e = std::getenv("HP_PIPE_DEBUG");
        return e && *e && *e != '0';
    }();
    return on;
}
#define PDBG(...)                                             \
    do {                                                      \
        if (pipe_debug()) {                                   \
            std::fprintf(stderr, "[hp pipe r%d] ", rank);     \
            std::fprintf(stderr, __VA_ARGS__);                \
            std::fputc('\n', stderr);                        \
            std::fflush(stderr);                              \
        }                                                     \
    } while (0)

cudaError_t timing_record(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaError_t r = cudaStreamIsCapturing(st, &cap);
    if (r != cudaSuccess) return r;
    if (cap == cudaStreamCaptureStatusActive)
        return cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    return cudaEventRecord(e, st);
}

uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// oracle/synth.py seed_for(*parts, base=...): the chain starts at the
// options' seed (default 2403, the value the fixtures and tests use)
uint64_t seed_for(uint64_t base, std::initializer_list<uint64_t> parts) {
    uint64_t s = base;
    for (uint64_t p : parts) s = splitmix(s ^ p);
    return s;
}

struct op_shape {
    int64_t n, k;
};

// K3 bytes for one op at `bits`, m tokens
double k3_bytes(op_shape o, int bits, int scheme, int64_t m) {
    const double w = static_cast<double>(o.n) * o.k;
    double b = bits == 16 ? 2.0 * w : std::ceil(w * bits / 8.0) + 4.0 * w / 128.0 *
                                                                       (scheme == 0 ? 2 : 1);
    return b + 2.0 * m * (o.k + o.n);
}

}  // namespace

std::vector<std::vector<unit_ref>> static_unit_order(const plan_io::plan_document& plan,
                                                     const model_spec& m) {
    const auto& p = plan.p;
    const int S = static_cast<int>(p.stages.size());
    const double P = 4.0 * m.h1 * m.h1 + 2.0 * m.h1 * m.h2;
    const double s = plan.load.prompt_len;
    std::vector<pipesim::stage_cost> cost(S);
    for (int j = 0; j < S; ++j) {
        for (int l = p.stages[j].begin; l < p.stages[j].end; ++l) {
            const int b = p.layer_bits[l];
            cost[j].pre_s += 2.0 * P * p.eta * s / 1.2e15 + 5e-6;
            cost[j].dec_s += P * (b / 8.0 + (b == 16 ? 0.0 : 4.0 / 128.0)) / 5.5e12 + 1.2e-5;
        }
        if (j + 1 < S) {
            cost[j].comm_pre_s = 2.0 * p.eta * s * m.h1 / 7.0e11 + 1e-5;
            cost[j].comm_dec_s = 2.0 * p.xi * m.h1 / 7.0e11 + 1e-5;
        }
    }
    const auto sched = pipesim::make_schedule(plan.load.global_bz, p.eta, p.xi);
    const auto rep = pipesim::simulate(cost, sched, plan.load.gen_len, true);
    std::vector<std::vector<unit_ref>> order(S);
    // timeline is sorted by (start, stage, kind, index, token)
    for (const auto& e : rep.timeline) order[e.stage].push_back({e.kind, e.index, e.token});
    return order;
}

struct pipeline::impl {
    plan_io::plan_document plan;
    model_spec model;
    int rank = 0, world = 1;
    pipeline_options opt;
    int begin = 0, end = 0;
    std::vector<int> bits;
    int B = 0, s = 0, n = 0, eta = 0, xi = 0;
    int64_t h1 = 0, h2 = 0;
    pipesim::microbatch_schedule sched;
    std::vector<unit_ref> units;      // this stage, execution order
    std::vector<unit_ref> prev_units; // previous stage's order (recv order), rank > 0
    std::vector<unit_ref> last_units; // last stage's order (feedback order)
    std::vector<int> group_size;      // requests per decode group
    std::vector<int> group_first;     // first request of each group

    cudaStream_t cs = nullptr, ss = nullptr, rs = nullptr;
    ncclComm_t c_in = nullptr, c_out = nullptr;  // link from prev / to next
    bool graph_ready = false;
    cudaGraphExec_t graph = nullptr;

    struct opw {
        hp_qweight w{};
        void* packed = nullptr;
        float* scale = nullptr;
        float* zero = nullptr;
    };
    struct layer {
        opw ops[4];
        void* ln[4] = {nullptr, nullptr, nullptr, nullptr};
        int bits = 16;
    };
    std::vector<layer> layers;
    void* prompt = nullptr;      // [B*s x h1] working prompt / prefill activations
    void* pristine = nullptr;    // rank 0 synthetic prompt
    void* scr_a = nullptr;       // [M x h1]
    void* scr_qkv = nullptr;     // [M x 3h1]
    void* scr_f = nullptr;       // [M x h2]
    std::vector<void*> dec_x;    // per group [xi_g x h1]
    std::vector<void*> fb;       // last rank (world > 1): gather target per group
    // K3 fused (option decode_fused): one hp_decode_plan per decode group, bound to
    // dec_x[g]; a decode unit = one persistent launch per bit-width run of
    // the stage's layers (k3_stage.cu) instead of 6 launches per layer
    std::vector<hp_decode_plan*> dplans;
    int dplan_runs = 0;              // kernel launches per fused decode unit
    cudaEvent_t dec_ev[2] = {nullptr, nullptr};  // instrumented fused unit
    void* ws = nullptr;
    size_t ws_bytes = 0;
    int64_t weight_bytes = 0;

    // events
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join_s = nullptr, ev_join_r = nullptr;
    std::vector<cudaEvent_t> unit_ev;        // 2 per unit
    std::vector<cudaEvent_t> recv_ev;        // per incoming message
    std::vector<cudaEvent_t> comp_ev;        // per outgoing message
    size_t comp_used = 0;
    bool timed_out = false;
    std::vector<cudaEvent_t> op_ev[2];       // instrumented unit per phase
    std::vector<cudaEvent_t> lay_ev[2];      // whole layer (LN + 4 ops), same unit
    std::vector<double> layer_s[2];          // last instrumented run, per layer
    int instr_unit[2] = {-1, -1};
    kernel_stats kstats[2];
    std::vector<double> unit_s;
    int launches_per_round = 0;

    void* alloc(size_t bytes) {
        void* p = nullptr;
        cuda_ok(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "cudaMalloc");
        return p;
    }

    int prefill_rows(int k) const { return sched.prefill_sizes[k] * s; }
    void* prefill_ptr(int k) const {
        return static_cast<char*>(prompt) + static_cast<size_t>(k) * eta * s * h1 * 2;
    }

    void build(const std::vector<std::array<char, 128>>& ids) {
        const auto slice = plan_io::slice_for_stage(plan, rank);
        begin = slice.begin;
        end = slice.end;
        bits = slice.bits;
        B = plan.load.global_bz;
        s = plan.load.prompt_len;
        n = plan.load.gen_len;
        eta = plan.p.eta;
        xi = plan.p.xi;
        h1 = model.h1;
        h2 = model.h2;
        sched = pipesim::make_schedule(B, eta, xi);
        for (int g = 0; g < sched.num_groups; ++g) {
            group_first.push_back(g * xi);
            group_size.push_back(std::min(xi, B - g * xi));
        }
        const auto order = static_unit_order(plan, model);
        units = order[rank];
        if (rank > 0) prev_units = order[rank - 1];
        last_units = order[world - 1];

        cuda_ok(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream");
        cuda_ok(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking), "stream");
        cuda_ok(cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking), "stream");
        if (opt.sm_budget > 0) hp_set_sm_budget(opt.sm_budget);

        if (world > 1) {
            // NCCL's send/recv kernels occupy their SMs (one CTA per channel)
            // for as long as a message is outstanding -- a posted receive
            // spins through the whole previous stage's unit. With NCCL's
            // default P2P channel count they took enough SMs that the
            // persistent 1-CTA-per-SM K3/K4 grids ran partly serialised
            // (OPT-13B 2-stage bench: K4 786 TF/s, 36.3k tok/s). Two
            // channels per link move the 21 MB prefill messages in well
            // under a unit and leave the grid its SMs (K4 1208 TF/s, 52.7k
            // tok/s; 4 stages 70k -> 99.5k). The caller's own setting wins.
            // NCCL caches its parameters at its first initialisation in the
            // process, so a host that initialised NCCL before (torch.distributed
            // with the nccl backend) must export it itself (bench.py does).
            setenv("NCCL_MAX_P2P_NCHANNELS", "2", 0);
            // link l: rank l -> rank (l+1) % world; ids[l] names link l
            nccl_ok(ncclGroupStart(), "group");
            const int prev = (rank - 1 + world) % world;
            ncclUniqueId id_out, id_in;
            std::memcpy(&id_out, ids.at(rank).data(), sizeof id_out);
            std::memcpy(&id_in, ids.at(prev).data(), sizeof id_in);
            nccl_ok(ncclCommInitRank(&c_out, 2, id_out, 0), "init out");
            nccl_ok(ncclCommInitRank(&c_in, 2, id_in, 1), "init in");
            nccl_ok(ncclGroupEnd(), "group end");
        }

        // ---- weights: synthetic bf16 generated on device, packed by K1 ------
        const op_shape shp[4] = {{3 * h1, h1}, {h1, h1}, {h2, h1}, {h1, h2}};
        void* tmp = alloc(static_cast<size_t>(h2) * h1 * 2);
        layers.resize(end - begin);
        for (int l = begin; l < end; ++l) {
            layer& L = layers[l - begin];
            L.bits = bits[l - begin];
            for (int o = 0; o < 4; ++o) {
                opw& w = L.ops[o];
                const int64_t nn = shp[o].n, kk = shp[o].k;
                cuda_ok(hp::launch_synth(tmp, nn * kk, seed_for(opt.seed, {1, uint64_t(l), uint64_t(o)}),
                                         0.0, opt.weight_std, cs),
                        "synth weights");
                const int64_t pb = hp_packed_bytes(nn, kk, L.bits);
                w.packed = alloc(pb);
                weight_bytes += pb;
                if (L.bits != 16) {
                    const int64_t sc = hp_scale_count(nn, kk);
                    w.scale = static_cast<float*>(alloc(sc * 4));
                    weight_bytes += sc * 4;
                    if (opt.scheme == HP_ASYMMETRIC) {
                        w.zero = static_cast<float*>(alloc(sc * 4));
                        weight_bytes += sc * 4;
                    }
                }
                hp_ok(hp_quant_pack(tmp, nn, kk, kk, L.bits, opt.scheme, HP_NEAREST, w.packed,
                                    w.scale, w.zero, nullptr, nullptr, cs),
                      "quant_pack");
                w.w = hp_qweight{nn, kk, L.bits, opt.scheme, w.packed, w.scale, w.zero};
            }
            for (int j = 0; j < 4; ++j) {  // LN gain ~ 1, bias ~ 0 (synthetic)
                L.ln[j] = alloc(h1 * 2);
                cuda_ok(hp::launch_synth(L.ln[j], h1, seed_for(opt.seed, {4, uint64_t(l), uint64_t(j)}),
                                         (j % 2 == 0) ? 1.0 : 0.0, 0.02, cs),
                        "synth ln");
            }
        }
        cuda_ok(cudaStreamSynchronize(cs), "weights");
        cudaFree(tmp);

        // ---- activations -------------------------------------------------
        const int64_t M = static_cast<int64_t>(eta) * s;
        prompt = alloc(static_cast<size_t>(B) * s * h1 * 2);
        if (rank == 0) {
            pristine = alloc(static_cast<size_t>(B) * s * h1 * 2);
            cuda_ok(hp::launch_synth(pristine, int64_t(B) * s * h1, seed_for(opt.seed, {3}), 0.0, 1.0, cs),
                    "synth prompt");
        }
        const int64_t Mx = std::max<int64_t>(M, xi);
        scr_a = alloc(Mx * h1 * 2);
        scr_qkv = alloc(Mx * 3 * h1 * 2);
        scr_f = alloc(Mx * h2 * 2);
        for (int g = 0; g < sched.num_groups; ++g) {
            dec_x.push_back(alloc(static_cast<size_t>(group_size[g]) * h1 * 2));
            cuda_ok(cudaMemsetAsync(dec_x.back(), 0, group_size[g] * h1 * 2, cs), "memset");
            if (world > 1 && rank == world - 1)
                fb.push_back(alloc(static_cast<size_t>(group_size[g]) * h1 * 2));
        }
        // split-K workspace: max over this stage's ops and every (rows, phase)
        // the round launches -- a ragged last prefill micro-batch (B % eta != 0)
        // or a short last decode group can need MORE stream-K workspace than
        // the full-size one (fewer tiles -> more segments per tile)
        for (const auto& sh : round_shapes())
            for (const layer& L : layers)
                for (const opw& w : L.ops)
                    ws_bytes = std::max(ws_bytes,
                                        hp_qlinear_workspace_bytes(&w.w, sh.first, sh.second));
        if (ws_bytes) {
            ws = alloc(ws_bytes);
            cuda_ok(cudaMemsetAsync(ws, 0, ws_bytes, cs), "ws");
        }

        if (opt.decode_fused) {
            std::vector<hp_decoder_layer> dl(layers.size());
            for (size_t li = 0; li < layers.size(); ++li) {
                for (int o = 0; o < 4; ++o) dl[li].ops[o] = layers[li].ops[o].w;
                for (int j = 0; j < 4; ++j) dl[li].ln[j] = layers[li].ln[j];
                if (li == 0 || layers[li].bits != layers[li - 1].bits) ++dplan_runs;
            }
            for (int g = 0; g < sched.num_groups; ++g) {
                hp_decode_plan* dp = nullptr;
                hp_ok(hp_decode_plan_create(dl.data(), static_cast<int>(dl.size()), dec_x[g],
                                            group_size[g], &dp),
                      "decode_plan_create");
                dplans.push_back(dp);
            }
            for (cudaEvent_t* e : {&dec_ev[0], &dec_ev[1]}) cuda_ok(cudaEventCreate(e), "ev");
        }

        load_kernels();
        if (world > 1) connect_links();

        // ---- events ------------------------------------------------------
        cuda_ok(cudaEventCreate(&ev_t0), "ev");
        cuda_ok(cudaEventCreate(&ev_t1), "ev");
        for (cudaEvent_t* e : {&ev_fork, &ev_join_s, &ev_join_r})
            cuda_ok(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "ev");
        unit_ev.resize(2 * units.size());
        for (auto& e : unit_ev) cuda_ok(cudaEventCreate(&e), "ev");
        const size_t n_in = rank > 0 ? prev_units.size() : feedback_order().size();
        recv_ev.resize(n_in);
        for (auto& e : recv_ev) cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ev");
        comp_ev.resize(units.size() + sched.num_groups + 1);
        for (auto& e : comp_ev) cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ev");
        // instrumented units: first prefill, middle decode token of group 0
        for (size_t u = 0; u < units.size(); ++u) {
            if (units[u].kind == pipesim::unit_kind::prefill && instr_unit[0] < 0)
                instr_unit[0] = static_cast<int>(u);
            if (units[u].kind == pipesim::unit_kind::decode && units[u].index == 0 &&
                units[u].token == std::max(1, (n - 1) / 2))
                instr_unit[1] = static_cast<int>(u);
        }
        for (int ph = 0; ph < 2; ++ph) {
            op_ev[ph].resize(static_cast<size_t>(layers.size()) * 4 * 2);
            for (auto& e : op_ev[ph]) cuda_ok(cudaEventCreate(&e), "ev");
            lay_ev[ph].resize(static_cast<size_t>(layers.size()) * 2);
            for (auto& e : lay_ev[ph]) cuda_ok(cudaEventCreate(&e), "ev");
            layer_s[ph].assign(layers.size(), 0.0);
        }
        cuda_ok(cudaStreamSynchronize(cs), "init");
    }

    // feedback messages last -> 0, in the last stage's emission order
    std::vector<unit_ref> feedback_order() const {
        std::vector<unit_ref> out;
        if (world == 1) return out;
        std::vector<int> left(sched.num_groups, 0);
        for (int g : sched.group_of_prefill) ++left[g];
        for (const unit_ref& u : last_units) {
            if (u.kind == pipesim::unit_kind::prefill) {
                const int g = sched.group_of_prefill[u.index];
                if (--left[g] == 0 && n >= 2) out.push_back({pipesim::unit_kind::decode, g, 1});
            } else if (u.token + 1 <= n - 1) {
                out.push_back({pipesim::unit_kind::decode, u.index, u.token + 1});
            }
        }
        return out;
    }

    void qlin(const opw& w, const void* x, int64_t ldx, int64_t m, void* y, int64_t ldy,
              const void* res, int epi, int phase, cudaEvent_t* evs) {
        if (evs) cuda_ok(timing_record(evs[0], cs), "ev");
        hp_ok(hp_qlinear(&w.w, x, ldx, m, y, ldy, res, res ? ldy : 0, epi, phase, ws, ws_bytes,
                         cs),
              "qlinear");
        if (evs) cuda_ok(timing_record(evs[1], cs), "ev");
    }

    // forward of this stage's layers, in place on x [m x h1]; a decode unit
    // of group g >= 0 runs the group's K3-fused plan (bound to dec_x[g])
    void forward(void* x, int64_t m, int phase, bool instrument, int group = -1) {
        if (phase == HP_DECODE && group >= 0 && !dplans.empty()) {
            if (instrument) cuda_ok(timing_record(dec_ev[0], cs), "ev");
            hp_ok(hp_decode_plan_run(dplans[group], cs), "decode_plan_run");
            if (instrument) cuda_ok(timing_record(dec_ev[1], cs), "ev");
            return;
        }
        for (size_t li = 0; li < layers.size(); ++li) {
            const layer& L = layers[li];
            cudaEvent_t* ev = instrument ? &op_ev[phase][li * 8] : nullptr;
            if (instrument) cuda_ok(timing_record(lay_ev[phase][2 * li], cs), "ev");
            cuda_ok(hp::launch_layernorm(x, h1, m, static_cast<int>(h1), L.ln[0], L.ln[1], scr_a,
                                         h1, cs),
                    "ln1");
            qlin(L.ops[0], scr_a, h1, m, scr_qkv, 3 * h1, nullptr, HP_EPI_NONE, phase, ev);
            // self-only attention: output = V slice of qkv
            qlin(L.ops[1], static_cast<char*>(scr_qkv) + 2 * h1 * 2, 3 * h1, m, x, h1, x,
                 HP_EPI_NONE, phase, ev ? ev + 2 : nullptr);
            cuda_ok(hp::launch_layernorm(x, h1, m, static_cast<int>(h1), L.ln[2], L.ln[3], scr_a,
                                         h1, cs),
                    "ln2");
            qlin(L.ops[2], scr_a, h1, m, scr_f, h2, nullptr, HP_EPI_RELU, phase, ev ? ev + 4 : nullptr);
            qlin(L.ops[3], scr_f, h2, m, x, h1, x, HP_EPI_NONE, phase, ev ? ev + 6 : nullptr);
            if (instrument) cuda_ok(timing_record(lay_ev[phase][2 * li + 1], cs), "ev");
        }
    }

    // CUDA loads a kernel's module lazily at its first launch, and that load
    // waits for the device: issued while an NCCL recv kernel spins on rs (it
    // waits for a message this very stage must first compute and send) it
    // never returns. So run every (phase, rows) forward the round will use,
    // plus the gather, once on scratch before any NCCL operation is posted.
    // every distinct (rows, phase) the round's units run with
    std::vector<std::pair<int64_t, int>> round_shapes() const {
        std::vector<std::pair<int64_t, int>> shapes;
        for (int k = 0; k < static_cast<int>(sched.prefill_sizes.size()); ++k)
            shapes.push_back({prefill_rows(k), HP_PREFILL});
        for (int g = 0; g < sched.num_groups; ++g) shapes.push_back({group_size[g], HP_DECODE});
        std::sort(shapes.begin(), shapes.end());
        shapes.erase(std::unique(shapes.begin(), shapes.end()), shapes.end());
        return shapes;
    }

    void load_kernels() {
        const auto shapes = round_shapes();
        int64_t rows = 1;
        for (const auto& sh : shapes) rows = std::max(rows, sh.first);
        void* x = nullptr;
        cuda_ok(cudaMalloc(&x, static_cast<size_t>(rows) * h1 * 2 * 2), "cudaMalloc scratch");
        cuda_ok(hp::launch_synth(x, rows * h1, seed_for(opt.seed, {5}), 0.0, 1.0, cs), "synth scratch");
        for (const auto& sh : shapes) forward(x, sh.first, sh.second, false);
        for (int g = 0; g < static_cast<int>(dplans.size()); ++g) {
            forward(dec_x[g], group_size[g], HP_DECODE, false, g);
            cuda_ok(cudaMemsetAsync(dec_x[g], 0, static_cast<size_t>(group_size[g]) * h1 * 2, cs),
                    "memset");
        }
        cuda_ok(hp::launch_gather_rows(x, h1, 1, 0, 1, static_cast<int>(h1),
                                       static_cast<char*>(x) + static_cast<size_t>(rows) * h1 * 2, h1,
                                       cs),
                "gather");
        cuda_ok(cudaStreamSynchronize(cs), "load kernels");
        cuda_ok(cudaFree(x), "cudaFree scratch");
        if (ws_bytes) cuda_ok(cudaMemsetAsync(ws, 0, ws_bytes, cs), "ws");
    }

    // NCCL connects P2P channels lazily, host-blocking, on the first
    // send/recv that needs them (how many channels / which protocol depends
    // on the message size) and needs the peer to connect the SAME link
    // concurrently. A round posts rank 0's feedback recvs (link world-1)
    // first while rank 1 waits on link 0 -> a cycle of blocked hosts. So
    // exchange one message of every size the round uses on each link here,
    // in ascending link order (rank r: link r-1 then link r; rank 0: link 0
    // then link world-1) -- a chain, which cannot deadlock.
    std::vector<size_t> link_counts(int l) const {
        std::vector<size_t> c;
        if (l < world - 1) {
            for (int k = 0; k < static_cast<int>(sched.prefill_sizes.size()); ++k)
                c.push_back(static_cast<size_t>(prefill_rows(k)) * h1);
        }
        for (int g = 0; g < sched.num_groups; ++g) c.push_back(static_cast<size_t>(group_size[g]) * h1);
        std::sort(c.begin(), c.end());
        c.erase(std::unique(c.begin(), c.end()), c.end());
        return c;
    }
    void connect_links() {
        const int prev = (rank - 1 + world) % world;
        size_t maxc = 0;
        for (int l : {rank, prev})
            for (size_t c : link_counts(l)) maxc = std::max(maxc, c);
        void* probe = nullptr;
        cuda_ok(cudaMalloc(&probe, maxc * 2), "cudaMalloc probe");
        auto link = [&](bool out) {
            for (size_t c : link_counts(out ? rank : prev)) {
                PDBG("connect %s count %zu", out ? "out" : "in", c);
                if (out)
                    nccl_ok(ncclSend(probe, c, ncclBfloat16, /*peer=*/1, c_out, cs), "connect send");
                else
                    nccl_ok(ncclRecv(probe, c, ncclBfloat16, /*peer=*/0, c_in, cs), "connect recv");
                cuda_ok(cudaStreamSynchronize(cs), "connect");
            }
        };
        if (rank == 0) {
            link(true);
            link(false);
        } else {
            link(false);
            link(true);
        }
        cuda_ok(cudaFree(probe), "cudaFree probe");
    }

    // Enqueue one whole round on (cs, ss, rs). Capturable.
    void enqueue_round() {
        // fork side streams off the compute stream (joins them into a capture)
        cuda_ok(cudaEventRecord(ev_fork, cs), "ev");
        cuda_ok(cudaStreamWaitEvent(ss, ev_fork, 0), "wait");
        cuda_ok(cudaStreamWaitEvent(rs, ev_fork, 0), "wait");

        // post every receive in the sender's order
        if (world > 1) {
            const std::vector<unit_ref> incoming = rank > 0 ? prev_units : feedback_order();
            for (size_t i = 0; i < incoming.size(); ++i) {
                const unit_ref& u = incoming[i];
                void* dst;
                size_t count;
                if (rank > 0 && u.kind == pipesim::unit_kind::prefill) {
                    dst = prefill_ptr(u.index);
                    count = static_cast<size_t>(prefill_rows(u.index)) * h1;
                } else {
                    dst = dec_x[u.index];
                    count = static_cast<size_t>(group_size[u.index]) * h1;
                }
                PDBG("recv %zu (kind %d idx %d tok %d) count %zu", i, static_cast<int>(u.kind), u.index, u.token, count);
                nccl_ok(ncclRecv(dst, count, ncclBfloat16, /*peer=*/0, c_in, rs), "recv");
                cuda_ok(cudaEventRecord(recv_ev[i], rs), "ev");
            }
        }
        // map unit -> its recv index
        std::map<std::tuple<int, int, int>, int> recv_idx;
        if (world > 1) {
            const std::vector<unit_ref> incoming = rank > 0 ? prev_units : feedback_order();
            for (size_t i = 0; i < incoming.size(); ++i)
                recv_idx[{static_cast<int>(incoming[i].kind), incoming[i].index,
                          incoming[i].token}] = static_cast<int>(i);
        }
        std::vector<int> left(sched.num_groups, 0);
        for (int g : sched.group_of_prefill) ++left[g];
        int comp_i = 0;
        const bool last = rank == world - 1;

        for (size_t ui = 0; ui < units.size(); ++ui) {
            const unit_ref& u = units[ui];
            const bool pre = u.kind == pipesim::unit_kind::prefill;
            PDBG("unit %zu (kind %d idx %d tok %d)", ui, static_cast<int>(u.kind), u.index, u.token);
            // ---- input dependency
            const bool needs_recv = world > 1 && (rank > 0 || !pre);
            if (needs_recv) {
                auto it = recv_idx.find({static_cast<int>(u.kind), u.index, u.token});
                if (it == recv_idx.end()) throw std::logic_error("pipeline: unit without recv");
                cuda_ok(cudaStreamWaitEvent(cs, recv_ev[it->second], 0), "wait");
            }
            void* x = pre ? prefill_ptr(u.index) : dec_x[u.index];
            const int64_t m = pre ? prefill_rows(u.index) : group_size[u.index];
            const int phase = pre ? HP_PREFILL : HP_DECODE;
            cuda_ok(timing_record(unit_ev[2 * ui], cs), "ev");
            forward(x, m, phase, opt.instrument && instr_unit[phase] == static_cast<int>(ui),
                    pre ? -1 : u.index);
            cuda_ok(timing_record(unit_ev[2 * ui + 1], cs), "ev");

            // ---- output
            if (!last) {
                cuda_ok(cudaEventRecord(comp_ev[comp_i], cs), "ev");
                cuda_ok(cudaStreamWaitEvent(ss, comp_ev[comp_i++], 0), "wait");
                PDBG("send unit %zu count %zu", ui, static_cast<size_t>(m) * h1);
                nccl_ok(ncclSend(x, static_cast<size_t>(m) * h1, ncclBfloat16, /*peer=*/1, c_out, ss),
                        "send");
                PDBG("send unit %zu posted", ui);
                continue;
            }
            if (pre) {
                // last position of each request -> its decode group's input
                const int g = sched.group_of_prefill[u.index];
                const int req0 = u.index * eta;
                void* dst_base = world > 1 ? fb[g] : dec_x[g];
                const int row0 = req0 - group_first[g];
                // a prefill batch may straddle a group boundary: split
                int r = 0;
                while (r < sched.prefill_sizes[u.index]) {
                    const int req = req0 + r;
                    const int gg = req / xi;
                    const int take = std::min(sched.prefill_sizes[u.index] - r,
                                              group_first[gg] + group_size[gg] - req);
                    void* dst = world > 1 ? fb[gg] : dec_x[gg];
                    cuda_ok(hp::launch_gather_rows(x, h1, s, static_cast<int64_t>(r) * s + s - 1, take,
                                                   static_cast<int>(h1),
                                                   static_cast<char*>(dst) +
                                                       static_cast<size_t>(req - group_first[gg]) * h1 * 2,
                                                   h1, cs),
                            "gather");
                    r += take;
                }
                (void)dst_base;
                (void)row0;
                if (--left[g] == 0 && n >= 2 && world > 1) {
                    cuda_ok(cudaEventRecord(comp_ev[comp_i], cs), "ev");
                    cuda_ok(cudaStreamWaitEvent(ss, comp_ev[comp_i++], 0), "wait");
                    PDBG("send fb group %d count %zu", g, static_cast<size_t>(group_size[g]) * h1);
                    nccl_ok(ncclSend(fb[g], static_cast<size_t>(group_size[g]) * h1, ncclBfloat16,
                                     /*peer=*/1, c_out, ss),
                            "send fb");
                }
            } else if (world > 1 && u.token + 1 <= n - 1) {
                cuda_ok(cudaEventRecord(comp_ev[comp_i], cs), "ev");
                cuda_ok(cudaStreamWaitEvent(ss, comp_ev[comp_i++], 0), "wait");
                PDBG("send fb unit %zu count %zu", ui, static_cast<size_t>(m) * h1);
                nccl_ok(ncclSend(x, static_cast<size_t>(m) * h1, ncclBfloat16, /*peer=*/1, c_out, ss),
                        "send fb");
            }
        }
        comp_used = static_cast<size_t>(comp_i);
        // join side streams back into the compute stream
        cuda_ok(cudaEventRecord(ev_join_s, ss), "ev");
        cuda_ok(cudaStreamWaitEvent(cs, ev_join_s, 0), "wait");
        cuda_ok(cudaEventRecord(ev_join_r, rs), "ev");
        cuda_ok(cudaStreamWaitEvent(cs, ev_join_r, 0), "wait");
    }

    // Block until cs drains; with opt.timeout_s > 0 poll instead and, on
    // expiry, throw pipeline_timeout naming how far each stream got.
    void wait_round(const char* what) {
        PDBG("wait %s", what);
        if (opt.timeout_s <= 0) {
            cuda_ok(cudaStreamSynchronize(cs), what);
            return;
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            const cudaError_t e = cudaStreamQuery(cs);
            if (e == cudaSuccess) return;
            if (e != cudaErrorNotReady) cuda_ok(e, what);
            const double dt =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (dt > opt.timeout_s) break;
            std::this_thread::sleep_for(std::chrono::microseconds(dt < 0.01 ? 20 : 2000));
        }
        auto done = [](cudaEvent_t ev) { return cudaEventQuery(ev) == cudaSuccess; };
        size_t u_done = 0, r_done = 0, c_done = 0;
        while (u_done < units.size() && done(unit_ev[2 * u_done + 1])) ++u_done;
        while (r_done < recv_ev.size() && done(recv_ev[r_done])) ++r_done;
        while (c_done < comp_used && done(comp_ev[c_done])) ++c_done;
        std::string msg = std::string("pipeline: ") + what + " exceeded " +
                          std::to_string(opt.timeout_s) + " s on rank " + std::to_string(rank) +
                          ": units done " + std::to_string(u_done) + "/" +
                          std::to_string(units.size()) + ", recvs done " + std::to_string(r_done) +
                          "/" + std::to_string(recv_ev.size()) + ", sends ready " +
                          std::to_string(c_done) + "/" + std::to_string(comp_used);
        if (u_done < units.size()) {
            const unit_ref& u = units[u_done];
            msg += ", stuck at unit (" + std::string(u.kind == pipesim::unit_kind::prefill ? "prefill" : "decode") +
                   " " + std::to_string(u.index) + " token " + std::to_string(u.token) + ")";
        }
        timed_out = true;
        throw pipeline_timeout(msg);
    }

    void capture() {
        cudaGraph_t g = nullptr;
        cuda_ok(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "capture");
        enqueue_round();
        cuda_ok(cudaStreamEndCapture(cs, &g), "end capture");
        cuda_ok(cudaGraphInstantiate(&graph, g, 0), "instantiate");
        cudaGraphDestroy(g);
        graph_ready = true;
    }

    run_timing run(const void* host_prompt, void* host_out) {
        run_timing t;
        cuda_ok(cudaEventRecord(ev_t0, cs), "ev");
        if (rank == 0) {
            const size_t bytes = static_cast<size_t>(B) * s * h1 * 2;
            if (host_prompt)
                cuda_ok(cudaMemcpyAsync(prompt, host_prompt, bytes, cudaMemcpyHostToDevice, cs), "h2d");
            else
                cuda_ok(cudaMemcpyAsync(prompt, pristine, bytes, cudaMemcpyDeviceToDevice, cs), "d2d");
        }
        if (opt.use_graphs) {
            if (!graph_ready) {
                enqueue_round();  // eager warm-up (sets kernel attributes)
                wait_round("warm-up round");
                if (rank == 0) {
                    const size_t bytes = static_cast<size_t>(B) * s * h1 * 2;
                    cuda_ok(cudaMemcpyAsync(prompt, host_prompt ? host_prompt : pristine, bytes,
                                            host_prompt ? cudaMemcpyHostToDevice
                                                        : cudaMemcpyDeviceToDevice,
                                            cs),
                            "reload");
                }
                capture();
            }
            cuda_ok(cudaGraphLaunch(graph, cs), "graph launch");
        } else {
            enqueue_round();
        }
        if (rank == world - 1 && host_out) {
            for (int g = 0; g < sched.num_groups; ++g) {
                const void* src = (n >= 2 || world == 1) ? dec_x[g] : fb[g];
                cuda_ok(cudaMemcpyAsync(static_cast<char*>(host_out) +
                                            static_cast<size_t>(group_first[g]) * h1 * 2,
                                        src, static_cast<size_t>(group_size[g]) * h1 * 2,
                                        cudaMemcpyDeviceToHost, cs),
                        "d2h");
            }
        }
        cuda_ok(cudaEventRecord(ev_t1, cs), "ev");
        wait_round("round");
        float ms = 0.f;
        cuda_ok(cudaEventElapsedTime(&ms, ev_t0, ev_t1), "elapsed");
        t.makespan_s = ms * 1e-3;
        unit_s.assign(units.size(), 0.0);
        for (size_t ui = 0; ui < units.size(); ++ui) {
            cuda_ok(cudaEventElapsedTime(&ms, unit_ev[2 * ui], unit_ev[2 * ui + 1]), "elapsed");
            unit_s[ui] = ms * 1e-3;
            (units[ui].kind == pipesim::unit_kind::prefill ? t.prefill_s : t.decode_s) += unit_s[ui];
        }
        t.io_s = std::max(0.0, t.makespan_s - t.prefill_s - t.decode_s);
        if (opt.instrument) collect_kernel_stats();
        return t;
    }

    void collect_kernel_stats() {
        const op_shape shp[4] = {{3 * h1, h1}, {h1, h1}, {h2, h1}, {h1, h2}};
        for (int ph = 0; ph < 2; ++ph) {
            const int ui = instr_unit[ph];
            if (ui < 0) continue;
            const unit_ref& u = units[ui];
            const int64_t m = ph == 0 ? prefill_rows(u.index) : group_size[u.index];
            if (ph == 1 && !dplans.empty()) {
                // K3 fused: one timed span over the unit's launches; per-layer
                // decode costs need per-op decode (tools/layer_costs.py)
                float ms = 0.f;
                cuda_ok(cudaEventElapsedTime(&ms, dec_ev[0], dec_ev[1]), "elapsed fused");
                double info[4];
                hp_ok(hp_decode_plan_info(dplans[u.index], info), "decode_plan_info");
                kernel_stats& k = kstats[1];
                k.launches += dplan_runs;
                k.seconds += ms * 1e-3;
                k.bytes += info[1];
                for (size_t li = 0; li < layers.size(); ++li) {
                    layer_s[1][li] = 0.0;
                    for (int o = 0; o < 4; ++o) k.flops += 2.0 * m * shp[o].n * shp[o].k;
                }
                continue;
            }
            for (size_t li = 0; li < layers.size(); ++li) {
                float ms = 0.f;
                cuda_ok(cudaEventElapsedTime(&ms, lay_ev[ph][2 * li], lay_ev[ph][2 * li + 1]),
                        "elapsed layer");
                layer_s[ph][li] = ms * 1e-3;
            }
            for (size_t li = 0; li < layers.size(); ++li)
                for (int o = 0; o < 4; ++o) {
                    float ms = 0.f;
                    cuda_ok(cudaEventElapsedTime(&ms, op_ev[ph][li * 8 + 2 * o],
                                                 op_ev[ph][li * 8 + 2 * o + 1]),
                            "elapsed op");
                    kernel_stats& k = kstats[ph];
                    ++k.launches;
                    k.seconds += ms * 1e-3;
                    k.bytes += k3_bytes(shp[o], layers[li].bits, opt.scheme, m);
                    k.flops += 2.0 * m * shp[o].n * shp[o].k;
                }
        }
    }

    ~impl() {
        if (graph) cudaGraphExecDestroy(graph);
        // Destroy finalizes with the peer: same chain order as connect_links
        // (rank 0: link 0 then link world-1; rank r: link r-1 then link r).
        // After a timeout the round is still stuck on the device: abort.
        auto close = [&](ncclComm_t c) {
            if (!c) return;
            if (timed_out)
                ncclCommAbort(c);
            else
                ncclCommDestroy(c);
        };
        if (rank == 0) {
            close(c_out);
            close(c_in);
        } else {
            close(c_in);
            close(c_out);
        }
        auto f = [](void* p) {
            if (p) cudaFree(p);
        };
        for (layer& L : layers) {
            for (opw& w : L.ops) {
                f(w.packed);
                f(w.scale);
                f(w.zero);
            }
            for (void* p : L.ln) f(p);
        }
        f(prompt);
        f(pristine);
        f(scr_a);
        f(scr_qkv);
        f(scr_f);
        for (void* p : dec_x) f(p);
        for (void* p : fb) f(p);
        f(ws);
        for (hp_decode_plan* dp : dplans) hp_decode_plan_destroy(dp);
        for (cudaEvent_t e : dec_ev)
            if (e) cudaEventDestroy(e);
        for (auto* v : {&unit_ev, &recv_ev, &comp_ev, &op_ev[0], &op_ev[1], &lay_ev[0], &lay_ev[1]})
            for (cudaEvent_t e : *v) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_t0, ev_t1, ev_fork, ev_join_s, ev_join_r})
            if (e) cudaEventDestroy(e);
        for (cudaStream_t st : {cs, ss, rs})
            if (st) cudaStreamDestroy(st);
    }
};

pipeline::pipeline(const plan_io::plan_document& plan, const model_spec& model, int rank,
                   int world, const std::vector<std::array<char, 128>>& nccl_ids,
                   const pipeline_options& opt)
    : p_(std::make_unique<impl>()) {
    plan_io::validate(plan);
    if (static_cast<int>(plan.p.stages.size()) != world)
        throw std::invalid_argument("pipeline: plan has " + std::to_string(plan.p.stages.size()) +
                                    " stages but world size is " + std::to_string(world));
    if (rank < 0 || rank >= world) throw std::invalid_argument("pipeline: bad rank");
    if (plan.has_quant && plan.quant.scheme != opt.scheme)
        throw std::invalid_argument("pipeline: the plan's quant.scheme differs from the options' scheme");
    if (model.num_layers != plan.num_layers)
        throw std::invalid_argument("pipeline: model/plan layer count mismatch");
    if (world > 1 && static_cast<int>(nccl_ids.size()) < world)
        throw std::invalid_argument("pipeline: need one NCCL id per link");
    p_->plan = plan;
    p_->model = model;
    p_->rank = rank;
    p_->world = world;
    p_->opt = opt;
    p_->build(nccl_ids);
}

pipeline::~pipeline() = default;

run_timing pipeline::run(const void* host_prompt, void* host_out) {
    return p_->run(host_prompt, host_out);
}

pipesim::stage_cost pipeline::measured_cost() const {
    pipesim::stage_cost c;
    double pre = 0, dec = 0;
    int np = 0, nd = 0;
    for (size_t i = 0; i < p_->units.size() && i < p_->unit_s.size(); ++i) {
        if (p_->units[i].kind == pipesim::unit_kind::prefill) {
            pre += p_->unit_s[i];
            ++np;
        } else {
            dec += p_->unit_s[i];
            ++nd;
        }
    }
    c.pre_s = np ? pre / np : 0.0;
    c.dec_s = nd ? dec / nd : 0.0;
    return c;
}

const kernel_stats& pipeline::stats(int phase) const { return p_->kstats[phase ? 1 : 0]; }

const std::vector<double>& pipeline::layer_costs(int phase) const {
    return p_->layer_s[phase ? 1 : 0];
}

void pipeline::reset_stats() {
    p_->kstats[0] = kernel_stats{};
    p_->kstats[1] = kernel_stats{};
}

std::int64_t pipeline::weight_bytes() const { return p_->weight_bytes; }

int pipeline::num_kernel_launches_per_round() const {
    int n = 0;
    for (const unit_ref& u : p_->units)
        n += (u.kind == pipesim::unit_kind::decode && !p_->dplans.empty())
                 ? p_->dplan_runs
                 : static_cast<int>(p_->layers.size()) * 6;
    if (p_->rank == p_->world - 1)
        for (const unit_ref& u : p_->units)
            if (u.kind == pipesim::unit_kind::prefill) ++n;  // gather (>=1)
    return n;
}

}  // namespace hetplan::runtime
