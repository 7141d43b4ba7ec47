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
//     graph per rank after an eager warm-up round;
//   * weights are loaded once, through the binned H2D + K1 loader below.
#include "hetplan/runtime/pipeline.hpp"
#include "hetplan/runtime/microbatch.hpp"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <cmath>
#include <cstring>
#include <fcntl.h>
#include <map>
#include <unistd.h>
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
cudaError_t launch_embed(const int32_t* tok, int rows, int pos0, int pos_per_req, int s_tokens,
                         const void* E, const void* P, int pos_s, int h, int64_t vocab, void* x,
                         cudaStream_t st);
cudaError_t launch_attn_prefill(const void* qkv, int reqs, int s, int h, int D, void* out, void* kc,
                                void* vc, int req0, int S_max, cudaStream_t st);
cudaError_t launch_attn_decode(const void* qkv, int rows, int h, int D, int p, void* out, void* kc,
                               void* vc, int req0, int S_max, cudaStream_t st, void* ws, int split);
size_t attn_decode_workspace(int rows, int h, int D, int split);
cudaError_t launch_argmax(const void* logits, int64_t ld, int rows, int64_t vocab, int32_t* tok,
                          int32_t* tok2, int64_t tok2_stride, cudaStream_t st);
cudaError_t launch_synth_tokens(int32_t* out, int64_t n, uint64_t seed, int64_t vocab,
                                cudaStream_t st);
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

namespace {

// ---- the weight loader: host memory / disk -> pinned bins -> device, K1 on
// each bin while the next one is copied. Two
// device bins and two pinned host bins; a bin's device buffer is reused only
// after its consumer (K1 or a device copy on the compute stream) finished,
// a host bin only after its H2D copy finished.
class bin_loader {
public:
    bin_loader(cudaStream_t compute, int64_t bin_bytes) : cs_(compute), bin_(bin_bytes) {
        cuda_ok(cudaStreamCreateWithFlags(&cp_, cudaStreamNonBlocking), "loader stream");
        for (int i = 0; i < 2; ++i) {
            cuda_ok(cudaMalloc(&dev_[i], static_cast<size_t>(bin_)), "loader bin");
            cuda_ok(cudaEventCreateWithFlags(&ev_copy_[i], cudaEventDisableTiming), "ev");
            cuda_ok(cudaEventCreateWithFlags(&ev_used_[i], cudaEventDisableTiming), "ev");
        }
    }
    ~bin_loader() {
        cudaStreamSynchronize(cs_);
        cudaStreamSynchronize(cp_);
        for (int i = 0; i < 2; ++i) {
            cudaFree(dev_[i]);
            if (host_[i]) cudaFreeHost(host_[i]);
            cudaEventDestroy(ev_copy_[i]);
            cudaEventDestroy(ev_used_[i]);
        }
        for (auto& kv : fds_) ::close(kv.second);
        cudaStreamDestroy(cp_);
    }
    int64_t bin_bytes() const { return bin_; }
    double source_bytes() const { return bytes_; }
    int64_t bins() const { return bins_; }

    // Bytes [off, off + len) of src (len <= bin) into a device bin; the
    // compute stream is ordered after the copy. Returns the device pointer;
    // the caller enqueues its consumer on the compute stream, then release().
    void* fetch(const tensor_source& src, int64_t off, int64_t len) {
        if (len > bin_) throw std::logic_error("loader: chunk larger than a bin");
        slot_ = static_cast<int>(bins_++ & 1);
        cuda_ok(cudaStreamWaitEvent(cp_, ev_used_[slot_], 0), "loader wait");
        if (src.host && pinned(src.host)) {
            cuda_ok(cudaMemcpyAsync(dev_[slot_], static_cast<const char*>(src.host) + off,
                                    static_cast<size_t>(len), cudaMemcpyHostToDevice, cp_),
                    "loader h2d");
        } else {
            if (!host_[slot_])
                cuda_ok(cudaMallocHost(&host_[slot_], static_cast<size_t>(bin_)), "loader pinned bin");
            // the H2D copy that last read this host bin must be done
            cuda_ok(cudaEventSynchronize(ev_copy_[slot_]), "loader host bin");
            if (src.host) {
                std::memcpy(host_[slot_], static_cast<const char*>(src.host) + off, static_cast<size_t>(len));
            } else {
                read_file(src.path, src.offset + off, host_[slot_], len);
            }
            cuda_ok(cudaMemcpyAsync(dev_[slot_], host_[slot_], static_cast<size_t>(len),
                                    cudaMemcpyHostToDevice, cp_),
                    "loader h2d");
        }
        cuda_ok(cudaEventRecord(ev_copy_[slot_], cp_), "ev");
        cuda_ok(cudaStreamWaitEvent(cs_, ev_copy_[slot_], 0), "loader wait");
        bytes_ += static_cast<double>(len);
        return dev_[slot_];
    }
    void release() { cuda_ok(cudaEventRecord(ev_used_[slot_], cs_), "ev"); }

private:
    static bool pinned(const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    }
    void read_file(const std::string& path, int64_t off, void* dst, int64_t len) {
        auto it = fds_.find(path);
        if (it == fds_.end()) {
            const int fd = ::open(path.c_str(), O_RDONLY);
            if (fd < 0) throw std::invalid_argument("pipeline: cannot open weight file " + path);
            it = fds_.emplace(path, fd).first;
        }
        int64_t done = 0;
        while (done < len) {
            const ssize_t r = ::pread(it->second, static_cast<char*>(dst) + done,
                                      static_cast<size_t>(len - done), off + done);
            if (r <= 0)
                throw std::invalid_argument("pipeline: short read from " + path + " at byte " +
                                            std::to_string(off + done));
            done += r;
        }
    }

    cudaStream_t cs_ = nullptr, cp_ = nullptr;
    int64_t bin_ = 0;
    void* dev_[2] = {nullptr, nullptr};
    void* host_[2] = {nullptr, nullptr};
    cudaEvent_t ev_copy_[2] = {nullptr, nullptr}, ev_used_[2] = {nullptr, nullptr};
    int slot_ = 0;
    int64_t bins_ = 0;
    double bytes_ = 0.0;
    std::map<std::string, int> fds_;
};

}  // namespace

struct pipeline::impl {
    plan_io::plan_document plan;
    model_spec model;
    int rank = 0, world = 1;
    pipeline_options opt;
    int begin = 0, end = 0;
    std::vector<int> bits;
    int B = 0, s = 0, n = 0, eta = 0, xi = 0, S_max = 0;
    int64_t h1 = 0, h2 = 0, vocab = 0;
    int heads = 0, hd = 0;  // attention heads, head dim
    pipesim::microbatch_schedule sched;
    std::vector<unit_ref> units;      // this stage, execution order
    std::vector<unit_ref> prev_units; // previous stage's order (recv order), rank > 0
    std::vector<unit_ref> last_units; // last stage's order (feedback order)
    std::vector<int> group_size;      // requests per decode group
    std::vector<int> group_first;     // first request of each group
    bool first = false, last = false; // stage 0 (embedding) / last stage (LM head)

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
        void* kv = nullptr;  // K cache [B][S_max][h1], then V cache, bf16
        int bits = 16;
    };
    std::vector<layer> layers;
    // stage 0: embedding, positions, prompt token ids
    void* embed = nullptr;       // [vocab x h1] (rank 0 and the last rank)
    void* pos_emb = nullptr;     // [pos_s x h1] (rank 0)
    int32_t* prompt_tok = nullptr;    // [B x s] working prompt ids (rank 0)
    int32_t* pristine_tok = nullptr;  // [B x s] synthetic prompt ids (rank 0)
    // last stage: final LN, tied LM head, generated tokens
    void* lnf[2] = {nullptr, nullptr};
    opw lm;                      // 16-bit packed embedding (hp_qlinear LM head)
    void* lm_x = nullptr;        // [xi x h1] gathered last positions
    void* lm_a = nullptr;        // [xi x h1] final-LN output
    void* logits = nullptr;      // [xi x vocab]
    int32_t* out_tok = nullptr;  // [B x n] generated ids (last rank)
    int32_t* cur_tok = nullptr;  // [B] each request's latest token (rank 0 and last rank)
    // activations
    void* prompt = nullptr;      // [B*s x h1] prefill activations
    void* scr_a = nullptr;       // [M x h1] LN / attention output
    void* scr_qkv = nullptr;     // [M x 3h1]
    void* scr_f = nullptr;       // [M x h2]
    std::vector<void*> dec_x;    // per group [xi_g x h1]
    void* ws = nullptr;
    size_t ws_bytes = 0;
    // decode attention: the context is split over attn_split CTAs per
    // (request, head) only when the (request, head) pairs alone would not
    // fill the SMs (~8 resident CTAs each); with the head-major cache one
    // CTA per pair streams contiguous rows at ~0.92 of HBM
    int attn_split = 1;
    void* attn_ws = nullptr;
    int64_t weight_bytes = 0;
    load_stats lstats;

    // events
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join_s = nullptr, ev_join_r = nullptr;
    std::vector<cudaEvent_t> unit_ev;        // 2 per unit
    std::vector<cudaEvent_t> recv_ev;        // per incoming message
    std::vector<cudaEvent_t> comp_ev;        // per outgoing message
    size_t comp_used = 0;
    bool timed_out = false;
    std::vector<cudaEvent_t> op_ev[2];       // instrumented unit per phase: 4 ops + attention
    std::vector<cudaEvent_t> lay_ev[2];      // whole layer, same unit
    std::vector<double> layer_s[2];          // last instrumented run, per layer
    int instr_unit[2] = {-1, -1};
    kernel_stats kstats[4];
    std::vector<double> unit_s;

    void* alloc(size_t bytes) {
        void* p = nullptr;
        cuda_ok(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "cudaMalloc");
        return p;
    }

    int prefill_rows(int k) const { return sched.prefill_sizes[k] * s; }
    void* prefill_ptr(int k) const {
        return static_cast<char*>(prompt) + static_cast<size_t>(k) * eta * s * h1 * 2;
    }
    void* kcache(const layer& L) const { return L.kv; }
    void* vcache(const layer& L) const {
        return static_cast<char*>(L.kv) + static_cast<size_t>(B) * S_max * h1 * 2;
    }

    // ---- weights -----------------------------------------------------------
    const tensor_source* source(const std::vector<tensor_source>& v, size_t i) const {
        if (!opt.weights || i >= v.size() || v[i].empty()) return nullptr;
        return &v[i];
    }
    const tensor_source* source(const tensor_source& t) const {
        return opt.weights && !t.empty() ? &t : nullptr;
    }

    // bf16 [n x k] -> packed op (tile layout, K1), from a source (binned) or
    // the seeded synthetic generator
    void load_linear(bin_loader& ld, const tensor_source* src, uint64_t seed, int64_t nn,
                     int64_t kk, int b, opw& w, void* tmp) {
        const int64_t pb = hp_packed_bytes(nn, kk, b);
        w.packed = alloc(pb);
        weight_bytes += pb;
        if (b != 16) {
            const int64_t sc = hp_scale_count(nn, kk);
            w.scale = static_cast<float*>(alloc(sc * 4));
            weight_bytes += sc * 4;
            if (opt.scheme == HP_ASYMMETRIC) {
                w.zero = static_cast<float*>(alloc(sc * 4));
                weight_bytes += sc * 4;
            }
        }
        w.w = hp_qweight{nn, kk, b, opt.scheme, w.packed, w.scale, w.zero};
        if (!src) {
            cuda_ok(hp::launch_synth(tmp, nn * kk, seed, 0.0, opt.weight_std, cs), "synth weights");
            hp_ok(hp_quant_pack(tmp, nn, kk, kk, b, opt.scheme, HP_NEAREST, w.packed, w.scale,
                                w.zero, nullptr, nullptr, cs),
                  "quant_pack");
            return;
        }
        // bins of whole 128-row tiles: a row block's codes/scales are
        // contiguous in the tile layout (layout.cuh)
        const int64_t G = (kk + 127) / 128;
        int64_t rows = ld.bin_bytes() / (kk * 2) / 128 * 128;
        if (rows < 128) throw std::invalid_argument("pipeline: bin_bytes below one 128-row block");
        for (int64_t r0 = 0; r0 < nn; r0 += rows) {
            const int64_t rr = std::min(rows, nn - r0);
            void* bin = ld.fetch(*src, r0 * kk * 2, rr * kk * 2);
            const int64_t t0 = r0 / 128;
            hp_ok(hp_quant_pack(bin, rr, kk, kk, b, opt.scheme, HP_NEAREST,
                                static_cast<char*>(w.packed) + t0 * G * b * 2048,
                                w.scale ? w.scale + t0 * G * 128 : nullptr,
                                w.zero ? w.zero + t0 * G * 128 : nullptr, nullptr, nullptr, cs),
                  "quant_pack (bin)");
            ld.release();
        }
    }
    // plain bf16 tensor [elems] -> device
    void* load_plain(bin_loader& ld, const tensor_source* src, uint64_t seed, int64_t elems,
                     double mean, double std_) {
        void* d = alloc(elems * 2);
        weight_bytes += elems * 2;
        if (!src) {
            cuda_ok(hp::launch_synth(d, elems, seed, mean, std_, cs), "synth");
            return d;
        }
        for (int64_t off = 0; off < elems * 2; off += ld.bin_bytes()) {
            const int64_t len = std::min<int64_t>(ld.bin_bytes(), elems * 2 - off);
            void* bin = ld.fetch(*src, off, len);
            cuda_ok(cudaMemcpyAsync(static_cast<char*>(d) + off, bin, len, cudaMemcpyDeviceToDevice, cs),
                    "loader d2d");
            ld.release();
        }
        return d;
    }

    void load_weights() {
        const auto t0 = std::chrono::steady_clock::now();
        const op_shape shp[4] = {{3 * h1, h1}, {h1, h1}, {h2, h1}, {h1, h2}};
        const int64_t bin = opt.weights ? std::max<int64_t>(opt.weights->bin_bytes, 1 << 20) : (64 << 20);
        bin_loader ld(cs, bin);
        void* tmp = alloc(static_cast<size_t>(h2) * h1 * 2);  // synthetic staging (largest op)
        const std::vector<tensor_source> none;
        const auto& lin = opt.weights ? opt.weights->linear : none;
        const auto& nrm = opt.weights ? opt.weights->norm : none;
        layers.resize(end - begin);
        for (int l = begin; l < end; ++l) {
            layer& L = layers[l - begin];
            L.bits = bits[l - begin];
            for (int o = 0; o < 4; ++o)
                load_linear(ld, source(lin, static_cast<size_t>(l) * 4 + o),
                            seed_for(opt.seed, {1, uint64_t(l), uint64_t(o)}), shp[o].n, shp[o].k,
                            L.bits, L.ops[o], tmp);
            for (int j = 0; j < 4; ++j)  // LN gain ~ 1, bias ~ 0 (synthetic)
                L.ln[j] = load_plain(ld, source(nrm, static_cast<size_t>(l) * 4 + j),
                                     seed_for(opt.seed, {4, uint64_t(l), uint64_t(j)}), h1,
                                     (j % 2 == 0) ? 1.0 : 0.0, 0.02);
            L.kv = alloc(static_cast<size_t>(2) * B * S_max * h1 * 2);
        }
        if (first || last) {
            const tensor_source* es = opt.weights ? source(opt.weights->embed) : nullptr;
            embed = load_plain(ld, es, seed_for(opt.seed, {6}), vocab * h1, 0.0, 0.02);
        }
        if (first && model.pos_s > 2) {
            const tensor_source* ps = opt.weights ? source(opt.weights->pos) : nullptr;
            pos_emb = load_plain(ld, ps, seed_for(opt.seed, {7}), model.pos_s * h1, 0.0, 0.02);
        }
        if (last) {
            for (int j = 0; j < 2; ++j) {
                const tensor_source* fs = opt.weights ? source(opt.weights->final_norm[j]) : nullptr;
                lnf[j] = load_plain(ld, fs, seed_for(opt.seed, {8, uint64_t(j)}), h1, j == 0 ? 1.0 : 0.0,
                                    0.02);
            }
            // tied LM head: the embedding repacked by K1 at 16 bits (tile layout)
            const int64_t pb = hp_packed_bytes(vocab, h1, 16);
            lm.packed = alloc(pb);
            weight_bytes += pb;
            lm.w = hp_qweight{vocab, h1, 16, opt.scheme, lm.packed, nullptr, nullptr};
            hp_ok(hp_quant_pack(embed, vocab, h1, h1, 16, opt.scheme, HP_NEAREST, lm.packed, nullptr,
                                nullptr, nullptr, nullptr, cs),
                  "lm head pack");
            if (!first) {  // the last rank keeps only the packed copy
                cuda_ok(cudaStreamSynchronize(cs), "lm head");
                cudaFree(embed);
                weight_bytes -= vocab * h1 * 2;
                embed = nullptr;
            }
        }
        cuda_ok(cudaStreamSynchronize(cs), "weights");
        cudaFree(tmp);
        lstats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        lstats.source_bytes = ld.source_bytes();
        lstats.bins = ld.bins();
        lstats.packed_bytes = static_cast<double>(weight_bytes);
    }

    void build(const std::vector<std::array<char, 128>>& ids) {
        const auto slice = plan_io::slice_for_stage(plan, rank);
        begin = slice.begin;
        end = slice.end;
        bits = slice.bits;
        B = plan.load.global_bz;
        s = plan.load.prompt_len;
        n = plan.load.gen_len;
        S_max = s + n;
        eta = plan.p.eta;
        xi = plan.p.xi;
        h1 = model.h1;
        h2 = model.h2;
        vocab = model.vocab_s;
        heads = model.num_heads;
        first = rank == 0;
        last = rank == world - 1;
        if (heads <= 0 || h1 % heads) throw std::invalid_argument("pipeline: h1 % num_heads != 0");
        hd = static_cast<int>(h1 / heads);
        if (hd != 64 && hd != 128)
            throw std::invalid_argument("pipeline: attention head dim must be 64 or 128 (h1 / num_heads = " +
                                        std::to_string(hd) + ")");
        if (vocab <= 0 || vocab > (int64_t(1) << 31)) throw std::invalid_argument("pipeline: bad vocab_s");
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

        load_weights();

        // ---- activations and token buffers -----------------------------
        const int64_t M = static_cast<int64_t>(eta) * s;
        prompt = alloc(static_cast<size_t>(B) * s * h1 * 2);
        if (first) {
            prompt_tok = static_cast<int32_t*>(alloc(static_cast<size_t>(B) * s * 4));
            pristine_tok = static_cast<int32_t*>(alloc(static_cast<size_t>(B) * s * 4));
            cuda_ok(hp::launch_synth_tokens(pristine_tok, int64_t(B) * s, seed_for(opt.seed, {3}), vocab, cs),
                    "synth prompt");
        }
        if (first || last) {
            cur_tok = static_cast<int32_t*>(alloc(static_cast<size_t>(B) * 4));
            cuda_ok(cudaMemsetAsync(cur_tok, 0, static_cast<size_t>(B) * 4, cs), "memset");
        }
        if (last) {
            out_tok = static_cast<int32_t*>(alloc(static_cast<size_t>(B) * n * 4));
            lm_x = alloc(static_cast<size_t>(xi) * h1 * 2);
            lm_a = alloc(static_cast<size_t>(xi) * h1 * 2);
            logits = alloc(static_cast<size_t>(xi) * vocab * 2);
        }
        const int64_t Mx = std::max<int64_t>(M, xi);
        scr_a = alloc(Mx * h1 * 2);
        scr_qkv = alloc(Mx * 3 * h1 * 2);
        scr_f = alloc(Mx * h2 * 2);
        for (int g = 0; g < sched.num_groups; ++g) {
            dec_x.push_back(alloc(static_cast<size_t>(group_size[g]) * h1 * 2));
            cuda_ok(cudaMemsetAsync(dec_x.back(), 0, group_size[g] * h1 * 2, cs), "memset");
        }
        // split-K workspace: max over this stage's ops and every (rows, phase)
        // the round launches -- a ragged last prefill micro-batch (B % eta != 0)
        // or a short last decode group can need MORE stream-K workspace than
        // the full-size one (fewer tiles -> more segments per tile)
        for (const auto& sh : round_shapes()) {
            for (const layer& L : layers)
                for (const opw& w : L.ops)
                    ws_bytes = std::max(ws_bytes,
                                        hp_qlinear_workspace_bytes(&w.w, sh.first, sh.second));
        }
        if (last)
            for (int m = 1; m <= xi; ++m)
                ws_bytes = std::max(ws_bytes, hp_qlinear_workspace_bytes(&lm.w, m, HP_DECODE));
        if (ws_bytes) {
            ws = alloc(ws_bytes);
            cuda_ok(cudaMemsetAsync(ws, 0, ws_bytes, cs), "ws");
        }
        {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            int min_pairs = xi;  // the smallest decode group
            for (int gs : group_size) min_pairs = std::min(min_pairs, gs);
            min_pairs *= static_cast<int>(h1 / hd);
            attn_split = std::max(1, std::min(8, (8 * sms + min_pairs - 1) / std::max(1, min_pairs)));
        }
        if (const size_t ab = hp::attn_decode_workspace(xi, static_cast<int>(h1), hd, attn_split)) {
            attn_ws = alloc(ab);
            cuda_ok(cudaMemsetAsync(attn_ws, 0, ab, cs), "attention ws");
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
            op_ev[ph].resize(static_cast<size_t>(layers.size()) * 5 * 2);
            for (auto& e : op_ev[ph]) cuda_ok(cudaEventCreate(&e), "ev");
            lay_ev[ph].resize(static_cast<size_t>(layers.size()) * 2);
            for (auto& e : lay_ev[ph]) cuda_ok(cudaEventCreate(&e), "ev");
            layer_s[ph].assign(layers.size(), 0.0);
        }
        cuda_ok(cudaStreamSynchronize(cs), "init");
    }

    // feedback messages last -> 0 (token ids), in the last stage's emission
    // order: the micro-batch manager replays the last stage's completions
    // (a group's first tokens go out when its last prefill batch is done)
    std::vector<unit_ref> feedback_order() const {
        std::vector<unit_ref> out;
        if (world == 1) return out;
        microbatch_manager m(B, eta, xi, n);
        for (const unit_ref& u : last_units) {
            if (u.kind == pipesim::unit_kind::prefill) {
                const int g = m.prefill_done(u.index);
                if (g >= 0 && n >= 2) out.push_back({pipesim::unit_kind::decode, g, 1});
            } else {
                m.decode_done(u.index, u.token);
                if (u.token + 1 <= n - 1) out.push_back({pipesim::unit_kind::decode, u.index, u.token + 1});
            }
        }
        return out;
    }

    void record(cudaEvent_t* evs, int i) {
        if (evs) cuda_ok(timing_record(evs[i], cs), "ev");
    }

    // HP_PIPE_TRACE=1 (eager rounds only): an event after every launch, so
    // the watchdog can name the first kernel that did not complete
    bool trace_on = [] {
        const char* e = std::getenv("HP_PIPE_TRACE");
        return e && *e && *e != '0';
    }();
    std::vector<cudaEvent_t> trace_ev;
    std::vector<std::string> trace_what;
    size_t trace_n = 0;
    int trace_unit = -1;
    void tr(const char* what, int li = -1) {
        if (!trace_on) return;
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cuda_ok(cudaStreamIsCapturing(cs, &cap), "capture status");
        if (cap != cudaStreamCaptureStatusNone) return;
        if (trace_n == trace_ev.size()) {
            cudaEvent_t e;
            cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "trace ev");
            trace_ev.push_back(e);
            trace_what.emplace_back();
        }
        trace_what[trace_n] = "unit " + std::to_string(trace_unit) + " layer " + std::to_string(li) + " " + what;
        cuda_ok(cudaEventRecord(trace_ev[trace_n], cs), "trace ev");
        ++trace_n;
    }

    void qlin(const opw& w, const void* x, int64_t ldx, int64_t m, void* y, int64_t ldy,
              const void* res, int epi, int phase) {
        hp_ok(hp_qlinear(&w.w, x, ldx, m, y, ldy, res, res ? ldy : 0, epi, phase, ws, ws_bytes, cs),
              "qlinear");
    }

    // the requests / positions a unit works on (attention context)
    struct unit_ctx {
        int req0, nreq;
        int pos;  // decode: the new token's position; prefill: -1 (positions 0..s-1)
    };

    // forward of this stage's layers, in place on x [m x h1]
    void forward(void* x, int64_t m, int phase, bool instrument, const unit_ctx& u) {
        for (size_t li = 0; li < layers.size(); ++li) {
            const layer& L = layers[li];
            cudaEvent_t* ev = instrument ? &op_ev[phase][li * 10] : nullptr;
            if (instrument) cuda_ok(timing_record(lay_ev[phase][2 * li], cs), "ev");
            cuda_ok(hp::launch_layernorm(x, h1, m, static_cast<int>(h1), L.ln[0], L.ln[1], scr_a,
                                         h1, cs),
                    "ln1");
            tr("ln1", static_cast<int>(li));
            record(ev, 0);
            qlin(L.ops[0], scr_a, h1, m, scr_qkv, 3 * h1, nullptr, HP_EPI_NONE, phase);
            tr("qkv", static_cast<int>(li));
            record(ev, 1);
            // causal multi-head attention over the KV cache -> scr_a
            if (phase == HP_PREFILL) {
                cuda_ok(hp::launch_attn_prefill(scr_qkv, u.nreq, s, static_cast<int>(h1), hd, scr_a,
                                                kcache(L), vcache(L), u.req0, S_max, cs),
                        "attention (prefill)");
            } else {
                cuda_ok(hp::launch_attn_decode(scr_qkv, u.nreq, static_cast<int>(h1), hd, u.pos, scr_a,
                                               kcache(L), vcache(L), u.req0, S_max, cs, attn_ws,
                                               attn_split),
                        "attention (decode)");
            }
            tr("attention", static_cast<int>(li));
            record(ev, 8);
            record(ev, 2);
            qlin(L.ops[1], scr_a, h1, m, x, h1, x, HP_EPI_NONE, phase);
            tr("out", static_cast<int>(li));
            record(ev, 3);
            cuda_ok(hp::launch_layernorm(x, h1, m, static_cast<int>(h1), L.ln[2], L.ln[3], scr_a,
                                         h1, cs),
                    "ln2");
            tr("ln2", static_cast<int>(li));
            record(ev, 4);
            qlin(L.ops[2], scr_a, h1, m, scr_f, h2, nullptr, HP_EPI_RELU, phase);
            tr("fc1", static_cast<int>(li));
            record(ev, 5);
            record(ev, 6);
            qlin(L.ops[3], scr_f, h2, m, x, h1, x, HP_EPI_NONE, phase);
            tr("fc2", static_cast<int>(li));
            record(ev, 7);
            if (instrument) cuda_ok(timing_record(lay_ev[phase][2 * li + 1], cs), "ev");
        }
    }
    // attention span of the instrumented layer: events 1 (after qkv) .. 8
    // (after attention); op spans: (0,1) qkv, (2,3) out, (4,5) fc1, (6,7) fc2

    // stage 0: token ids -> x (token embedding + learned position)
    void embed_prefill(int k) {
        cuda_ok(hp::launch_embed(prompt_tok + static_cast<size_t>(k) * eta * s, prefill_rows(k), 0, 1, s,
                                 embed, pos_emb, static_cast<int>(model.pos_s), static_cast<int>(h1),
                                 vocab, prefill_ptr(k), cs),
                "embed");
    }
    void embed_decode(int g, int tok) {
        cuda_ok(hp::launch_embed(cur_tok + group_first[g], group_size[g], s + tok - 1, 0, 1, embed, pos_emb,
                                 static_cast<int>(model.pos_s), static_cast<int>(h1), vocab, dec_x[g], cs),
                "embed");
    }
    // last stage: final LN + tied LM head + argmax of `rows` hidden rows at
    // x (row stride ldx, first row offset `off`), requests req0.. -> cur_tok
    // and out_tok[:, col]
    void lm_head(const void* x, int64_t stride, int64_t off, int rows, int req0, int col) {
        cuda_ok(hp::launch_gather_rows(x, h1, stride, off, rows, static_cast<int>(h1), lm_x, h1, cs),
                "gather");
        tr("gather");
        cuda_ok(hp::launch_layernorm(lm_x, h1, rows, static_cast<int>(h1), lnf[0], lnf[1], lm_a, h1, cs),
                "final ln");
        tr("final ln");
        qlin(lm, lm_a, h1, rows, logits, vocab, nullptr, HP_EPI_NONE, HP_DECODE);
        tr("lm head");
        cuda_ok(hp::launch_argmax(logits, vocab, rows, vocab, cur_tok + req0,
                                  out_tok + static_cast<size_t>(req0) * n + col, n, cs),
                "argmax");
        tr("argmax");
    }

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

    // CUDA loads a kernel's module lazily at its first launch, and that load
    // waits for the device: issued while an NCCL recv kernel spins on rs (it
    // waits for a message this very stage must first compute and send) it
    // never returns. So run every (phase, rows) forward the round will use,
    // and the glue, once on scratch before any NCCL operation is posted.
    void load_kernels() {
        const auto shapes = round_shapes();
        int64_t rows = 1;
        for (const auto& sh : shapes) rows = std::max(rows, sh.first);
        void* x = nullptr;
        cuda_ok(cudaMalloc(&x, static_cast<size_t>(rows) * h1 * 2), "cudaMalloc scratch");
        cuda_ok(hp::launch_synth(x, rows * h1, seed_for(opt.seed, {5}), 0.0, 1.0, cs), "synth scratch");
        for (const auto& sh : shapes) {
            const bool pre = sh.second == HP_PREFILL;
            forward(x, sh.first, sh.second, false, {0, pre ? static_cast<int>(sh.first / s) : static_cast<int>(sh.first), pre ? -1 : s});
        }
        if (first) embed_decode(0, 1);
        if (last) {
            for (int g = 0; g < sched.num_groups; ++g) lm_head(x, 1, 0, group_size[g], 0, 0);
            for (int k = 0; k < static_cast<int>(sched.prefill_sizes.size()); ++k)
                lm_head(x, 1, 0, sched.prefill_sizes[k], 0, 0);
        }
        cuda_ok(cudaStreamSynchronize(cs), "load kernels");
        cuda_ok(cudaFree(x), "cudaFree scratch");
        if (ws_bytes) cuda_ok(cudaMemsetAsync(ws, 0, ws_bytes, cs), "ws");
        if (cur_tok) cuda_ok(cudaMemsetAsync(cur_tok, 0, static_cast<size_t>(B) * 4, cs), "memset");
        for (const layer& L : layers)  // scratch forwards wrote cache rows
            cuda_ok(cudaMemsetAsync(L.kv, 0, static_cast<size_t>(2) * B * S_max * h1 * 2, cs), "kv");
        cuda_ok(cudaStreamSynchronize(cs), "load kernels");
    }

    // NCCL connects P2P channels lazily, host-blocking, on the first
    // send/recv that needs them (how many channels / which protocol depends
    // on the message size) and needs the peer to connect the SAME link
    // concurrently. A round posts rank 0's feedback recvs (link world-1)
    // first while rank 1 waits on link 0 -> a cycle of blocked hosts. So
    // exchange one message of every size the round uses on each link here,
    // in ascending link order (rank r: link r-1 then link r; rank 0: link 0
    // then link world-1) -- a chain, which cannot deadlock.
    // Messages: bf16 activations on links l < world-1; int32 token ids on
    // the feedback link world-1 -> 0. Returns (count, is_tokens).
    std::vector<std::pair<size_t, bool>> link_msgs(int l) const {
        std::vector<std::pair<size_t, bool>> c;
        if (l < world - 1) {
            for (int k = 0; k < static_cast<int>(sched.prefill_sizes.size()); ++k)
                c.push_back({static_cast<size_t>(prefill_rows(k)) * h1, false});
            for (int g = 0; g < sched.num_groups; ++g) c.push_back({static_cast<size_t>(group_size[g]) * h1, false});
        } else {
            for (int g = 0; g < sched.num_groups; ++g) c.push_back({static_cast<size_t>(group_size[g]), true});
        }
        std::sort(c.begin(), c.end());
        c.erase(std::unique(c.begin(), c.end()), c.end());
        return c;
    }
    void connect_links() {
        const int prev = (rank - 1 + world) % world;
        size_t maxb = 0;
        for (int l : {rank, prev})
            for (const auto& c : link_msgs(l)) maxb = std::max(maxb, c.first * (c.second ? 4 : 2));
        void* probe = nullptr;
        cuda_ok(cudaMalloc(&probe, maxb), "cudaMalloc probe");
        auto link = [&](bool out) {
            for (const auto& c : link_msgs(out ? rank : prev)) {
                const ncclDataType_t t = c.second ? ncclInt32 : ncclBfloat16;
                PDBG("connect %s count %zu", out ? "out" : "in", c.first);
                if (out)
                    nccl_ok(ncclSend(probe, c.first, t, /*peer=*/1, c_out, cs), "connect send");
                else
                    nccl_ok(ncclRecv(probe, c.first, t, /*peer=*/0, c_in, cs), "connect recv");
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

    void send_after_compute(const void* buf, size_t count, ncclDataType_t t, int& comp_i) {
        cuda_ok(cudaEventRecord(comp_ev[comp_i], cs), "ev");
        cuda_ok(cudaStreamWaitEvent(ss, comp_ev[comp_i++], 0), "wait");
        nccl_ok(ncclSend(buf, count, t, /*peer=*/1, c_out, ss), "send");
    }

    // Enqueue one whole round on (cs, ss, rs). Capturable.
    void enqueue_round() {
        // fork side streams off the compute stream (joins them into a capture)
        cuda_ok(cudaEventRecord(ev_fork, cs), "ev");
        cuda_ok(cudaStreamWaitEvent(ss, ev_fork, 0), "wait");
        cuda_ok(cudaStreamWaitEvent(rs, ev_fork, 0), "wait");

        // post every receive in the sender's order
        std::map<std::tuple<int, int, int>, int> recv_idx;
        if (world > 1) {
            const std::vector<unit_ref> incoming = rank > 0 ? prev_units : feedback_order();
            for (size_t i = 0; i < incoming.size(); ++i) {
                const unit_ref& u = incoming[i];
                PDBG("recv %zu (kind %d idx %d tok %d)", i, static_cast<int>(u.kind), u.index, u.token);
                if (rank > 0 && u.kind == pipesim::unit_kind::prefill) {
                    nccl_ok(ncclRecv(prefill_ptr(u.index), static_cast<size_t>(prefill_rows(u.index)) * h1,
                                     ncclBfloat16, /*peer=*/0, c_in, rs),
                            "recv");
                } else if (rank > 0) {
                    nccl_ok(ncclRecv(dec_x[u.index], static_cast<size_t>(group_size[u.index]) * h1,
                                     ncclBfloat16, /*peer=*/0, c_in, rs),
                            "recv");
                } else {  // stage 0: the group's next token ids from the last stage
                    nccl_ok(ncclRecv(cur_tok + group_first[u.index], static_cast<size_t>(group_size[u.index]),
                                     ncclInt32, /*peer=*/0, c_in, rs),
                            "recv tokens");
                }
                cuda_ok(cudaEventRecord(recv_ev[i], rs), "ev");
                recv_idx[{static_cast<int>(u.kind), u.index, u.token}] = static_cast<int>(i);
            }
        }
        trace_n = 0;
        microbatch_manager mbm(B, eta, xi, n);  // the round's status table
        int comp_i = 0;

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
            const unit_ctx ctx = pre ? unit_ctx{u.index * eta, sched.prefill_sizes[u.index], -1}
                                     : unit_ctx{group_first[u.index], group_size[u.index], s + u.token - 1};
            cuda_ok(timing_record(unit_ev[2 * ui], cs), "ev");
            trace_unit = static_cast<int>(ui);
            if (first) {
                if (pre) embed_prefill(u.index);
                else embed_decode(u.index, u.token);
                tr("embed");
            }
            forward(x, m, phase, opt.instrument && instr_unit[phase] == static_cast<int>(ui), ctx);
            if (last) {
                if (pre) lm_head(x, s, s - 1, sched.prefill_sizes[u.index], ctx.req0, 0);
                else lm_head(x, 1, 0, group_size[u.index], ctx.req0, u.token);
            }
            cuda_ok(timing_record(unit_ev[2 * ui + 1], cs), "ev");

            // ---- output
            if (!last) {
                PDBG("send unit %zu count %zu", ui, static_cast<size_t>(m) * h1);
                send_after_compute(x, static_cast<size_t>(m) * h1, ncclBfloat16, comp_i);
                continue;
            }
            // a prefill batch may straddle a group boundary: the group's
            // tokens are complete once the manager marks its last batch done
            const int ready = pre ? mbm.prefill_done(u.index) : -1;
            if (!pre) mbm.decode_done(u.index, u.token);
            if (world == 1) continue;
            if (pre) {
                if (ready >= 0 && n >= 2)
                    send_after_compute(cur_tok + group_first[ready], static_cast<size_t>(group_size[ready]),
                                       ncclInt32, comp_i);
            } else if (u.token + 1 <= n - 1) {
                send_after_compute(cur_tok + group_first[u.index], static_cast<size_t>(group_size[u.index]),
                                   ncclInt32, comp_i);
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
        if (trace_n) {
            size_t t = 0;
            while (t < trace_n && done(trace_ev[t])) ++t;
            msg += t < trace_n ? ", first pending launch: " + trace_what[t] +
                                     (t ? " (last completed: " + trace_what[t - 1] + ")" : std::string())
                               : std::string(", every traced launch completed");
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

    void load_prompt(const int32_t* host_tokens) {
        if (!first) return;
        const size_t bytes = static_cast<size_t>(B) * s * 4;
        if (host_tokens)
            cuda_ok(cudaMemcpyAsync(prompt_tok, host_tokens, bytes, cudaMemcpyHostToDevice, cs), "h2d");
        else
            cuda_ok(cudaMemcpyAsync(prompt_tok, pristine_tok, bytes, cudaMemcpyDeviceToDevice, cs), "d2d");
    }

    run_timing run(const int32_t* host_tokens, int32_t* host_out) {
        run_timing t;
        cuda_ok(cudaEventRecord(ev_t0, cs), "ev");
        load_prompt(host_tokens);
        // HP_EAGER_PDL=0: launch the eager (uncaptured) rounds without
        // programmatic dependent launch (diagnostic for the eager-round stall,
        // DESIGN §8); captured rounds keep it
        struct pdl_off {
            bool on;
            explicit pdl_off(bool e) : on(e) { if (on) hp_set_pdl(0); }
            ~pdl_off() { if (on) hp_set_pdl(1); }
        };
        static const bool eager_no_pdl = [] {
            const char* e = std::getenv("HP_EAGER_PDL");
            return e && *e == '0';
        }();
        if (opt.use_graphs) {
            if (!graph_ready) {
                {
                    pdl_off g(eager_no_pdl);
                    enqueue_round();  // eager warm-up (sets kernel attributes)
                }
                wait_round("warm-up round");
                load_prompt(host_tokens);
                capture();
            }
            cuda_ok(cudaGraphLaunch(graph, cs), "graph launch");
        } else {
            pdl_off g(eager_no_pdl);
            enqueue_round();
        }
        if (last && host_out)
            cuda_ok(cudaMemcpyAsync(host_out, out_tok, static_cast<size_t>(B) * n * 4,
                                    cudaMemcpyDeviceToHost, cs),
                    "d2h");
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

    void final_hidden(void* host) const {
        if (!last) throw std::invalid_argument("pipeline: final_hidden is on the last rank");
        for (int g = 0; g < sched.num_groups; ++g)
            cuda_ok(cudaMemcpy(static_cast<char*>(host) + static_cast<size_t>(group_first[g]) * h1 * 2,
                               n >= 2 ? dec_x[g] : prompt, static_cast<size_t>(group_size[g]) * h1 * 2,
                               cudaMemcpyDeviceToHost),
                    "final hidden");
    }

    void collect_kernel_stats() {
        const op_shape shp[4] = {{3 * h1, h1}, {h1, h1}, {h2, h1}, {h1, h2}};
        const int pairs[4][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}};
        for (int ph = 0; ph < 2; ++ph) {
            const int ui = instr_unit[ph];
            if (ui < 0) continue;
            const unit_ref& u = units[ui];
            const int64_t m = ph == 0 ? prefill_rows(u.index) : group_size[u.index];
            const int nreq = ph == 0 ? sched.prefill_sizes[u.index] : group_size[u.index];
            const double ctx = ph == 0 ? s : s + u.token;  // keys per query (decode) / prompt
            for (size_t li = 0; li < layers.size(); ++li) {
                float ms = 0.f;
                cuda_ok(cudaEventElapsedTime(&ms, lay_ev[ph][2 * li], lay_ev[ph][2 * li + 1]),
                        "elapsed layer");
                layer_s[ph][li] = ms * 1e-3;
                for (int o = 0; o < 4; ++o) {
                    cuda_ok(cudaEventElapsedTime(&ms, op_ev[ph][li * 10 + pairs[o][0]],
                                                 op_ev[ph][li * 10 + pairs[o][1]]),
                            "elapsed op");
                    kernel_stats& k = kstats[ph];
                    ++k.launches;
                    k.seconds += ms * 1e-3;
                    k.bytes += k3_bytes(shp[o], layers[li].bits, opt.scheme, m);
                    k.flops += 2.0 * m * shp[o].n * shp[o].k;
                }
                cuda_ok(cudaEventElapsedTime(&ms, op_ev[ph][li * 10 + 1], op_ev[ph][li * 10 + 8]),
                        "elapsed attention");
                kernel_stats& a = kstats[2 + ph];
                ++a.launches;
                a.seconds += ms * 1e-3;
                if (ph == 0) {  // causal: s(s+1)/2 score rows x hd, QK^T and PV
                    a.flops += 4.0 * nreq * heads * hd * (static_cast<double>(s) * (s + 1) / 2);
                    a.bytes += 2.0 * m * 3 * h1 + 2.0 * m * h1 + 2.0 * 2 * m * h1;  // qkv in, out, K/V cache write
                } else {  // K and V rows 0..p of every request, + qkv in, out
                    a.bytes += 2.0 * 2 * nreq * ctx * h1 + 2.0 * m * 3 * h1 + 2.0 * m * h1;
                    a.flops += 4.0 * nreq * heads * hd * ctx;
                }
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
            f(L.kv);
        }
        for (void* p : {embed, pos_emb, static_cast<void*>(prompt_tok), static_cast<void*>(pristine_tok),
                        lnf[0], lnf[1], lm.packed, lm_x, lm_a, logits, static_cast<void*>(out_tok),
                        static_cast<void*>(cur_tok), prompt, scr_a, scr_qkv, scr_f, ws, attn_ws})
            f(p);
        for (void* p : dec_x) f(p);
        for (auto* v : {&unit_ev, &recv_ev, &comp_ev, &op_ev[0], &op_ev[1], &lay_ev[0], &lay_ev[1], &trace_ev})
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
    if (opt.weights) {
        const size_t L4 = static_cast<size_t>(plan.num_layers) * 4;
        if ((!opt.weights->linear.empty() && opt.weights->linear.size() != L4) ||
            (!opt.weights->norm.empty() && opt.weights->norm.size() != L4))
            throw std::invalid_argument("pipeline: weight set needs num_layers*4 linear / norm entries");
    }
    p_->plan = plan;
    p_->model = model;
    p_->rank = rank;
    p_->world = world;
    p_->opt = opt;
    p_->build(nccl_ids);
    p_->opt.weights = nullptr;  // the caller's set is read during construction only
}

pipeline::~pipeline() = default;

run_timing pipeline::run(const std::int32_t* host_tokens, std::int32_t* host_out) {
    return p_->run(host_tokens, host_out);
}

void pipeline::final_hidden(void* host) const { p_->final_hidden(host); }

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

const kernel_stats& pipeline::stats(int kind) const { return p_->kstats[std::clamp(kind, 0, 3)]; }

const std::vector<double>& pipeline::layer_costs(int phase) const {
    return p_->layer_s[phase ? 1 : 0];
}

void pipeline::reset_stats() {
    for (auto& k : p_->kstats) k = kernel_stats{};
}

std::int64_t pipeline::weight_bytes() const { return p_->weight_bytes; }

const load_stats& pipeline::loading() const { return p_->lstats; }

int pipeline::num_kernel_launches_per_round() const {
    int n = 0;
    const int per_layer = 7;  // LN1, qkv, attention, out, LN2, fc1, fc2
    for (const unit_ref& u : p_->units) {
        n += static_cast<int>(p_->layers.size()) * per_layer;
        if (p_->first) ++n;                                            // embedding
        if (p_->last) n += 4;                                          // gather, LN, LM head, argmax
        (void)u;
    }
    return n;
}

}  // namespace hetplan::runtime
