// Pipeline schedule + discrete-event timing model (B200 build).
//
// make_schedule follows /root/reference/proj/src/pipesim.cpp:22-46; the
// simulator reproduces the reference engine's semantics (:86-248) — events
// ordered by (time, arrival-before-completion, stage, unit), all events of
// one instant applied before the touched stages dispatch (FIFO by (ready,
// kind, index, token)), one transfer at a time per link overlapped with
// compute — so makespans agree bit-for-bit. The B200 executor
// (csrc/host/pipeline.cpp) walks the same schedule.
#include "hetplan/pipesim/pipesim.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>
#include <stdexcept>
#include <tuple>

#include <json.hpp>

#include "hetplan/types.hpp"

namespace hetplan::pipesim {

namespace {

[[noreturn]] void reject(const std::string& what) {
    throw std::invalid_argument(what);
}

struct unit {
    unit_kind kind;
    int index;
    int token;
    auto key() const { return std::make_tuple(kind, index, token); }
};

struct waiting {  // unit queued at a stage
    double ready;
    unit u;
    bool operator<(const waiting& o) const {
        return std::make_tuple(ready, u.key()) < std::make_tuple(o.ready, o.u.key());
    }
};

struct event {
    double at;
    int type;  // 0 = arrival, 1 = compute finished
    int stage;
    unit u;
    bool operator<(const event& o) const {
        return std::make_tuple(at, type, stage, u.key()) <
               std::make_tuple(o.at, o.type, o.stage, o.u.key());
    }
};

class engine {
public:
    engine(const std::vector<stage_cost>& c, const microbatch_schedule& s, int n, bool tl)
        : cost_(c), sched_(s), n_(n), keep_(tl), S_(static_cast<int>(c.size())),
          queues_(S_), free_at_(S_, 0.0), busy_(S_, 0.0),
          link_free_(std::max(0, S_ - 1), 0.0), pending_(s.num_groups, 0) {
        for (int g : s.group_of_prefill) ++pending_[g];
        for (int k = 0; k < static_cast<int>(s.prefill_sizes.size()); ++k)
            events_.insert({0.0, 0, 0, {unit_kind::prefill, k, 0}});
    }

    void run() {
        while (!events_.empty()) {
            const double now = events_.begin()->at;
            for (;;) {
                std::set<int> touched;
                bool any = false;
                while (!events_.empty() && events_.begin()->at == now) {
                    const event e = *events_.begin();
                    events_.erase(events_.begin());
                    handle(e, touched);
                    any = true;
                }
                for (int j : touched) dispatch(j, now);
                if (!any) break;
            }
        }
    }

    double makespan = 0.0;
    std::int64_t finished = 0;
    std::vector<timeline_event> timeline;
    const std::vector<double>& busy() const { return busy_; }

private:
    double compute(int j, const unit& u) const {
        return u.kind == unit_kind::prefill ? cost_[j].pre_s : cost_[j].dec_s;
    }
    double transfer(int j, const unit& u) const {
        return u.kind == unit_kind::prefill ? cost_[j].comm_pre_s : cost_[j].comm_dec_s;
    }

    void leave_pipeline(const unit& u, double t) {
        makespan = std::max(makespan, t);
        ++finished;
        if (u.kind == unit_kind::prefill) {
            const int g = sched_.group_of_prefill[u.index];
            if (--pending_[g] == 0 && n_ >= 2)
                events_.insert({t, 0, 0, {unit_kind::decode, g, 1}});
        } else if (u.token + 1 <= n_ - 1) {
            events_.insert({t, 0, 0, {unit_kind::decode, u.index, u.token + 1}});
        }
    }

    void handle(const event& e, std::set<int>& touched) {
        touched.insert(e.stage);
        if (e.type == 0) {
            queues_[e.stage].insert({e.at, e.u});
            return;
        }
        if (e.stage == S_ - 1) {
            leave_pipeline(e.u, e.at);
            return;
        }
        const double start = std::max(e.at, link_free_[e.stage]);
        link_free_[e.stage] = start + transfer(e.stage, e.u);
        events_.insert({link_free_[e.stage], 0, e.stage + 1, e.u});
    }

    void dispatch(int j, double now) {
        if (queues_[j].empty() || free_at_[j] > now) return;
        const waiting w = *queues_[j].begin();
        queues_[j].erase(queues_[j].begin());
        const double c = compute(j, w.u);
        free_at_[j] = now + c;
        busy_[j] += c;
        if (keep_) timeline.push_back({j, w.u.kind, w.u.index, w.u.token, now, now + c});
        events_.insert({now + c, 1, j, w.u});
    }

    const std::vector<stage_cost>& cost_;
    const microbatch_schedule& sched_;
    int n_;
    bool keep_;
    int S_;
    std::set<event> events_;
    std::vector<std::set<waiting>> queues_;
    std::vector<double> free_at_, busy_, link_free_;
    std::vector<int> pending_;
};

}  // namespace

microbatch_schedule make_schedule(int global_bz, int eta, int xi) {
    if (global_bz <= 0) reject("schedule: B must be positive");
    if (eta < 1 || eta > xi || xi > global_bz)
        reject("schedule: need 1 <= eta <= xi <= B (eta=" + std::to_string(eta) +
               " xi=" + std::to_string(xi) + " B=" + std::to_string(global_bz) + ")");
    microbatch_schedule s;
    s.global_bz = global_bz;
    s.eta = eta;
    s.xi = xi;
    const int batches = static_cast<int>(ceil_div(global_bz, eta));
    s.prefill_sizes.reserve(batches);
    for (int k = 0, first = 0; k < batches; ++k, first += eta) {
        s.prefill_sizes.push_back(std::min(eta, global_bz - first));
        s.group_of_prefill.push_back(first / xi);  // group of its first request
    }
    s.num_groups = static_cast<int>(ceil_div(global_bz, xi));
    if (s.group_of_prefill.back() != s.num_groups - 1)
        reject("schedule: decode group " + std::to_string(s.num_groups - 1) +
               " would own no prefill batch");
    return s;
}

sim_report simulate(const std::vector<stage_cost>& stages,
                    const microbatch_schedule& sched, int gen_len, bool keep_timeline) {
    if (stages.empty()) reject("simulate: no stages");
    for (size_t j = 0; j < stages.size(); ++j)
        for (double v : {stages[j].pre_s, stages[j].dec_s, stages[j].comm_pre_s,
                         stages[j].comm_dec_s})
            if (!(v >= 0.0) || !std::isfinite(v))
                reject("simulate: stage " + std::to_string(j) + " cost negative or non-finite");
    if (gen_len < 1) reject("simulate: gen_len must be >= 1");
    const microbatch_schedule want = make_schedule(sched.global_bz, sched.eta, sched.xi);
    if (want.prefill_sizes != sched.prefill_sizes ||
        want.group_of_prefill != sched.group_of_prefill || want.num_groups != sched.num_groups)
        reject("simulate: schedule inconsistent with (B, eta, xi)");

    engine e(stages, sched, gen_len, keep_timeline);
    e.run();
    const std::int64_t expect = static_cast<std::int64_t>(sched.prefill_sizes.size()) +
                                (gen_len >= 2 ? static_cast<std::int64_t>(sched.num_groups) *
                                                    (gen_len - 1)
                                              : 0);
    if (e.finished != expect) throw std::logic_error("simulate: unit count mismatch");

    sim_report r;
    r.makespan_s = e.makespan;
    r.stage_busy_s = e.busy();
    double tot = 0.0;
    for (double b : r.stage_busy_s) tot += b;
    r.bubble_fraction =
        e.makespan > 0.0 ? 1.0 - tot / (static_cast<double>(stages.size()) * e.makespan) : 0.0;
    r.timeline = std::move(e.timeline);
    std::sort(r.timeline.begin(), r.timeline.end(), [](const timeline_event& a,
                                                       const timeline_event& b) {
        return std::make_tuple(a.start, a.stage, a.kind, a.index, a.token) <
               std::make_tuple(b.start, b.stage, b.kind, b.index, b.token);
    });
    return r;
}

double analytic_latency(const std::vector<stage_cost>& stages, int global_bz, int eta,
                        int xi, int gen_len) {
    if (stages.empty()) reject("analytic_latency: no stages");
    double worst_pre = 0.0, worst_dec = 0.0, sum_pre = 0.0, sum_dec = 0.0;
    for (const stage_cost& c : stages) {
        worst_pre = std::max({worst_pre, c.pre_s, c.comm_pre_s});
        worst_dec = std::max({worst_dec, c.dec_s, c.comm_dec_s});
        sum_pre += c.pre_s;
        sum_dec += c.dec_s;
    }
    return static_cast<double>(bubble_count(global_bz, eta)) * worst_pre +
           static_cast<double>(bubble_count(global_bz, xi)) * (gen_len - 1) * worst_dec +
           sum_pre + sum_dec;
}

std::string serialize_report(const sim_report& r, double analytic_s) {
    nlohmann::ordered_json j;
    j["format_version"] = 1;
    j["makespan_s"] = r.makespan_s;
    j["analytic_s"] = analytic_s;
    j["gap_s"] = r.makespan_s - analytic_s;
    j["bubble_fraction"] = r.bubble_fraction;
    j["stage_busy_s"] = r.stage_busy_s;
    j["timeline_events"] = r.timeline.size();
    return j.dump(2) + "\n";
}

std::string timeline_csv(const sim_report& r) {
    std::string s = "stage,kind,index,token,start,end\n";
    char buf[160];
    for (const timeline_event& e : r.timeline) {
        std::snprintf(buf, sizeof buf, "%d,%s,%d,%d,%.17g,%.17g\n", e.stage,
                      e.kind == unit_kind::prefill ? "prefill" : "decode", e.index, e.token,
                      e.start, e.end);
        s += buf;
    }
    return s;
}

}  // namespace hetplan::pipesim
