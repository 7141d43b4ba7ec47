// Thread-safe micro-batch manager (include/hetplan/runtime/microbatch.hpp;
// PAPER.md:798-804). Group membership of the prefill micro-batches comes
// from pipesim::make_schedule (pipesim.cpp:22-46): batch k -> group of its
// first request.
#include "hetplan/runtime/microbatch.hpp"

#include <stdexcept>
#include <string>

namespace hetplan::runtime {

microbatch_manager::microbatch_manager(int B, int eta, int xi, int n)
    : sched_(pipesim::make_schedule(B, eta, xi)), n_(n) {
    if (n < 1) throw std::invalid_argument("microbatch_manager: n must be >= 1");
    reset();
}

int microbatch_manager::num_prefill() const { return static_cast<int>(sched_.prefill_sizes.size()); }
int microbatch_manager::num_groups() const { return sched_.num_groups; }
int microbatch_manager::group_of_prefill(int k) const { return sched_.group_of_prefill.at(k); }

void microbatch_manager::reset() {
    std::lock_guard<std::mutex> g(mu_);
    prefill_.assign(sched_.prefill_sizes.size(), status::pending);
    left_.assign(sched_.num_groups, 0);
    for (int grp : sched_.group_of_prefill) ++left_[grp];
    decoded_.assign(sched_.num_groups, 0);
    queue_.clear();
}

int microbatch_manager::prefill_done(int k) {
    std::lock_guard<std::mutex> g(mu_);
    if (k < 0 || k >= static_cast<int>(prefill_.size()))
        throw std::invalid_argument("microbatch_manager: prefill batch " + std::to_string(k) +
                                    " out of range");
    if (prefill_[k] == status::done) return -1;
    prefill_[k] = status::done;
    const int grp = sched_.group_of_prefill[k];
    if (--left_[grp] != 0) return -1;
    if (n_ >= 2) queue_.push_back({grp, 1});
    return grp;
}

bool microbatch_manager::decode_done(int group, int token) {
    std::lock_guard<std::mutex> g(mu_);
    if (group < 0 || group >= sched_.num_groups)
        throw std::invalid_argument("microbatch_manager: group out of range");
    if (left_[group] != 0)
        throw std::logic_error("microbatch_manager: decode reported before the group's prefill finished");
    if (token != decoded_[group] + 1 || token > n_ - 1)
        throw std::logic_error("microbatch_manager: decode token " + std::to_string(token) +
                               " of group " + std::to_string(group) + " out of order");
    decoded_[group] = token;
    if (token + 1 <= n_ - 1) queue_.push_back({group, token + 1});
    return token == n_ - 1;
}

bool microbatch_manager::next_decode(decode_item& out) {
    std::lock_guard<std::mutex> g(mu_);
    if (queue_.empty()) return false;
    out = queue_.front();
    queue_.pop_front();
    return true;
}

microbatch_manager::status microbatch_manager::prefill_status(int k) const {
    std::lock_guard<std::mutex> g(mu_);
    return prefill_.at(k);
}

bool microbatch_manager::group_ready(int group) const {
    std::lock_guard<std::mutex> g(mu_);
    return left_.at(group) == 0;
}

bool microbatch_manager::all_done() const {
    std::lock_guard<std::mutex> g(mu_);
    for (int l : left_)
        if (l) return false;
    for (int d : decoded_)
        if (d != n_ - 1) return false;
    return true;
}

}  // namespace hetplan::runtime
