#pragma once
// Micro-batch manager ("Microbatch Manager"): a
// thread-safe status table of one serving round's micro-batches. Every
// prefill micro-batch (eta requests) belongs to the decode micro-batch group
// (xi requests) of its first request (pipesim.cpp:34-44); a group is
// enqueued for the decode phase only when ALL its prefill micro-batches are
// marked done, and each decode token of a group is enqueued when the
// previous one is done, until n - 1 decode tokens ran. One lock guards the
// table, so stage threads, NCCL completion callbacks or a serving front-end
// may report completions concurrently.
//
// The pipeline executor uses it on the last stage to decide when a group's
// first next-token ids are complete (the feedback send to stage 0) and to
// derive the decode unit order; tests drive it from many threads.

#include <cstdint>
#include <deque>
#include <mutex>
#include <vector>

#include "hetplan/pipesim/pipesim.hpp"

namespace hetplan::runtime {

class microbatch_manager {
public:
    enum class status : std::uint8_t { pending, running, done };
    struct decode_item {
        int group;
        int token;  // 1 .. n-1
    };

    // B requests, prefill micro-batch eta, decode micro-batch xi, n tokens
    // per request (make_schedule semantics, pipesim.cpp:22-46).
    microbatch_manager(int B, int eta, int xi, int n);

    int num_prefill() const;
    int num_groups() const;
    int group_of_prefill(int k) const;

    // Prefill micro-batch k finished. Returns the group made ready by it
    // (its first decode token was enqueued), or -1. Idempotent per k: a
    // second report of the same batch returns -1 and changes nothing.
    int prefill_done(int k);
    // Decode token `token` of `group` finished; enqueues token + 1 when
    // token + 1 <= n - 1. Returns true if the group has finished decoding.
    bool decode_done(int group, int token);
    // Pop the next enqueued decode item (FIFO in readiness order).
    bool next_decode(decode_item& out);

    status prefill_status(int k) const;
    bool group_ready(int group) const;
    bool all_done() const;
    void reset();  // a new round

private:
    mutable std::mutex mu_;
    pipesim::microbatch_schedule sched_;
    int n_ = 0;
    std::vector<status> prefill_;
    std::vector<int> left_;        // prefill batches still running per group
    std::vector<int> decoded_;     // decode tokens finished per group
    std::deque<decode_item> queue_;
};

}  // namespace hetplan::runtime
