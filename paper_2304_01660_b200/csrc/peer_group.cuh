// In-process rank group over peer device memory (one host thread per rank).
//
// The alternative to NCCL for a single process driving several GPUs (or, for
// testing, several contexts on one GPU): an all-reduce is one kernel per rank
// that reads every rank's buffer directly (peer pointers over NVLink / the
// same HBM), so no staging copy or proxy thread is involved.  Host threads
// meet at a barrier only to exchange pointers and stream events; the GPU
// ordering comes from cross-stream event waits.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <mutex>
#include <stdexcept>
#include <vector>

namespace tsd {

constexpr int kMaxGroup = 8;

struct PeerPtrs {
    const void* p[kMaxGroup];
};

// out[i] = reduce_r in_r[i]; kind 0: u8 min, 1: u32 max, 2: u64 min
void launch_peer_reduce(int kind, PeerPtrs in, int nranks, void* out, size_t cnt, cudaStream_t st);

class HostBarrier {
public:
    explicit HostBarrier(int n) : n_(n) {}
    // throws once any rank has failed (so no thread waits forever on a dead rank)
    void wait() {
        std::unique_lock<std::mutex> lk(mu_);
        if (broken_) throw std::runtime_error("peer group: another rank failed");
        const unsigned long long gen = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            cv_.notify_all();
            return;
        }
        cv_.wait(lk, [&] { return gen != gen_ || broken_; });
        if (broken_) throw std::runtime_error("peer group: another rank failed");
    }
    void fail() {
        std::lock_guard<std::mutex> lk(mu_);
        broken_ = true;
        cv_.notify_all();
    }
    void reset() {
        std::lock_guard<std::mutex> lk(mu_);
        broken_ = false;
        count_ = 0;
    }

private:
    std::mutex mu_;
    std::condition_variable cv_;
    int n_, count_ = 0;
    unsigned long long gen_ = 0;
    bool broken_ = false;
};

struct PeerGroup {
    int n = 0;
    HostBarrier bar;
    std::vector<const void*> ptrs;
    std::vector<cudaEvent_t> ev_in, ev_red;
    explicit PeerGroup(int ranks) : n(ranks), bar(ranks), ptrs(ranks), ev_in(ranks), ev_red(ranks) {}
};

}  // namespace tsd
