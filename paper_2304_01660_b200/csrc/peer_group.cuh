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

#include <chrono>
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

// every rank's barrier flag array (kMaxGroup u64 slots, one per rank)
struct FlagPtrs {
    unsigned long long* p[kMaxGroup];
};
// device-side barrier of `world` ranks: all ranks' preceding stream work done
void launch_flag_barrier(const FlagPtrs& f, int world, int rank, unsigned long long epoch, cudaStream_t st);

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
        // a rank that never arrives (diverged control flow) must fail the call,
        // not hang it
        if (!cv_.wait_for(lk, std::chrono::seconds(120), [&] { return gen != gen_ || broken_; })) {
            broken_ = true;
            cv_.notify_all();
            throw std::runtime_error("peer group: barrier timeout");
        }
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
    bool distinct = false;  // every rank on its own device (device barriers allowed)
    HostBarrier bar;
    std::vector<const void*> ptrs;
    std::vector<void*> p_alive, p_ymax, p_emax, p_nnkey;  // fused transport: every rank's arrays
    std::vector<unsigned long long*> p_flags;                // device barrier flags of every rank
    std::vector<cudaEvent_t> ev_in, ev_red;
    explicit PeerGroup(int ranks)
        : n(ranks), bar(ranks), ptrs(ranks), p_alive(ranks), p_ymax(ranks), p_emax(ranks), p_nnkey(ranks),
          p_flags(ranks), ev_in(ranks), ev_red(ranks) {}
};

}  // namespace tsd

// ---------------------------------------------------------------------------
// Cross-process ranks (one process per GPU, e.g. under torchrun): the same
// fused peer stores, with the arrays shared through CUDA IPC memory handles,
// the per-rank barrier events through CUDA IPC event handles, and the host
// barrier in a POSIX shared-memory segment of the node.
#include <fcntl.h>
#include <stdio.h>
#include <stdlib.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <string>

namespace tsd {

struct ShmBarrierState {
    std::atomic<int> count;
    std::atomic<int> gen;
    std::atomic<int> broken;
};

class ShmBarrier {
public:
    ShmBarrier(const std::string& name, int world, bool create) : name_(name), n_(world) {
        const int fd = shm_open(name.c_str(), O_RDWR | (create ? O_CREAT : 0), 0600);
        if (fd < 0) throw std::runtime_error("shm_open " + name + " failed");
        if (create && ftruncate(fd, sizeof(ShmBarrierState)) != 0) {
            close(fd);
            throw std::runtime_error("ftruncate " + name + " failed");
        }
        void* p = mmap(nullptr, sizeof(ShmBarrierState), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) throw std::runtime_error("mmap " + name + " failed");
        st_ = static_cast<ShmBarrierState*>(p);
        if (create) {
            st_->count.store(0);
            st_->gen.store(0);
            st_->broken.store(0);
        }
        owner_ = create;
    }
    ~ShmBarrier() {
        munmap(st_, sizeof(ShmBarrierState));
        if (owner_) shm_unlink(name_.c_str());
    }
    void wait() {
        static const double timeout_s = std::getenv("TSD_BARRIER_TIMEOUT") ? std::atof(std::getenv("TSD_BARRIER_TIMEOUT"))
                                                                          : 120.0;
        ++waits_;
        if (std::getenv("TSD_DEBUG_BARRIER")) fprintf(stderr, "[ipc] pid %d barrier #%ld\n", (int)getpid(), waits_);
        if (st_->broken.load()) throw std::runtime_error("ipc group: another rank failed");
        const int g = st_->gen.load(std::memory_order_acquire);
        if (st_->count.fetch_add(1) + 1 == n_) {
            st_->count.store(0);
            st_->gen.fetch_add(1, std::memory_order_release);
            return;
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (unsigned spin = 0; st_->gen.load(std::memory_order_acquire) == g; ++spin) {
            if (st_->broken.load()) throw std::runtime_error("ipc group: another rank failed");
            if ((spin & 1023u) == 1023u) {
                sched_yield();
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
                    st_->broken.store(1);
                    throw std::runtime_error("ipc group: barrier timeout");
                }
            }
        }
    }
    void fail() { st_->broken.store(1); }

private:
    std::string name_;
    int n_;
    long waits_ = 0;
    ShmBarrierState* st_ = nullptr;
    bool owner_ = false;
};

}  // namespace tsd
