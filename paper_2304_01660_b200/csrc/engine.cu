// Host engine + C-ABI of libtsdiscord_b200.so.
//
// The control flow mirrors the reference exactly where it is observable
// (validation, MERLIN's length loop and threshold schedule, record order,
// error kinds); the scan itself is re-designed for B200:
//
//   pardrag(m, r^2)  (reference: src/pardrag.cpp:421-434)
//     dense  : band tiles k in [m, m + b*kW) over all rows, both ends of every
//              certain pair are killed (select + neighbour clearing, Alg. 3)
//     sparse : full rows (both sides) for the remaining candidates, with kills,
//              plus a lower bound of every live row's max correlation (Alg. 4)
//     exact  : survivors' near-minimum pairs re-evaluated with the reference's
//              FP64 znormalize + sq_ed (pardrag.cpp:378-416)
//   merlin (src/merlin.cpp:57-132): sequential lengths, Eq. 7-8 stats on the
//   device, adaptive r; only (count, survivors) cross to the host per try.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tsdiscord_b200.h"
#include "common.cuh"
#include "engine_internal.h"
#include "nccl_shim.h"
#include "peer_group.cuh"
#include "tile_space.cuh"

using namespace tsd;

namespace {

thread_local std::string g_create_err;

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(TSD_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    void ensure(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
        cap = n;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

template <typename T>
struct HBuf {
    T* p = nullptr;
    size_t cap = 0;
    void ensure(size_t n) {
        if (n <= cap) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        ck(cudaMallocHost(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMallocHost");
        cap = n;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

constexpr int kQueueCap = 1 << 22;
constexpr int kCollCap = 1 << 23;

}  // namespace

struct tsd_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    cudaStream_t st2 = nullptr;  // side stream (resident seeds built beside init_stats)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string err;

    // series
    int64_t n = 0;
    std::vector<double> h_t;
    DBuf<double> t;

    // per-length state
    int64_t stats_m = -1;  // length the device mu/sig currently hold (-1: none)
    DBuf<double> mu, sig, scr_a, scr_b;
    int64_t derived_m = -1;
    DBuf<float> df, dg, nrm;
    DBuf<int> crange;  // per-length slot of the derived length (k_derive; common.cuh kCrInts), two parity slots
    // double-double prefix sums of t and t^2 (statistics error, common.cuh)
    DBuf<double2> pfx1, pfx2, pfx_tot1, pfx_tot2;
    DBuf<int> deg;     // degenerate rows (sigma < eps) of the derived length
    DBuf<int> degc, deg2;  // ... split: one-pass constant (conventions) / the others (exact)

    // scan state
    DBuf<uint8_t> alive;
    DBuf<int2> queue, coll;
    DBuf<unsigned> ymax, emax;
    DBuf<double> bnd_lo, bnd_hi;
    // resident band-0 seed rows (length recurrence), valid for length seed_m
    DBuf<double> seedqt;
    int64_t seed_m = -1;
    int seed_L = 0, seed_kA = 0, seed_nb = 0, seed_bstep = 1;
    int seed_ustep = 1;  // entry stride of the resident rows: 9 when pass 0 reads slot 0 only (half_pk 20)
    bool seed_pair = false;  // band 0 of this run walks both sides together (k_band0_pair)
    DBuf<int> cand;
    DBuf<float> ythr;
    DBuf<unsigned long long> nnkey, acc;  // acc: [0] cells, [1] seeds
    DBuf<int> blk, list;
    // per-(row, band) corr upper bounds of the full-row stage (collection skip)
    DBuf<unsigned long long> ubk;
    DBuf<int> exli;
    int collect_skip = 1;
    // kill witnesses across tries (ScanParams::wit): int per series index
    // row cache (ScanParams::rcqt): resident raw QT rows of anchor rows next to
    // the previous tries' exact-nn rows, advanced with the lengths
    int row_cache = 1;
    DBuf<double> rcqt;
    DBuf<int> surv;  // every survivor of the try (k_survivors), read back for the anchors
    RcRows rc{};
    int rc_age[kRcSlots] = {};
    int64_t rc_m = -1;  // length every filled slot holds (-1: none)
    int64_t rc_fills = 0;
    int rc_keep = 2;  // tries a slot survives without being needed
    // Short windows seed cheaply (m FMA per diagonal) while a fill costs N m
    // FMA and every slot N FMA per length: the cache pays from m ~ 384 on
    // (measured with the cache at every length: C4 -5%, C5 -1.4%, C3 +1.6%,
    // C2 +1%).
    int64_t rc_min_m = 384;
    bool rc_on(int64_t m) const { return row_cache && m >= rc_min_m; }
    void rc_reset() {
        rc_m = -1;
        rc.n = kRcSlots;
        for (int s = 0; s < kRcSlots; ++s) {
            rc.row[s] = -1;
            rc_age[s] = 0;
        }
    }
    // stats went m -> m+1: advance the slots with them (or drop them)
    void rc_step(int64_t m) {
        if (rc_m != m) return;
        const int64_t N1 = n - m;
        bool any = false;
        for (int s = 0; s < kRcSlots; ++s) {
            if (rc.row[s] >= N1) rc.row[s] = -1;
            any |= rc.row[s] >= 0;
        }
        if (!any) {
            rc_m = -1;
            return;
        }
        launch_rc_advance(t.p, (int)n, (int)m, rc, (long long)n, rcqt.p, st);
        ck(cudaGetLastError(), "rc advance");
        ctr.kernel_launches += 1;
        rc_m = m + 1;
    }
    // after a MERLIN try at length m: anchors just before / after every
    // cluster of the exact-nn rows (the discord regions recur from length to
    // length); a missing anchor evicts the least recently needed slot and is
    // filled at m (N m FMA, once per region)
    static constexpr int kRcMargin = 16, kRcTol = 48, kRcGap = 64;
    void rc_update(int64_t m, const int* ex, int ec) {
        if (!rc_on(m) || ec <= 0) {
            if (rc_m >= 0 && !rc_on(m + 1)) rc_reset();  // below the length gate: nothing to carry
            return;
        }
        const int N = (int)(n - m + 1);
        if (rc_m != m) {
            for (int s = 0; s < kRcSlots; ++s) rc.row[s] = -1;
            rc_m = m;
        }
        rc.n = kRcSlots;
        std::vector<int> v(ex, ex + ec);
        std::sort(v.begin(), v.end());
        std::vector<std::pair<int, int>> cl;  // clusters (lo, hi)
        for (int x : v) {
            if (!cl.empty() && x - cl.back().second <= kRcGap) cl.back().second = x;
            else cl.push_back({x, x});
        }
        std::stable_sort(cl.begin(), cl.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) {
            return x.second - x.first > y.second - y.first;
        });
        bool used[kRcSlots] = {};
        int wanted = 0;
        for (const auto& c2 : cl) {
            if (wanted + 2 > kRcSlots) break;
            for (int side = 0; side < 2; ++side) {
                ++wanted;
                int hit = -1;
                for (int s = 0; s < kRcSlots; ++s) {
                    const int r = rc.row[s];
                    if (r < 0) continue;
                    const int d = side == 0 ? c2.first - r : r - c2.second;
                    if (d >= 0 && d <= kRcTol) hit = s;
                }
                if (hit < 0) {
                    int best = -1;
                    for (int s = 0; s < kRcSlots; ++s)
                        if (!used[s] && (best < 0 || rc.row[s] < 0 && rc.row[best] >= 0 ||
                                         (rc.row[s] < 0) == (rc.row[best] < 0) && rc_age[s] > rc_age[best]))
                            best = s;
                    if (best < 0) continue;
                    hit = best;
                    rc.row[hit] = side == 0 ? std::max(0, c2.first - kRcMargin) : std::min(N - 1, c2.second + kRcMargin);
                    rcqt.ensure((size_t)kRcSlots * (size_t)n);
                    launch_rc_fill(t.p, (int)n, (int)m, rc.row[hit], rcqt.p + (size_t)hit * (size_t)n, st);
                    ck(cudaGetLastError(), "rc fill");
                    ctr.kernel_launches += 1;
                    ++rc_fills;
                }
                used[hit] = true;
            }
        }
        for (int s = 0; s < kRcSlots; ++s) {
            rc_age[s] = used[s] ? 0 : rc_age[s] + 1;
            if (rc_age[s] > rc_keep) rc.row[s] = -1;  // not needed lately: stop advancing it
        }
    }
    DBuf<int> wit;
    // run-seed cache of the witness test (ScanParams::wc_*)
    int wit_cache = 1;
    DBuf<double> wc_qt;
    DBuf<int> wc_m, wc_q;
    DBuf<unsigned long long> dbgc;  // TSD_DEBUG slot counters (ScanParams::dbg)
    DBuf<int4> wl;  // the try's witness candidate runs (first row, length, witness)
    DBuf<int2> wl2;  // rows left for the 9-diagonal phase (row, witness)
    int witness = 1;
    long long ub_entries = 1ll << 22;  // 32 MB
    DBuf<double> nnout;
    DBuf<int2> groups, slots;  // groups of the current stage; per-span candidate groups
    DBuf<double> bcost;        // per-CTA span costs of a compaction
    DBuf<TryCtl> ctl;  // device-resident control block of the current try
    DBuf<unsigned long long> lbstat;  // compaction look-back status words
    unsigned epoch = 0;
    HBuf<TryCtl> h_ctl;
    HBuf<int> h_int, h_ex, h_surv;
    HBuf<unsigned long long> h_acc;
    HBuf<double> h_nn;

    // tuning
    bool debug = std::getenv("TSD_DEBUG") != nullptr;
    int dense_rows = 0;  // rows per band-0 block; 0: auto (block_rows)
    int sparse_rows = 0;   // 0: choose by cost model (on the device)
    // Bands of a later band pass: at least enough to fill band_fill waves of
    // the scan grid (the compaction sizes the pass from its group count).
    // Measured: more bands per pass kill more rows before the full rows; the
    // best factor grows with the series (C2: 6 -> 33.3 ms vs 35.4 ms at 1;
    // C4: 24 -> 768 ms vs 878 ms; C3 / C5 flat from 16 on).  0: automatic.
    double band_fill = 0.0;
    int band_slots(int64_t N) const {
        const double f = band_fill > 0.0 ? band_fill : (N < (1 << 18) ? 6.0 : 24.0);
        return (int)std::max(1.0, f * (double)scan_slots_prune());
    }
    int band_passes = 6;  // cap on band passes (incl. pass 0) per try; full rows cover the rest (measured: C4 914 -> 896 ms vs 40)
    int band_hint = 0;     // adaptive count: passes the previous try needed (0: none yet)
    int track_hint = 0;    // ... and tracked chunks (plus the catch-all launch)
    int track_chunks = 1;  // cap on tracked launches per try (1: the catch-all alone)
    int band0_sides = 2;   // band 0 on both sides of every row, or the positive side only
    // band-pass evaluation density, 1 cell in N (kills stay certain; a row a pass
    // misses is walked again later).  Measured: C2 41.0 -> 39.5 ms, C4 1060 ->
    // 1013 ms with 1/3 in pass 0 and 1/2 in the later band passes.
    // later band passes: 20 = the middle slot of every thread's 9 diagonals
    // only (every 9th diagonal, fully; the other slots' walks and seeds are
    // dead code): C4 476 -> 427 ms, C5 629 -> 582 ms (3: every slot, 1 step in 3)
    int half_pass0 = 3, half_bands = 20;
    long long half_bands_m = 128;
    int pass0_pk = 1;  // band 0 walks every pair once and kills both ends (k_band0_pk)
    int pk_rows = 0;   // rows per block of the pair-kill walk (0: by the grid's waves)
    int64_t pk_min_n = 1 << 15;  // the pair-kill walk from this many subsequences on (C2: 32.2 -> 30.4 ms; C1: 8.8 -> 9.3 ms, so not below)
    int half_pk = 20;  // pass-0 pattern (pk_sampled): 20 = slot 0 of every thread, every step (C4 480 -> 466 ms,
                       // C5 663 -> 627 ms); 6 = even slots, (j + 2 step) % 6; 12 = slots 0/3/6, one per step
    int pair_band0 = 1;  // both sides of band 0 in one packed-FP32x2 walk  // later passes use half_bands only from this length on
    int seed32_track = 1;    // FP32 seeds in the full-row launch (wider error band, half the seed cost; C4 -3.4%)
    int seed32_collect = 1;  // ... and in the collection launch
    float band_keep = 0.85f;  // band loop stops when a pass leaves more than this fraction alive
    float seed_w = 0.25f;  // grouping cost: one group-diagonal seed = seed_w*m walked row-diagonals (FP32 seeds)
    int band_few = 256;       // ... or when at most max(band_few, N/4096) rows are left (C2: 64 -> 41.8 ms, 256 -> 41.2 ms)
    // With kill witnesses the rows left after pass 0 are few but mostly have
    // near killers: the band passes go on down to band_few_wit rows (the full
    // rows walk far diagonals first and would seed every far tile of them).
    // Measured (rows left after which the band passes stop): C4 720 / 702 /
    // 772 ms at 16 / 64 / 256, C3 432 / 426 ms at 16 / 64, C2 33.4 / 32.5 /
    // 31.2 ms at 16 / 64 / 256.  0: automatic (256 below N = 2^18, else 64).
    // With the one-slot band passes (half_bands 20) a pass costs about a ninth
    // of its seeds, so from m = few_m on (where full-row seeds are longest)
    // the passes go on down to few_lo rows: C4 417 -> 367 ms; below it 64
    // stays best (C5 583 vs 594 ms at 2, C3 376 vs 380 ms).
    int band_few_wit = 0;
    int64_t few_m = 512;
    int few_lo = 2;
    int few_rows(int64_t N, int64_t m) const {
        if (!witness) return std::max<int>(band_few, (int)(N / 4096));
        if (band_few_wit > 0) return band_few_wit;
        if (N < (1 << 18)) return 256;
        return m >= few_m ? few_lo : 64;
    }
    int result_prefix = 1024;  // records copied back with the try's single round trip
    // knife-edge queue / near-pair buffer capacities (settable below the
    // allocation for tests of the overflow fallback)
    int queue_cap = kQueueCap, coll_cap = kCollCap;
    double err_k = 4.0;

    // accounting
    tsd_counters ctr{};
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;

    // heatmap (device-resident score matrix)
    DBuf<double> hm;
    int64_t hm_min = 0, hm_max = -1, hm_n = 0;
    DBuf<HmCol> hm_cols;
    DBuf<unsigned long long> hm_cnt;
    DBuf<int64_t> hm_rows, hm_idx;
    DBuf<double> hm_vals;

    // multi-GPU (segment-sharded tiles; flags / maxima / minima all-reduced)
    int rank = 0, world = 1;
    void* comm = nullptr;

    // ------------------------------------------------------------------
    static double now_ms() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
            .count();
    }
    void sync() {
        const double t0 = now_ms();
        ck(cudaStreamSynchronize(st), "stream sync");
        ctr.host_wait_ms += now_ms() - t0;
        ctr.host_syncs += 1;
    }

    // Reductions across ranks: NCCL (one process per GPU) or the in-process
    // peer group (peer_group.cuh).  Every rank reaches them in the same order
    // with identical sizes: the host control flow depends only on reduced data.
    PeerGroup* group = nullptr;
    DBuf<unsigned char> red_tmp;

    void allreduce(void* p, size_t cnt, int kind, size_t esize) {
        if (world <= 1) return;
        if (group) {
            peer_allreduce(p, cnt, kind, esize);
            return;
        }
        if (!nccl_allreduce(comm, p, cnt, kind, st)) fail(TSD_ECUDA, "ncclAllReduce failed");
    }
    void peer_allreduce(void* p, size_t cnt, int kind, size_t esize) {
        PeerGroup& g = *group;
        g.ptrs[rank] = p;
        ck(cudaEventRecord(g.ev_in[rank], st), "event");
        g.bar.wait();  // every rank's input pointer and event are published
        PeerPtrs in{};
        for (int r = 0; r < g.n; ++r) {
            in.p[r] = g.ptrs[r];
            if (r != rank) ck(cudaStreamWaitEvent(st, g.ev_in[r], 0), "event wait");
        }
        red_tmp.ensure(cnt * esize);
        launch_peer_reduce(kind, in, g.n, red_tmp.p, cnt, st);
        ck(cudaGetLastError(), "peer reduce");
        ck(cudaEventRecord(g.ev_red[rank], st), "event");
        g.bar.wait();  // no rank overwrites its input before every rank has read it
        for (int r = 0; r < g.n; ++r)
            if (r != rank) ck(cudaStreamWaitEvent(st, g.ev_red[r], 0), "event wait");
        ck(cudaMemcpyAsync(p, red_tmp.p, cnt * esize, cudaMemcpyDeviceToDevice, st), "D2D");
        ctr.kernel_launches += 1;
    }
    // Fused transport (peer group): the kernels store kills and row maxima into
    // every rank's arrays (Peers), so an "all-reduce" of alive / ymax / emax is
    // only an event barrier between the ranks' streams.
    bool fused = true;
    Peers peers{};
    // cross-process ranks (tsd_ipc_*): peers fixed at join, barrier in shared memory
    ShmBarrier* ipc_bar = nullptr;
    cudaEvent_t ipc_ev = nullptr;                  // this rank's exported barrier event
    std::vector<cudaEvent_t> ipc_peer_ev;          // every rank's event (own included)
    std::vector<void*> ipc_opened;                 // peer mappings to close
    int64_t ipc_rows = 0;                          // capacity of the shared arrays
    bool ipc_host_sync = std::getenv("TSD_IPC_SYNC") != nullptr;
    // Device-side barriers (k_flag_barrier): every rank owns kMaxGroup u64
    // flag slots in device memory (in-process groups: `bflags`; IPC: the tail
    // of the shared nnkey array), and a barrier is one single-thread kernel per
    // rank that publishes an epoch into every rank's slot and spins on its own
    // slots, so the host never blocks on the other ranks.  dev_barrier: 1 on,
    // 0 off (host barrier + cross-stream event waits), -1 auto (on).
    int dev_barrier = -1;
    bool use_dev_bar = false;
    DBuf<unsigned long long> bflags;
    FlagPtrs fptr{};
    unsigned long long bar_epoch = 0;
    void peer_publish() {
        if (ipc_bar) return;  // fixed at join
        peers.n = 0;
        if (!group || !fused || world <= 1) return;
        PeerGroup& g = *group;
        if (!bflags.p) {
            // zeroed before any rank can see the pointer (else a peer's early
            // epoch store could be wiped by this memset)
            bflags.ensure(kMaxGroup);
            ck(cudaMemsetAsync(bflags.p, 0, kMaxGroup * sizeof(unsigned long long), st), "memset");
            sync();
        }
        g.p_alive[rank] = alive.p;
        g.p_ymax[rank] = ymax.p;
        g.p_emax[rank] = emax.p;
        g.p_nnkey[rank] = nnkey.p;
        g.p_flags[rank] = bflags.p;
        g.bar.wait();
        peers.n = g.n;
        for (int r = 0; r < g.n; ++r) {
            peers.alive[r] = static_cast<uint8_t*>(g.p_alive[r]);
            peers.ymax[r] = static_cast<unsigned*>(g.p_ymax[r]);
            peers.emax[r] = static_cast<unsigned*>(g.p_emax[r]);
            peers.nnkey[r] = static_cast<unsigned long long*>(g.p_nnkey[r]);
            fptr.p[r] = g.p_flags[r];
        }
        // In one process, ranks sharing a device cannot use device barriers: an
        // implicitly device-synchronising call (cudaFree) on one rank's thread
        // would wait for another rank's barrier kernel, which waits for this
        // rank's next enqueue.  Distinct devices (and separate processes) are safe.
        use_dev_bar = dev_barrier == 1 || (dev_barrier == -1 && g.distinct);
        g.bar.wait();  // the tables stay put until every rank has read them
    }
    void peer_barrier() {  // every rank's preceding kernels (and their remote stores) are done
        if (use_dev_bar) {
            launch_flag_barrier(fptr, world, rank, ++bar_epoch, st);
            ck(cudaGetLastError(), "flag barrier");
            ctr.kernel_launches += 1;
            return;
        }
        if (ipc_bar) {
            ck(cudaEventRecord(ipc_ev, st), "event");
            if (ipc_host_sync) sync();  // this rank's work done on the device before the host barrier
            ipc_bar->wait();
            if (!ipc_host_sync)
                for (int r = 0; r < world; ++r)
                    if (r != rank) ck(cudaStreamWaitEvent(st, ipc_peer_ev[r], 0), "event wait");
            ipc_bar->wait();
            return;
        }
        PeerGroup& g = *group;
        ck(cudaEventRecord(g.ev_in[rank], st), "event");
        g.bar.wait();
        for (int r = 0; r < g.n; ++r)
            if (r != rank) ck(cudaStreamWaitEvent(st, g.ev_in[r], 0), "event wait");
        g.bar.wait();  // nobody re-records its event before every rank has waited on it
    }
    void reduce_alive(int64_t N) {
        if (peers.n > 1) peer_barrier();
        else allreduce_min_u8(alive.p, N);
    }
    void reduce_maxima(int64_t N) {  // after reduce_alive of the same scan
        if (peers.n > 1) return;
        allreduce_max_u32(ymax.p, N);
        allreduce_max_u32(emax.p, N);
    }
    void allreduce_min_u8(uint8_t* p, size_t cnt) { allreduce(p, cnt, 0 /*u8 min*/, 1); }
    void allreduce_max_u32(unsigned* p, size_t cnt) { allreduce(p, cnt, 1 /*u32 max*/, 4); }
    void allreduce_min_u64(unsigned long long* p, size_t cnt) { allreduce(p, cnt, 2 /*u64 min*/, 8); }

    // ---- statistics --------------------------------------------------
    void init_stats_dev(int64_t m) {
        mu.ensure(n);
        sig.ensure(n);
        scr_a.ensure(n);
        scr_b.ensure(n);
        launch_init_stats(t.p, (int)n, (int)m, mu.p, sig.p, scr_a.p, scr_b.p, st);
        ctr.kernel_launches += 2;
        ck(cudaGetLastError(), "init_stats");
        stats_m = m;
        derived_m = -1;
    }
    void advance_stats_dev() {
        launch_advance_stats(t.p, (int)n, (int)stats_m, mu.p, sig.p, st);
        ctr.kernel_launches += 1;
        ck(cudaGetLastError(), "advance_stats");
        ++stats_m;
        derived_m = -1;
    }
    void derive(int64_t m) {
        if (derived_m == m) return;
        const int64_t N = n - m + 1;
        df.ensure(N);
        dg.ensure(N);
        nrm.ensure(N);
        crange.ensure(2 * kCrInts);
        deg.ensure(N);
        // both parity slots cleared: the fused length step after this one uses the other
        ck(cudaMemsetAsync(crange.p, 0, 2 * kCrInts * sizeof(int), st), "memset");
        cr_cur = crange.p + kCrInts * (m & 1);
        degc.ensure(N);
        deg2.ensure(N);
        launch_derive(t.p, (int)m, (int)N, mu.p, sig.p, df.p, dg.p, nrm.p, cr_cur, deg.p, pfx1.p, pfx2.p, degc.p,
                      deg2.p, st);
        ctr.kernel_launches += 1;
        ck(cudaGetLastError(), "derive");
        derived_m = m;
    }
    // MERLIN length step m -> m+1 in one launch: stats (ping-pong buffers),
    // derived operands of m+1 and, when resident, the seed rows
    int* cr_cur = nullptr;  // constant-row range of derived_m
    DBuf<double> mu2, sig2;
    void next_length(bool with_seed) {
        const int64_t m = stats_m, m1 = m + 1, N1 = n - m;
        mu2.ensure(n);
        sig2.ensure(n);
        df.ensure(N1);
        dg.ensure(N1);
        nrm.ensure(N1);
        if (derived_m != m || !cr_cur) derive(m);  // establishes the parity slots
        int* cr = crange.p + kCrInts * (m1 & 1);
        int* crn = crange.p + kCrInts * ((m1 + 1) & 1);
        deg.ensure(N1);
        degc.ensure(N1);
        deg2.ensure(N1);
        launch_next_length(t.p, (int)n, (int)m, mu.p, sig.p, mu2.p, sig2.p, df.p, dg.p, nrm.p, cr, crn, seed_L, seed_kA,
                           seed_nb, seed_bstep, seed_ustep, with_seed ? seedqt.p : nullptr, deg.p, pfx1.p, pfx2.p, degc.p,
                           deg2.p, st);
        ck(cudaGetLastError(), "next length");
        ctr.kernel_launches += 1;
        std::swap(mu.p, mu2.p);
        std::swap(mu.cap, mu2.cap);
        std::swap(sig.p, sig2.p);
        std::swap(sig.cap, sig2.cap);
        stats_m = m1;
        derived_m = m1;
        cr_cur = cr;
        if (with_seed) seed_m = m1;
    }

    // Rows per band-0 block: 512 when the blocks fill the persistent grid, else
    // smaller blocks (256/128) so that small series still occupy every SM
    // (measured at C2: 256 rows 55.5 ms, 128 rows 56.8 ms, 512 rows 57.8 ms).
    // Rows per block of the pair-kill walk: the slots (block pairs) should fill
    // the persistent grid to just past a whole number of waves (a last, sparse
    // wave runs at a higher per-CTA rate) or just below one wave.  Measured:
    // C4 (N = 1e6) 384 rows 620 ms / 448: 648 / 512: 649; C3 (N = 5e5) 448
    // rows 421 ms / 384: 464 / 512: 428; C5 (N = 2e6) 512 rows 800 ms / 384:
    // 807.  The first target wave count with L <= 512 (nearest multiple of 32) wins.
    int pk_block_rows(int64_t N) const {
        if (N < (1 << 18)) return 256;  // below a wave anyway (C2: 256 rows 30.4 ms, 128: 30.5, 512: 31.2)
        const double g = (double)band0_pk_slots();
        for (double w : {0.9, 2.2, 3.3, 4.4, 5.5, 6.6, 7.7}) {
            const int L = (int)std::lround((double)N / (2.0 * g * w) / 32.0) * 32;
            if (L <= kMaxRows && L >= 128) return L;
            if (L < 128) break;
        }
        return kMaxRows;
    }
    int block_rows(int64_t N, bool paired = false) const {
        if (dense_rows > 0) return dense_rows;
        // ~one wave of the band-pass scan grid: two tiles per block (one per
        // side), or one when both sides walk together (k_band0_pair)
        const int64_t want = (4 * (int64_t)(paired ? band0_pair_slots() : scan_slots_prune())) / 5;
        const int per = paired ? 1 : 2;
        for (int L = kMaxRows; L > 128; L /= 2)
            if (per * ((N + L - 1) / L) >= want) return L;
        return 128;
    }

    // ---- resident seed rows ----------------------------------------------
    void seed_init(int64_t m, int64_t kA) {
        const int64_t N = n - m + 1;
        // the paired walk only when its largest blocks still fill a wave
        // (measured: C4 / C5 gain 1-2%; at C2 the smaller blocks it would need
        // cost more in staging than the walk saves)
        if (pass0_pk && pair_band0 != 0 && band0_sides == 2 && N >= pk_min_n) {
            // pair-kill walk: a slot is two blocks' positive sides
            seed_pair = true;
            seed_L = pk_rows > 0 ? pk_rows : pk_block_rows(N);
            seed_bstep = 2;  // the walk reads the positive-side rows only
            seed_ustep = half_pk == 20 ? kDiag : 1;  // ... and, for pattern 20, slot 0 of every thread
        } else {
            seed_pair = pair_band0 != 0 && band0_sides == 2 && block_rows(N, true) == kMaxRows;
            seed_L = block_rows(N, seed_pair);
            seed_bstep = 1;
            seed_ustep = 1;
        }
        seed_kA = (int)kA;
        seed_nb = 2 * (int)((N + seed_L - 1) / seed_L);
        seedqt.ensure((size_t)seed_nb * kW);
        launch_seed_init(t.p, (int)n, (int)m, seed_L, seed_kA, seed_nb, seed_bstep, seed_ustep, seedqt.p, st);
        ck(cudaGetLastError(), "seed init");
        ctr.kernel_launches += 1;
        seed_m = m;
    }
    void seed_advance() {  // seed_m -> seed_m + 1
        launch_seed_advance(t.p, (int)n, (int)seed_m, seed_L, seed_kA, seed_nb, seed_bstep, seed_ustep, seedqt.p, st);
        ck(cudaGetLastError(), "seed advance");
        ctr.kernel_launches += 1;
        ++seed_m;
    }

    // ---- scan helpers ---------------------------------------------------
    ScanParams params(int64_t m, double r_sq) {
        ScanParams p{};
        p.t = t.p;
        p.mu = mu.p;
        p.sig = sig.p;
        p.df = df.p;
        p.dg = dg.p;
        p.nrm = nrm.p;
        p.n = (int)n;
        p.m = (int)m;
        p.N = (int)(n - m + 1);
        p.r_sq = r_sq;
        p.thr0 = 1.0 - r_sq / (2.0 * (double)m);
        p.err_k = err_k;
        p.alive = alive.p;
        p.queue = queue.p;
        p.queue_count = &ctl.p->queue;
        p.queue_cap = queue_cap;
        p.ymax = ymax.p;
        p.emax = emax.p;
        p.seedqt = seedqt.p;
        p.cr = cr_cur;
        p.ythr = ythr.p;
        p.coll = coll.p;
        p.coll_count = &ctl.p->coll;
        p.coll_cap = coll_cap;
        p.ctl = ctl.p;
        p.groups = groups.p;
        p.rank = rank;
        p.world = world;
        p.acc = acc.p;
        p.peers = peers;
        p.pfx1 = pfx1.p;
        if (debug) {
            if (dbgc.cap < 16) {
                dbgc.ensure(16);
                ck(cudaMemset(dbgc.p, 0, 16 * sizeof(unsigned long long)), "memset");
            }
            p.dbg = dbgc.p;
        }
        return p;
    }

    // scan launches of one try are bracketed by pooled events (harvested after
    // the try's single sync)
    struct EvPair {
        cudaEvent_t a, b;
        int mode;
    };
    std::vector<EvPair> ev_pool;
    size_t ev_used = 0;

    // bracket every scan with events (per-phase kernel time for the roofline).
    // Off by default: an event between two kernels breaks the programmatic
    // dependent launch chain (C2: 53.7 ms with events, 43.1 ms without)
    bool scan_events = false;
    int scan_idx = 0;  // scan launches of the current try (slot counter index)
    void scan(int mode, const ScanParams& p0) {
        ScanParams p = p0;
        if (scan_idx >= 32) fail(TSD_ERUNTIME, "too many scan launches in one try");
        p.next = &ctl.p->slotc[scan_idx++];
        if (!scan_events) {
            launch_scan(mode, p, st);
            ck(cudaGetLastError(), "scan launch");
            ctr.scan_launches += 1;
            ctr.kernel_launches += 1;
            return;
        }
        if (ev_used == ev_pool.size()) {
            EvPair e{};
            ck(cudaEventCreate(&e.a), "event");
            ck(cudaEventCreate(&e.b), "event");
            ev_pool.push_back(e);
        }
        EvPair& e = ev_pool[ev_used++];
        e.mode = mode;
        ck(cudaEventRecord(e.a, st), "event");
        launch_scan(mode, p, st);
        ck(cudaGetLastError(), "scan launch");
        ck(cudaEventRecord(e.b, st), "event");
        ctr.scan_launches += 1;
        ctr.kernel_launches += 1;
    }

    // after a full sync: fold the scan launch times of this call into ctr
    void harvest_events() {
        for (size_t i = 0; i < ev_used; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev_pool[i].a, ev_pool[i].b);
            ctr.scan_ms += ms;
            if (ev_pool[i].mode == kPrune) ctr.dense_ms += ms;
            else if (ev_pool[i].mode == kPruneTrack) ctr.sparse_ms += ms;
            else ctr.collect_ms += ms;
        }
        ev_used = 0;
    }

    // alive flags -> sorted list, break rule (band passes), groups of the list
    void compact(int N, int gate, int64_t m) {
        const size_t nb = (size_t)compact_blocks(N);
        if (lbstat.cap < nb) {
            lbstat.ensure(nb);
            ck(cudaMemsetAsync(lbstat.p, 0, nb * sizeof(unsigned long long), st), "memset");
            epoch = 0;
        }
        if (++epoch >= (1u << 30)) {
            ck(cudaMemsetAsync(lbstat.p, 0, lbstat.cap * sizeof(unsigned long long), st), "memset");
            epoch = 1;
        }
        slots.ensure(group_slots(N));
        bcost.ensure((size_t)compact_blocks(N) * 6);
        launch_compact_group(alive.p, N, list.p, lbstat.p, epoch, ctl.p, gate, groups.p, slots.p, (int)m,
                             sparse_rows, band_keep, few_rows(N, m), seed_w, bcost.p, band_slots(N), st);
        ck(cudaGetLastError(), "compact");
        ctr.kernel_launches += 1;
        // fused peers: no rank's next scan may store kills into this rank's
        // flags before this compaction has read them (the lists must agree)
        if (peers.n > 1) peer_barrier();
    }

    // debug trace: one host round trip per stage (TSD_DEBUG only)
    void trace(const char* what, int64_t m, double r_sq, int pass) {
        if (!debug) return;
        ck(cudaMemcpyAsync(h_ctl.p, ctl.p, sizeof(TryCtl), cudaMemcpyDeviceToHost, st), "D2H");
        sync();
        const TryCtl& c = *h_ctl.p;
        if (dbgc.p) {
            unsigned long long d[16] = {};
            ck(cudaMemcpy(d, dbgc.p, sizeof d, cudaMemcpyDeviceToHost), "D2H");
            fprintf(stderr, "[tsd] slots prune %llu/%llu track %llu/%llu collect %llu/%llu witness runs %llu cached %llu\n",
                    d[1], d[0], d[3], d[2], d[5], d[4], d[6], d[7]);
            fprintf(stderr, "[tsd] track tiles: row-cache %llu direct %llu resident %llu rows %llu\n", d[8], d[9], d[11],
                    d[10]);
            fprintf(stderr, "[tsd] slowest collection tile: %llu cycles, rows %llu k0 %lld evals %llu\n", d[12], d[13],
                    (long long)d[14] - (1ll << 30), d[15]);
            unsigned long long z = 0;
            ck(cudaMemcpy(dbgc.p + 12, &z, sizeof z, cudaMemcpyHostToDevice), "H2D");
        }
        fprintf(stderr,
                "[tsd] m=%lld r2=%.6g %s pass=%d groups=%d span=%d alive=%d stop=%d queue=%d band=[%d,+%d) "
                "track=[%d,+%d) phase=%d\n",
                (long long)m, r_sq, what, pass, c.G, c.span, c.alive, c.stop == INT_MAX ? -1 : c.stop, c.queue,
                c.bK0, c.bnb * kW, c.tK0, c.tnb * kW, c.tphase);
    }

    void ensure_scan_buffers(int N) {
        if (ipc_bar && N > ipc_rows) fail(TSD_EINVAL, "ipc group: series longer than at tsd_ipc_export");
        alive.ensure(N);
        queue.ensure(kQueueCap);
        coll.ensure(kCollCap);
        ymax.ensure(N);
        emax.ensure(N);
        bnd_lo.ensure(N);
        bnd_hi.ensure(N);
        cand.ensure(N);
        ythr.ensure(N);
        nnkey.ensure(N);
        acc.ensure(5);
        surv.ensure(N);
        wl.ensure(N);
        wl2.ensure(N);
        if (wit.cap < (size_t)n) {
            wit.ensure((size_t)n);
            ck(cudaMemsetAsync(wit.p, 0x80, (size_t)n * sizeof(int), st), "memset");  // kNoWit
        }
        nnout.ensure(N);
        list.ensure(N);
        exli.ensure(N);
        if (collect_skip && !ubk.p) {
            ubk.ensure((size_t)ub_entries);
            // epoch-tagged entries: zero is older than every try
            ck(cudaMemsetAsync(ubk.p, 0, (size_t)ub_entries * sizeof(unsigned long long), st), "memset");
        }
        groups.ensure(N);
        if (!ctl.p) {
            ctl.ensure(1);
            ck(cudaMemsetAsync(ctl.p, 0, sizeof(TryCtl), st), "memset");  // self-resetting tickets start at 0
        }
        h_ctl.ensure(1);
        h_int.ensure(8);
        h_acc.ensure(5);
        h_ex.ensure(result_prefix);
        h_surv.ensure(result_prefix);
        h_nn.ensure(result_prefix);
    }

    // fold the device work counters of the current call into ctr
    void harvest(int64_t m) {
        const unsigned long long* hacc = h_acc.p;
        ctr.cells += hacc[0];
        ctr.cells_eval += hacc[1];
        ctr.seed_dots += hacc[2];
        ctr.seed_flops += hacc[2] * 2ull * (unsigned long long)m;
        ctr.wit_tests += hacc[3];
        ctr.wit_kills += hacc[4];
    }

    // Core PD3: survivors {c : nn(c)^2 >= r_sq} with exact nn, sorted like
    // sort_discords.  If `all_nn` is given (r_sq must be 0) it receives nn for
    // every index.
    // need_top > 0 (MERLIN): only the records that can be in the top need_top
    // get exact distances; last_count still receives the full survivor count.
    //
    // The whole try is enqueued on the stream without a host round trip: every
    // count a later stage needs lives in the device control block (TryCtl) and
    // the kernels gate themselves on it.  The host reads back once, at the end.
    int last_count = 0;
    int enq_passes = 0;
    std::vector<tsd_record> pardrag_core(int64_t m, double r_sq, double* all_nn = nullptr,
                                         int64_t need_top = 0) {
        const double t_start = now_ms();
        struct WallGuard {
            tsd_ctx* c;
            double t0;
            ~WallGuard() { c->ctr.host_wall_ms += now_ms() - t0; }
        } wall_guard{this, t_start};
        const int N = (int)(n - m + 1);
        derive(m);
        ensure_scan_buffers(N);
        ev_used = 0;
        scan_idx = 0;
        ctr.pardrag_calls += 1;
        peer_publish();
        TryCtl* C = ctl.p;
        // band 0 is the band at kA (resident seed rows) or at m; later passes
        // continue from its end, with the device choosing their widths
        const bool seeded = seed_m == m;
        const long long k_max = (long long)N - 1;
        const long long K1 = seeded ? (long long)seed_kA + kW : (long long)m + kW;
        launch_try_init(alive.p, ymax.p, emax.p, ythr.p, nnkey.p, N, C, acc.p, (int)std::min<long long>(K1, INT_MAX),
                        st);
        ck(cudaGetLastError(), "try init");
        ctr.kernel_launches += 1;
        // fused peers: another rank's kills must not land before this rank's reset
        if (peers.n > 1) peer_barrier();
        const ScanParams P = params(m, r_sq);
        std::vector<tsd_record> out;
        int* const W = witness && m <= kWitMaxM ? wit.p : nullptr;

        // ---- band passes (PD3 selection): diagonals |k| in [K0, K0 + nb*kW) on
        // both sides of every undecided row; only certain FP32 kills.  Pass 0
        // tiles all rows in aligned blocks; later passes tile the device-built
        // groups of the remaining rows over a device-chosen number of bands.  The
        // break rule (nothing / few left, < 15% killed, no diagonals left) is
        // applied on the device; passes after it are no-ops.
        enq_passes = 0;
        if (r_sq > 0.0) {
            // passes after the device-side break rule are no-ops but still cost
            // their launches: enqueue what the previous try needed (consecutive
            // lengths behave alike), growing while the cap is what stopped it
            const int want = band_hint > 0 ? std::min(band_hint, band_passes) : std::min(4, band_passes);
            for (int pass = 0; pass < want && (pass == 0 || K1 <= k_max); ++pass) {
                ++enq_passes;
                ScanParams q = P;
                q.pass = pass;
                if (pass == 0 && seeded) {
                    // band 0 at the fixed offset kA (>= m for every length of the run)
                    // seeded from the resident rows: no direct dot products
                    q.space = kSpaceSeed;
                    q.L = seed_L;
                    q.kA = seed_kA;
                    q.nb = band0_sides;
                    q.pair = seed_pair ? (pass0_pk ? 2 : 1) : 0;
                } else if (pass == 0) {
                    q.space = kSpaceBlocks;
                    q.L = block_rows(N);
                    q.K0 = (int)m;
                    q.nb = 1;
                } else {
                    q.space = kSpaceBand;  // groups and bands set by the previous compaction
                }
                q.half = pass == 0 ? (q.pair == 2 ? half_pk : half_pass0) : (m >= half_bands_m ? half_bands : 1);
                q.wit = pass == 0 ? nullptr : W;
                scan(kPrune, q);
                if (pass == 0 && W) {
                    // rows killed after pass 0 in earlier tries test their killer
                    // before the later bands are walked (k_witness)
                    ScanParams w = P;
                    w.wit = W;
                    if (wit_cache) {
                        if (wc_m.cap < (size_t)n) {
                            wc_m.ensure((size_t)n);
                            ck(cudaMemsetAsync(wc_m.p, 0, (size_t)n * sizeof(int), st), "memset");  // empty
                        }
                        wc_qt.ensure((size_t)n);
                        wc_q.ensure((size_t)n);
                        w.wc_qt = wc_qt.p;
                        w.wc_m = wc_m.p;
                        w.wc_q = wc_q.p;
                        w.pfx1 = pfx1.p;
                    }
                    launch_witness(w, wl.p, wl2.p, st);
                    ck(cudaGetLastError(), "witness");
                    ctr.kernel_launches += N < (1 << 18) ? 2 : 3;
                }
                reduce_alive(N);
                compact(N, pass, m);
                trace("band", m, r_sq, pass);
            }
        } else {
            compact(N, kGateNone, m);
        }

        // ---- full rows (PD3 refinement) for every remaining candidate: prune,
        // queue knife edges, and track a lower bound of each row's best corr.
        // The diagonals are swept as tracked chunks with a compaction (and new
        // groups) after each: first the far diagonals the band passes never
        // reached, doubling, where the remaining non-discords die, then the
        // near chunk [m, kend) for the rows still undecided.  The last launch
        // covers whatever chunks the enqueued count did not reach.
        ScanParams q = P;
        q.seed32 = seed32_track;
        q.wit = W;
        if (rc_on(m) && need_top > 0 && rc_m == m) {  // full rows + collection seed from the row cache
            q.rcqt = rcqt.p;
            q.rc_stride = (long long)n;
            q.rc_n = kRcSlots;
            for (int s = 0; s < kRcSlots; ++s) q.rc_row[s] = rc.row[s] < N ? rc.row[s] : -1;
        }
        // collection skip: single catch-all full-row launch, one rank (a row's
        // band may span two tiles dealt to different ranks)
        if (collect_skip && ubk.p && world == 1 && (track_chunks <= 1)) {
            q.ub = ubk.p;
            q.ub_cap = (long long)ubk.cap;
            q.list = list.p;
            q.exli = exli.p;
        }
        launch_track_init(C, N, (int)m, r_sq > 0.0 && enq_passes > 0, st);
        ck(cudaGetLastError(), "track init");
        ctr.kernel_launches += 1;
        // Measured: separate tracked chunks cost a launch latency each (C4:
        // 505 us per try in 6 chunks vs 346 us in one launch), so by default
        // the whole stage is the single catch-all launch; track_chunks > 1
        // enables the chunked schedule (experiments).
        const int twant = track_chunks <= 1 ? 1 : std::max(1, std::min(track_hint > 0 ? track_hint : 4, track_chunks));
        for (int j = 0; j + 1 < twant; ++j) {
            q.space = kSpaceTrack;
            scan(kPruneTrack, q);
            reduce_alive(N);
            compact(N, kGateTrack, m);
            trace("tracked", m, r_sq, j);
        }
        q.space = kSpaceTrackRest;
        scan(kPruneTrack, q);
        reduce_alive(N);
        reduce_maxima(N);
        // knife edges: the reference's FP64 distance decides (pardrag.cpp:255);
        // degenerate rows: every pair with one is decided exactly.  One launch.
        launch_recheck(t.p, (int)m, N, queue.p, &C->queue, queue_cap, list.p, C, cr_cur, degc.p, deg2.p, nrm.p,
                       r_sq, alive.p,
                       nnkey.p, rank, world, peers, W, st);
        ck(cudaGetLastError(), "recheck");
        reduce_alive(N);

        // ---- survivors: exact nearest neighbours (pardrag.cpp:378-416).  One
        // CTA filters the list to the survivors, applies the MERLIN top-k
        // filter, resets their keys and groups them.
        launch_survivors(list.p, alive.p, C, ymax.p, emax.p, nrm.p, cr_cur, N, (int)m, (int)need_top, bnd_lo.p,
                         bnd_hi.p, cand.p, ythr.p, nnkey.p, groups.p, sparse_rows, seed_w, exli.p, rc_on(m) ? surv.p : nullptr, st);
        ck(cudaGetLastError(), "survivors");
        const int* ex = cand.p;  // rows whose exact nn is computed (count: C->ec)
        q.space = kSpaceFull;  // every diagonal of the exact-nn rows' groups
        q.seed32 = seed32_collect;
        q.wit = nullptr;
        scan(kCollect, q);
        trace("collected", m, r_sq, 0);
        launch_ref_pairs(1, t.p, (int)m, coll.p, &C->coll, coll_cap, r_sq, alive.p, nnkey.p, C,
                         world == 1 ? ex : nullptr, nnout.p, peers, st);
        ck(cudaGetLastError(), "exact");
        if (world > 1) {
            if (peers.n > 1) peer_barrier();  // every rank's exact pairs reached every nnkey
            else allreduce_min_u64(nnkey.p, N);
            launch_gather_nn(ex, &C->ec, nnkey.p, nnout.p, st);
            ck(cudaGetLastError(), "gather");
            ctr.kernel_launches += 1;
        }
        ctr.kernel_launches += 3;  // recheck, survivors, exact pairs

        // ---- the try's single round trip: control block, counters and a
        // bounded prefix of the records (the rest only if there are more)
        const int pf = std::min(N, result_prefix);
        ck(cudaMemcpyAsync(h_ctl.p, C, sizeof(TryCtl), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(h_acc.p, acc.p, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(h_ex.p, ex, pf * sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        if (rc_on(m) && need_top > 0)
            ck(cudaMemcpyAsync(h_surv.p, surv.p, pf * sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(h_nn.p, nnout.p, pf * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        sync();
        const TryCtl hc = *h_ctl.p;
        if (hc.queue > queue_cap || hc.coll > coll_cap) {
            // degenerate inputs (exact ties by the thousand, e.g. an exactly
            // periodic series): finish the try with the exact pass over every
            // live row instead of failing, as the reference does
            harvest(m);
            harvest_events();
            ctr.rechecks += (unsigned long long)std::min(hc.queue, queue_cap);
            ctr.exact_pairs += (unsigned long long)std::min(hc.coll, coll_cap);
            ctr.fallbacks += 1;
            out = exact_fallback(m, r_sq, all_nn, N);
            last_count = (int)out.size();
            return out;
        }
        ctr.rechecks += (unsigned long long)hc.queue;
        ctr.exact_pairs += (unsigned long long)hc.coll;
        last_count = hc.sc;
        // tracked chunks: run them one by one next time as far as this try needed
        track_hint = hc.tphase >= 2 ? hc.tpasses + 1 : std::min(16, std::max(track_hint, 4) + 2);
        if (r_sq > 0.0 && enq_passes > 0) {
            // cut off by the count: allow more; otherwise (passes stopped paying,
            // or rows ran out) enqueue what this try used: the passes after the
            // device-side break are no-op launches (measured: C2 35.7 -> 35.4 ms,
            // C3 631 -> 626 ms against keeping the largest count seen)
            if (hc.stop == INT_MAX) band_hint = enq_passes + 2;
            else band_hint = std::max(1, hc.passes);
        }
        const int ec = hc.ec;
        if (debug)
            fprintf(stderr, "[tsd] m=%lld r2=%.6g done passes=%d survivors=%d exact=%d queue=%d coll=%d\n",
                    (long long)m, r_sq, hc.passes, hc.sc, ec, hc.queue, hc.coll);
        const int* hex = h_ex.p;
        const double* hnn = h_nn.p;
        std::vector<int> ex_big;
        std::vector<double> nn_big;
        if (ec > pf) {
            ex_big.resize(ec);
            nn_big.resize(ec);
            ck(cudaMemcpyAsync(ex_big.data(), ex, ec * sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(nn_big.data(), nnout.p, ec * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
            sync();
            hex = ex_big.data();
            hnn = nn_big.data();
        }
        if (need_top > 0 && rc_on(m)) rc_update(m, h_surv.p, std::min(hc.sc, pf));
        out.reserve(ec);
        for (int e = 0; e < ec; ++e) {
            const int c = hex[e];
            const double d = hnn[e];
            if (all_nn) all_nn[c] = d;
            out.push_back(tsd_record{(int64_t)c + 1, d, std::sqrt(d)});
        }
        // sort_discords: nn_dist_sq desc, index asc (src/types.cpp:15-20)
        std::sort(out.begin(), out.end(), [](const tsd_record& a, const tsd_record& b) {
            if (a.nn_dist_sq != b.nn_dist_sq) return a.nn_dist_sq > b.nn_dist_sq;
            return a.index < b.index;
        });
        return finish(m, out);
    }

    // Overflow fallback (src/pardrag.cpp:142-149,388-407): the rows still alive
    // get the exact pass against every admissible q.  Kills made so far are
    // certain, and a dropped knife-edge pair can only have left a row alive
    // wrongly, so the exact pass over the live rows decides them all; the
    // exact-nn keys it lowers are the survivors' nn.  Records sorted like
    // sort_discords, every survivor included (the MERLIN count stays exact).
    std::vector<tsd_record> exact_fallback(int64_t m, double r_sq, double* all_nn, int N) {
        compact(N, kGateNone, m);  // list + ctl->alive from the current flags
        launch_exact_rows(t.p, (int)m, N, list.p, ctl.p, r_sq, alive.p, nnkey.p, rank, world, peers, st);
        ck(cudaGetLastError(), "exact rows");
        ctr.kernel_launches += 1;
        reduce_alive(N);
        if (world > 1) {
            if (peers.n > 1) peer_barrier();
            else allreduce_min_u64(nnkey.p, N);
        }
        ck(cudaMemcpyAsync(h_ctl.p, ctl.p, sizeof(TryCtl), cudaMemcpyDeviceToHost, st), "D2H");
        sync();
        const int cnt = h_ctl.p->alive;
        std::vector<int> rows(cnt);
        std::vector<uint8_t> al(N);
        std::vector<unsigned long long> keys(N);
        if (cnt > 0) ck(cudaMemcpyAsync(rows.data(), list.p, cnt * sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(al.data(), alive.p, N, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(keys.data(), nnkey.p, N * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st), "D2H");
        sync();
        std::vector<tsd_record> out;
        for (int c : rows) {
            if (!al[c]) continue;
            double d;
            std::memcpy(&d, &keys[c], sizeof d);
            if (all_nn) all_nn[c] = d;
            out.push_back(tsd_record{(int64_t)c + 1, d, std::sqrt(d)});
        }
        std::sort(out.begin(), out.end(), [](const tsd_record& a, const tsd_record& b) {
            if (a.nn_dist_sq != b.nn_dist_sq) return a.nn_dist_sq > b.nn_dist_sq;
            return a.index < b.index;
        });
        return out;
    }

    // end of a pardrag call (the stream is idle): fold in counters and timings
    std::vector<tsd_record>& finish(int64_t m, std::vector<tsd_record>& out) {
        harvest(m);
        harvest_events();
        return out;
    }
};

// ---------------------------------------------------------------------------
// host arithmetic shared with the C++ API (bit-exact restatements)
namespace {

void layout(int64_t n, int64_t m, int64_t seglen, int64_t out[4]) {
    // src/types.cpp:26-39
    if (m < 3) fail(TSD_EINVAL, "subsequence length must be at least 3");
    if (m > n - 2) fail(TSD_EINVAL, "subsequence length too large for series");
    if (seglen < m) fail(TSD_EINVAL, "segment length must be at least the subsequence length");
    if (n < seglen) fail(TSD_EINVAL, "series shorter than one segment");
    const int64_t seg_n = seglen - m + 1, cnt = n - m + 1;
    const int64_t num_seg = (cnt + seg_n - 1) / seg_n;
    out[0] = seglen;
    out[1] = seg_n;
    out[2] = num_seg;
    out[3] = num_seg * seg_n + 2 * (m - 1) - n;
}

double window_mean(const double* h, int64_t len) {
    if (len < 5) fail(TSD_ELOGIC, "threshold history window too short");
    double s = 0.0;
    for (int64_t k = len - 5; k < len; ++k) s += h[k];
    return s / 5.0;
}

double window_std(const double* h, int64_t len) {
    const double mu = window_mean(h, len);
    double s = 0.0;
    for (int64_t k = len - 5; k < len; ++k) {
        const double d = h[k] - mu;
        s += d * d;
    }
    return std::sqrt(s / 5.0);
}

double next_thr(const double* h, int64_t len, int phase, int64_t min_len, double last_r, bool failed) {
    // src/merlin.cpp:35-55
    switch (phase) {
        case 0:
            return failed ? 0.5 * last_r : 2.0 * std::sqrt((double)min_len);
        case 1:
            if (!failed && len < 1) fail(TSD_ELOGIC, "threshold history is empty");
            return 0.99 * (failed ? last_r : h[len - 1]);
        case 2: {
            if (failed) {
                const double sigma = window_std(h, len);
                return last_r - std::max(sigma, 0.01 * last_r);
            }
            const double r = window_mean(h, len) - 2.0 * window_std(h, len);
            if (r <= 0.0) return 0.01 * h[len - 1];
            return r;
        }
        default:
            fail(TSD_ELOGIC, "unreachable");
    }
}

template <typename F>
int guard(tsd_ctx* ctx, F&& f) {
    try {
        f();
        if (ctx) ctx->err.clear();
        return TSD_OK;
    } catch (const Fail& e) {
        if (ctx) ctx->err = e.msg;
        else g_create_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        if (ctx) ctx->err = "out of host memory";
        return TSD_ERUNTIME;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return TSD_ERUNTIME;
    }
}

void need_series(tsd_ctx* c) {
    if (c->n <= 0) fail(TSD_EINVAL, "no series set");
}

}  // namespace

// ===========================================================================
extern "C" {

const char* tsd_create_error(void) { return g_create_err.c_str(); }

int tsd_ctx_create(int device, tsd_ctx** out) {
    *out = nullptr;
    tsd_ctx* c = new tsd_ctx();
    const int rc = guard(nullptr, [&] {
        int cnt = 0;
        ck(cudaGetDeviceCount(&cnt), "cudaGetDeviceCount");
        if (device < 0 || device >= cnt) fail(TSD_ECUDA, "no such CUDA device");
        c->device = device;
        ck(cudaSetDevice(device), "cudaSetDevice");
        ck(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreate(&c->ev_a), "event");
        ck(cudaEventCreate(&c->ev_b), "event");
        ck(cudaEventCreate(&c->ev_t0), "event");
        ck(cudaEventCreate(&c->ev_t1), "event");
        scan_configure();
        ck(cudaGetLastError(), "configure");
    });
    if (rc != TSD_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return TSD_OK;
}

void tsd_ctx_destroy(tsd_ctx* c) {
    if (!c) return;
    if (c->debug)
        fprintf(stderr, "[tsd] host ms: wall %.1f wait %.1f\n", c->ctr.host_wall_ms, c->ctr.host_wait_ms);
    cudaSetDevice(c->device);
    if (c->comm) nccl_destroy(c->comm);
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    for (int r = 0; r < (int)c->ipc_peer_ev.size(); ++r)
        if (r != c->rank && c->ipc_peer_ev[r]) cudaEventDestroy(c->ipc_peer_ev[r]);
    if (c->ipc_ev) cudaEventDestroy(c->ipc_ev);
    if (c->st2) cudaStreamDestroy(c->st2);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    delete c->ipc_bar;
    c->t.release();
    c->mu.release();
    c->sig.release();
    c->scr_a.release();
    c->scr_b.release();
    c->df.release();
    c->dg.release();
    c->nrm.release();
    c->crange.release();
    c->pfx1.release();
    c->pfx2.release();
    c->pfx_tot1.release();
    c->pfx_tot2.release();
    c->deg.release();
    c->degc.release();
    c->deg2.release();
    c->mu2.release();
    c->sig2.release();
    c->lbstat.release();
    c->alive.release();
    c->queue.release();
    c->coll.release();
    c->ymax.release();
    c->emax.release();
    c->seedqt.release();
    c->bnd_lo.release();
    c->bnd_hi.release();
    c->cand.release();
    c->ythr.release();
    c->nnkey.release();
    c->acc.release();
    c->blk.release();
    c->list.release();
    c->ubk.release();
    c->exli.release();
    c->nnout.release();
    c->groups.release();
    c->slots.release();
    c->bcost.release();
    c->hm.release();
    c->hm_cols.release();
    c->hm_cnt.release();
    c->hm_rows.release();
    c->hm_idx.release();
    c->hm_vals.release();
    c->red_tmp.release();
    c->ctl.release();
    c->h_ctl.release();
    c->h_ex.release();
    c->h_surv.release();
    c->surv.release();
    c->rcqt.release();
    c->wit.release();
    c->wl.release();
    c->wl2.release();
    c->bflags.release();
    c->wc_qt.release();
    c->wc_m.release();
    c->wc_q.release();
    c->h_nn.release();
    c->h_int.release();
    c->h_acc.release();
    for (auto& e : c->ev_pool) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    if (c->ev_a) cudaEventDestroy(c->ev_a);
    if (c->ev_b) cudaEventDestroy(c->ev_b);
    if (c->ev_t0) cudaEventDestroy(c->ev_t0);
    if (c->ev_t1) cudaEventDestroy(c->ev_t1);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

const char* tsd_last_error(const tsd_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int tsd_nccl_unique_id(uint8_t out[128]) {
    return guard(nullptr, [&] {
        if (!nccl_get_unique_id(out)) fail(TSD_ECUDA, "ncclGetUniqueId failed (NCCL unavailable?)");
    });
}

int tsd_ctx_join(tsd_ctx* c, int rank, int world, const uint8_t id[128]) {
    return guard(c, [&] {
        if (world < 1 || rank < 0 || rank >= world) fail(TSD_EINVAL, "bad rank/world");
        c->rank = rank;
        c->world = world;
        if (world == 1) return;
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        c->comm = nccl_init(id, rank, world);
        if (!c->comm) fail(TSD_ECUDA, "ncclCommInitRank failed");
    });
}

int tsd_series_set(tsd_ctx* c, const double* v, int64_t n) {
    return guard(c, [&] {
        // src/types.cpp:8-13
        if (n < 3) fail(TSD_EINVAL, "time series needs at least 3 points");
        for (int64_t i = 0; i < n; ++i)
            if (!std::isfinite(v[i])) fail(TSD_EINVAL, "time series contains a non-finite value");
        if (n > (int64_t)INT32_MAX / 2) fail(TSD_EINVAL, "series too long for 32-bit device indexing");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        c->h_t.assign(v, v + n);
        c->n = n;
        c->t.ensure(n);
        ck(cudaMemcpyAsync(c->t.p, v, n * sizeof(double), cudaMemcpyHostToDevice, c->st), "series H2D");
        c->pfx1.ensure(n + 1);
        c->pfx2.ensure(n + 1);
        c->pfx_tot1.ensure(dd_prefix_blocks((int)n));
        c->pfx_tot2.ensure(dd_prefix_blocks((int)n));
        launch_dd_prefix(c->t.p, (int)n, c->pfx_tot1.p, c->pfx_tot2.p, c->pfx1.p, c->pfx2.p, c->st);
        ck(cudaGetLastError(), "prefix sums");
        c->ctr.kernel_launches += 3;
        c->sync();
        c->stats_m = -1;
        c->derived_m = -1;
        c->seed_m = -1;
        if (c->wit.p) ck(cudaMemset(c->wit.p, 0x80, c->wit.cap * sizeof(int)), "memset");  // witnesses of the old series
        c->rc_reset();
        if (c->wc_m.p) ck(cudaMemset(c->wc_m.p, 0, c->wc_m.cap * sizeof(int)), "memset");
    });
}

int64_t tsd_series_len(const tsd_ctx* c) { return c ? c->n : 0; }

int tsd_init_stats(tsd_ctx* c, int64_t m, double* mu, double* sigma) {
    return guard(c, [&] {
        need_series(c);
        // src/stats.cpp:9
        if (m < 2 || m > c->n - 1) fail(TSD_EINVAL, "init_stats: length out of range");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        c->init_stats_dev(m);
        const int64_t N = c->n - m + 1;
        ck(cudaMemcpyAsync(mu, c->mu.p, N * sizeof(double), cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaMemcpyAsync(sigma, c->sig.p, N * sizeof(double), cudaMemcpyDeviceToHost, c->st), "D2H");
        c->sync();
    });
}

int tsd_advance_stats(tsd_ctx* c, int64_t m, const double* mu_in, const double* sigma_in,
                      double* mu_out, double* sigma_out) {
    return guard(c, [&] {
        need_series(c);
        // src/stats.cpp:41
        if (m + 1 > c->n - 1) fail(TSD_EINVAL, "advance_stats: next length out of range");
        if (m < 2) fail(TSD_EINVAL, "advance_stats: length out of range");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const int64_t N = c->n - m + 1;
        c->mu.ensure(c->n);
        c->sig.ensure(c->n);
        ck(cudaMemcpyAsync(c->mu.p, mu_in, N * sizeof(double), cudaMemcpyHostToDevice, c->st), "H2D");
        ck(cudaMemcpyAsync(c->sig.p, sigma_in, N * sizeof(double), cudaMemcpyHostToDevice, c->st), "H2D");
        c->stats_m = m;
        c->advance_stats_dev();
        ck(cudaMemcpyAsync(mu_out, c->mu.p, (N - 1) * sizeof(double), cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaMemcpyAsync(sigma_out, c->sig.p, (N - 1) * sizeof(double), cudaMemcpyDeviceToHost, c->st),
           "D2H");
        c->sync();
    });
}

int tsd_compute_layout(int64_t n, int64_t m, int64_t seglen, int64_t out[4]) {
    return guard(nullptr, [&] { layout(n, m, seglen, out); });
}

int tsd_next_threshold(const double* h, int64_t len, int phase, int64_t min_len, double last_r,
                       int failed, double* out) {
    return guard(nullptr, [&] { *out = next_thr(h, len, phase, min_len, last_r, failed != 0); });
}

namespace {
// One device try for the pardrag-family entry points: validates like the
// reference call, installs the caller's stats (or computes init_stats(m) on
// the device) and runs pardrag_core.  all_nn (nullable, N entries) receives
// the exact nn of every survivor.
std::vector<tsd_record> run_try(tsd_ctx* c, int64_t m, double r_sq, int64_t seglen, const double* mu,
                                const double* sigma, double* all_nn = nullptr) {
    need_series(c);
    int64_t lay[4];
    layout(c->n, m, seglen, lay);  // same preconditions as the reference call
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    ck(cudaEventRecord(c->ev_t0, c->st), "event");
    c->seed_m = -1;
    const int64_t N = c->n - m + 1;
    if (mu && sigma) {
        c->mu.ensure(c->n);
        c->sig.ensure(c->n);
        ck(cudaMemcpyAsync(c->mu.p, mu, N * sizeof(double), cudaMemcpyHostToDevice, c->st), "H2D");
        ck(cudaMemcpyAsync(c->sig.p, sigma, N * sizeof(double), cudaMemcpyHostToDevice, c->st), "H2D");
        c->stats_m = m;
        c->derived_m = -1;
    } else if (c->stats_m != m) {
        c->init_stats_dev(m);
    }
    auto recs = c->pardrag_core(m, r_sq, all_nn);
    ck(cudaEventRecord(c->ev_t1, c->st), "event");
    c->sync();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1);
    c->ctr.total_ms = ms;
    return recs;
}

void copy_out(const std::vector<tsd_record>& recs, tsd_record* out, int64_t cap, int64_t* count) {
    *count = (int64_t)recs.size();
    const int64_t k = std::min<int64_t>(cap, (int64_t)recs.size());
    if (k > 0) std::memcpy(out, recs.data(), k * sizeof(tsd_record));
}
}  // namespace

int tsd_pardrag(tsd_ctx* c, int64_t m, double r_sq, int64_t seglen, const double* mu,
                const double* sigma, tsd_record* out, int64_t cap, int64_t* count) {
    return guard(c, [&] { copy_out(run_try(c, m, r_sq, seglen, mu, sigma), out, cap, count); });
}

int tsd_par_select(tsd_ctx* c, int64_t m, double r_sq, int64_t seglen, const double* mu, const double* sigma,
                   uint8_t* cand, double* nn) {
    return guard(c, [&] {
        need_series(c);
        const int64_t N = c->n - m + 1;
        if (r_sq < 0.0) fail(TSD_EINVAL, "par_select: negative threshold");
        // survivors receive their exact nn (possibly +inf: no admissible
        // partner); the rows the try killed keep the NaN marker
        std::vector<double> all((size_t)std::max<int64_t>(N, 1), NAN);
        run_try(c, m, r_sq, seglen, mu, sigma, all.data());
        for (int64_t i = 0; i < N; ++i) {
            const double d = all[(size_t)i];
            cand[i] = std::isnan(d) ? 0 : 1;
            nn[i] = std::isnan(d) ? INFINITY : d;
        }
    });
}

int tsd_par_refine(tsd_ctx* c, int64_t m, double r_sq, int64_t seglen, const double* mu, const double* sigma,
                   const uint8_t* cand, tsd_record* out, int64_t cap, int64_t* count) {
    return guard(c, [&] {
        if (r_sq < 0.0) fail(TSD_EINVAL, "par_refine: negative threshold");
        need_series(c);
        const int64_t N = c->n - m + 1;
        bool any = false;
        for (int64_t i = 0; i < N && !any; ++i) any = cand[i] != 0;
        if (!any) {  // nothing to refine (pardrag_test.cpp: "no surviving candidates")
            int64_t lay[4];
            layout(c->n, m, seglen, lay);
            *count = 0;
            return;
        }
        auto recs = run_try(c, m, r_sq, seglen, mu, sigma);
        std::vector<tsd_record> kept;
        kept.reserve(recs.size());
        for (const auto& r : recs)
            if (cand[r.index - 1]) kept.push_back(r);
        copy_out(kept, out, cap, count);
    });
}

int tsd_stats_walk(tsd_ctx* c, int64_t m0, int64_t m1, int fused, double* mu, double* sigma) {
    return guard(c, [&] {
        need_series(c);
        if (m0 < 2 || m1 < m0 || m1 > c->n - 1) fail(TSD_EINVAL, "stats_walk: length out of range");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        c->init_stats_dev(m0);
        c->seed_m = -1;
        // the MERLIN set-up: resident seed rows at kA = m1 when the band fits
        if (fused && m0 >= 3 && m1 + kW < c->n - m1 + 1) c->seed_init(m0, m1);
        for (int64_t m = m0; m < m1; ++m) {
            if (fused) c->next_length(c->seed_m == m);
            else c->advance_stats_dev();
        }
        const int64_t N = c->n - m1 + 1;
        ck(cudaMemcpyAsync(mu, c->mu.p, N * sizeof(double), cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaMemcpyAsync(sigma, c->sig.p, N * sizeof(double), cudaMemcpyDeviceToHost, c->st), "D2H");
        c->sync();
    });
}

int tsd_seed_rows(tsd_ctx* c, double* out, int64_t cap, int64_t info[4]) {
    return guard(c, [&] {
        info[0] = c->seed_m;
        info[1] = c->seed_L;
        info[2] = c->seed_kA;
        info[3] = c->seed_m < 0 ? 0 : c->seed_nb;
        const int64_t cnt = info[3] * (int64_t)kW;
        if (out && cnt > 0 && cap >= cnt) {
            ck(cudaSetDevice(c->device), "cudaSetDevice");
            ck(cudaMemcpyAsync(out, c->seedqt.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, c->st), "D2H");
            c->sync();
        }
    });
}

int tsd_brute_force_nn(tsd_ctx* c, int64_t m, double* out) {
    return guard(c, [&] {
        need_series(c);
        if (m < 3 || m > c->n - 2) fail(TSD_EINVAL, "brute_force_nn: length out of range");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (c->stats_m != m) c->init_stats_dev(m);
        c->seed_m = -1;
        const int64_t N = c->n - m + 1;
        for (int64_t i = 0; i < N; ++i) out[i] = INFINITY;
        c->pardrag_core(m, 0.0, out);
    });
}

int tsd_merlin(tsd_ctx* c, int64_t min_len, int64_t max_len, const tsd_merlin_opts* o,
               int64_t* counts, tsd_record* recs, double* final_r, int64_t* retries, uint8_t* failed) {
    return guard(c, [&] {
        need_series(c);
        const int64_t n = c->n;
        const int64_t top_k = o ? o->top_k : 1;
        const int64_t seglen_opt = o ? o->seglen : 512;
        const int64_t max_retries = o ? o->max_retries : 100;
        const bool reuse = o ? o->reuse_stats != 0 : true;
        // src/merlin.cpp:60-62
        if (min_len < 3 || min_len > max_len || 2 * max_len > n)
            fail(TSD_EINVAL, "merlin: length range out of bounds (need 3 <= minL <= maxL <= n/2)");
        if (top_k < 1) fail(TSD_EINVAL, "merlin: topK must be positive");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaEventRecord(c->ev_t0, c->st), "event");

        std::vector<double> history;
        // band-0 seeds resident for the whole run when the band fits (kA = maxL
        // keeps every band-0 diagonal a non-self match at every length); they
        // depend on the series only, so they are built on a side stream while
        // the single-threaded Eq. 4 running sums of init_stats run
        c->seed_m = -1;
        const bool seeded = (int64_t)max_len + kW < n - max_len + 1;
        if (seeded) {
            if (!c->st2) ck(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking), "stream");
            if (!c->ev_fork) ck(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "event");
            if (!c->ev_join) ck(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "event");
            ck(cudaEventRecord(c->ev_fork, c->st), "event");
            ck(cudaStreamWaitEvent(c->st2, c->ev_fork, 0), "event wait");
            std::swap(c->st, c->st2);
            c->seed_init(min_len, max_len);  // on the side stream
            std::swap(c->st, c->st2);
            ck(cudaEventRecord(c->ev_join, c->st2), "event");
        }
        c->init_stats_dev(min_len);
        if (seeded) ck(cudaStreamWaitEvent(c->st, c->ev_join, 0), "event wait");
        c->rc_reset();
        // every discovery starts from scratch: no kill witnesses from an earlier call
        if (c->wit.p) ck(cudaMemsetAsync(c->wit.p, 0x80, c->wit.cap * sizeof(int), c->st), "memset");
        if (c->wc_m.p) ck(cudaMemsetAsync(c->wc_m.p, 0, c->wc_m.cap * sizeof(int), c->st), "memset");
        for (int64_t m = min_len; m <= max_len; ++m) {
            const int64_t k = m - min_len;
            counts[k] = 0;
            failed[k] = 0;
            if (m > min_len) {
                if (reuse) {
                    c->next_length(c->seed_m == m - 1);
                } else {
                    c->init_stats_dev(m);
                    if (c->seed_m == m - 1) c->seed_advance();
                }
                c->rc_step(m - 1);
            }
            const int phase = m == min_len ? 0 : (m < min_len + 5 ? 1 : 2);
            if (phase != 0 && history.empty()) {
                failed[k] = 1;
                final_r[k] = 0.0;
                retries[k] = 0;
                continue;
            }
            int64_t lay[4];
            layout(n, m, std::min(std::max(seglen_opt, 2 * m), n), lay);  // src/merlin.cpp:86-87

            double r = next_thr(history.data(), (int64_t)history.size(), phase, min_len, 0.0, false);
            std::vector<tsd_record> got;
            int64_t tries = 0;
            bool success = false;
            for (;;) {
                const double r_sq = r > 0.0 ? r * r : 0.0;
                got = c->pardrag_core(m, r_sq, nullptr, top_k);
                const int64_t found = c->last_count;  // every survivor counts (merlin.cpp:100)
                if (found >= top_k) {
                    success = true;
                    break;
                }
                if (tries >= max_retries) {
                    success = found > 0;
                    break;
                }
                ++tries;
                r = next_thr(history.data(), (int64_t)history.size(), phase, min_len, r, true);
            }
            final_r[k] = r;
            retries[k] = tries;
            if (!success) {
                failed[k] = 1;
                continue;
            }
            if ((int64_t)got.size() > top_k) got.resize(top_k);
            double mn = got.front().nn_dist;
            for (const auto& g : got) mn = std::min(mn, g.nn_dist);
            history.push_back(mn);
            counts[k] = (int64_t)got.size();
            for (size_t j = 0; j < got.size(); ++j) recs[k * top_k + (int64_t)j] = got[j];
        }
        ck(cudaEventRecord(c->ev_t1, c->st), "event");
        c->sync();
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1);
        c->ctr.total_ms = ms;
    });
}

namespace {
// Heatmap(minL, maxL, n) preconditions (src/heatmap.cpp:12-13)
void hm_shape(tsd_ctx* c, int64_t min_len, int64_t max_len, int64_t n) {
    if (min_len < 3 || min_len > max_len || max_len >= n) fail(TSD_EINVAL, "heatmap: invalid length range");
    const int64_t rows = max_len - min_len + 1, cols = n - min_len;
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    c->hm.ensure((size_t)(rows * cols));
    c->hm_min = min_len;
    c->hm_max = max_len;
    c->hm_n = n;
}
}  // namespace

int tsd_heatmap_build(tsd_ctx* c, int64_t min_len, int64_t max_len, int64_t n, const int64_t* lengths,
                      const tsd_record* recs, int64_t count, double* scores_out) {
    return guard(c, [&] {
        hm_shape(c, min_len, max_len, n);
        const int64_t rows = max_len - min_len + 1, cols = n - min_len;
        ck(cudaMemsetAsync(c->hm.p, 0, (size_t)(rows * cols) * sizeof(double), c->st), "memset");
        // cells in record order; a later record of the same cell wins (set_score
        // overwrites), so duplicates are resolved here and the scatter is conflict-free
        std::vector<int64_t> r, i;
        std::vector<double> v;
        std::vector<std::pair<int64_t, int64_t>> order;  // (cell, position)
        for (int64_t e = 0; e < count; ++e) {
            const int64_t m = lengths[e], idx = recs[e].index;
            if (m < min_len || m > max_len || idx < 1)
                fail(TSD_EINVAL, "heatmap: record outside the matrix");
            if (idx > cols) continue;  // src/heatmap.cpp:26-27
            order.emplace_back((m - min_len) * cols + (idx - 1), e);
        }
        std::stable_sort(order.begin(), order.end(),
                         [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t k = 0; k < order.size(); ++k) {
            if (k + 1 < order.size() && order[k + 1].first == order[k].first) continue;  // keep the last
            const int64_t e = order[k].second, m = lengths[e];
            r.push_back(m - min_len);
            i.push_back(recs[e].index - 1);
            v.push_back(recs[e].nn_dist_sq / (2.0 * (double)m));
        }
        const int64_t u = (int64_t)r.size();
        if (u > 0) {
            c->hm_rows.ensure(u);
            c->hm_idx.ensure(u);
            c->hm_vals.ensure(u);
            ck(cudaMemcpyAsync(c->hm_rows.p, r.data(), u * sizeof(int64_t), cudaMemcpyHostToDevice, c->st), "H2D");
            ck(cudaMemcpyAsync(c->hm_idx.p, i.data(), u * sizeof(int64_t), cudaMemcpyHostToDevice, c->st), "H2D");
            ck(cudaMemcpyAsync(c->hm_vals.p, v.data(), u * sizeof(double), cudaMemcpyHostToDevice, c->st), "H2D");
            launch_hm_scatter(c->hm_rows.p, c->hm_idx.p, c->hm_vals.p, u, cols, c->hm.p, c->st);
            ck(cudaGetLastError(), "heatmap scatter");
        }
        if (scores_out)
            ck(cudaMemcpyAsync(scores_out, c->hm.p, (size_t)(rows * cols) * sizeof(double), cudaMemcpyDeviceToHost,
                               c->st),
               "D2H");
        c->sync();
    });
}

int tsd_heatmap_set(tsd_ctx* c, int64_t min_len, int64_t max_len, int64_t n, const double* scores) {
    return guard(c, [&] {
        hm_shape(c, min_len, max_len, n);
        const int64_t rows = max_len - min_len + 1, cols = n - min_len;
        ck(cudaMemcpyAsync(c->hm.p, scores, (size_t)(rows * cols) * sizeof(double), cudaMemcpyHostToDevice, c->st),
           "H2D");
        c->sync();
    });
}

int tsd_heatmap_rank(tsd_ctx* c, int64_t k, tsd_ranked* out, int64_t* count) {
    return guard(c, [&] {
        if (k < 1) fail(TSD_EINVAL, "rank_discords: k must be positive");
        if (c->hm_max < c->hm_min) fail(TSD_EINVAL, "rank_discords: no heatmap built");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const int64_t rows = c->hm_max - c->hm_min + 1, cols = c->hm_n - c->hm_min;
        c->hm_cols.ensure((size_t)cols);
        c->hm_cnt.ensure(1);
        ck(cudaMemsetAsync(c->hm_cnt.p, 0, sizeof(unsigned long long), c->st), "memset");
        ck(cudaEventRecord(c->ev_a, c->st), "event");
        launch_hm_colmax(c->hm.p, rows, cols, c->hm_min, c->hm_cols.p, c->hm_cnt.p, c->st);
        ck(cudaGetLastError(), "heatmap colmax");
        ck(cudaEventRecord(c->ev_b, c->st), "event");
        unsigned long long nz = 0;
        ck(cudaMemcpyAsync(&nz, c->hm_cnt.p, sizeof(nz), cudaMemcpyDeviceToHost, c->st), "D2H");
        c->sync();
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev_a, c->ev_b);
        c->ctr.heatmap_ms = ms;
        std::vector<HmCol> v((size_t)nz);
        if (nz)
            ck(cudaMemcpyAsync(v.data(), c->hm_cols.p, nz * sizeof(HmCol), cudaMemcpyDeviceToHost, c->st), "D2H");
        c->sync();
        // ranking order (src/heatmap.cpp:48-53)
        std::sort(v.begin(), v.end(), [](const HmCol& a, const HmCol& b) {
            if (a.score != b.score) return a.score > b.score;
            if (a.index != b.index) return a.index < b.index;
            return a.length < b.length;
        });
        const int64_t keep = std::min<int64_t>(k, (int64_t)v.size());
        for (int64_t e = 0; e < keep; ++e) out[e] = tsd_ranked{v[e].index, v[e].length, v[e].score};
        *count = keep;
    });
}

// ---- cross-process ranks over CUDA IPC -------------------------------------------
int tsd_ipc_export(tsd_ctx* c, int64_t rows, uint8_t out[5 * 64]) {
    return guard(c, [&] {
        if (rows < 1) fail(TSD_EINVAL, "ipc export: rows must be positive");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        // the shared arrays are allocated once, at their final size
        c->alive.release();
        c->ymax.release();
        c->emax.release();
        c->nnkey.release();
        c->alive.ensure(rows);
        c->ymax.ensure(rows);
        c->emax.ensure(rows);
        c->nnkey.ensure(rows + kMaxGroup);  // + the device barrier's flag slots (same rows on every rank)
        ck(cudaMemset(c->nnkey.p + rows, 0, kMaxGroup * sizeof(unsigned long long)), "memset");
        ck(cudaDeviceSynchronize(), "sync");  // zeroed before the handles are shared
        c->ipc_rows = rows;
        if (!c->ipc_ev)
            ck(cudaEventCreateWithFlags(&c->ipc_ev, cudaEventDisableTiming | cudaEventInterprocess), "ipc event");
        void* ptrs[4] = {c->alive.p, c->ymax.p, c->emax.p, c->nnkey.p};
        for (int k = 0; k < 4; ++k) {
            cudaIpcMemHandle_t h;
            ck(cudaIpcGetMemHandle(&h, ptrs[k]), "cudaIpcGetMemHandle");
            std::memcpy(out + 64 * k, &h, sizeof(h) < 64 ? sizeof(h) : 64);
        }
        cudaIpcEventHandle_t eh;
        ck(cudaIpcGetEventHandle(&eh, c->ipc_ev), "cudaIpcGetEventHandle");
        std::memcpy(out + 256, &eh, sizeof(eh) < 64 ? sizeof(eh) : 64);
    });
}

static int64_t rows_of(const tsd_ctx* c) { return c->ipc_rows; }

int tsd_ipc_join(tsd_ctx* c, int rank, int world, const uint8_t* handles, const char* shm_name) {
    return guard(c, [&] {
        if (world < 2 || world > kMaxPeers || rank < 0 || rank >= world) fail(TSD_EINVAL, "bad rank/world");
        if (c->ipc_rows == 0 || !c->ipc_ev) fail(TSD_EINVAL, "ipc join: call tsd_ipc_export first");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        c->rank = rank;
        c->world = world;
        c->peers = Peers{};
        c->peers.n = world;
        c->ipc_peer_ev.assign(world, nullptr);
        for (int r = 0; r < world; ++r) {
            const uint8_t* h = handles + (size_t)r * 320;
            void* p[4];
            if (r == rank) {
                p[0] = c->alive.p;
                p[1] = c->ymax.p;
                p[2] = c->emax.p;
                p[3] = c->nnkey.p;
                c->ipc_peer_ev[r] = c->ipc_ev;
            } else {
                for (int k = 0; k < 4; ++k) {
                    cudaIpcMemHandle_t mh;
                    std::memcpy(&mh, h + 64 * k, sizeof(mh) < 64 ? sizeof(mh) : 64);
                    ck(cudaIpcOpenMemHandle(&p[k], mh, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
                    c->ipc_opened.push_back(p[k]);
                }
                cudaIpcEventHandle_t eh;
                std::memcpy(&eh, h + 256, sizeof(eh) < 64 ? sizeof(eh) : 64);
                ck(cudaIpcOpenEventHandle(&c->ipc_peer_ev[r], eh), "cudaIpcOpenEventHandle");
            }
            c->peers.alive[r] = static_cast<uint8_t*>(p[0]);
            c->peers.ymax[r] = static_cast<unsigned*>(p[1]);
            c->peers.emax[r] = static_cast<unsigned*>(p[2]);
            c->peers.nnkey[r] = static_cast<unsigned long long*>(p[3]);
        }
        c->ipc_bar = new ShmBarrier(shm_name ? shm_name : "/tsd_ipc", world, rank == 0);
        for (int r = 0; r < world; ++r) c->fptr.p[r] = c->peers.nnkey[r] + rows_of(c);
        c->use_dev_bar = c->dev_barrier != 0;
        c->bar_epoch = 0;
    });
}

// ---- in-process rank group ---------------------------------------------------
struct tsd_group {
    std::vector<tsd_ctx*> ctx;
    PeerGroup* pg = nullptr;
    std::string err;
};

int tsd_group_create(const int* devices, int n, tsd_group** out) {
    *out = nullptr;
    if (n < 1 || n > kMaxGroup) {
        g_create_err = "group size must be 1.." + std::to_string(kMaxGroup);
        return TSD_EINVAL;
    }
    tsd_group* g = new tsd_group();
    g->pg = new PeerGroup(n);
    g->pg->distinct = true;
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < a; ++b)
            if (devices[a] == devices[b]) g->pg->distinct = false;
    for (int r = 0; r < n; ++r) {
        tsd_ctx* c = nullptr;
        const int rc = tsd_ctx_create(devices[r], &c);
        if (rc != TSD_OK) {
            tsd_group_destroy(g);
            return rc;
        }
        g->ctx.push_back(c);
        c->rank = r;
        c->world = n;
        c->group = g->pg;
        cudaSetDevice(c->device);
        if (cudaEventCreateWithFlags(&g->pg->ev_in[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->pg->ev_red[r], cudaEventDisableTiming) != cudaSuccess) {
            g_create_err = "event creation failed";
            tsd_group_destroy(g);
            return TSD_ECUDA;
        }
    }
    // peer access between distinct devices (same device: plain pointers)
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            const int da = g->ctx[a]->device, db = g->ctx[b]->device;
            if (da == db) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, da, db);
            if (!can) {
                g_create_err = "devices " + std::to_string(da) + " and " + std::to_string(db) + " lack peer access";
                tsd_group_destroy(g);
                return TSD_ECUDA;
            }
            cudaSetDevice(da);
            const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                g_create_err = std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e);
                tsd_group_destroy(g);
                return TSD_ECUDA;
            }
            cudaGetLastError();
        }
    *out = g;
    return TSD_OK;
}

void tsd_group_destroy(tsd_group* g) {
    if (!g) return;
    for (size_t r = 0; r < g->ctx.size(); ++r) {
        if (g->pg->ev_in[r]) cudaEventDestroy(g->pg->ev_in[r]);
        if (g->pg->ev_red[r]) cudaEventDestroy(g->pg->ev_red[r]);
        tsd_ctx_destroy(g->ctx[r]);
    }
    delete g->pg;
    delete g;
}

const char* tsd_group_last_error(const tsd_group* g) { return g ? g->err.c_str() : g_create_err.c_str(); }
int tsd_group_size(const tsd_group* g) { return g ? (int)g->ctx.size() : 0; }
tsd_ctx* tsd_group_ctx(tsd_group* g, int rank) {
    return (g && rank >= 0 && rank < (int)g->ctx.size()) ? g->ctx[rank] : nullptr;
}

}  // extern "C"
namespace {
// runs f(rank) on one host thread per rank; a failing rank releases the others
template <typename F>
int group_run(tsd_group* g, F&& f) {
    const int n = (int)g->ctx.size();
    std::vector<int> rc(n, TSD_OK);
    g->pg->bar.reset();
    std::vector<std::thread> th;
    for (int r = 0; r < n; ++r)
        th.emplace_back([&, r] {
            rc[r] = f(r);
            if (rc[r] != TSD_OK) g->pg->bar.fail();
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < n; ++r)
        if (rc[r] != TSD_OK) {
            g->err = "rank " + std::to_string(r) + ": " + tsd_last_error(g->ctx[r]);
            return rc[r];
        }
    g->err.clear();
    return TSD_OK;
}
}  // namespace
extern "C" {

int tsd_group_series_set(tsd_group* g, const double* v, int64_t n) {
    return group_run(g, [&](int r) { return tsd_series_set(g->ctx[r], v, n); });
}

int tsd_group_merlin(tsd_group* g, int64_t min_len, int64_t max_len, const tsd_merlin_opts* o, int64_t* counts,
                     tsd_record* recs, double* final_r, int64_t* retries, uint8_t* failed) {
    const int n = (int)g->ctx.size();
    const int64_t L = std::max<int64_t>(max_len - min_len + 1, 1);
    const int64_t k = std::max<int64_t>(o ? o->top_k : 1, 1);
    struct Out {
        std::vector<int64_t> counts, retries;
        std::vector<tsd_record> recs;
        std::vector<double> final_r;
        std::vector<uint8_t> failed;
    };
    std::vector<Out> outs(n);
    for (auto& x : outs) {
        x.counts.assign(L, 0);
        x.retries.assign(L, 0);
        x.recs.assign(L * k, tsd_record{});
        x.final_r.assign(L, 0.0);
        x.failed.assign(L, 0);
    }
    const int rc = group_run(g, [&](int r) {
        Out& x = outs[r];
        return tsd_merlin(g->ctx[r], min_len, max_len, o, x.counts.data(), x.recs.data(), x.final_r.data(),
                          x.retries.data(), x.failed.data());
    });
    if (rc != TSD_OK) return rc;
    // every rank holds the same reduced state, hence the same records
    for (int r = 1; r < n; ++r)
        if (outs[r].counts != outs[0].counts || outs[r].failed != outs[0].failed ||
            std::memcmp(outs[r].recs.data(), outs[0].recs.data(), L * k * sizeof(tsd_record)) != 0) {
            g->err = "ranks diverged";
            return TSD_ERUNTIME;
        }
    std::copy(outs[0].counts.begin(), outs[0].counts.end(), counts);
    std::copy(outs[0].retries.begin(), outs[0].retries.end(), retries);
    std::copy(outs[0].final_r.begin(), outs[0].final_r.end(), final_r);
    std::copy(outs[0].failed.begin(), outs[0].failed.end(), failed);
    std::copy(outs[0].recs.begin(), outs[0].recs.end(), recs);
    return TSD_OK;
}

int tsd_group_pardrag(tsd_group* g, int64_t m, double r_sq, int64_t seglen, tsd_record* out, int64_t cap,
                      int64_t* count) {
    const int n = (int)g->ctx.size();
    std::vector<std::vector<tsd_record>> bufs(n, std::vector<tsd_record>(std::max<int64_t>(cap, 1)));
    std::vector<int64_t> cnt(n, 0);
    const int rc = group_run(g, [&](int r) {
        return tsd_pardrag(g->ctx[r], m, r_sq, seglen, nullptr, nullptr, bufs[r].data(), cap, &cnt[r]);
    });
    if (rc != TSD_OK) return rc;
    for (int r = 1; r < n; ++r)
        if (cnt[r] != cnt[0] ||
            std::memcmp(bufs[r].data(), bufs[0].data(), std::min(cnt[0], cap) * sizeof(tsd_record)) != 0) {
            g->err = "ranks diverged";
            return TSD_ERUNTIME;
        }
    *count = cnt[0];
    std::copy(bufs[0].begin(), bufs[0].begin() + std::min(cnt[0], cap), out);
    return TSD_OK;
}

int tsd_matrix_profile_fp64(tsd_ctx* c, int64_t m, double* out) {
    return guard(c, [&] {
        need_series(c);
        if (m < 3 || m > c->n - 2) fail(TSD_EINVAL, "matrix_profile: length out of range");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const int64_t n = c->n, N = n - m + 1;
        double gm = 0.0;
        for (double v : c->h_t) gm += v;
        gm /= (double)n;
        DBuf<double> scratch, res;
        DBuf<unsigned long long> keys;
        scratch.ensure((size_t)(2 * n + 4 * N));
        keys.ensure((size_t)(2 * N));
        res.ensure((size_t)N);
        ck(cudaEventRecord(c->ev_a, c->st), "event");
        mp_fp64(c->t.p, (int)n, (int)m, gm, scratch.p, keys.p, res.p, c->st);
        ck(cudaGetLastError(), "matrix profile");
        ck(cudaEventRecord(c->ev_b, c->st), "event");
        ck(cudaMemcpyAsync(out, res.p, (size_t)N * sizeof(double), cudaMemcpyDeviceToHost, c->st), "D2H");
        c->sync();
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev_a, c->ev_b);
        c->ctr.total_ms = ms;
        scratch.release();
        keys.release();
        res.release();
    });
}

int tsd_gen_randomwalk(int64_t n, uint64_t seed, double* out) {
    return guard(nullptr, [&] {
        // src/io.cpp:110-119 — same engine and distribution (libstdc++)
        if (n < 3) fail(TSD_EINVAL, "gen_randomwalk: n must be at least 3");
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> step(0.0, 1.0);
        out[0] = 0.0;
        for (int64_t i = 1; i < n; ++i) out[i] = out[i - 1] + step(rng);
    });
}

int tsd_get_counters(const tsd_ctx* c, tsd_counters* out) {
    if (!c || !out) return TSD_EINVAL;
    *out = c->ctr;
    return TSD_OK;
}

int tsd_reset_counters(tsd_ctx* c) {
    if (!c) return TSD_EINVAL;
    c->ctr = tsd_counters{};
    return TSD_OK;
}

int tsd_tile_plan(int space, int64_t N, int64_t m, int64_t L, int64_t kA, int64_t nb, int64_t K0,
                  const int32_t* groups, int64_t G, int rank, int world, int32_t* out, int64_t cap,
                  int64_t* count) {
    return guard(nullptr, [&] {
        if (world < 1 || rank < 0 || rank >= world) fail(TSD_EINVAL, "bad rank/world");
        if (N < 1 || m < 1) fail(TSD_EINVAL, "bad N/m");
        ScanParams p{};
        p.N = (int)N;
        p.m = (int)m;
        p.L = (int)L;
        p.kA = (int)kA;
        p.nb = (int)nb;
        p.K0 = (int)K0;
        p.rank = rank;
        p.world = world;
        p.groups = reinterpret_cast<const int2*>(groups);
        TileCtx c{0, 0, 0, 0};
        switch (space) {
            case 0:  // band 0 at kA over L-row blocks (resident seeds), nb sides
                p.space = kSpaceSeed;
                c.slots = nb * ((N + L - 1) / L);
                break;
            case 1:  // band [K0, K0 + nb kW) over L-row blocks
                p.space = kSpaceBlocks;
                c.G = (N + L - 1) / L;
                c.slots = 2 * nb * c.G;
                c.k0 = K0;
                break;
            case 2:  // band [K0, K0 + nb kW) over the groups
                if (!groups || G < 1) fail(TSD_EINVAL, "groups required");
                p.space = kSpaceBand;
                c.G = G;
                c.slots = 2 * nb * G;
                c.k0 = K0;
                break;
            case 3: {  // every diagonal |k| >= m of the groups (full rows)
                if (!groups || G < 1) fail(TSD_EINVAL, "groups required");
                p.space = kSpaceFull;
                c.G = G;
                const int64_t maxc = (N - m + kW - 1) / kW;
                c.slots = maxc > 0 ? 2 * maxc * G : 0;
                break;
            }
            default:
                fail(TSD_EINVAL, "unknown tile space");
        }
        // the kernels' cyclic deal: rank r fetches slots r, r + world, ...
        const long long mine = world > 1 ? (c.slots > rank ? (c.slots - rank + world - 1) / world : 0) : c.slots;
        int64_t k = 0;
        for (long long f = 0; f < mine; ++f) {
            TileDesc td;
            if (!tile_decode(p, c, f * world + rank, td)) continue;
            if (k < cap) {
                int32_t* o = out + 5 * k;
                o[0] = td.r0;
                o[1] = td.rows;
                o[2] = td.k0;
                o[3] = td.dir;
                o[4] = td.seed;
            }
            ++k;
        }
        *count = k;
    });
}

int tsd_set_param(tsd_ctx* c, const char* key, double v) {
    return guard(c, [&] {
        const std::string k = key ? key : "";
        if (k == "dense_rows") c->dense_rows = v <= 0 ? 0 : std::max(16, std::min(kMaxRows, (int)v));
        else if (k == "sparse_rows") c->sparse_rows = std::max(0, std::min(kMaxRows, (int)v));
        else if (k == "err_scale") c->err_k = v;
        else if (k == "scan_events") c->scan_events = v != 0.0;
        else if (k == "fused_peers") c->fused = v != 0.0;
        else if (k == "seed32_track") c->seed32_track = v != 0.0;
        else if (k == "seed32_collect") c->seed32_collect = v != 0.0;
        else if (k == "band0_sides") c->band0_sides = v <= 1.0 ? 1 : 2;
        else if (k == "track_chunks") c->track_chunks = std::max(1, std::min(16, (int)v));
        else if (k == "band_few") c->band_few = std::max(0, (int)v);
        else if (k == "half_pass0") c->half_pass0 = v >= 6 ? 6 : std::max(1, std::min(3, (int)v));
        else if (k == "half_bands") c->half_bands = v == 20 ? 20 : std::max(1, std::min(3, (int)v));
        else if (k == "half_bands_m") c->half_bands_m = (long long)v;
        else if (k == "pair_band0") c->pair_band0 = v != 0.0;
        else if (k == "pass0_pk") c->pass0_pk = v != 0.0;
        else if (k == "half_pk")
            c->half_pk = (v == 12 || v == 16 || v == 20) ? (int)v
                         : v >= 9 ? 9 : (v >= 6 ? 6 : std::max(1, std::min(3, (int)v)));
        else if (k == "pk_min_n") c->pk_min_n = (int64_t)v;
        else if (k == "pk_rows") c->pk_rows = v <= 0 ? 0 : std::max(16, std::min(kMaxRows, (int)v));
        else if (k == "seed_w") c->seed_w = (float)std::max(0.01, v);
        else if (k == "band_keep") c->band_keep = (float)std::max(0.0, std::min(1.0, v));
        else if (k == "band_fill") c->band_fill = std::max(0.0, v);
        else if (k == "band_passes") c->band_passes = std::max(1, std::min(64, (int)v));
        else if (k == "result_prefix") c->result_prefix = std::max(16, std::min(1 << 20, (int)v));
        else if (k == "collect_skip") c->collect_skip = v != 0.0;
        else if (k == "witness") c->witness = v != 0.0;
        else if (k == "row_cache") c->row_cache = v != 0.0;
        else if (k == "wit_cache") c->wit_cache = v != 0.0;
        else if (k == "few_m") c->few_m = (int64_t)v;
        else if (k == "few_lo") c->few_lo = std::max(1, (int)v);
        else if (k == "dev_barrier") {
            c->dev_barrier = v < 0 ? -1 : (v != 0.0 ? 1 : 0);
            c->use_dev_bar = c->world > 1 && c->peers.n > 1 && c->dev_barrier != 0;
        }
        else if (k == "rc_min_m") c->rc_min_m = (int64_t)v;
        else if (k == "band_few_wit") c->band_few_wit = std::max(0, (int)v);
        else if (k == "queue_cap") c->queue_cap = std::max(1, std::min(kQueueCap, (int)v));
        else if (k == "coll_cap") c->coll_cap = std::max(1, std::min(kCollCap, (int)v));
        else fail(TSD_EINVAL, "unknown parameter " + k);
    });
}

}  // extern "C"
