// Shared device-side definitions for the PALMAD engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tsd {

// include/tsdiscord/stats.hpp:11 — a subsequence with sigma below this is constant.
constexpr double kSigmaEps = 1e-12;

// ---- statistics error of the FP32 filter ("Statistics error") --
// The FP32 walk normalises with the reference's rolling mu / sigma (Eq. 4 /
// 7-8), while the exact distance it certifies against uses each window's
// one-pass statistics (znormalize).  Both deviate from the window's true
// moments by an amount that grows like mu^2 / sigma^2 (DC offsets).  Per
// length, k_derive / k_next_length measure the rolling statistics against
// double-double prefix sums and bound the one-pass ones a priori; the
// per-length maxima (over windows the filter keeps) widen every certified band.
// A window whose statistics error exceeds kStatsUnreliable (flat stretches
// with a spurious rolling sigma, extreme offsets) is decided exactly, like a
// sigma < eps window.
constexpr double kEps64 = 1.1102230246251565e-16;  // 2^-53
constexpr double kStatsUnreliable = 1e-3;          // corr units
constexpr double kStatsRows = 1040.0;              // 2 (kMaxRows + 8): walk steps a mean error acts over
// per-length slot (two parity slots of kCrInts ints): [0] max(N - i), [1] max(i + 1)
// over degenerate rows, [2] their count (listed in deg), [3] bits of the max
// statistics error a_i (float >= 0), [4] bits of the max 1 + mu_i^2 / sigma_i^2,
// [5] max(N - i) and [6] max(i + 1) over the degenerate windows whose one-pass
// statistics are constant too (znormalize gives all zeros: the 0 / 2m
// conventions decide their pairs), [7] their count (listed in degc), [8] the
// count of the other degenerate windows (listed in deg2; decided exactly)
constexpr int kCrInts = 9;

// The reference's znormalize test for a window (src/distance.cpp:8-22):
// sequential sums in index order, no contraction; true when z is all zeros.
__device__ __forceinline__ bool onepass_const(const double* __restrict__ w, int m) {
    double s = 0.0, q = 0.0;
    for (int k = 0; k < m; ++k) {
        const double v = w[k];
        s = __dadd_rn(s, v);
        q = __dadd_rn(q, __dmul_rn(v, v));
    }
    const double mean = __ddiv_rn(s, (double)m);
    const double var = __dsub_rn(__ddiv_rn(q, (double)m), __dmul_rn(mean, mean));
    return __dsqrt_rn(var > 0.0 ? var : 0.0) < kSigmaEps;
}

struct dd {  // double-double (unevaluated sum hi + lo)
    double hi, lo;
};
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return dd{s, e};
}
__device__ __forceinline__ dd dd_fast(double a, double b) {  // |a| >= |b|
    const double s = __dadd_rn(a, b);
    return dd{s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = dd_two_sum(a.hi, b.hi);
    const dd t = dd_two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = dd_fast(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return dd_fast(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sq(double a) {  // exact a*a
    const double p = __dmul_rn(a, a);
    return dd{p, fma(a, a, -p)};
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    const double p = __dmul_rn(a.hi, b.hi);
    double e = fma(a.hi, b.hi, -p);
    e = fma(a.hi, b.lo, fma(a.lo, b.hi, e));
    return dd_fast(p, e);
}
__device__ __forceinline__ dd dd_div_d(dd a, double b) {
    const double q1 = __ddiv_rn(a.hi, b);
    const double r = __dadd_rn(fma(-q1, b, a.hi), a.lo);
    return dd_fast(q1, __ddiv_rn(r, b));
}

// ---- tile-scan geometry ----------------------------------------------------
// One CTA sweeps a parallelogram of the distance matrix: `rows` consecutive
// candidates c (walk order given by dir) x W consecutive diagonals k = q - c.
// Each thread owns D adjacent diagonals and walks them down (dir=+1, k >= m)
// or up (dir=-1, k <= -m) with the FP32 centered-covariance recurrence, so
// every invalid cell (q outside [0,N)) lies at the far end of its walk.
constexpr int kThreads = 128;            // threads per scan CTA
constexpr int kDiag = 9;                 // diagonals per thread (odd: conflict-free strided smem)
constexpr int kW = kThreads * kDiag;     // 1152 diagonals per tile
constexpr int kMaxRows = 512;            // max rows per tile
constexpr int kSeedChunk = 512;          // seed dot products are staged m in chunks of this

struct TileDesc {
    int r0;    // first row (0-based candidate index)
    int rows;  // number of rows (<= kMaxRows), all < N
    int k0;    // lowest diagonal of the tile; the tile covers [k0, k0 + kW)
    int dir;   // +1: positive side walked downward; -1: negative side walked upward
    int seed;  // >= 0: seed row kept resident across lengths (ScanParams::seedqt), else -1
};

// Tile spaces: how a persistent scan CTA turns a fetched slot index into a tile.
enum TileSpace : int {
    kSpaceSeed = 0,    // band 0 at offset kA over aligned L-row blocks, seeded from resident rows
    kSpaceBlocks = 1,  // band [K0, K0 + nb*kW) over aligned L-row blocks (FP32 / FP64 direct seeds)
    kSpaceBand = 2,    // band [K0, K0 + nb*kW) over the device-built groups (TryCtl::G)
    kSpaceFull = 3,    // every diagonal |k| >= m of the device-built groups, near-first
    kSpaceTrack = 4,   // tracked full-row chunk [tK0, tK0 + tnb*kW) over the groups (TryCtl)
    kSpaceTrackRest = 5  // every tracked chunk not yet run (far rest + near), in one launch
};

// Device-resident control block of one DRAG try: every count the host used to
// read back between passes lives here, so a whole try is enqueued without a
// host round trip (kernels gate themselves on these fields).
struct TryCtl {
    int alive;      // undecided rows after the latest compaction
    int prev;       // the count before it (band-pass break rule)
    int stop;       // band passes with index > stop are skipped (INT_MAX: none yet)
    int G;          // groups of the current stage (ScanParams::groups)
    int slotc[32];  // persistent-scan slot counters, one per scan launch of the try (k_try_init zeroes them)
    int queue;      // knife-edge pairs queued
    int coll;       // near pairs collected
    int crange[2];  // first / last constant row
    int sc;         // range-discord survivors (after the knife-edge recheck)
    int ec;         // rows whose exact nn is computed (MERLIN top-k filter)
    int passes;     // band passes that ran
    int span;       // group span of the current stage
    int cticket;    // compaction: CTA order tickets (self-resetting)
    int cdone;      // compaction: finished CTAs (self-resetting)
    int ctotal;     // compaction: total of the latest launch
    int xdone;      // exact pass: finished CTAs (self-resetting)
    int stop_why;   // band loop: 1 nothing / few rows / no diagonals left, 2 a pass killed too few
    int bK0;        // band passes >= 1: first diagonal of the next pass
    int bnb;        // ... and its number of kW-wide bands (set by the compaction before it)
    // full rows as tracked chunks: far chunks [kend, N) first (doubling), then
    // the near chunk [m, kend) that the band passes covered without tracking
    int kend;       // end of the band passes' coverage
    int tK0, tnb;   // next tracked chunk
    int tphase;     // 0 far chunks, 1 near chunk, 2 done
    int tpasses;    // tracked chunks that ran
    unsigned tepoch;  // try counter (k_try_init): tags the per-(row, band) bounds of this try
    int wn;         // kill-witness candidates listed after band pass 0 (k_witness_list)
    int wn2;        // ... rows left for the 9-diagonal phase (k_witness9)
    int wrun, wrun2;  // witness phases: runs / rows fetched (dynamic)
    double lk;      // top-k filter: need_top-th largest nn lower bound
    double cost[6]; // compaction: grouping cost per span (16..512), self-resetting
};

// compaction / grouping gates: a band pass index (>= 0: skipped once the band
// passes stopped before it), or one of these
constexpr int kGateNone = -1;   // always runs
constexpr int kGateTrack = -3;  // tracked chunks: skipped once the chunks are done

enum ScanMode : int {
    kPrune = 0,       // dense band: kill both ends of any pair with d^2 < r^2
    kPruneTrack = 1,  // sparse rows: prune + track a lower bound of each live row's max corr
    kCollect = 2      // survivors: push every pair that may attain the row's exact minimum
};

// Fused rank reduction over peer memory (in-process rank group): a kernel that
// kills a row, or raises a row maximum, stores into EVERY rank's array (peer
// stores / atomics over NVLink, plain ones on a shared device).  Kills are
// monotone byte stores and maxima are atomicMax, so the stores themselves are
// the AND / MAX all-reduce; the ranks only meet at an event barrier afterwards.
constexpr int kMaxPeers = 8;
struct Peers {
    uint8_t* alive[kMaxPeers];
    unsigned* ymax[kMaxPeers];
    unsigned* emax[kMaxPeers];
    unsigned long long* nnkey[kMaxPeers];
    int n;  // 0: local only
};

__device__ __forceinline__ void peer_min_key(const Peers& P, unsigned long long* local, int c,
                                             unsigned long long v) {
    if (P.n > 1) {
#pragma unroll 1
        for (int r = 0; r < P.n; ++r) atomicMin(&P.nnkey[r][c], v);
    } else {
        atomicMin(&local[c], v);
    }
}

__device__ __forceinline__ void peer_kill(const Peers& P, uint8_t* local, int c) {
    if (P.n > 1) {
#pragma unroll 1
        for (int r = 0; r < P.n; ++r) P.alive[r][c] = 0;
    } else {
        local[c] = 0;
    }
}

struct ScanParams {
    const double* t;     // series (n)
    const double* mu;    // FP64 rolling mean, length m (N)
    const double* sig;   // FP64 rolling std (N)
    const float* df;     // FP32 (t[i+m-1]-t[i-1])/2             (N; [0] unused)
    const float* dg;     // FP32 (t[i+m-1]-mu_i)+(t[i-1]-mu_{i-1}) (N; [0] unused)
    const float* nrm;    // FP32 1/(sqrt(m)*sigma_i), 0 if constant (N)
    int n, m, N;
    double r_sq;         // squared threshold
    double thr0;         // 1 - r_sq/(2m): corr > thr0  <=>  d^2 < r^2
    double err_k;        // error model: |cov_fp32 - cov| <= err_k*eps*m*smax_c*smax_q*(rows+8)
    uint8_t* alive;      // candidate flags (N); 1 = may still be a range discord
    int2* queue;         // knife-edge pairs for the exact FP64 recheck
    int* queue_count;
    int queue_cap;
    unsigned* ymax;      // kPruneTrack: ordered-float key of the row's max route value x = cov*qn
    unsigned* emax;      // kPruneTrack: bits of the largest tile error term E*qn_max seen by the row
    const float* ythr;   // kCollect: per-row collection threshold (decoded ymax)
    int2* coll;          // kCollect output pairs
    int* coll_count;
    int coll_cap;
    // tile space of this launch (persistent CTAs fetch slots from *next, a
    // counter of its own: no exit ticket, no reset)
    TryCtl* ctl;
    int* next;
    const int2* groups;  // kSpaceBand / kSpaceFull: (first, last) row of each group
    int space;           // TileSpace
    int pass;            // band pass index (kSpaceBand: skipped when ctl->stop < pass)
    int K0, nb;          // kSpaceBlocks: diagonals [K0, K0 + nb*kW) on both sides (kSpaceBand: TryCtl)
    int L, kA;           // kSpaceSeed / kSpaceBlocks: block rows; kSpaceSeed: band offset
    int rank, world;     // tiles are dealt cyclically across ranks
    int seed32;          // FP32 direct seeds (with their error term in E) outside the band passes too
    Peers peers;         // fused cross-rank kills / maxima (n > 1), else local
    int half;            // band passes: evaluate 1 cell in `half` (1: all)
    int pair;            // band 0 (kSpaceSeed, both sides): one paired walk per row block (k_band0_pair)
    const double* seedqt;  // resident raw dot products QT(i, i+k) of the band-0 tiles (kW per tile)
    const int* cr;         // per-length slot of this length (kCrInts ints; statistics error in [3], [4])
    // per-(row, band) correlation upper bounds of the full-row stage, read by the
    // collection to skip bands that cannot hold a row's nearest neighbour
    // (nullptr: off).  Entry ((li * 2 + side) * nbands + band) for the row at
    // list index li; value (tepoch << 32) | f2key(bound).
    unsigned long long* ub;
    long long ub_cap;      // entries available
    const int* list;       // the sorted list of the full-row stage (ctl->alive rows)
    int* exli;             // survivors' list index by row (k_survivors), read by the collection
    unsigned long long* acc;  // accounting: [0] cells walked, [1] cells evaluated, [2] seed dots,
                              // [3] witness rows tested, [4] witness kills
    // Kill witnesses (MERLIN's consecutive tries): per row, the first of 9
    // diagonals k (q = c + k .. c + k + 8) that killed it in an earlier try, or
    // kNoWit.  Written by the stages after band pass 0 (nullptr: not recorded),
    // tested by k_witness at the start of the next try.  Hints only: a witness
    // kill is certified like any other, so stale entries cost a test, nothing else.
    int* wit;
    // run-seed cache of the witness test (k_witness): per row, the raw FP64
    // dot product QT(c, wc_q[c]) at length wc_m[c] (0: none); with pfx1, the
    // double-double prefix sums of t that convert it to the shifted seed
    double* wc_qt;
    int* wc_m;
    int* wc_q;
    const double2* pfx1;
    unsigned long long* dbg;  // TSD_DEBUG: [mode*2] slots fetched, [mode*2+1] slots with work (nullptr: off)
    // Row cache (full rows / collection): resident raw QT rows of up to
    // kRcSlots anchor rows near the previous tries' survivors, valid for this
    // length (rc_n = 0: none); slot s holds QT(rc_row[s], q) at rcqt[s * rc_stride + q]
    const double* rcqt;
    long long rc_stride;
    int rc_n;
    int rc_row[8];
};
constexpr int kRcSlots = 8;
struct RcRows {  // the anchor rows of the row-cache slots (-1: empty)
    int row[kRcSlots];
    int n;
};

constexpr int kNoWit = (int)0x80808080;  // memset byte 0x80
constexpr int kWitMaxM = 1024;           // witness tests stage whole windows: lengths up to this

// canonical diagonal band of |k| for the per-(row, band) bounds: [m + b kW, m + (b+1) kW)
__host__ __device__ __forceinline__ int ub_nbands(int N, int m) { return N > m ? (N - m + kW - 1) / kW : 0; }

// Widening of every certified band of this length (correlation units) for
// the statistics error: twice the largest per-window error a_i, plus, for
// tiles seeded from the resident raw dot products QT (no centring), their FP64
// accumulation error (m + 4) u sqrt((1 + Om_c)(1 + Om_q)) and the rolling
// means' error acting on m mu_c mu_q (a_i bounds 1040 |mu err| / sigma).
__device__ __forceinline__ double stats_band(const ScanParams& p, bool resident_seed) {
    const double a = (double)__int_as_float(p.cr[3]);
    double x = 2.0 * a;
    if (resident_seed) {
        const double b2 = (double)__int_as_float(p.cr[4]);
        x += 2.0 * (double)(p.m + 4) * kEps64 * b2 + 4.0 * a * sqrt(b2) / kStatsRows;
    }
    return x;
}

// Programmatic dependent launch: every kernel of the try chain is launched
// with programmatic stream serialization (launch_pdl), waits here for its
// predecessor's completion and memory, then lets its own successor launch, so
// the successor's CTAs are resident when this grid ends (no launch gap).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// GPU-scope memory-model helpers.  Cross-CTA hand-offs use a release/acquire
// atomic by one thread after a CTA barrier (cumulative through bar.sync)
// instead of a sequentially consistent fence in every thread.
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Order-preserving float <-> uint32 map (for atomicMax on floats of any sign).
__device__ __forceinline__ unsigned f2key(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

}  // namespace tsd
