/*
 * tsdiscord_b200.h — C-ABI of the B200-native PALMAD / MERLIN library
 * (libtsdiscord_b200.so).  Plain pointers and sizes only; no torch or C++ types.
 *
 * Every entry point replaces one function of the reference's C++ discord API
 * (/root/reference/proj/include/tsdiscord); the C++ drop-in headers in
 * include/tsdiscord/ are implemented on top of this layer and rethrow the
 * status codes as the reference's exception types:
 *
 *   TSD_EINVAL   -> std::invalid_argument  (preconditions: src/types.cpp:9-11,27-30,
 *                                           src/stats.cpp:9,41, src/merlin.cpp:60-62)
 *   TSD_ELOGIC   -> std::logic_error       (src/merlin.cpp:19,54)
 *   TSD_ERUNTIME -> std::runtime_error     (I/O, src/io.cpp)
 *   TSD_ECUDA    -> std::runtime_error     (device failure; never a silent CPU fallback)
 *
 * Indices in and out are 1-based, like the reference (types.hpp:11).
 * A context owns one CUDA device, its stream, the resident series and all
 * device-side state; contexts are not thread-safe (one per calling thread).
 */
#ifndef TSDISCORD_B200_H
#define TSDISCORD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TSD_OK = 0,
    TSD_EINVAL = 1,
    TSD_ELOGIC = 2,
    TSD_ERUNTIME = 3,
    TSD_ECUDA = 4
};

typedef struct tsd_ctx tsd_ctx;

/* One discord: replaces tsdiscord::DiscordRecord (include/tsdiscord/types.hpp:50-54). */
typedef struct {
    int64_t index;     /* 1-based start */
    double nn_dist_sq; /* squared z-normalised ED to the nearest non-self match */
    double nn_dist;    /* sqrt(nn_dist_sq) */
} tsd_record;

/* Replaces tsdiscord::MerlinOptions (include/tsdiscord/merlin.hpp:32-38).
 * `workers` is accepted for source compatibility and ignored (the device
 * schedules itself; results never depend on it, as in the reference). */
typedef struct {
    int64_t top_k;       /* default 1 */
    int64_t seglen;      /* default 512; only validated, the device tiling is its own */
    int64_t workers;     /* default 1; ignored */
    int64_t max_retries; /* default 100 */
    int32_t reuse_stats; /* default 1: advance stats with Eq. 7-8 instead of recomputing */
} tsd_merlin_opts;

/* Per-run counters (device-side work accounting, for the roofline). */
typedef struct {
    uint64_t cells;         /* (candidate, subsequence) cells walked by the FP32 recurrence (2 FFMA) */
    uint64_t cells_eval;    /* of which evaluated against the threshold (+1 FMUL, +1 FMNMX) */
    uint64_t seed_dots;     /* directly seeded dot products (m FMAs each, FP64) */
    uint64_t seed_flops;    /* sum over seeds of 2*m */
    uint64_t rechecks;      /* knife-edge pairs resolved with the exact FP64 distance */
    uint64_t exact_pairs;   /* near-minimum pairs rebuilt exactly for survivors */
    uint64_t pardrag_calls; /* DRAG tries */
    uint64_t scan_launches; /* launches of the tile scan kernel */
    uint64_t kernel_launches; /* all kernel launches issued by the library */
    uint64_t host_syncs;    /* stream synchronisations (host round trips) */
    double scan_ms;         /* device time inside the scan kernel (CUDA events) */
    double dense_ms;        /* ... of which dense band phase */
    double sparse_ms;       /* ... of which sparse full-row phase */
    double collect_ms;      /* ... of which survivor near-pair collection */
    double total_ms;        /* device time of the last merlin/pardrag call (CUDA events) */
    double host_wall_ms;    /* host wall time inside DRAG tries */
    double host_wait_ms;    /* ... of which blocked in stream synchronisation */
    double heatmap_ms;      /* device time of the last heatmap column-max pass */
    uint64_t fallbacks;     /* tries that overflowed the knife-edge queue or the near-pair
                               buffer and finished with the exact pass over their live rows */
    uint64_t wit_tests;     /* rows that tested the kill witness of an earlier try */
    uint64_t wit_kills;     /* ... and were killed by it (before any walk) */
} tsd_counters;

/* ---- context ------------------------------------------------------------ */
int tsd_ctx_create(int device, tsd_ctx** out);
void tsd_ctx_destroy(tsd_ctx* ctx);
const char* tsd_last_error(const tsd_ctx* ctx); /* message of the last failing call */
/* Message of a failed tsd_ctx_create (no context to attach it to). */
const char* tsd_create_error(void);

/* Multi-GPU: join a segment-sharded group of `world` contexts (one process per
 * GPU).  `nccl_id` is the 128-byte ncclUniqueId produced by tsd_nccl_unique_id
 * on rank 0 and broadcast by the caller.  With world == 1 this is a no-op. */
int tsd_nccl_unique_id(uint8_t out[128]);
int tsd_ctx_join(tsd_ctx* ctx, int rank, int world, const uint8_t nccl_id[128]);

/* ---- series (replaces tsdiscord::TimeSeries, types.hpp:16-32) ------------
 * Validates n >= 3 and finiteness (src/types.cpp:8-13), uploads once. */
int tsd_series_set(tsd_ctx* ctx, const double* values, int64_t n);
int64_t tsd_series_len(const tsd_ctx* ctx);

/* ---- rolling statistics (stats.hpp:29,33; src/stats.cpp:7-58) -------------
 * init: Eq. 4 running sums for length m; mu/sigma receive n-m+1 values.
 * advance: Eq. 7-8 from length m to m+1 given mu/sigma of length m
 * (n-m+1 values in); writes n-m values.  Both run on the device and are
 * bit-identical to the reference's FP64 arithmetic. */
int tsd_init_stats(tsd_ctx* ctx, int64_t m, double* mu, double* sigma);
int tsd_advance_stats(tsd_ctx* ctx, int64_t m, const double* mu_in, const double* sigma_in,
                      double* mu_out, double* sigma_out);

/* ---- layout and threshold schedule (host arithmetic, bit-exact) ----------
 * compute_layout: src/types.cpp:26-39 -> out = {seglen, seg_n, num_seg, pad}.
 * next_threshold: src/merlin.cpp:35-55; phase 0 first, 1 warmup, 2 steady;
 * history = per-length minimal nn distances (unsquared). */
int tsd_compute_layout(int64_t n, int64_t m, int64_t seglen, int64_t out[4]);
int tsd_next_threshold(const double* history, int64_t history_len, int phase, int64_t min_len,
                       double last_r, int failed, double* out);

/* ---- PD3 range-discord scan (pardrag.hpp:87-93; src/pardrag.cpp:421-434) --
 * Returns every subsequence whose exact nearest-neighbour distance^2 is
 * >= r_sq, with that exact distance, sorted (nn desc, index asc).
 * `seglen` is validated with compute_layout exactly like the reference.
 * mu/sigma (nullable): caller-supplied stats for length m (n-m+1 values);
 * NULL means "compute init_stats(m) on the device".
 * *count receives the number of records; at most `cap` are written. */
int tsd_pardrag(tsd_ctx* ctx, int64_t m, double r_sq, int64_t seglen, const double* mu,
                const double* sigma, tsd_record* out, int64_t cap, int64_t* count);

/* ---- the two PD3 phases (pardrag.hpp:68-84; src/pardrag.cpp:339-419) -------
 * On the device a try is one stream-ordered sequence (band passes, full rows,
 * knife-edge recheck, exact nn), so the selection phase already decides every
 * row exactly.  par_select: cand[i] (N = n-m+1 entries) is 1 for every
 * subsequence with nn^2 >= r_sq (a candidate set with no false positives) and
 * nn[i] its exact nn^2 (+inf for pruned rows: the device keeps no partial
 * route minima).  par_refine: the records of the candidates still set in
 * `cand` (callers may clear entries between the phases, as
 * tests/pardrag_test.cpp:178-189 does), exact nn, sorted like sort_discords;
 * a candidate-free state returns no records without a device pass. */
int tsd_par_select(tsd_ctx* ctx, int64_t m, double r_sq, int64_t seglen, const double* mu,
                   const double* sigma, uint8_t* cand, double* nn);
int tsd_par_refine(tsd_ctx* ctx, int64_t m, double r_sq, int64_t seglen, const double* mu,
                   const double* sigma, const uint8_t* cand, tsd_record* out, int64_t cap,
                   int64_t* count);

/* ---- the tile deal of the multi-rank scan (host side, no device needed) ----
 * Decodes the tile slots rank `rank` of `world` fetches in one scan launch,
 * with the kernels' own decoder (tile_space.cuh): space 0 = band 0 at offset
 * kA over L-row blocks (nb sides, resident seeds), 1 = band [K0, K0+nb*1152)
 * over L-row blocks, 2 = the same band over `groups` (G pairs first,last row),
 * 3 = every diagonal |k| >= m of the groups (full rows).  out receives 5 ints
 * per tile {r0, rows, k0, dir, seed}; *count the tiles (at most cap written).
 * tests/test_multirank.py deals tiles to gloo ranks with it. */
int tsd_tile_plan(int space, int64_t N, int64_t m, int64_t L, int64_t kA, int64_t nb, int64_t K0,
                  const int32_t* groups, int64_t G, int rank, int world, int32_t* out, int64_t cap,
                  int64_t* count);

/* ---- MERLIN's length step, exposed for checking ----------------------------
 * stats_walk: init_stats(m0) on the device, then m1-m0 length steps exactly as
 * tsd_merlin runs them (fused != 0: the one-launch k_next_length step with the
 * resident seed rows at kA = m1 when they fit; 0: the plain Eq. 7-8 advance).
 * mu/sigma receive the n-m1+1 values of length m1 (src/stats.cpp:38-58 bit for
 * bit).  seed_rows: the resident rows (info = {m, L, kA, nb}; out, if cap >=
 * nb*1152, the raw dot products QT_m(i, i +- (kA+u)) row-major). */
int tsd_stats_walk(tsd_ctx* ctx, int64_t m0, int64_t m1, int fused, double* mu, double* sigma);
int tsd_seed_rows(tsd_ctx* ctx, double* out, int64_t cap, int64_t info[4]);

/* ---- MERLIN (merlin.hpp:50-54; src/merlin.cpp:57-137) ---------------------
 * Arrays have L = max_len-min_len+1 entries (recs: L*top_k, row-major).
 * counts[k]  records kept for length min_len+k (0 for failed lengths)
 * failed[k]  1 if the length is in failed_lengths
 * final_r[k], retries[k] as MerlinReport. */
int tsd_merlin(tsd_ctx* ctx, int64_t min_len, int64_t max_len, const tsd_merlin_opts* opts,
               int64_t* counts, tsd_record* recs, double* final_r, int64_t* retries,
               uint8_t* failed);

/* ---- exact nearest-neighbour profile on the device -----------------------
 * brute_force_nn (drag.hpp:38; src/drag.cpp:137-149): exact nn^2 of every
 * subsequence (n-m+1 values) with the reference arithmetic. */
int tsd_brute_force_nn(tsd_ctx* ctx, int64_t m, double* out);

/* ---- in-process rank group (single process, several GPUs) ----------------
 * The alternative to tsd_ctx_join + NCCL when one process drives several
 * devices: rank r owns devices[r] (repeats allowed: several ranks may share a
 * GPU, which is how the sharded path is tested on one device).  The scan tiles
 * are dealt cyclically over the ranks and the kill flags / route maxima /
 * exact-nn keys are all-reduced by one kernel per rank reading every rank's
 * buffer through peer memory.  Results equal the single-rank ones bit for bit;
 * the group entry points check that every rank produced the same records
 * (TSD_ERUNTIME "ranks diverged" otherwise). */
typedef struct tsd_group tsd_group;
int tsd_group_create(const int* devices, int n, tsd_group** out);
void tsd_group_destroy(tsd_group* g);
const char* tsd_group_last_error(const tsd_group* g);
int tsd_group_size(const tsd_group* g);
tsd_ctx* tsd_group_ctx(tsd_group* g, int rank); /* per-rank counters / params */
int tsd_group_series_set(tsd_group* g, const double* values, int64_t n);
int tsd_group_merlin(tsd_group* g, int64_t min_len, int64_t max_len, const tsd_merlin_opts* opts,
                     int64_t* counts, tsd_record* recs, double* final_r, int64_t* retries, uint8_t* failed);
int tsd_group_pardrag(tsd_group* g, int64_t m, double r_sq, int64_t seglen, tsd_record* out, int64_t cap,
                      int64_t* count);

/* ---- cross-process ranks over CUDA IPC (one process per GPU) ---------------
 * The fused peer-store transport of tsd_group_* between processes: every rank
 *  1. calls tsd_ipc_export(ctx, rows, h) after tsd_series_set (rows >= the series
 *     length; the shared kill-flag / row-max / exact-nn arrays are allocated
 *     once at that size) and gets 320 bytes of CUDA IPC handles;
 *  2. gathers all ranks' 320-byte blocks in rank order (e.g. all_gather_object);
 *  3. rank 0 calls tsd_ipc_join first (it creates the shared-memory barrier
 *     `shm_name`), then the others, with identical shm_name;
 *  4. runs tsd_merlin / tsd_pardrag with identical arguments on every rank.
 * Ranks may share a GPU.  tsd_ctx_join (NCCL) is the alternative transport. */
int tsd_ipc_export(tsd_ctx* ctx, int64_t rows, uint8_t out_handles[320]);
int tsd_ipc_join(tsd_ctx* ctx, int rank, int world, const uint8_t* all_handles, const char* shm_name);

/* ---- heatmap / ranking on the device (heatmap.hpp) ------------------------
 * One ranked column: replaces tsdiscord::RankedDiscord (include/tsdiscord/heatmap.hpp:35-39). */
typedef struct {
    int64_t index;  /* 1-based start index */
    int64_t length; /* length of the column maximum (smallest on ties) */
    double score;   /* nn_dist_sq / (2m) */
} tsd_ranked;

/* Builds the score matrix of a discord set on the device and keeps it there
 * (build_heatmap, src/heatmap.cpp:18-31; Heatmap(minL, maxL, n) preconditions
 * src/heatmap.cpp:10-15 -> TSD_EINVAL).  Records: `count` entries, lengths[e]
 * the discord length of recs[e]; a record whose index exceeds n-minL is
 * dropped, later duplicates of a cell win.  scores_out (nullable) receives the
 * (maxL-minL+1) x (n-minL) row-major matrix. */
int tsd_heatmap_build(tsd_ctx* ctx, int64_t min_len, int64_t max_len, int64_t n, const int64_t* lengths,
                      const tsd_record* recs, int64_t count, double* scores_out);
/* Replaces the device score matrix with a host one (same shape rules). */
int tsd_heatmap_set(tsd_ctx* ctx, int64_t min_len, int64_t max_len, int64_t n, const double* scores);
/* rank_discords (src/heatmap.cpp:33-57): per-column maximum over lengths on
 * the device, columns ordered by (score desc, index asc, length asc), at most
 * k, non-zero only.  k < 1 -> TSD_EINVAL.  `out` must hold min(k, n-minL). */
int tsd_heatmap_rank(tsd_ctx* ctx, int64_t k, tsd_ranked* out, int64_t* count);

/* ---- independent FP64 matrix profile (checker) ----------------------------
 * nn^2 of every subsequence (n-m+1 values, +inf without a non-self match) by
 * a different algorithm than the product path: the FP64 STOMP diagonal
 * recurrence over every cell, no pruning.  Agrees with brute_force_nn to
 * ~1e-10 relative; meant for parity checks at sizes where the reference's
 * O(N^2 m) brute_force_nn (src/drag.cpp:137-149) is out of reach. */
int tsd_matrix_profile_fp64(tsd_ctx* ctx, int64_t m, double* out);

/* ---- host utilities the reference API also exposes (io.hpp) --------------
 * gen_randomwalk: src/io.cpp:110-119 (libstdc++ mt19937_64 + normal_distribution). */
int tsd_gen_randomwalk(int64_t n, uint64_t seed, double* out);

/* ---- accounting ---------------------------------------------------------- */
int tsd_get_counters(const tsd_ctx* ctx, tsd_counters* out);
int tsd_reset_counters(tsd_ctx* ctx);
/* Diagnostic: FP32 FFMA throughput of `device` (TFLOP/s, 2 flops per FFMA),
 * measured with a dependent-chain-free FFMA loop over all SMs. */
int tsd_fp32_peak_probe(int device, double* tflops);
/* Tuning knobs (testing and tuning only).  Except err_scale, they change the
 * schedule, never the results.  Returns TSD_EINVAL for an unknown key.  Keys:
 *   dense_rows      rows per band-0 block (0: auto)
 *   sparse_rows     fixed group span (0: cost model)
 *   err_scale       err_k of the FP32 error bound (default 4; a smaller value
 *                   voids the bound's proof)
 *   band_passes     cap on band passes per try;  band_few / band_keep: break rule
 *   half_pass0, half_bands, half_bands_m   reduced-density evaluation patterns
 *                   (half_bands 20: the middle slot of every thread only, the
 *                   default; 2 / 3: every slot, 1 step in 2 / 3)
 *   pair_band0      paired both-sides band-0 walk for large series (1)
 *   band0_sides     sides of band 0 (2)
 *   seed_w          cost-model weight of a seed element vs a walked row
 *   seed32_track, seed32_collect           FP32 seeds in those launches
 *   track_chunks    tracked full-row chunks (1: one catch-all launch)
 *   witness         kill witnesses of earlier tries, tested right after band pass 0 (1)
 *   wit_cache       the witness test's run-seed cache (1)
 *   band_few_wit    with witnesses: band passes stop at this many rows (0: auto:
 *                   256 below N = 2^18, else few_lo from m = few_m on, else 64)
 *   few_m, few_lo   (512, 2)
 *   pass0_pk        band 0 walks every pair once, both ends killed (1)
 *   pk_min_n, pk_rows, half_pk   its minimum N, block rows (0: auto), pattern
 *                   (20: slot 0 of every thread, the default; 6 / 9: strides;
 *                   12, 16: three slots)
 *   row_cache, rc_min_m          resident full rows of anchors next to the
 *                   previous tries' survivors (1, from m = 384)
 *   dev_barrier     rank groups: device flag barriers (-1 auto, 0 host, 1 device)
 *   fused_peers     rank groups: peer stores inside the kernels (1)
 *   scan_events     bracket scans with events (per-phase timing; slower)
 *   result_prefix   records copied back with the try's single sync */
int tsd_set_param(tsd_ctx* ctx, const char* key, double value);

#ifdef __cplusplus
}
#endif
#endif
