// PD3 scan kernels for sm_100a (north_star (b), (c)).
//
// k_scan<MODE> is the hot path: persistent CTAs that fetch parallelogram tiles
// of the distance matrix (TileDesc) and replace the reference's per-segment
// scan_chunk loop (src/pardrag.cpp:157-282) with a B200 layout:
//   * seeds: the covariances of the tile's first row, from resident FP64 seed
//     rows carried across lengths (band 0), or as FP32 dot products over the
//     series staged in shared memory with their rounding in the error bound
//     (the reference seeds row+column per chunk, pardrag.cpp:162-182; a
//     parallelogram needs only the row);
//   * walk: every thread advances kDiag adjacent diagonals with the FP32
//     centered-covariance recurrence cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i
//     (2 FFMA per cell; the q-side operands slide through registers, the
//     c-side operand is a shared-memory broadcast);
//   * decision: x = cov * nrm_q is compared with the row's threshold
//     (corr > 1 - r^2/(2m) widened by the proven FP32 error bound).  Band
//     passes only make certain kills (aggregated per warp); the full rows also
//     queue knife-edge pairs for the exact FP64 recheck (the analogue of
//     pardrag.cpp:255) and track each row's maximum for its nn bounds.
// k_band0_pair walks both sides of a band-0 row block in one CTA on packed
// FP32x2 registers (FFMA2), with k_scan's per-side arithmetic.
// Kills are monotone byte stores, so the final state is schedule-independent.
//
// k_ref_pairs evaluates reference_sq_dist (pardrag.cpp:57-69 -> znormalize +
// sq_ed, distance.cpp:8-33) bit-exactly, one warp per pair: the reference's
// sequential sums stay sequential (lanes 0/1), only the element-wise loads and
// z-normalised terms are computed in parallel.
#include <float.h>
#include <limits.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "engine_internal.h"
#include "tile_space.cuh"

namespace tsd {

constexpr float kEps32 = 5.9604645e-08f;  // 2^-24
constexpr double kSlack = 1e-9;           // absolute corr slack around the threshold

// rows are padded to a multiple of kDiag (+1 for the one-step prefetch); padded
// rows carry zero operands (exact no-op increments) and are never evaluated
constexpr int kRowsPad = kMaxRows + kDiag + 1;
constexpr int kQPad = kMaxRows + kDiag + kW + kDiag;

// Per-mode shared memory: the band passes need neither the collection
// thresholds nor the row-max keys, which frees 4 KB per CTA (6 band-pass CTAs per
// SM fit at 80 registers; 7 were measured slower).
template <int MODE>
struct __align__(16) ScanSmem {
    float4 crow[kRowsPad];                           // per row: {cdf, cdg, tc, cn}
    float cy[MODE == kCollect ? kRowsPad : 1];       // kCollect: per-row collection threshold
    unsigned ykey[MODE == kPruneTrack ? kRowsPad : 1];  // kPruneTrack: row max keys
    union {
        struct {
            float2 qd[kQPad];  // (df, dg) of the q side
            float qn[kQPad];   // norm of the q side (NaN: invalid q)
        } walk;
        struct {
            double a[kSeedChunk];
            double win[kW + kSeedChunk];
        } seed;
        struct {
            float a[kSeedChunk];
            float win[kW + kSeedChunk];
        } seed32;
    } u;
    float red[7][kThreads / 32];
    int flag[2];
    int2 span[2][kThreads / 32];  // per warp: first / last undecided row of the tile (double-buffered)
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ TileCtx load_ctx(const ScanParams& p) {
    const TryCtl* ctl = p.ctl;
    TileCtx c{0, 0, 0, 0};
    switch (p.space) {
        case kSpaceSeed: c.slots = (long long)p.nb * ((p.N + p.L - 1) / p.L); break;  // nb = sides (1 or 2)
        case kSpaceBlocks:
            c.G = (p.N + p.L - 1) / p.L;
            c.slots = 2ll * p.nb * c.G;
            c.k0 = p.K0;
            break;
        case kSpaceBand:
            c.G = ctl->G;
            c.k0 = ctl->bK0;
            c.slots = ctl->stop < p.pass ? 0 : 2ll * ctl->bnb * c.G;
            break;
        case kSpaceTrack:
            c.G = ctl->G;
            c.k0 = ctl->tK0;
            c.slots = ctl->tphase >= 2 ? 0 : 2ll * ctl->tnb * c.G;
            break;
        case kSpaceTrackRest: {
            // bands left for the catch-all: the far rest [tK0, N) when the far
            // chunks are unfinished, and the near chunk [m, kend) unless it ran
            const long long k_max = (long long)p.N - 1;
            long long nf = 0, nn = 0;
            const int ph = ctl->tphase;
            if (ph == 0) {
                if ((long long)ctl->tK0 <= k_max) nf = (k_max - ctl->tK0 + kW) / kW;
                if (ctl->kend > p.m) nn = ((long long)ctl->kend - p.m + kW - 1) / kW;
            } else if (ph == 1) {
                nn = ctl->tnb;  // the pending near chunk starts at m
            }
            c.G = ctl->G;
            c.nf = nf;
            c.k0 = ctl->tK0;
            c.slots = 2ll * (nf + nn) * c.G;
            break;
        }
        default: {  // full rows: the farthest group needs ceil((N - m) / kW) tiles a side
            c.G = ctl->G;
            const long long maxc = ((long long)p.N - p.m + kW - 1) / kW;
            c.slots = maxc > 0 ? 2ll * maxc * c.G : 0;
        }
    }
    return c;
}

struct F9 {
    float v[kDiag];
};

// Full-row slow path of one walk step (row c, diagonals u0 .. u0+kDiag-1): the
// exact constant conventions, certain kills of the row candidate and knife-edge
// pairs for the FP64 recheck.  Only the row candidate is killed (the pair's
// other end is decided by its own row), so a decided row never re-enters.
// Kept out of line: it runs on a few steps only and would otherwise bloat the
// unrolled walk.
__device__ __noinline__ void slow_track(const F9 x, const F9 qn, float tz, float cw, int c, int u0, int dir,
                                        int qbase, int N, int m, double r_sq, double thr0, double E, double xs,
                                        uint8_t* alive, uint8_t* const* peer_alive, int npeer, int2* queue,
                                        int* queue_count, int queue_cap, int* wit) {
    double best = 0.0;  // largest kill margin of this call (its diagonal becomes the witness)
    int best_q = -1;
#pragma unroll
    for (int j = 0; j < kDiag; ++j) {
        if (!(x.v[j] > tz)) continue;
        const int u = u0 + j;
        const int q = dir > 0 ? qbase + u : qbase - u;
        if (q < 0 || q >= N) continue;
        const float qj = qn.v[j];
        if (cw == 0.f || qj == 0.f) {
            const double d = (cw == 0.f && qj == 0.f) ? 0.0 : 2.0 * (double)m;
            if (d < r_sq) {
                if (npeer > 1) for (int r = 0; r < npeer; ++r) peer_alive[r][c] = 0;
                else alive[c] = 0;
            }
            continue;
        }
        const double corr = (double)x.v[j] * (double)cw;
        const double ec = E * (double)cw * (double)qj + kSlack + xs;
        if (corr - ec > thr0) {
            if (npeer > 1) for (int r = 0; r < npeer; ++r) peer_alive[r][c] = 0;
            else alive[c] = 0;
            if (corr - ec - thr0 > best) {
                best = corr - ec - thr0;
                best_q = q;
            }
        } else if (corr + ec >= thr0) {
            const int at = atomicAdd(queue_count, 1);
            if (at < queue_cap) queue[at] = make_int2(c, q);
        }
    }
    if (wit && best_q >= 0) wit[c] = best_q - c - kDiag / 2;  // the killer in the middle of the next try's 9
}

// FP64 direct seeds: cov(c_first, q) for this thread's kDiag diagonals, q =
// qbase + u (dir > 0) or qbase - u (dir < 0), u = tid*kDiag + j.
// cov = sum_p (t[c+p]-mu_c) t[q+p] - mu_q * sum_p (t[c+p]-mu_c).  sa / swin:
// shared scratch of kSeedChunk and kW + kSeedChunk doubles; every thread of
// the CTA calls it (it synchronises).
__device__ __forceinline__ void seed_fp64(const ScanParams& p, int c_first, int qbase, int dir, double* sa,
                                          double* swin, float (&cov)[kDiag]) {
    const int tid = threadIdx.x;
    const int N = p.N, m = p.m;
    const int qlo = dir > 0 ? qbase : qbase - (kW - 1);
    const int o_t = dir > 0 ? tid * kDiag : kW - kDiag - tid * kDiag;  // lowest window offset
    double acc[kDiag];
#pragma unroll
    for (int i = 0; i < kDiag; ++i) acc[i] = 0.0;
    double delta = 0.0;
    const double mu_c = p.mu[c_first];
    for (int pc = 0; pc < m; pc += kSeedChunk) {
        const int len = min(kSeedChunk, m - pc);
        __syncthreads();
#pragma unroll 4
        for (int x = tid; x < len; x += kThreads) sa[x] = p.t[c_first + pc + x] - mu_c;
#pragma unroll 4
        for (int x = tid; x < kW + len - 1; x += kThreads) {
            const int g = qlo + pc + x;
            swin[x] = (g >= 0 && g < p.n) ? p.t[g] : 0.0;
        }
        __syncthreads();
        double w[kDiag];
#pragma unroll
        for (int i = 0; i < kDiag - 1; ++i) w[i] = swin[o_t + i];
        int pp = 0;
        for (; pp + kDiag <= len; pp += kDiag) {
#pragma unroll
            for (int uu = 0; uu < kDiag; ++uu) {
                // ring: window value for offset o_t + pp + uu + i lives in w[(uu + i) % kDiag]
                w[(uu + kDiag - 1) % kDiag] = swin[o_t + pp + uu + kDiag - 1];
                const double av = sa[pp + uu];
                delta += av;
#pragma unroll
                for (int i = 0; i < kDiag; ++i) acc[i] = fma(av, w[(uu + i) % kDiag], acc[i]);
            }
        }
        for (; pp < len; ++pp) {
            const double av = sa[pp];
            delta += av;
#pragma unroll
            for (int i = 0; i < kDiag; ++i) acc[i] = fma(av, swin[o_t + pp + i], acc[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < kDiag; ++i) {
        const int q = qlo + o_t + i;
        acc[i] = (q >= 0 && q < N) ? acc[i] - p.mu[q] * delta : 0.0;
    }
    if (dir > 0) {
#pragma unroll
        for (int j = 0; j < kDiag; ++j) cov[j] = (float)acc[j];
    } else {
#pragma unroll
        for (int j = 0; j < kDiag; ++j) cov[j] = (float)acc[kDiag - 1 - j];
    }
}

// Band-pass evaluation pattern: cell (slot j, step uu) of the thread's 9
// diagonals.  STRIDE 2 / 3: (j + step) % STRIDE, every slot.  STRIDE 20: the
// middle slot only, every step -- every 9th diagonal of the band, each fully;
// the other 8 slots are never read, so the compiler drops their walks AND their
// m-long seeds (the middle slot reads the same seed on both sides).
template <int STRIDE>
__device__ __forceinline__ constexpr bool scan_sampled(int j, int uu) {
    return STRIDE == 20 ? j == kDiag / 2 : (j + uu) % STRIDE == 0;
}
template <int STRIDE>
__device__ __forceinline__ constexpr int scan_walked_slots() {
    return STRIDE == 20 ? 1 : kDiag;
}
template <int STRIDE>
__device__ __forceinline__ constexpr int scan_evals_per_row() {  // per thread-slice of 9 diagonals, x kThreads / 9
    int n = 0;
    for (int j = 0; j < kDiag; ++j)
        for (int uu = 0; uu < kDiag; ++uu) n += scan_sampled<STRIDE>(j, uu) ? 1 : 0;
    return n * kThreads / kDiag;
}

template <int MODE, int STRIDE = 1>
__global__ void __launch_bounds__(kThreads, MODE == kPruneTrack ? 4 : 6) k_scan(const ScanParams p) {
    pdl_enter();
    // static shared memory (33 KB): CTA-relative LDS addressing, no shared
    // window base to rematerialise inside the walk
    __shared__ ScanSmem<MODE> S;
    __shared__ uint8_t* s_peer_alive[kMaxPeers];  // slow path: peer pointers without a param copy
    if (threadIdx.x < kMaxPeers) s_peer_alive[threadIdx.x] = p.peers.alive[threadIdx.x];
    const int tid = threadIdx.x;
    const TileCtx cx = load_ctx(p);
    const long long slots = cx.slots;
    // persistent CTAs: slots are fetched dynamically; rank r owns slots r, r+world, ...
    const long long mine = p.world > 1 ? (slots > p.rank ? (slots - p.rank + p.world - 1) / p.world : 0) : slots;
    // first round static (CTA b takes slot b: the hardware spreads consecutive
    // CTAs over the SMs, so a launch with fewer tiles than CTAs stays balanced),
    // then dynamic.  Per slot, the next slot's fetch, the decode and the
    // all-decided test overlap and share one barrier, which also retires the
    // previous tile's shared memory; the fetched slot lands in S.flag[par],
    // which is not rewritten before the next iteration's barrier.
    int par = 0;
    for (long long f = blockIdx.x;; par ^= 1) {
    if (f >= mine) break;
    if (tid == 0) S.flag[par] = atomicAdd(p.next, 1);
    TileDesc td;
    const bool valid = tile_decode(p, cx, f * p.world + p.rank, td);
    bool work;
    if (MODE == kCollect || p.space == kSpaceSeed) {
        int any = 0;
        if (valid) {  // tiles whose rows are all decided are skipped
            if (MODE == kCollect && p.ub != nullptr) {
                // ... and so are bands that cannot hold any of its rows' nearest
                // neighbours: the full-row stage's upper bound of corr over the
                // band is below the row's lower bound of its best corr
                const int nbands = ub_nbands(p.N, p.m);
                const long long nlist = p.ctl->alive;
                const bool ub_on = nlist * 2 * nbands <= p.ub_cap;
                const int kf = td.dir > 0 ? td.k0 : -(td.k0 + kW - 1);
                const int b = (kf - p.m) / kW;
                const unsigned long long etag = (unsigned long long)p.ctl->tepoch << 32;
                for (int s = tid; s < td.rows; s += kThreads) {
                    const int c = td.r0 + s;
                    if (!p.alive[c]) continue;
                    const float th = p.ythr[c];
                    if (th == FLT_MAX) continue;  // not a collection row
                    bool need = true;
                    if (ub_on && b >= 0 && b < nbands) {
                        const unsigned long long v =
                            p.ub[((long long)p.exli[c] * 2 + (td.dir < 0)) * nbands + b];
                        if ((v & 0xffffffff00000000ull) == etag) {
                            const float lb = th * p.nrm[c];  // corr lower bound of the row's best q
                            need = key2f((unsigned)v) >= lb - fabsf(lb) * 4.8e-7f - 1e-7f;
                        }
                    }
                    any |= need;
                }
            } else {
                for (int s = tid; s < td.rows; s += kThreads) any |= p.alive[td.r0 + s];
            }
        }
        work = __syncthreads_or(any);
    } else {
        // directly seeded tiles shrink to their first..last undecided row:
        // rows only die, and the seed is taken at the new first row
        int lo = INT_MAX, hi = -1;
        if (valid)
            for (int s = tid; s < td.rows; s += kThreads)
                if (p.alive[td.r0 + s]) {
                    lo = min(lo, s);
                    hi = s;
                }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if ((tid & 31) == 0) S.span[par][tid >> 5] = make_int2(lo, hi);
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
            lo = min(lo, S.span[par][w].x);
            hi = max(hi, S.span[par][w].y);
        }
        work = hi >= 0;
        if (work) {
            td.r0 += lo;
            td.rows = hi - lo + 1;
        }
    }
    f = (long long)S.flag[par] + gridDim.x;
    if (p.dbg && tid == 0) {
        if (valid) atomicAdd(&p.dbg[2 * MODE], 1ull);
        if (work) atomicAdd(&p.dbg[2 * MODE + 1], 1ull);
    }
    if (!work) continue;
#ifdef TSD_TILE_TIMING
    const long long t_start = (MODE == kCollect && p.dbg) ? clock64() : 0;
#endif
    // Row cache (full rows / collection): a resident raw QT row of an anchor
    // row at most min(m/2, room) rows before the tile's first row (dir > 0) or
    // after its last (dir < 0) replaces the tile's m-long direct seeds; the
    // `ext` rows in between are only walked (2 FFMA per cell: cheaper than
    // a seed while ext < m/2)
    int rc = -1, ext = 0;
    if (MODE != kPrune && p.rc_n > 0) {
        const int gap = min(p.m / 2, kMaxRows - td.rows);
        for (int s2 = 0; s2 < p.rc_n; ++s2) {
            const int ar = p.rc_row[s2];
            if (ar < 0) continue;  // empty slot
            const int d = td.dir > 0 ? td.r0 - ar : ar - (td.r0 + td.rows - 1);
            if (d >= 0 && d <= gap && (rc < 0 || d < ext)) {
                rc = s2;
                ext = d;
            }
        }
        if (rc >= 0) {
            if (td.dir > 0) td.r0 -= ext;
            td.rows += ext;
        } else {
            ext = 0;
        }
    }
    if (MODE == kPruneTrack && p.dbg && tid == 0) {
        atomicAdd(&p.dbg[rc >= 0 ? 8 : (td.seed >= 0 ? 11 : 9)], 1ull);
        atomicAdd(&p.dbg[10], (unsigned long long)td.rows);
    }
    const int rows = td.rows;
    const int dir = td.dir;
    const int N = p.N;
    const int m = p.m;
    const int r_end = td.r0 + rows - 1;
    const int c_first = dir > 0 ? td.r0 : r_end;
    // local q coordinate u: step s, slot j of thread t sits at u = s + t*kDiag + j
    const int qbase = dir > 0 ? td.r0 + td.k0 : r_end + td.k0 + kW - 1;
    const int nq = rows - 1 + kW;


    // ---- 1. seeds: cov(c_first, q) for this thread's kDiag diagonals --------
    float cov[kDiag];
    double e_seed = 0.0;  // absolute error bound of FP32 seeds (0 for FP64 / resident seeds)
    if (rc >= 0) {
        // row-cache anchor: QT(c_first, q) for every q, carried across lengths
        // like the band-0 rows (k_rc_advance): cov = QT - m mu_c mu_q
        const double* qt = p.rcqt + (size_t)rc * (size_t)p.rc_stride;
        const double mmu = (double)m * p.mu[c_first];
#pragma unroll
        for (int j = 0; j < kDiag; ++j) {
            const int u = tid * kDiag + j;
            const int q = dir > 0 ? qbase + u : qbase - u;
            cov[j] = (q >= 0 && q < N) ? (float)(qt[q] - mmu * p.mu[q]) : 0.f;
        }
    } else if (td.seed >= 0) {
        // resident seed row, carried across lengths by the dot-product length
        // recurrence (k_seed_advance): cov = QT - m mu_c mu_q
        const double* qt = p.seedqt + (size_t)td.seed * kW + tid * kDiag;
        const double mmu = (double)m * p.mu[c_first];
#pragma unroll
        for (int j = 0; j < kDiag; ++j) {
            const int u = tid * kDiag + j;
            const int q = dir > 0 ? qbase + u : qbase - u;
            cov[j] = (q >= 0 && q < N) ? (float)(qt[j] - mmu * p.mu[q]) : 0.f;
        }
    } else if (MODE == kPrune || p.seed32) {
        // band passes only make certain kills, so their seeds may be FP32: the
        // rounding of a = t[c+p]-mu_c, w = t[q+p]-anchor and of the m-term sums is
        // bounded by E_seed (added to the tile's error bound below)
        const int qlo = dir > 0 ? qbase : qbase - (kW - 1);
        const int o_t = dir > 0 ? tid * kDiag : kW - kDiag - tid * kDiag;
        const int qmid = min(max(qlo + kW / 2, 0), N - 1);
        const double anchor = p.mu[qmid];
        const double mu_c = p.mu[c_first];
        float acc[kDiag];
#pragma unroll
        for (int i = 0; i < kDiag; ++i) acc[i] = 0.f;
        float wmax = 0.f;
        // sum_p (t[c+p] - mu_c) exactly from the double-double prefix sums (no
        // FADD per element in the loop; its rounding, ~u (|S_c| + m |mu_c|), is
        // orders below kSlack in correlation units)
        const double2 pc1 = p.pfx1[c_first + m], pc0 = p.pfx1[c_first];
        const double delta = ((pc1.x - pc0.x) + (pc1.y - pc0.y)) - (double)m * mu_c;
        for (int pc = 0; pc < m; pc += kSeedChunk) {
            const int len = min(kSeedChunk, m - pc);
            __syncthreads();
#pragma unroll 4
            for (int x = tid; x < len; x += kThreads) S.u.seed32.a[x] = (float)(p.t[c_first + pc + x] - mu_c);
#pragma unroll 4
            for (int x = tid; x < kW + len - 1; x += kThreads) {
                const int g = qlo + pc + x;
                const float w = (g >= 0 && g < p.n) ? (float)(p.t[g] - anchor) : 0.f;
                S.u.seed32.win[x] = w;
                wmax = fmaxf(wmax, fabsf(w));
            }
            __syncthreads();
            float w[kDiag];
#pragma unroll
            for (int i = 0; i < kDiag - 1; ++i) w[i] = S.u.seed32.win[o_t + i];
            int pp = 0;
            // 18 elements per iteration: the broadcast row values as 9 float2
            // loads (pp stays a multiple of 18, so 8-byte aligned)
            for (; pp + 2 * kDiag <= len; pp += 2 * kDiag) {
                float2 a2[kDiag];
#pragma unroll
                for (int i = 0; i < kDiag; ++i) a2[i] = reinterpret_cast<const float2*>(S.u.seed32.a + pp)[i];
#pragma unroll
                for (int uu = 0; uu < 2 * kDiag; ++uu) {
                    w[(uu + kDiag - 1) % kDiag] = S.u.seed32.win[o_t + pp + uu + kDiag - 1];
                    const float av = (uu & 1) ? a2[uu >> 1].y : a2[uu >> 1].x;
#pragma unroll
                    for (int i = 0; i < kDiag; ++i) acc[i] = fmaf(av, w[(uu + i) % kDiag], acc[i]);
                }
            }
            for (; pp < len; ++pp) {
                const float av = S.u.seed32.a[pp];
#pragma unroll
                for (int i = 0; i < kDiag; ++i) acc[i] = fmaf(av, S.u.seed32.win[o_t + pp + i], acc[i]);
            }
        }
        wmax = warp_max(wmax);
        if ((tid & 31) == 0) S.red[0][tid >> 5] = wmax;
        __syncthreads();
        wmax = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < kThreads / 32; ++w2) wmax = fmaxf(wmax, S.red[0][w2]);
        // |seed error| <= (m + 4) eps * sum|a| * wmax, sum|a| <= m sigma_c
        e_seed = (double)(m + 4) * (double)kEps32 * (double)m * p.sig[c_first] * (double)wmax;
        double seedv[kDiag];
#pragma unroll
        for (int i = 0; i < kDiag; ++i) {
            const int q = qlo + o_t + i;
            seedv[i] = (q >= 0 && q < N) ? (double)acc[i] - (p.mu[q] - anchor) * delta : 0.0;
        }
        if (dir > 0) {
#pragma unroll
            for (int j = 0; j < kDiag; ++j) cov[j] = (float)seedv[j];
        } else {
#pragma unroll
            for (int j = 0; j < kDiag; ++j) cov[j] = (float)seedv[kDiag - 1 - j];
        }
    } else {
        seed_fp64(p, c_first, qbase, dir, S.u.seed.a, S.u.seed.win, cov);
    }
    __syncthreads();  // seed buffers are reused below

    // ---- 2. stage the walk operands ---------------------------------------
    // Every iteration's global loads are independent (no load behind a
    // branch on another load) and the loops are unrolled, so a thread keeps
    // several loads in flight: the prologue is latency-bound otherwise.  The
    // largest sigma of each side comes from the smallest non-zero norm,
    // sigma = 1/(sqrt(m) nrm) up to the FP32 rounding of nrm (factor below).
    float cn_min = FLT_MAX, qn_min = FLT_MAX, qn_max = 0.f;
    float dc = 0.f, gc = 0.f, dq = 0.f, gq = 0.f;  // max |df|, |dg| walked on each side
#pragma unroll 4
    for (int s = tid; s < rows; s += kThreads) {
        const int c = dir > 0 ? td.r0 + s : r_end - s;
        const int ci = dir > 0 ? c : min(c + 1, N - 1);  // s == 0 takes no increment
        float4 v;
        const float a = p.df[ci], b = p.dg[ci];
        v.x = s == 0 ? 0.f : (dir > 0 ? a : -a);
        v.y = s == 0 ? 0.f : (dir > 0 ? b : -b);
        v.w = p.nrm[c];
        v.z = 0.f;
        if (v.w != 0.f) cn_min = fminf(cn_min, v.w);
        dc = fmaxf(dc, fabsf(v.x));
        gc = fmaxf(gc, fabsf(v.y));
        S.crow[s] = v;
    }
    const int rows_p = (rows + kDiag - 1) / kDiag * kDiag;
    for (int s = rows + tid; s <= rows_p; s += kThreads) S.crow[s] = make_float4(0.f, 0.f, FLT_MAX, 0.f);
#pragma unroll 4
    for (int u = tid; u < rows_p + kW + kDiag; u += kThreads) {
        const int q = dir > 0 ? qbase + u : qbase - u;
        const bool valid = u < nq && q >= 0 && q < N;
        const int qc = valid ? q : 0;
        const int qi = dir > 0 ? qc : min(qc + 1, N - 1);
        float a = p.df[qi], b = p.dg[qi];
        const float nn = p.nrm[qc];
        if (!valid || (dir < 0 && qc + 1 >= N)) {
            a = 0.f;
            b = 0.f;
        }
        if (valid && nn != 0.f) {
            qn_min = fminf(qn_min, nn);
            qn_max = fmaxf(qn_max, nn);
        }
        dq = fmaxf(dq, fabsf(a));
        gq = fmaxf(gq, fabsf(b));
        S.u.walk.qd[u] = make_float2(a, b);
        // an invalid q gets a NaN norm: its x = cov*qn is NaN, which never passes a
        // threshold test and is ignored by fmaxf (a constant q keeps qn = 0, x = 0)
        // (a degenerate q, sigma < eps, is NaN too: its reference distances are
        // not what the FP32 model predicts, every pair with it is decided exactly)
        S.u.walk.qn[u] = (valid && nn != 0.f) ? nn : __int_as_float(0x7fffffff);
    }
    cn_min = -warp_max(-cn_min);
    qn_min = -warp_max(-qn_min);
    qn_max = warp_max(qn_max);
    dc = warp_max(dc);
    gc = warp_max(gc);
    dq = warp_max(dq);
    gq = warp_max(gq);
    if ((tid & 31) == 0) {
        S.red[0][tid >> 5] = cn_min;
        S.red[1][tid >> 5] = qn_min;
        S.red[2][tid >> 5] = qn_max;
        S.red[3][tid >> 5] = dc;
        S.red[4][tid >> 5] = gc;
        S.red[5][tid >> 5] = dq;
        S.red[6][tid >> 5] = gq;
    }
    __syncthreads();
    cn_min = FLT_MAX;
    qn_min = FLT_MAX;
    qn_max = 0.f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        cn_min = fminf(cn_min, S.red[0][w]);
        qn_min = fminf(qn_min, S.red[1][w]);
        qn_max = fmaxf(qn_max, S.red[2][w]);
        dc = fmaxf(dc, S.red[3][w]);
        gc = fmaxf(gc, S.red[4][w]);
        dq = fmaxf(dq, S.red[5][w]);
        gq = fmaxf(gq, S.red[6][w]);
    }
    const double inv_sqm = 1.0 / sqrt((double)m);
    const double smax_c = cn_min < FLT_MAX ? inv_sqm / (double)cn_min * (1.0 + 1e-6) : 0.0;
    const double smax_q = qn_min < FLT_MAX ? inv_sqm / (double)qn_min * (1.0 + 1e-6) : 0.0;
    // Absolute FP32 covariance error bound for every cell of this tile.  One
    // walk step is two FFMA on FP32-rounded operands: rounding <= u(|a| + |b|)
    // with |a|, |b| <= m smax_c smax_q (Cauchy-Schwarz) + the increment, and the
    // operands' own rounding <= 2u per product, so one step errs by at most
    // u (2 m smax_c smax_q + 3 P), P = max|df_c||dg_q| + max|df_q||dg_c| over the
    // walked rows and q.  err_k = 4 doubles that first-order bound (margin for
    // second-order terms and the FP64 statistics' rounding) over rows + 8 steps;
    // e_seed bounds the seed (0 for FP64 / resident seeds).
    const double P = (double)dc * (double)gq + (double)dq * (double)gc;
    const double E =
        p.err_k * (double)kEps32 * (double)(rows + 8) * ((double)m * smax_c * smax_q + 1.5 * P) + e_seed;
    const float Ef = (float)E;
    // statistics error of this length (correlation units; resident raw seeds add theirs)
    const double xs = stats_band(p, td.seed >= 0 || rc >= 0);
    // Row thresholds.  crow.z = tc: a live row's cells with x = cov*qn > tc may be
    // within the error band of d^2 = r^2 (slow path); kNoEval marks rows whose
    // cells are only walked (already decided, or not a survivor in kCollect).
    constexpr float kNoEval = FLT_MAX;
    int evals = 0;
    for (int s = tid; s < rows; s += kThreads) {
        const int c = dir > 0 ? td.r0 + s : r_end - s;
        const float cn = S.crow[s].w;
        const bool live = s >= ext && p.alive[c] != 0;  // anchor rows before the tile: walked only
        float tc;
        if (MODE == kCollect) {
            // the row's best lower bound, lowered by the statistics band (x units)
            S.cy[s] = (live && cn != 0.f) ? p.ythr[c] - (float)(xs / (double)cn) * (1.f + 2.4e-7f) : FLT_MAX;
            tc = S.cy[s] < FLT_MAX ? 0.f : kNoEval;
        } else if (!live) {
            tc = kNoEval;
        } else if (cn == 0.f) {
            // degenerate row (sigma < eps): decided exactly against every q
            // (k_recheck), never by the FP32 walk
            tc = kNoEval;
        } else if (MODE == kPrune) {
            // band passes only make certain kills: every cell with x > tk has
            // corr - eps_cell > thr0 (eps_cell <= eps_row); knife edges are left
            // to the full-row pass
            const double eps_row = E * (double)cn * (double)qn_max + kSlack + 8.0 * (double)kEps32 + xs;
            const double tk = (p.thr0 + eps_row) / (double)cn;
            tc = (float)tk;
            tc = tc + fabsf(tc) * 2.4e-7f;  // round toward +inf (conservative)
        } else {
            const double eps_row = E * (double)cn * (double)qn_max + kSlack + 8.0 * (double)kEps32 + xs;
            tc = (float)((p.thr0 - eps_row) / (double)cn);
            tc = tc - fabsf(tc) * 2.4e-7f;  // round toward -inf (conservative)
        }
        S.crow[s].z = tc;
        evals += tc != kNoEval;
        if (MODE == kPruneTrack) S.ykey[s] = (live && cn != 0.f) ? 1u : 0u;  // 0 = untracked
    }
    evals = __syncthreads_count(evals);

    // ---- 3. walk ----------------------------------------------------------
    // Step s: row c(s) against q(u), u = s + t*kDiag + j.  The q-side operands of
    // slot j at step s live in ring[(j + s) % kDiag]; rows are padded so the
    // loop runs in whole kDiag blocks with compile-time ring indices and no
    // bounds checks.  Step 0 carries zero row operands (no increment).
    float2 rd[kDiag];
    float rn[kDiag];
    const int ub = tid * kDiag;
    const float2* qdp = S.u.walk.qd + ub;
    const float* qnp = S.u.walk.qn + ub;
    const float4* crp = S.crow;
#pragma unroll
    for (int j = 0; j < kDiag; ++j) {
        rd[j] = qdp[j];
        rn[j] = qnp[j];
    }
    const int lane = tid & 31;

    float4 cr_next = crp[0];  // row operands are prefetched one step ahead
    for (int s0 = 0; s0 < rows_p; s0 += kDiag) {
        unsigned hit = 0u;  // kPrune: steps of this block whose row is certainly killed
#pragma unroll
        for (int uu = 0; uu < kDiag; ++uu) {
            const int ss = s0 + uu;
            const float4 cr = cr_next;
            cr_next = crp[ss + 1];
#pragma unroll
            for (int j = 0; j < kDiag; ++j) {
                const int rj = (j + uu) % kDiag;
                cov[j] = fmaf(cr.x, rd[rj].y, cov[j]);
                cov[j] = fmaf(rd[rj].x, cr.y, cov[j]);
            }
            if (MODE == kPrune) {
                // band passes evaluate every step branch-free: a decided row has
                // tc = kNoEval (never exceeded), and the kill stores wait for the
                // end of the 9-step block.  The max is a depth-2 FMNMX3 tree.
                float x[kDiag];
                float mx;
                if (STRIDE > 1) {
                    // reduced-density evaluation: cell (step, j) only when
                    // (j + step) % STRIDE == 0, so each row tests 1/STRIDE of its
                    // band.  Kills stay certain; a row missed here is walked again
                    // by the next pass.  The walk (2 FFMA per cell) is unchanged.
                    mx = -FLT_MAX;
#pragma unroll
                    for (int j = 0; j < kDiag; ++j)
                        if (scan_sampled<STRIDE>(j, uu)) mx = fmaxf(mx, cov[j] * rn[(j + uu) % kDiag]);
                } else {
#pragma unroll
                    for (int j = 0; j < kDiag; ++j) x[j] = cov[j] * rn[(j + uu) % kDiag];
                    mx = fmaxf(fmaxf(fmaxf(fmaxf(x[0], x[1]), x[2]), fmaxf(fmaxf(x[3], x[4]), x[5])),
                               fmaxf(fmaxf(x[6], x[7]), x[8]));
                }
                hit |= (mx > cr.z ? 1u : 0u) << uu;
            } else if (cr.z != kNoEval) {  // CTA-uniform branch: the row is undecided
                float x[kDiag];
                float mx = -FLT_MAX;
#pragma unroll
                for (int j = 0; j < kDiag; ++j) {
                    x[j] = cov[j] * rn[(j + uu) % kDiag];
                    mx = fmaxf(mx, x[j]);
                }
                if (MODE == kPruneTrack) {
                    if (mx > cr.z) {
                        // rare: kills, knife edges, constant conventions (out of line)
                        F9 xv, qv;
#pragma unroll
                        for (int j = 0; j < kDiag; ++j) {
                            xv.v[j] = x[j];
                            qv.v[j] = rn[(j + uu) % kDiag];
                        }
                        slow_track(xv, qv, cr.z, cr.w, dir > 0 ? td.r0 + ss : r_end - ss, ss + ub, dir, qbase, N,
                                   m, p.r_sq, p.thr0, E, xs, p.alive, s_peer_alive, p.peers.n, p.queue,
                                   p.queue_count, p.queue_cap, p.wit);
                    }
                    if (S.ykey[ss] != 0u) {
                        // row max of the FP32 route value x = cov*qn over valid q (NaN for
                        // invalid q is ignored by fmaxf; a constant q contributes exactly
                        // 0); the tile's error term E*qn_max is folded in at the end
                        // (keys are order-preserving and mx is never NaN: one REDUX
                        // gives the key of the warp max)
                        const unsigned yk = __reduce_max_sync(0xffffffffu, f2key(mx));
                        if (lane == 0 && yk > f2key(-FLT_MAX)) atomicMax(&S.ykey[ss], yk);
                    }
                }
                if (MODE == kCollect) {
                    const float th = S.cy[ss];
                    const int c = dir > 0 ? td.r0 + ss : r_end - ss;
#pragma unroll
                    for (int j = 0; j < kDiag; ++j) {
                        // upper bound (cov + E) * qn reaches the row's best lower bound
                        // (NaN for an invalid q fails the comparison)
                        if (fmaf(Ef, rn[(j + uu) % kDiag], x[j]) >= th) {
                            const int u = ss + ub + j;
                            const int q = dir > 0 ? qbase + u : qbase - u;
                            const int at = atomicAdd(p.coll_count, 1);
                            if (at < p.coll_cap) p.coll[at] = make_int2(c, q);
                        }
                    }
                }
            }
            // slide: slot kDiag-1 of step ss+1 is u = ss + 1 + ub + kDiag - 1
            rd[uu % kDiag] = qdp[ss + kDiag];
            rn[uu % kDiag] = qnp[ss + kDiag];
        }
        if (MODE == kPrune) {
            // certain kills of the row candidates (FP32 only), warp-aggregated:
            // lane b stores the row of step s0 + b if any lane killed it
            const unsigned h = __reduce_or_sync(0xffffffffu, hit);
            if (lane < kDiag && ((h >> lane) & 1u)) {
                const int ss = s0 + lane;
                peer_kill(p.peers, p.alive, dir > 0 ? td.r0 + ss : r_end - ss);
            }
            if (p.wit != nullptr && hit != 0u) {
                // witnesses for the next try: this thread's 9 diagonals killed the
                // rows of its hit steps (benign races: any killer will do)
                const int kb = dir > 0 ? td.k0 + ub : td.k0 + kW - kDiag - ub;
                unsigned hh = hit;
                while (hh) {
                    const int ss = s0 + __ffs(hh) - 1;
                    hh &= hh - 1u;
                    if (ss < rows) p.wit[dir > 0 ? td.r0 + ss : r_end - ss] = kb;
                }
            }
        }
    }

    if (MODE == kPruneTrack) {
        __syncthreads();
        // per-(row, band) bounds for the collection: the tile covers the canonical
        // bands b_lo..b_hi of |k| on its side
        const int nbands = ub_nbands(N, m);
        const long long nlist = p.ctl->alive;
        const bool ub_on = p.ub != nullptr && nlist * 2 * nbands <= p.ub_cap;
        const int kf = dir > 0 ? td.k0 : -(td.k0 + kW - 1);  // smallest |k| of the tile
        const int b_lo = max(0, (kf - m) / kW), b_hi = min(nbands - 1, (kf + kW - 1 - m) / kW);
        const unsigned long long etag = (unsigned long long)p.ctl->tepoch << 32;
        for (int s = tid; s < rows; s += kThreads) {
            const unsigned k = S.ykey[s];
            if (k > 1u) {
                const int c = dir > 0 ? td.r0 + s : r_end - s;
                if (ub_on) {
                    // list index of c (sorted list): binary search
                    int lo = 0, hi = (int)nlist - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (p.list[mid] < c) lo = mid + 1;
                        else hi = mid;
                    }
                    if (hi >= 0 && p.list[lo] == c) {
                        // corr upper bound of every q of this tile for row c
                        const float ubc = (float)(((double)key2f(k) + E * (double)qn_max) * (double)S.crow[s].w + xs) *
                                              (1.f + 4.8e-7f) + 1e-7f;
                        const unsigned long long v = etag | f2key(ubc);
                        for (int b = b_lo; b <= b_hi; ++b)
                            atomicMax(&p.ub[((long long)lo * 2 + (dir < 0)) * nbands + b], v);
                    }
                }
                // the tile's error term in x units of this row: E*qn_max + xs/cn (>= 0: bit order)
                const unsigned ekey =
                    __float_as_uint((float)(E * (double)qn_max + xs / (double)S.crow[s].w) * (1.f + 4.8e-7f));
                if (p.peers.n > 1) {
                    for (int r = 0; r < p.peers.n; ++r) {
                        atomicMax(&p.peers.ymax[r][c], k);
                        atomicMax(&p.peers.emax[r][c], ekey);
                    }
                } else {
                    atomicMax(&p.ymax[c], k);
                    atomicMax(&p.emax[c], ekey);
                }
            }
        }
    }
    if (tid == 0) {
        // walked cells, evaluated cells and direct seed dots actually computed
        // (slots a pattern never reads are neither walked nor seeded)
        constexpr int kWalked = MODE == kPrune ? scan_walked_slots<STRIDE>() * kThreads : kW;
        constexpr int kEvals = MODE == kPrune && STRIDE > 1 ? scan_evals_per_row<STRIDE>() : kW / STRIDE;
        atomicAdd(&p.acc[0], (unsigned long long)rows * (unsigned long long)kWalked);
        atomicAdd(&p.acc[1], (unsigned long long)evals * (unsigned long long)kEvals);
        if (td.seed < 0 && rc < 0) atomicAdd(&p.acc[2], (unsigned long long)kWalked);
#ifdef TSD_TILE_TIMING
        if (MODE == kCollect && p.dbg) {  // build flag + TSD_DEBUG: the slowest collection tile
            const unsigned long long dt = (unsigned long long)(clock64() - t_start);
            if (dt > p.dbg[12]) {
                p.dbg[12] = dt;
                p.dbg[13] = (unsigned long long)rows;
                p.dbg[14] = (unsigned long long)(td.k0 + (1 << 30));
                p.dbg[15] = (unsigned long long)evals;
            }
        }
#endif
    }
    }  // persistent tile loop
}

// ---------------------------------------------------------------------------
// Band 0 with both sides in one walk (packed FP32x2).
//
// A band-0 tile of k_scan walks one side of one row block.  Here one CTA walks
// both sides of row block j together: lane .x of every register pair is the
// positive side (rows a + s, q = c + kA + u, resident seed row 2j), lane .y the
// negative side (rows e - s, q = c - kA - u, seed row 2j+1), so each step is
// FFMA2 / FMUL2 on pairs.  Per side the arithmetic is exactly k_scan's: the
// same operands, the same two roundings per cell in the same order, the same
// kill rule, so the kills are identical and the error bound E (taken over
// both sides' maxima) stays valid.  Half the issue slots of the walk.
struct __align__(16) PairSmem {
    float4 crow[kRowsPad];  // per row step: {cdf+, cdf-, cdg+, cdg-}
    float2 ctc[kRowsPad];   // per row step: thresholds {tc+, tc-} (first: norms)
    union {
        struct {
            float4 qd[kQPad];  // per q step: {qdf+, qdf-, qdg+, qdg-}
            float2 qn[kQPad];  // per q step: norms (NaN: invalid q)
        } walk;
        struct {
            double a[kSeedChunk];
            double win[kW + kSeedChunk];
        } seed;
    } u;
    float red[7][kThreads / 32];
    int flag[2];
};

template <int STRIDE>
__global__ void __launch_bounds__(kThreads, 4) k_band0_pair(const ScanParams p) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char pair_smem[];
    PairSmem& S = *reinterpret_cast<PairSmem*>(pair_smem);
    const int tid = threadIdx.x;
    const int N = p.N, m = p.m, L = p.L, kA = p.kA;
    const long long slots = (N + L - 1) / L;
    const long long mine = p.world > 1 ? (slots > p.rank ? (slots - p.rank + p.world - 1) / p.world : 0) : slots;
    int par = 0;
    for (long long f = blockIdx.x;; par ^= 1) {
    if (f >= mine) break;
    if (tid == 0) S.flag[par] = atomicAdd(p.next, 1);
    const int jb = (int)(f * p.world + p.rank);
    const int a = jb * L, e = min(N, a + L) - 1, rows = e - a + 1;
    const bool v0 = (long long)a + kA < N, v1 = (long long)e - kA >= 0;
    int any = 0;
    if (v0 || v1)
        for (int s = tid; s < rows; s += kThreads) any |= p.alive[a + s];
    const bool work = __syncthreads_or(any);
    f = (long long)S.flag[par] + gridDim.x;
    if (!work) continue;
    const int qb0 = a + kA, qb1 = e - kA;  // q of step 0, u = 0 on each side
    const int nq = rows - 1 + kW;

    // ---- seeds (resident rows; the partial last block's negative side direct)
    float2 cov[kDiag];
    bool direct1 = false;
    {
        float c0[kDiag], c1[kDiag];
        const double* qt0 = p.seedqt + (size_t)(2 * jb) * kW + tid * kDiag;
        const double mm0 = (double)m * p.mu[a];
#pragma unroll
        for (int j = 0; j < kDiag; ++j) {
            const int q = qb0 + tid * kDiag + j;
            c0[j] = (v0 && q < N) ? (float)(qt0[j] - mm0 * p.mu[q]) : 0.f;
        }
        if (rows == L) {
            const double* qt1 = p.seedqt + (size_t)(2 * jb + 1) * kW + tid * kDiag;
            const double mm1 = (double)m * p.mu[e];
#pragma unroll
            for (int j = 0; j < kDiag; ++j) {
                const int q = qb1 - tid * kDiag - j;
                c1[j] = (v1 && q >= 0) ? (float)(qt1[j] - mm1 * p.mu[q]) : 0.f;
            }
        } else if (v1) {
            seed_fp64(p, e, qb1, -1, S.u.seed.a, S.u.seed.win, c1);
            direct1 = true;
            __syncthreads();  // seed scratch is reused below
        } else {
#pragma unroll
            for (int j = 0; j < kDiag; ++j) c1[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < kDiag; ++j) cov[j] = make_float2(c0[j], c1[j]);
    }

    // ---- stage the walk operands of both sides (k_scan's staging, per side)
    float cn_min = FLT_MAX, qn_min = FLT_MAX, qn_max = 0.f;
    float dc = 0.f, gc = 0.f, dq = 0.f, gq = 0.f;
#pragma unroll 4
    for (int s = tid; s < rows; s += kThreads) {
        const int c0 = a + s, c1 = e - s;
        const int ci1 = min(c1 + 1, N - 1);  // s == 0 takes no increment
        float4 v;
        v.x = (s == 0 || !v0) ? 0.f : p.df[c0];
        v.z = (s == 0 || !v0) ? 0.f : p.dg[c0];
        v.y = (s == 0 || !v1) ? 0.f : -p.df[ci1];
        v.w = (s == 0 || !v1) ? 0.f : -p.dg[ci1];
        const float n0 = p.nrm[c0];
        if (n0 != 0.f) cn_min = fminf(cn_min, n0);  // both sides walk the rows [a, e]
        dc = fmaxf(dc, fmaxf(fabsf(v.x), fabsf(v.y)));
        gc = fmaxf(gc, fmaxf(fabsf(v.z), fabsf(v.w)));
        S.crow[s] = v;
        S.ctc[s] = make_float2(n0, p.nrm[c1]);
    }
    const int rows_p = (rows + kDiag - 1) / kDiag * kDiag;
    for (int s = rows + tid; s <= rows_p; s += kThreads) {
        S.crow[s] = make_float4(0.f, 0.f, 0.f, 0.f);
        S.ctc[s] = make_float2(FLT_MAX, FLT_MAX);
    }
    const float qnan = __int_as_float(0x7fffffff);
#pragma unroll 4
    for (int u = tid; u < rows_p + kW + kDiag; u += kThreads) {
        const int q0 = qb0 + u, q1 = qb1 - u;
        const bool ok0 = v0 && u < nq && q0 < N;
        const bool ok1 = v1 && u < nq && q1 >= 0;
        const int qc0 = ok0 ? q0 : 0, qc1 = ok1 ? q1 : 0;
        const int qi1 = min(qc1 + 1, N - 1);
        float a0 = p.df[qc0], b0 = p.dg[qc0], a1 = p.df[qi1], b1 = p.dg[qi1];
        const float n0 = p.nrm[qc0], n1 = p.nrm[qc1];
        if (!ok0) a0 = b0 = 0.f;
        if (!ok1 || qc1 + 1 >= N) a1 = b1 = 0.f;
        if (ok0 && n0 != 0.f) {
            qn_min = fminf(qn_min, n0);
            qn_max = fmaxf(qn_max, n0);
        }
        if (ok1 && n1 != 0.f) {
            qn_min = fminf(qn_min, n1);
            qn_max = fmaxf(qn_max, n1);
        }
        dq = fmaxf(dq, fmaxf(fabsf(a0), fabsf(a1)));
        gq = fmaxf(gq, fmaxf(fabsf(b0), fabsf(b1)));
        S.u.walk.qd[u] = make_float4(a0, a1, b0, b1);
        S.u.walk.qn[u] = make_float2((ok0 && n0 != 0.f) ? n0 : qnan, (ok1 && n1 != 0.f) ? n1 : qnan);
    }
    cn_min = -warp_max(-cn_min);
    qn_min = -warp_max(-qn_min);
    qn_max = warp_max(qn_max);
    dc = warp_max(dc);
    gc = warp_max(gc);
    dq = warp_max(dq);
    gq = warp_max(gq);
    if ((tid & 31) == 0) {
        S.red[0][tid >> 5] = cn_min;
        S.red[1][tid >> 5] = qn_min;
        S.red[2][tid >> 5] = qn_max;
        S.red[3][tid >> 5] = dc;
        S.red[4][tid >> 5] = gc;
        S.red[5][tid >> 5] = dq;
        S.red[6][tid >> 5] = gq;
    }
    __syncthreads();
    cn_min = FLT_MAX;
    qn_min = FLT_MAX;
    qn_max = 0.f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        cn_min = fminf(cn_min, S.red[0][w]);
        qn_min = fminf(qn_min, S.red[1][w]);
        qn_max = fmaxf(qn_max, S.red[2][w]);
        dc = fmaxf(dc, S.red[3][w]);
        gc = fmaxf(gc, S.red[4][w]);
        dq = fmaxf(dq, S.red[5][w]);
        gq = fmaxf(gq, S.red[6][w]);
    }
    const double inv_sqm = 1.0 / sqrt((double)m);
    const double smax_c = cn_min < FLT_MAX ? inv_sqm / (double)cn_min * (1.0 + 1e-6) : 0.0;
    const double smax_q = qn_min < FLT_MAX ? inv_sqm / (double)qn_min * (1.0 + 1e-6) : 0.0;
    // k_scan's bound over the union of both sides' operands; the direct FP64
    // seed and the resident seeds carry no seed error term
    const double P = (double)dc * (double)gq + (double)dq * (double)gc;
    const double E = p.err_k * (double)kEps32 * (double)(rows + 8) * ((double)m * smax_c * smax_q + 1.5 * P);
    const double xs = stats_band(p, true);  // statistics error, resident raw seeds included
    constexpr float kNoEval = FLT_MAX;
    int evals = 0;
    for (int s = tid; s < rows; s += kThreads) {
        const float2 cn = S.ctc[s];
        float2 tc;
        const bool live0 = v0 && p.alive[a + s] != 0, live1 = v1 && p.alive[e - s] != 0;
        if (!live0 || cn.x == 0.f) {
            tc.x = kNoEval;
        } else {
            const double eps_row = E * (double)cn.x * (double)qn_max + kSlack + 8.0 * (double)kEps32 + xs;
            tc.x = (float)((p.thr0 + eps_row) / (double)cn.x);
            tc.x = tc.x + fabsf(tc.x) * 2.4e-7f;  // round toward +inf (conservative)
        }
        if (!live1 || cn.y == 0.f) {
            tc.y = kNoEval;
        } else {
            const double eps_row = E * (double)cn.y * (double)qn_max + kSlack + 8.0 * (double)kEps32 + xs;
            tc.y = (float)((p.thr0 + eps_row) / (double)cn.y);
            tc.y = tc.y + fabsf(tc.y) * 2.4e-7f;
        }
        S.ctc[s] = tc;
        evals += (tc.x != kNoEval) + (tc.y != kNoEval);
    }
    evals = __syncthreads_count(evals);

    // ---- walk: k_scan's ring, on pairs
    float4 rd[kDiag];
    float2 rn[kDiag];
    const int ub = tid * kDiag;
    const float4* qdp = S.u.walk.qd + ub;
    const float2* qnp = S.u.walk.qn + ub;
#pragma unroll
    for (int j = 0; j < kDiag; ++j) {
        rd[j] = qdp[j];
        rn[j] = qnp[j];
    }
    float4 cr_next = S.crow[0];
    float2 tc_next = S.ctc[0];
    // hit masks cover kAgg walk blocks (27 steps) between two aggregations:
    // in pass 0 nearly every row dies, and the reduction's latency per block
    // was ~15% of the stall samples at one aggregation per 9 steps
    constexpr int kAgg = 3;
    unsigned hit0 = 0u, hit1 = 0u;
    int hb = 0;  // walk blocks in the current masks
    for (int s0 = 0; s0 < rows_p; s0 += kDiag) {
        const int sh = hb * kDiag;
#pragma unroll
        for (int uu = 0; uu < kDiag; ++uu) {
            const int ss = s0 + uu;
            const float4 cr = cr_next;
            const float2 tc = tc_next;
            cr_next = S.crow[ss + 1];
            tc_next = S.ctc[ss + 1];
            const float2 cdf = make_float2(cr.x, cr.y), cdg = make_float2(cr.z, cr.w);
#pragma unroll
            for (int j = 0; j < kDiag; ++j) {
                const int rj = (j + uu) % kDiag;
                cov[j] = __ffma2_rn(cdf, make_float2(rd[rj].z, rd[rj].w), cov[j]);
                cov[j] = __ffma2_rn(make_float2(rd[rj].x, rd[rj].y), cdg, cov[j]);
            }
            float mx0 = -FLT_MAX, mx1 = -FLT_MAX;
#pragma unroll
            for (int j = 0; j < kDiag; ++j)
                if ((j + uu) % STRIDE == 0) {
                    const float2 x = __fmul2_rn(cov[j], rn[(j + uu) % kDiag]);
                    mx0 = fmaxf(mx0, x.x);
                    mx1 = fmaxf(mx1, x.y);
                }
            hit0 |= (mx0 > tc.x ? 1u : 0u) << (sh + uu);
            hit1 |= (mx1 > tc.y ? 1u : 0u) << (sh + uu);
            rd[uu % kDiag] = qdp[ss + kDiag];
            rn[uu % kDiag] = qnp[ss + kDiag];
        }
        // warp-aggregated kills every kAgg blocks: lane b stores the row of
        // step sb + b of each side if any lane killed it (one store per row and
        // warp instead of one per thread and hit)
        if (++hb == kAgg || s0 + kDiag >= rows_p) {
            const unsigned h0 = __reduce_or_sync(0xffffffffu, hit0), h1 = __reduce_or_sync(0xffffffffu, hit1);
            const int lane = tid & 31, sb = s0 - (hb - 1) * kDiag;
            if ((h0 >> lane) & 1u) peer_kill(p.peers, p.alive, a + sb + lane);
            if ((h1 >> lane) & 1u) peer_kill(p.peers, p.alive, e - (sb + lane));
            hit0 = hit1 = 0u;
            hb = 0;
        }
    }
    if (tid == 0) {
        atomicAdd(&p.acc[0], (unsigned long long)rows * (unsigned long long)kW * (unsigned long long)(v0 + v1));
        atomicAdd(&p.acc[1], (unsigned long long)evals * (unsigned long long)(kW / STRIDE));
        if (direct1) atomicAdd(&p.acc[2], (unsigned long long)kW);
    }
    }  // persistent tile loop
}

// Sampled cells of the pair-kill walk: slot j (diagonal ub + j of the thread)
// at step uu of a 9-step block.  A slot that no pattern ever samples is never
// read, so the compiler drops its walk too: STRIDE 6 samples the even slots
// only (5 of 9 walked), 12 / 16 three slots (slots 0, 3, 6), 20 slot 0 alone.
// Every pattern meets each partner q of a walked slot once per 9 steps.
template <int STRIDE>
__device__ __forceinline__ constexpr bool pk_sampled(int j, int uu) {
    return STRIDE == 20   ? (j == 0)
           : STRIDE == 12 ? (j % 3 == 0 && (j / 3 + uu) % 3 == 0)
           : STRIDE == 16 ? (j % 3 == 0 && (j / 3 + uu) % 3 != 2)
           : STRIDE >= 6  ? (j + 2 * uu) % STRIDE == 0
                          : (2 * j + uu) % STRIDE == 0;
}

template <int STRIDE>
__device__ __forceinline__ constexpr int pk_walked_slots() {
    int n = 0;
    for (int j = 0; j < kDiag; ++j) {
        bool any = false;
        for (int uu = 0; uu < kDiag; ++uu) any = any || pk_sampled<STRIDE>(j, uu);
        n += any ? 1 : 0;
    }
    return n;
}
template <int STRIDE>
__device__ __forceinline__ constexpr int pk_samples() {  // sampled (slot, step) pairs per 9-step block
    int n = 0;
    for (int j = 0; j < kDiag; ++j)
        for (int uu = 0; uu < kDiag; ++uu) n += pk_sampled<STRIDE>(j, uu) ? 1 : 0;
    return n;
}

// ---------------------------------------------------------------------------
// Band 0, every unordered pair once (pair-kill walk).
//
// A pair {c, q} with |q - c| in band 0 is a positive-side cell of c and a
// negative-side cell of q, so walking both sides of every row computes every
// pair twice.  Here each CTA walks the positive sides of two row blocks A and
// B together (lane .x of every register pair: block A, .y: block B; FFMA2 /
// FMUL2 on pairs as in k_band0_pair), and a certain hit at (c, q) kills both
// ends: d(c, q) < r means neither is a range discord.  The row kills are
// aggregated per warp as before; the partner kills are byte flags per q step
// in shared memory (plain racy stores of 1), written to `alive` after the walk.
// Every row is evaluated whether or not it is still alive: a dead row's cells
// still kill its partners.  The per-cell arithmetic, the error bound and the
// certainty rule are k_band0_pair's (the bound is symmetric in c and q: the
// tile's E covers the cell whichever end it is read from).  Half the walk of
// the two-sided band; the resident seed rows of the positive sides only.
struct __align__(16) PkSmem {
    float4 crow[kRowsPad];  // per row step: {cdf_A, cdf_B, cdg_A, cdg_B}
    float2 ctc[kRowsPad];   // per row step: thresholds {tc_A, tc_B} (first: norms)
    float4 qd[kQPad];       // per q step: {qdf_A, qdf_B, qdg_A, qdg_B}
    float2 qn[kQPad];       // per q step: norms (NaN: invalid q)
    unsigned char qhit[2][kQPad];  // per q step: killed as a partner (A, B)
    float red[7][kThreads / 32];
    int flag[2];
};

template <int STRIDE>
__global__ void __launch_bounds__(kThreads, 4) k_band0_pk(const ScanParams p) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char pk_smem[];
    PkSmem& S = *reinterpret_cast<PkSmem*>(pk_smem);
    const int tid = threadIdx.x;
    const int N = p.N, m = p.m, L = p.L, kA = p.kA;
    const int nblk = (N + L - 1) / L;
    const long long slots = (nblk + 1) / 2;
    const long long mine = p.world > 1 ? (slots > p.rank ? (slots - p.rank + p.world - 1) / p.world : 0) : slots;
    int par = 0;
    for (long long f = blockIdx.x;; par ^= 1) {
    if (f >= mine) break;
    if (tid == 0) S.flag[par] = atomicAdd(p.next, 1);
    const int jp = (int)(f * p.world + p.rank);
    const int bA = 2 * jp, bB = 2 * jp + 1;
    const bool hasB = bB < nblk;
    const int aA = bA * L, aB = bB * L;
    const int rowsA = min(N, aA + L) - aA, rowsB = hasB ? min(N, aB + L) - aB : 0;
    const bool vA = (long long)aA + kA < N, vB = hasB && (long long)aB + kA < N;
    int any = 0;
    if (vA)
        for (int s = tid; s < rowsA; s += kThreads) any |= p.alive[aA + s];
    if (vB)
        for (int s = tid; s < rowsB; s += kThreads) any |= p.alive[aB + s];
    const bool work = __syncthreads_or(any);
    f = (long long)S.flag[par] + gridDim.x;
    if (!work) continue;
    const int rows = rowsA;  // >= rowsB (B follows A)
    const int qbA = aA + kA, qbB = aB + kA;  // q of step 0, u = 0
    const int nqA = rowsA - 1 + kW, nqB = rowsB - 1 + kW;

    // ---- seeds: resident positive-side rows of both blocks
    float2 cov[kDiag];
    {
        const double* qtA = p.seedqt + (size_t)(2 * bA) * kW + tid * kDiag;
        const double* qtB = p.seedqt + (size_t)(2 * bB) * kW + tid * kDiag;
        const double mA = (double)m * p.mu[aA];
        const double mB = vB ? (double)m * p.mu[aB] : 0.0;
#pragma unroll
        for (int j = 0; j < kDiag; ++j) {
            const int qA = qbA + tid * kDiag + j, qB = qbB + tid * kDiag + j;
            const float x = (vA && qA < N) ? (float)(qtA[j] - mA * p.mu[qA]) : 0.f;
            const float y = (vB && qB < N) ? (float)(qtB[j] - mB * p.mu[qB]) : 0.f;
            cov[j] = make_float2(x, y);
        }
    }

    // ---- stage the walk operands of both blocks
    float cn_min = FLT_MAX, qn_min = FLT_MAX, qn_max = 0.f;
    float dc = 0.f, gc = 0.f, dq = 0.f, gq = 0.f;
#pragma unroll 4
    for (int s = tid; s < rows; s += kThreads) {
        const bool inB = s < rowsB;
        const int cA = aA + s, cB = inB ? aB + s : aA;
        float4 v;
        v.x = (s == 0 || !vA) ? 0.f : p.df[cA];
        v.z = (s == 0 || !vA) ? 0.f : p.dg[cA];
        v.y = (s == 0 || !vB || !inB) ? 0.f : p.df[cB];
        v.w = (s == 0 || !vB || !inB) ? 0.f : p.dg[cB];
        const float nA = p.nrm[cA], nB = inB ? p.nrm[cB] : 0.f;
        if (nA != 0.f) cn_min = fminf(cn_min, nA);
        if (nB != 0.f) cn_min = fminf(cn_min, nB);
        dc = fmaxf(dc, fmaxf(fabsf(v.x), fabsf(v.y)));
        gc = fmaxf(gc, fmaxf(fabsf(v.z), fabsf(v.w)));
        S.crow[s] = v;
        S.ctc[s] = make_float2(nA, nB);
    }
    const int rows_p = (rows + kDiag - 1) / kDiag * kDiag;
    for (int s = rows + tid; s <= rows_p; s += kThreads) {
        S.crow[s] = make_float4(0.f, 0.f, 0.f, 0.f);
        S.ctc[s] = make_float2(FLT_MAX, FLT_MAX);
    }
    const float qnan = __int_as_float(0x7fffffff);
#pragma unroll 4
    for (int u = tid; u < rows_p + kW + kDiag; u += kThreads) {
        const int qA = qbA + u, qB = qbB + u;
        const bool okA = vA && u < nqA && qA < N;
        const bool okB = vB && u < nqB && qB < N;
        const int qcA = okA ? qA : 0, qcB = okB ? qB : 0;
        float a0 = p.df[qcA], b0 = p.dg[qcA], a1 = p.df[qcB], b1 = p.dg[qcB];
        const float nA = p.nrm[qcA], nB = p.nrm[qcB];
        if (!okA) a0 = b0 = 0.f;
        if (!okB) a1 = b1 = 0.f;
        if (okA && nA != 0.f) {
            qn_min = fminf(qn_min, nA);
            qn_max = fmaxf(qn_max, nA);
        }
        if (okB && nB != 0.f) {
            qn_min = fminf(qn_min, nB);
            qn_max = fmaxf(qn_max, nB);
        }
        dq = fmaxf(dq, fmaxf(fabsf(a0), fabsf(a1)));
        gq = fmaxf(gq, fmaxf(fabsf(b0), fabsf(b1)));
        S.qd[u] = make_float4(a0, a1, b0, b1);
        S.qn[u] = make_float2((okA && nA != 0.f) ? nA : qnan, (okB && nB != 0.f) ? nB : qnan);
        S.qhit[0][u] = 0;
        S.qhit[1][u] = 0;
    }
    cn_min = -warp_max(-cn_min);
    qn_min = -warp_max(-qn_min);
    qn_max = warp_max(qn_max);
    dc = warp_max(dc);
    gc = warp_max(gc);
    dq = warp_max(dq);
    gq = warp_max(gq);
    if ((tid & 31) == 0) {
        S.red[0][tid >> 5] = cn_min;
        S.red[1][tid >> 5] = qn_min;
        S.red[2][tid >> 5] = qn_max;
        S.red[3][tid >> 5] = dc;
        S.red[4][tid >> 5] = gc;
        S.red[5][tid >> 5] = dq;
        S.red[6][tid >> 5] = gq;
    }
    __syncthreads();
    cn_min = FLT_MAX;
    qn_min = FLT_MAX;
    qn_max = 0.f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        cn_min = fminf(cn_min, S.red[0][w]);
        qn_min = fminf(qn_min, S.red[1][w]);
        qn_max = fmaxf(qn_max, S.red[2][w]);
        dc = fmaxf(dc, S.red[3][w]);
        gc = fmaxf(gc, S.red[4][w]);
        dq = fmaxf(dq, S.red[5][w]);
        gq = fmaxf(gq, S.red[6][w]);
    }
    const double inv_sqm = 1.0 / sqrt((double)m);
    const double smax_c = cn_min < FLT_MAX ? inv_sqm / (double)cn_min * (1.0 + 1e-6) : 0.0;
    const double smax_q = qn_min < FLT_MAX ? inv_sqm / (double)qn_min * (1.0 + 1e-6) : 0.0;
    const double P = (double)dc * (double)gq + (double)dq * (double)gc;
    const double E = p.err_k * (double)kEps32 * (double)(rows + 8) * ((double)m * smax_c * smax_q + 1.5 * P);
    const double xs = stats_band(p, true);  // statistics error, resident raw seeds included
    constexpr float kNoEval = FLT_MAX;
    int evals = 0;
    for (int s = tid; s < rows; s += kThreads) {
        // every row is evaluated, alive or not: its hits also kill the partners
        const float2 cn = S.ctc[s];
        float2 tc;
        if (!vA || cn.x == 0.f) {
            tc.x = kNoEval;
        } else {
            const double eps_row = E * (double)cn.x * (double)qn_max + kSlack + 8.0 * (double)kEps32 + xs;
            tc.x = (float)((p.thr0 + eps_row) / (double)cn.x);
            tc.x = tc.x + fabsf(tc.x) * 2.4e-7f;  // round toward +inf (conservative)
        }
        if (!vB || s >= rowsB || cn.y == 0.f) {
            tc.y = kNoEval;
        } else {
            const double eps_row = E * (double)cn.y * (double)qn_max + kSlack + 8.0 * (double)kEps32 + xs;
            tc.y = (float)((p.thr0 + eps_row) / (double)cn.y);
            tc.y = tc.y + fabsf(tc.y) * 2.4e-7f;
        }
        S.ctc[s] = tc;
        evals += (tc.x != kNoEval) + (tc.y != kNoEval);
    }
    evals = __syncthreads_count(evals);

    // ---- walk
    float4 rd[kDiag];
    float2 rn[kDiag];
    const int ub = tid * kDiag;
    const float4* qdp = S.qd + ub;
    const float2* qnp = S.qn + ub;
    unsigned char* const hA = S.qhit[0] + ub;
    unsigned char* const hB = S.qhit[1] + ub;
#pragma unroll
    for (int j = 0; j < kDiag; ++j) {
        rd[j] = qdp[j];
        rn[j] = qnp[j];
    }
    float4 cr_next = S.crow[0];
    float2 tc_next = S.ctc[0];
    constexpr int kAgg = 3;  // walk blocks per row-kill aggregation (27 steps)
    // partner-hit marks: any non-zero byte.  A per-thread register value
    // instead of the constant 1, which the compiler rematerialised before every
    // predicated store (25 moves per unrolled walk block; C5 681 -> 669 ms)
    const unsigned char mark = (unsigned char)((tid & 31) + 1);
    unsigned hit0 = 0u, hit1 = 0u;
    int hb = 0;
    for (int s0 = 0; s0 < rows_p; s0 += kDiag) {
        const int sh = hb * kDiag;
#pragma unroll
        for (int uu = 0; uu < kDiag; ++uu) {
            const int ss = s0 + uu;
            const float4 cr = cr_next;
            const float2 tc = tc_next;
            cr_next = S.crow[ss + 1];
            tc_next = S.ctc[ss + 1];
            const float2 cdf = make_float2(cr.x, cr.y), cdg = make_float2(cr.z, cr.w);
#pragma unroll
            for (int j = 0; j < kDiag; ++j) {
                const int rj = (j + uu) % kDiag;
                cov[j] = __ffma2_rn(cdf, make_float2(rd[rj].z, rd[rj].w), cov[j]);
                cov[j] = __ffma2_rn(make_float2(rd[rj].x, rd[rj].y), cdg, cov[j]);
            }
            bool h0 = false, h1 = false;
#pragma unroll
            for (int j = 0; j < kDiag; ++j)
                // sampled cells: (2j + step) % 3 == 0 spreads the samples over
                // every row's cells AND every partner's cells (a partner's
                // cells have j + step constant, so (j + step) % 3 would test
                // a third of the partners fully and the rest never)
                if (pk_sampled<STRIDE>(j, uu)) {
                    // (STRIDE 6 / 9: j + 2 step, also spread over rows and
                    // partners; step = 9 blk + uu keeps every pattern compile-time)
                    const float2 x = __fmul2_rn(cov[j], rn[(j + uu) % kDiag]);
                    // the row dies if any sampled cell passes (NaN never does),
                    // and the partner q of the cell (u = ss + ub + j) with it
                    const bool b0 = x.x > tc.x, b1 = x.y > tc.y;
                    if (b0) hA[ss + j] = mark;
                    if (b1) hB[ss + j] = mark;
                    h0 |= b0;
                    h1 |= b1;
                }
            hit0 |= (h0 ? 1u : 0u) << (sh + uu);
            hit1 |= (h1 ? 1u : 0u) << (sh + uu);
            rd[uu % kDiag] = qdp[ss + kDiag];
            rn[uu % kDiag] = qnp[ss + kDiag];
        }
        if (++hb == kAgg || s0 + kDiag >= rows_p) {
            const unsigned h0 = __reduce_or_sync(0xffffffffu, hit0), h1 = __reduce_or_sync(0xffffffffu, hit1);
            const int lane = tid & 31, sb = s0 - (hb - 1) * kDiag;
            if ((h0 >> lane) & 1u) peer_kill(p.peers, p.alive, aA + sb + lane);
            if ((h1 >> lane) & 1u) peer_kill(p.peers, p.alive, aB + sb + lane);
            hit0 = hit1 = 0u;
            hb = 0;
        }
    }
    __syncthreads();
    // partner kills (a hit needs a valid q: invalid q carry NaN norms)
    for (int u = tid; u < nqA; u += kThreads)
        if (S.qhit[0][u]) peer_kill(p.peers, p.alive, qbA + u);
    for (int u = tid; u < nqB; u += kThreads)
        if (S.qhit[1][u]) peer_kill(p.peers, p.alive, qbB + u);
    if (tid == 0) {
        // cells actually walked (slots that are never sampled are not walked)
        // and cells evaluated, per row of a walked side
        atomicAdd(&p.acc[0], (unsigned long long)(pk_walked_slots<STRIDE>() * kThreads) *
                                 (unsigned long long)((vA ? rowsA : 0) + (vB ? rowsB : 0)));
        atomicAdd(&p.acc[1], (unsigned long long)evals * (unsigned long long)(pk_samples<STRIDE>() * kThreads / kDiag));
    }
    }  // persistent tile loop
}

// ---------------------------------------------------------------------------
// reference_sq_dist, bit-exact, one warp per pair.  buf: 256 doubles per warp.
__device__ double ref_dist_warp(const double* __restrict__ t, int m, int i, int j, double* buf) {
    const int lane = threadIdx.x & 31;
    double mean = 0.0, sg = 0.0;
    {
        // window statistics: the warp stages 128-element chunks of both
        // windows in shared memory (coalesced, all loads in flight); lane 0
        // (window i) and lane 1 (window j) keep the reference's sequential sums
        double s = 0.0, q = 0.0;
        for (int base = 0; base < m; base += 128) {
            const int len = min(128, m - base);
            for (int k = lane; k < len; k += 32) {
                buf[k] = t[i + base + k];
                buf[128 + k] = t[j + base + k];
            }
            __syncwarp();
            if (lane < 2) {
                const double* x = buf + 128 * lane;
                for (int k = 0; k < len; ++k) {
                    const double v = x[k];
                    s = __dadd_rn(s, v);
                    q = __dadd_rn(q, __dmul_rn(v, v));
                }
            }
            __syncwarp();
        }
        if (lane < 2) {
            const double md = (double)m;
            mean = __ddiv_rn(s, md);
            const double var = __dsub_rn(__ddiv_rn(q, md), __dmul_rn(mean, mean));
            sg = __dsqrt_rn(var > 0.0 ? var : 0.0);
        }
    }
    const double mx = __shfl_sync(0xffffffffu, mean, 0), sx = __shfl_sync(0xffffffffu, sg, 0);
    const double my = __shfl_sync(0xffffffffu, mean, 1), sy = __shfl_sync(0xffffffffu, sg, 1);
    bool cx = sx < kSigmaEps, cy = sy < kSigmaEps;
    double acc = 0.0;
    if (!cx && !cy) {
        bool nzx = false, nzy = false;
        for (int base = 0; base < m; base += 256) {
            const int len = min(256, m - base);
            for (int k = lane; k < len; k += 32) {
                const double zx = __ddiv_rn(__dsub_rn(t[i + base + k], mx), sx);
                const double zy = __ddiv_rn(__dsub_rn(t[j + base + k], my), sy);
                nzx |= zx != 0.0;
                nzy |= zy != 0.0;
                const double d = __dsub_rn(zx, zy);
                buf[k] = __dmul_rn(d, d);
            }
            __syncwarp();
            if (lane == 0)
                for (int k = 0; k < len; ++k) acc = __dadd_rn(acc, buf[k]);
            __syncwarp();
        }
        cx = !__any_sync(0xffffffffu, nzx);
        cy = !__any_sync(0xffffffffu, nzy);
        acc = __shfl_sync(0xffffffffu, acc, 0);
    }
    if (cx && cy) return 0.0;
    if (cx || cy) return 2.0 * (double)m;
    return acc;
}

constexpr int kPairWarps = 8;

// mode 0: recheck (kill both ends when d < r^2); mode 1: exact nn (atomic min).
template <int MODE>
__global__ void __launch_bounds__(kPairWarps * 32) k_ref_pairs(const double* __restrict__ t, int m,
                                                               const int2* __restrict__ pairs,
                                                               const int* __restrict__ count,
                                                               int cap, double r_sq,
                                                               uint8_t* alive,
                                                               unsigned long long* nnkey,
                                                               TryCtl* ctl, const int* __restrict__ ex,
                                                               double* __restrict__ nnout, const Peers peers) {
    pdl_enter();
    __shared__ double buf[kPairWarps][256];
    const int w = threadIdx.x >> 5;
    const int total = min(*count, cap);
    for (int e = blockIdx.x * kPairWarps + w; e < total; e += gridDim.x * kPairWarps) {
        const int2 pr = pairs[e];
        if (MODE == 0 && !alive[pr.x] && !alive[pr.y]) continue;
        const double d = ref_dist_warp(t, m, pr.x, pr.y, buf[w]);
        if ((threadIdx.x & 31) == 0) {
            if (MODE == 0) {
                if (d < r_sq) {
                    peer_kill(peers, alive, pr.x);
                    peer_kill(peers, alive, pr.y);
                }
            } else {
                peer_min_key(peers, nnkey, pr.x, (unsigned long long)__double_as_longlong(d));
            }
        }
    }
    if (MODE == 1 && ex != nullptr) {
        // single-rank exact pass: the last CTA out gathers the survivors' nn
        __shared__ int s_last;
        __syncthreads();
        if (threadIdx.x == 0) s_last = atom_add_acq_rel(&ctl->xdone, 1) == (int)gridDim.x - 1;
        __syncthreads();
        if (!s_last) return;
        const int ec = ctl->ec;
        for (int e = threadIdx.x; e < ec; e += blockDim.x)
            nnout[e] = __longlong_as_double((long long)__ldcg(&nnkey[ex[e]]));
        if (threadIdx.x == 0) ctl->xdone = 0;
    }
}

// Degenerate rows (sigma < eps by the rolling statistics, or statistics too
// unreliable for the FP32 filter): the reference's distance for such a window
// depends on its own one-pass statistics (znormalize, src/distance.cpp:8-22:
// all-zero z -> the 0 / 2m conventions of reference_sq_dist,
// src/pardrag.cpp:57-69; else tiny equal z), so no pair with one goes through
// the FP32 model.  The windows were split per length (stats_kernels.cu
// degenerate_row):
//   one-pass constant (degc, cr[7]; their index range in cr[5], cr[6]): every
//     pair's distance is a convention -- 0 against another such window, 2m
//     against anything else -- so each row is decided in O(1):
//     A1  a listed regular row with such a partner at |c - q| >= m: d = 2m;
//     B1  such a row: nn = 0 if another one is at |c - q| >= m, else 2m if any
//         admissible q exists;
//   the others (deg2, cr[8]): the exact routine, one warp per pair:
//     A2  every listed regular row still alive x every such q;
//     B2  every such row still alive x every q (a dead row stops counting).
// d < r^2 kills the row; every d feeds its exact-nn key.  Dealt over the ranks.
__device__ __forceinline__ void degenerate_body(const double* __restrict__ t, int m, int N,
                                                const int* __restrict__ list, const TryCtl* __restrict__ ctl,
                                                const int* __restrict__ cr, const int* __restrict__ degc,
                                                const int* __restrict__ deg2, const float* __restrict__ nrm,
                                                double r_sq, uint8_t* alive, unsigned long long* nnkey, int rank,
                                                int world, const Peers& peers, double* buf) {
    if (cr[2] == 0) return;
    const int Dc = cr[7], D2 = cr[8];
    const int cmin = N - cr[5], cmax = cr[6] - 1;
    const long long nl = ctl->alive;
    const double two_m = 2.0 * (double)m;
    // A1 + B1: one thread per row
    const long long gt = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * world + rank;
    const long long gs = (long long)gridDim.x * blockDim.x * world;
    if (Dc > 0) {
        for (long long e = gt; e < nl; e += gs) {
            const int c = list[e];
            if (!alive[c] || nrm[c] == 0.f) continue;  // degenerate rows: B1 / B2
            if (c - cmin >= m || cmax - c >= m) {
                if (two_m < r_sq) peer_kill(peers, alive, c);
                peer_min_key(peers, nnkey, c, (unsigned long long)__double_as_longlong(two_m));
            }
        }
        for (long long e = gt; e < Dc; e += gs) {
            const int c = degc[e];
            if (!(c >= m || N - 1 - c >= m)) continue;  // no admissible partner: nn stays +inf
            const double d = (c - cmin >= m || cmax - c >= m) ? 0.0 : two_m;
            if (d < r_sq) peer_kill(peers, alive, c);
            peer_min_key(peers, nnkey, c, (unsigned long long)__double_as_longlong(d));
        }
    }
    if (D2 == 0) return;
    // A2 + B2: one warp per pair
    const long long totA = nl * D2, tot = totA + (long long)D2 * N;
    const int w = threadIdx.x >> 5;
    for (long long e = ((long long)blockIdx.x * kPairWarps + w) * world + rank; e < tot;
         e += (long long)gridDim.x * kPairWarps * world) {
        int c, q;
        if (e < totA) {
            c = list[e / D2];
            q = deg2[e % D2];
            if (!alive[c] || nrm[c] == 0.f) continue;
        } else {
            const long long f = e - totA;
            c = deg2[f / N];
            q = (int)(f % N);
            if (!alive[c]) continue;
        }
        if (abs(c - q) < m) continue;
        const double d = ref_dist_warp(t, m, c, q, buf);
        if ((threadIdx.x & 31) == 0) {
            if (d < r_sq) peer_kill(peers, alive, c);
            peer_min_key(peers, nnkey, c, (unsigned long long)__double_as_longlong(d));
        }
    }
}

// The knife-edge recheck and the degenerate pairs in
// one launch: both only kill rows or lower nn keys, so their order is free.
__global__ void __launch_bounds__(kPairWarps * 32) k_recheck(const double* __restrict__ t, int m, int N,
                                                             const int2* __restrict__ pairs,
                                                             const int* __restrict__ count, int cap,
                                                             const int* __restrict__ list,
                                                             const TryCtl* __restrict__ ctl,
                                                             const int* __restrict__ cr,
                                                             const int* __restrict__ degc,
                                                             const int* __restrict__ deg2,
                                                             const float* __restrict__ nrm, double r_sq,
                                                             uint8_t* alive, unsigned long long* nnkey,
                                                             int rank, int world, const Peers peers, int* wit) {
    pdl_enter();
    __shared__ double buf[kPairWarps][256];
    const int w = threadIdx.x >> 5;
    const int total = min(*count, cap);
    for (int e = blockIdx.x * kPairWarps + w; e < total; e += gridDim.x * kPairWarps) {
        const int2 pr = pairs[e];
        if (!alive[pr.x] && !alive[pr.y]) continue;
        const double d = ref_dist_warp(t, m, pr.x, pr.y, buf[w]);
        if ((threadIdx.x & 31) == 0 && d < r_sq) {
            peer_kill(peers, alive, pr.x);
            peer_kill(peers, alive, pr.y);
            if (wit) {
                wit[pr.x] = pr.y - pr.x - kDiag / 2;
                wit[pr.y] = pr.x - pr.y - kDiag / 2;
            }
        }
    }
    degenerate_body(t, m, N, list, ctl, cr, degc, deg2, nrm, r_sq, alive, nnkey, rank, world, peers, buf[w]);
}

// ---------------------------------------------------------------------------
// Kill witnesses (MERLIN: consecutive tries over lengths m, m+1, ... and the
// retries of one length see nearly the same distance matrix).  A row that was
// killed after band pass 0 in an earlier try remembers the 9 diagonals of its
// killer (ScanParams::wit: q = c + w .. c + w + 8).  Right after band pass 0 of
// the next try, the rows still alive that have a witness test those 9 cells
// before any later band is walked.  Witnesses come in runs (one diagonal
// kills consecutive rows), so k_witness_list cuts the candidates into runs of
// consecutive rows with the same witness (within 32-row chunks), and
// k_witness takes one run per warp (a variant staging each run with one
// round of cp.async copies, up to 200 KB of shared memory per SM, was 8%
// faster in isolation but made C4 30 ms slower end to end):
//   seed  QT(c0, q) = sum_p (t[c0+p] - A)(t[q+p] - B) at the run's first row
//         (A = mu_c0, B = mu of the middle q: small products under a DC
//         offset), the warp staging chunks of both windows in shared memory;
//   walk  lanes 0..8 carry one diagonal each down the run in FP64:
//         QT(c+1, q+1) = QT(c, q) - (t[c]-A)(t[q]-B) + (t[c+m]-A)(t[q+m]-B),
//         D(c+1) = D(c) - (t[c]-A) + (t[c+m]-A) with D(c) = sum_p (t[c+p]-A);
//   cov(c, q) = QT - (mu_q - B) D(c)  (exact identity with the true means; the
//         rolling means' error is in the statistics band), rounding bounded by
//         (m + 8 + 4 s) u m wa (wb + |mu_q - B|) + 4u(|QT| + |cov|), wa / wb the
//         largest |t - A| / |t - B| touched;
//   corr = cov / (m sigma_c sigma_q) kills c and q when
//         corr - (rounding + kSlack + statistics band) > thr0 (d(c, q) < r:
//         neither is a range discord), like a certain kill of the walk.
// Degenerate and constant windows never take part.  A row that survives its
// witness loses it.  The result is unchanged (every kill is certain); the later
// band passes and the full rows walk fewer groups, and the direct seeds those
// groups need are the bulk of their cost.
constexpr int kWitWarps = 8;
constexpr int kWitChunk = 256;

// candidate runs (first row, length): alive rows with the same witness,
// consecutive within a 32-row chunk (warp-aggregated append)
__global__ void k_witness_list(const ScanParams p, int4* __restrict__ wl) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    for (int c0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; c0 < p.N; c0 += gridDim.x * blockDim.x) {
        const int c = c0 + lane;
        const bool ok = c < p.N && p.alive[c] && p.nrm[c] > 0.f;  // alive, not constant / degenerate
        if (!__any_sync(0xffffffffu, ok)) continue;
        // a row without a witness borrows the nearest one of its chunk (before,
        // else after it): one diagonal often kills a run of consecutive rows
        const int own = c < p.N ? p.wit[c] : kNoWit;
        int wv = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, wv, o);
            if (wv == kNoWit && lane >= o) wv = u;
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_down_sync(0xffffffffu, wv, o);
            if (wv == kNoWit && lane + o < 32) wv = u;
        }
        const bool want = ok && wv != kNoWit;
        const unsigned wm = __ballot_sync(0xffffffffu, want);
        if (!wm) continue;
        const int pw = __shfl_up_sync(0xffffffffu, wv, 1);
        const bool pwant = __shfl_up_sync(0xffffffffu, want, 1);
        const bool start = want && (lane == 0 || !pwant || pw != wv);
        const unsigned sm = __ballot_sync(0xffffffffu, start);
        int at = 0;
        if (lane == 0) at = atomicAdd(&p.ctl->wn, __popc(sm));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (start) {
            const unsigned brk = lane < 31 ? (sm | ~wm) >> (lane + 1) : 0u;  // lanes that end the run
            const int len = brk ? __ffs(brk) : 32 - lane;
            wl[at + __popc(sm & ((1u << lane) - 1u))] = make_int4(c, len, wv, 0);
        }
    }
}

// The 9 diagonals q = c + kb .. c + kb + 8 of a run of L rows sharing the
// witness kb: seeds at the first row (both windows staged in shared memory in
// 256-element chunks; lane l: p = 4l .. 4l+3 of each 128-element half, 36 DFMA
// per 16 shared loads), then lanes 0..8 walk one diagonal each down the run.
__device__ __forceinline__ void wit_run9(const ScanParams& p, int c0, int L, int kb, double* sa, double* sw, double xs,
                                      unsigned long long& tests, unsigned long long& kills) {
    const int lane = threadIdx.x & 31;
    const int N = p.N, m = p.m;
        const int q0 = c0 + kb;
    const double A = p.mu[c0];
    const double B = p.mu[min(max(q0 + kDiag / 2, 0), N - 1)];
    double acc[kDiag];
#pragma unroll
    for (int j = 0; j < kDiag; ++j) acc[j] = 0.0;
    double delta = 0.0, wa = 0.0, wb = 0.0;
    for (int pc = 0; pc < m; pc += kWitChunk) {
        const int len = min(kWitChunk, m - pc);
        // all loads of the chunk in flight before the first shared store
        constexpr int kWv = (kWitChunk + 16 + 31) / 32;  // window loads per lane (ceil)
        double av[kWitChunk / 32], wv0[kWv];
#pragma unroll
        for (int i = 0; i < kWitChunk / 32; ++i) {
            const int x = lane + 32 * i;
            av[i] = x < len ? p.t[c0 + pc + x] - A : 0.0;
        }
#pragma unroll
        for (int i = 0; i < kWv; ++i) {
            const int x = lane + 32 * i;
            const int g = q0 + pc + x;
            wv0[i] = (x < len + kDiag - 1 && g >= 0 && g < p.n) ? p.t[g] - B : 0.0;
        }
#pragma unroll
        for (int i = 0; i < kWitChunk / 32; ++i) {
            sa[lane + 32 * i] = av[i];
            delta += av[i];
            wa = fmax(wa, fabs(av[i]));
        }
#pragma unroll
        for (int i = 0; i < kWv; ++i) {
            if (lane + 32 * i < kWitChunk + 16) sw[lane + 32 * i] = wv0[i];
            wb = fmax(wb, fabs(wv0[i]));
        }
        __syncwarp();
        // lane l: p = 4l .. 4l+3 of each 128-element half
#pragma unroll
        for (int h = 0; h < kWitChunk; h += 128) {
            double a4[4], w12[12];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const double2 v = reinterpret_cast<const double2*>(sa + h + 4 * lane)[i];
                a4[2 * i] = v.x;
                a4[2 * i + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const double2 v = reinterpret_cast<const double2*>(sw + h + 4 * lane)[i];
                w12[2 * i] = v.x;
                w12[2 * i + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < kDiag; ++j) acc[j] = fma(a4[i], w12[i + j], acc[j]);
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int j = 0; j < kDiag; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
        delta += __shfl_xor_sync(0xffffffffu, delta, o);
        wa = fmax(wa, __shfl_xor_sync(0xffffffffu, wa, o));
        wb = fmax(wb, __shfl_xor_sync(0xffffffffu, wb, o));
    }
    // lane j < 9 walks diagonal q = c + kb + j down the run
    double qt = 0.0;
#pragma unroll
    for (int j = 0; j < kDiag; ++j)
        if (j == lane) qt = acc[j];
    const double u_m = (double)m * kEps64;
    for (int s = 0; s < L; ++s) {
        const int c = c0 + s;
        const int q = c + kb + lane;
        if (s > 0) {
            const double to = p.t[c - 1] - A, tn = p.t[c + m - 1] - A;
            double qo = 0.0, qn = 0.0;
            if (lane < kDiag) {
                const int g0 = q - 1, g1 = q + m - 1;
                qo = (g0 >= 0 && g0 < p.n) ? p.t[g0] - B : 0.0;
                qn = (g1 >= 0 && g1 < p.n) ? p.t[g1] - B : 0.0;
            }
            qt = fma(tn, qn, fma(-to, qo, qt));
            delta = delta - to + tn;
            wa = fmax(wa, fabs(tn));
            wb = fmax(wb, fabs(qn));
        }
        if (!p.alive[c]) continue;  // killed meanwhile (warp-uniform)
        bool kill = false;
        double margin = -1.0;
        if (lane < kDiag && q >= 0 && q < N && abs(q - c) >= m && p.nrm[q] > 0.f) {
            const double dmu = p.mu[q] - B;
            const double cov = qt - dmu * delta;
            const double den = (double)m * p.sig[c] * p.sig[q];
            const double err = ((double)(m + 8 + 4 * s) * u_m * wa * (wb + fabs(dmu)) +
                                4.0 * kEps64 * (fabs(qt) + fabs(cov))) /
                               den;
            margin = cov / den - (err + xs) - p.thr0;
            kill = margin > 0.0;
        }
        const unsigned km = __ballot_sync(0xffffffffu, kill);
        if (km) {
            // the killer with the largest margin becomes the witness (the most
            // likely to kill again at the next length)
            int bl = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double om = __shfl_xor_sync(0xffffffffu, margin, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (om > margin || (om == margin && ol < bl)) {
                    margin = om;
                    bl = ol;
                }
            }
            if (lane == bl) {
                peer_kill(p.peers, p.alive, c);
                peer_kill(p.peers, p.alive, q);
                p.wit[c] = q - c - kDiag / 2;  // re-centred on the killing diagonal
                p.wit[q] = c - q - kDiag / 2;  // the partner's witness for the next try
            }
            ++kills;
        } else if (lane == 0) {
            p.wit[c] = kNoWit;
        }
        ++tests;
    }
    }

// One run per warp.  Phase 1 tests the middle diagonal of the 9 (a witness
// is re-centred on its killing diagonal, so this is usually the killer) for
// every row of the run at once: one m-long seed at the first row, the walk
// increments of rows 1..L-1 loaded by lane s and summed by a warp prefix scan
// (QT(c0+s) = QT(c0) + sum_{i<=s} ((t[c+m-1]-A)(t[q+m-1]-B) - (t[c-1]-A)(t[q-1]-B))),
// so every lane decides its own row.  The rows it does not kill take the
// 9-diagonal test (phase 2, wit_run9, one row at a time).  Rounding: the
// seed's m-term sum and the scan of s increments of at most 2 wa wb each are
// bounded by (m + 8 + 16 s) u m wa (wb + |mu_q - B|) + 4u (|QT| + |cov|).
template <bool INLINE2>
__global__ void __launch_bounds__(256) k_witness(const ScanParams p, const int4* __restrict__ wl,
                                                 int2* __restrict__ wl2) {
    pdl_enter();
    // INLINE2: the 9-diagonal phase in this kernel (small series: one launch
    // less per try); else deferred to k_witness9 (fewer registers here, more
    // warps for phase 1's load latency)
    __shared__ __align__(16) double s_a[INLINE2 ? 8 : 1][INLINE2 ? kWitChunk : 1];
    __shared__ __align__(16) double s_w[INLINE2 ? 8 : 1][INLINE2 ? kWitChunk + 16 : 1];
    const int lane = threadIdx.x & 31;
    const int N = p.N, m = p.m, n = p.n;
    const double xs = stats_band(p, false) + kSlack + 1e-12;
    const double xs_res = stats_band(p, true) + kSlack + 1e-12;  // cached raw seeds: the resident term
    const int total = p.ctl->wn;
    unsigned long long tests = 0, kills = 0;
    // runs are dealt one at a time per warp (their costs vary widely): the
    // first by warp index, the rest from a counter (one shared counter hit by
    // every warp of the grid serialised the whole kernel at C4)
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);;) {
        if (e >= total) break;
        const int4 run = wl[e];
        const int c0 = run.x, L = run.y, kb = run.z;  // kb: the run's (own or borrowed) witness
        const int qc = c0 + kb + kDiag / 2;  // middle diagonal's q of the first row
        const bool diag_ok = qc >= 0 && qc + L - 1 < N && abs(kb + kDiag / 2) >= m;  // warp-uniform
        const int c = c0 + lane;
        const bool mine = lane < L;
        bool alive = mine && p.alive[c] != 0;
        bool kill = false;
        if (diag_ok) {
            const double A = p.mu[c0], B = p.mu[qc];
            // ---- seed at the first row: from the run-seed cache (the raw dot
            // product QT(c0, qc) of an earlier length, advanced by the length
            // recurrence) or directly (shifted by A, B; the raw product is kept
            // for the next length)
            double acc, delta, e_seed, e_delta;
            bool cached = false;
            double wa = 0.0, wb = 0.0;
            if (p.wc_qt != nullptr) {
                const int cm = p.wc_m[c0];
                cached = p.wc_q[c0] == qc && cm > 0 && cm <= m && m - cm <= 32;
            }
            if (p.dbg && lane == 0) {
                atomicAdd(&p.dbg[6], 1ull);
                if (cached) atomicAdd(&p.dbg[7], 1ull);
            }
            if (cached) {
                const int cm = p.wc_m[c0];
                double tsum = lane < m - cm ? p.t[c0 + cm + lane] * p.t[qc + cm + lane] : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
                const double raw = p.wc_qt[c0] + tsum;  // QT_m(c0, qc) = QT_cm + sum_{l=cm}^{m-1} t t
                const double2 c1 = p.pfx1[c0 + m], c2 = p.pfx1[c0], q1 = p.pfx1[qc + m], q2 = p.pfx1[qc];
                const double Sc = (c1.x - c2.x) + (c1.y - c2.y), Sq = (q1.x - q2.x) + (q1.y - q2.y);
                const double mAB = (double)m * A * B;
                acc = raw - A * Sq - B * Sc + mAB;
                delta = Sc - (double)m * A;
                // conversion rounding (the raw value's own accumulated error is the
                // resident term of the statistics band, as for the band-0 rows)
                e_seed = 6.0 * kEps64 * (fabs(raw) + fabs(A * Sq) + fabs(B * Sc) + fabs(mAB));
                e_delta = 6.0 * kEps64 * (fabs(Sc) + fabs((double)m * A));
                if (lane == 0) p.wc_m[c0] = m;
                if (lane == 0) p.wc_qt[c0] = raw;
            } else {
                double raw = 0.0;
                acc = 0.0;
                delta = 0.0;
#pragma unroll 4
                for (int pp = lane; pp < m; pp += 32) {
                    const double tc = p.t[c0 + pp], tq = p.t[qc + pp];
                    const double a = tc - A, w = tq - B;
                    acc = fma(a, w, acc);
                    raw = fma(tc, tq, raw);
                    delta += a;
                    wa = fmax(wa, fabs(a));
                    wb = fmax(wb, fabs(w));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    raw += __shfl_xor_sync(0xffffffffu, raw, o);
                    delta += __shfl_xor_sync(0xffffffffu, delta, o);
                    wa = fmax(wa, __shfl_xor_sync(0xffffffffu, wa, o));
                    wb = fmax(wb, __shfl_xor_sync(0xffffffffu, wb, o));
                }
                e_seed = (double)(m + 8) * kEps64 * (double)m * wa * wb;
                e_delta = (double)(m + 8) * kEps64 * (double)m * wa;
                if (p.wc_qt != nullptr && lane == 0) {
                    p.wc_qt[c0] = raw;
                    p.wc_m[c0] = m;
                    p.wc_q[c0] = qc;
                }
            }
            // ---- walk increments of row s = lane, inclusive prefix scans of the
            // increments and of their magnitudes (the walk's rounding)
            const int q = qc + lane;
            double term = 0.0, dterm = 0.0, sabs = 0.0, dabs = 0.0;
            if (lane >= 1 && mine) {
                const double to = p.t[c - 1] - A, tn = p.t[c + m - 1] - A;
                const double qo = p.t[q - 1] - B, qn = p.t[q + m - 1] - B;
                term = fma(tn, qn, -to * qo);
                dterm = tn - to;
                sabs = fabs(tn * qn) + fabs(to * qo);
                dabs = fabs(tn) + fabs(to);
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double u1 = __shfl_up_sync(0xffffffffu, term, o), u2 = __shfl_up_sync(0xffffffffu, dterm, o);
                const double u3 = __shfl_up_sync(0xffffffffu, sabs, o), u4 = __shfl_up_sync(0xffffffffu, dabs, o);
                if (lane >= o) {
                    term += u1;
                    dterm += u2;
                    sabs += u3;
                    dabs += u4;
                }
            }
            if (alive && p.nrm[q] > 0.f) {
                const double qt = acc + term, dl = delta + dterm;
                const double dmu = p.mu[q] - B;
                const double cov = qt - dmu * dl;
                const double den = (double)m * p.sig[c] * p.sig[q];
                // seed + walk (each increment two roundings, a 6-level scan) + the
                // mean correction + the last operations
                const double ew = (double)(2 * lane + 12) * kEps64;
                const double err = (e_seed + ew * sabs + fabs(dmu) * (e_delta + ew * dabs) +
                                    4.0 * kEps64 * (fabs(qt) + fabs(cov) + fabs(dmu * dl))) /
                                   den;
                kill = cov / den - (err + (cached ? xs_res : xs)) > p.thr0;
            }
            if (kill) {
                peer_kill(p.peers, p.alive, c);
                peer_kill(p.peers, p.alive, q);
                p.wit[c] = kb;                 // (a borrowed witness becomes the row's own)
                p.wit[q] = c - q - kDiag / 2;  // the partner's witness for the next try
            }
            tests += __popc(__ballot_sync(0xffffffffu, alive));
            kills += __popc(__ballot_sync(0xffffffffu, kill));
        }
        // ---- the rest of the run goes to phase 2 (9 diagonals)
        unsigned rest = __ballot_sync(0xffffffffu, alive && !kill);
        if (diag_ok) tests -= __popc(rest);  // counted by phase 2
        if (INLINE2) {
            const int wp = threadIdx.x >> 5;
            while (rest) {
                const int s2 = __ffs(rest) - 1;
                rest &= rest - 1u;
                wit_run9(p, c0 + s2, 1, kb, s_a[wp], s_w[wp], xs, tests, kills);
            }
        } else if (rest) {
            int at = 0;
            if (lane == 0) at = atomicAdd(&p.ctl->wn2, __popc(rest));
            at = __shfl_sync(0xffffffffu, at, 0);
            if ((rest >> lane) & 1u) wl2[at + __popc(rest & ((1u << lane) - 1u))] = make_int2(c, kb);
        }
        if (total <= nwarps) break;  // one run per warp at most: no counter traffic
        if (lane == 0) e = nwarps + atomicAdd(&p.ctl->wrun, 1);
        e = __shfl_sync(0xffffffffu, e, 0);
    }
    if (lane == 0 && tests) {
        atomicAdd(&p.acc[3], tests);
        atomicAdd(&p.acc[4], kills);
    }
}

// Phase 2: the rows phase 1 left, all 9 diagonals of the witness, one warp
// per row (fetched dynamically), windows staged in shared memory.
__global__ void __launch_bounds__(kWitWarps * 32) k_witness9(const ScanParams p, const int2* __restrict__ wl2) {
    pdl_enter();
    __shared__ __align__(16) double s_a[kWitWarps][kWitChunk];
    __shared__ __align__(16) double s_w[kWitWarps][kWitChunk + 16];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const double xs = stats_band(p, false) + kSlack + 1e-12;
    const int total = p.ctl->wn2;
    unsigned long long tests = 0, kills = 0;
    const int nwarps = gridDim.x * kWitWarps;
    for (int e = blockIdx.x * kWitWarps + wp; e < total;) {  // first row by warp index, then a counter
        const int2 r = wl2[e];
        wit_run9(p, r.x, 1, r.y, s_a[wp], s_w[wp], xs, tests, kills);
        if (total <= nwarps) break;
        if (lane == 0) e = nwarps + atomicAdd(&p.ctl->wrun2, 1);
        e = __shfl_sync(0xffffffffu, e, 0);
    }
    if (lane == 0 && tests) {
        atomicAdd(&p.acc[3], tests);
        atomicAdd(&p.acc[4], kills);
    }
}

void launch_witness(const ScanParams& p, int4* wl, int2* wl2, cudaStream_t st) {
    launch_pdl(k_witness_list, std::max(1, std::min((p.N + 255) / 256, 148 * 8)), 256, st, p, wl);
    if (p.N < (1 << 18)) {
        launch_pdl(k_witness<true>, 148 * 2, 256, st, p, (const int4*)wl, wl2);
    } else {
        launch_pdl(k_witness<false>, 148 * 8, 256, st, p, (const int4*)wl, wl2);
        launch_pdl(k_witness9, 148 * 2, kWitWarps * 32, st, p, (const int2*)wl2);
    }
}

// Overflow fallback, the analogue of the reference's full exact pass for a
// candidate whose near-pair list would not stay bounded
// (src/pardrag.cpp:142-149,388-407): every listed row still alive against every
// admissible q by the exact routine.  d < r^2 kills the row; every d lowers its
// exact-nn key.  One warp per pair, dealt over the ranks.
__global__ void __launch_bounds__(kPairWarps * 32) k_exact_rows(const double* __restrict__ t, int m, int N,
                                                                const int* __restrict__ list,
                                                                const TryCtl* __restrict__ ctl, double r_sq,
                                                                uint8_t* alive, unsigned long long* nnkey, int rank,
                                                                int world, const Peers peers) {
    pdl_enter();
    __shared__ double buf[kPairWarps][256];
    const int w = threadIdx.x >> 5;
    const long long tot = (long long)ctl->alive * N;
    for (long long e = ((long long)blockIdx.x * kPairWarps + w) * world + rank; e < tot;
         e += (long long)gridDim.x * kPairWarps * world) {
        const int c = list[e / N], q = (int)(e % N);
        if (abs(c - q) < m || !alive[c]) continue;  // a dead row's nn is not needed
        const double d = ref_dist_warp(t, m, c, q, buf[w]);
        if ((threadIdx.x & 31) == 0) {
            if (d < r_sq) peer_kill(peers, alive, c);
            peer_min_key(peers, nnkey, c, (unsigned long long)__double_as_longlong(d));
        }
    }
}

// ---------------------------------------------------------------------------
// flags / compaction / grouping / survivor kernels.  None of them takes a
// count from the host: counts live in TryCtl, so one DRAG try is a single
// stream-ordered sequence with no host round trip.
constexpr int kSmallGrid = 148 * 2;  // grid-stride kernels over device-sized lists

// try start: every row undecided, counters reset, route maxima cleared
__global__ void k_try_init(uint8_t* __restrict__ alive, unsigned* __restrict__ ymax, unsigned* __restrict__ emax,
                           float* __restrict__ ythr, unsigned long long* __restrict__ nnkey, int N, TryCtl* ctl,
                           unsigned long long* acc, int band_k0) {
    pdl_enter();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        alive[i] = 1;
        ymax[i] = 0u;
        emax[i] = 0u;
        ythr[i] = FLT_MAX;  // collection off unless the row gets exact nn this try
        nnkey[i] = 0x7ff0000000000000ull;  // exact nn^2 (+inf), min-reduced by every exact pair
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->alive = N;
        ctl->prev = N;
        ctl->stop = INT_MAX;
        ctl->G = 0;
        ctl->queue = 0;
        ctl->coll = 0;
        ctl->crange[0] = N;
        ctl->crange[1] = -1;
        ctl->sc = 0;
        ctl->ec = 0;
        ctl->passes = 0;
        ctl->span = 0;
        ctl->stop_why = 0;
        ctl->bK0 = band_k0;
        ctl->bnb = 0;
        ctl->lk = 0.0;
        ctl->wn = 0;
        ctl->wn2 = 0;
        ctl->wrun = 0;
        ctl->wrun2 = 0;
        for (int k = 0; k < 32; ++k) ctl->slotc[k] = 0;
        ctl->tepoch += 1;
        acc[0] = acc[1] = acc[2] = acc[3] = acc[4] = 0ull;
    }
}

__device__ __forceinline__ bool gated_off(const TryCtl* ctl, int gate) {
    if (gate >= 0) return ctl->stop < gate;
    if (gate == kGateTrack) return ctl->tphase >= 2;
    return false;
}

constexpr int kCompactBlock = 1024;
constexpr int kCompactItems = 4;  // flags per thread
constexpr int kCompactTile = kCompactBlock * kCompactItems;
constexpr int kListPath = kCompactTile;  // list-path compaction up to this many previous rows

// block-wide exclusive scan of one int per thread (blockDim.x == 1024); returns
// the exclusive prefix, *total receives the block sum
__device__ __forceinline__ int block_exscan(int v, int* wsum, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int z = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        wsum[lane] = z;
    }
    __syncthreads();
    *total = wsum[(blockDim.x >> 5) - 1];
    return (w ? wsum[w - 1] : 0) + x - v;
}

// Groups of the listed rows for the next scan (single CTA).  Groups are the
// greedy spans of the sorted list: a group starts at a listed row a and takes
// every listed row < a + span.  A gap >= span between consecutive rows always
// starts a new group, so the greedy chain splits into independent segments at
// such gaps and every segment is walked by one thread.  The span minimises
// sum over groups of (2m seed work + 3 per walked row and diagonal).  Dense
// lists (>= 1 row in 64 undecided) take aligned 512-row blocks instead.
constexpr int kSpans = 6;  // 16, 32, ..., 512
// a list is "dense" (whole 512-row blocks, no cost model) only when it is long
// and >= 1 row in 64 is listed; a handful of clustered rows gets small spans
constexpr int kDenseMin = 4096;

// walks the segment starting at list index e (a segment start for `span`);
// calls emit(first_index, last_index) for each group
template <typename F>
__device__ __forceinline__ void walk_segment(const int* __restrict__ list, int cnt, int e, int span, F&& emit) {
    int j = e;
    for (;;) {
        const int g0 = j;
        const int lim = list[j] + span;
        ++j;
        while (j < cnt && list[j] < lim) ++j;
        emit(g0, j - 1);
        if (j >= cnt || list[j] - list[j - 1] >= span) return;
    }
}

constexpr int kGroupStage = 8192;  // list entries staged in smem (32 KB)
// whole-CTA (1024 threads) body; every thread must call it
__device__ void group_body(const int* __restrict__ list_g, const int cnt, int2* __restrict__ groups, TryCtl* ctl,
                           int m, int fixed_span, float seed_w) {
    __shared__ double costs[32][kSpans];
    __shared__ int wsum[32];
    __shared__ int s_span;
    __shared__ int s_list[kGroupStage];
    __syncthreads();  // callers may have used their own smem just before
    if (cnt == 0) {
        if (threadIdx.x == 0) ctl->G = 0;
        return;
    }
    // the greedy walks chase list entries one by one: stage the list in smem
    if (cnt <= kGroupStage) {
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) s_list[e] = list_g[e];
        __syncthreads();
    }
    const int* __restrict__ list = cnt <= kGroupStage ? s_list : list_g;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        int sp = fixed_span;
        if (sp <= 0 && cnt >= kDenseMin && (long long)cnt * 64 >= (long long)(list[cnt - 1] - list[0] + 1))
            sp = -kMaxRows;
        s_span = sp;
    }
    __syncthreads();
    if (s_span < 0) {  // dense: aligned blocks
        const int span = -s_span;
        int carry = 0;
        for (int base = 0; base < cnt; base += blockDim.x) {
            const int e = base + threadIdx.x;
            int r = 0, st = 0, en = 0;
            if (e < cnt) {
                r = list[e];
                st = (e == 0 || list[e - 1] / span != r / span);
                en = (e + 1 == cnt || list[e + 1] / span != r / span);
            }
            int tot;
            const int g = carry + block_exscan(st, wsum, &tot) + st - 1;  // group of entry e
            if (e < cnt) {
                if (st) groups[g].x = r;
                if (en) groups[g].y = r;
            }
            carry += tot;
        }
        if (threadIdx.x == 0) {
            ctl->G = carry;
            ctl->span = span;
        }
        return;
    }
    if (s_span == 0) {
        double c[kSpans];
#pragma unroll
        for (int k = 0; k < kSpans; ++k) c[k] = 0.0;
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            const int gap = e > 0 ? list[e] - list[e - 1] : INT_MAX;
#pragma unroll 1
            for (int k = 0; k < kSpans; ++k) {
                const int span = 16 << k;
                if (gap < span) continue;
                double acc = 0.0;
                walk_segment(list, cnt, e, span, [&](int i0, int i1) {
                    acc += seed_w * m + (double)(list[i1] - list[i0] + 1 + kDiag);
                });
                c[k] += acc;
            }
        }
#pragma unroll
        for (int k = 0; k < kSpans; ++k) {
            double v = c[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) costs[w][k] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double best = 1e300;
            int bs = 64;
            for (int k = 0; k < kSpans; ++k) {
                double v = 0.0;
                for (int x = 0; x < (int)(blockDim.x >> 5); ++x) v += costs[x][k];
                if (v < best) {
                    best = v;
                    bs = 16 << k;
                }
            }
            s_span = bs;
        }
        __syncthreads();
    }
    const int span = s_span;
    int carry = 0;
    for (int base = 0; base < cnt; base += blockDim.x) {
        const int e = base + threadIdx.x;
        const bool seg = e < cnt && (e == 0 || list[e] - list[e - 1] >= span);
        int ng = 0;
        if (seg) walk_segment(list, cnt, e, span, [&](int, int) { ++ng; });
        int tot;
        int g = carry + block_exscan(ng, wsum, &tot);
        if (seg)
            walk_segment(list, cnt, e, span, [&](int i0, int i1) { groups[g++] = make_int2(list[i0], list[i1]); });
        carry += tot;
    }
    if (threadIdx.x == 0) {
        ctl->G = carry;
        ctl->span = span;
    }
}

// One-kernel compaction of the alive flags into the sorted row list
// (decoupled look-back: a CTA's logical index comes from a ticket, so it only
// waits on CTAs that started before it), fused with the grouping of the new
// list for the next scan and, for band passes, the band-loop break rule.
//
// Groups are the non-empty aligned span-blocks of rows (span 16..512; a
// 4096-row compaction tile holds whole span-blocks, so every CTA sees its
// blocks completely).  Each CTA writes the (first, last) alive row of every
// span-block of its tile for all six spans (`slots`) and adds their cost
// sum(2m seed work + 3 per walked row and diagonal) per span; the last CTA to
// finish picks the span (dense lists: 512) and compacts that span's slots
// into the dense group array.
//
// status[] words: epoch (30 bits) | state (2: 1 aggregate, 2 inclusive) |
// value (32), so the array never needs clearing between launches.
__device__ __forceinline__ unsigned long long lb_word(unsigned epoch, unsigned state, unsigned v) {
    return ((unsigned long long)epoch << 34) | ((unsigned long long)state << 32) | v;
}
// offset of span k's slot region (tile b's span-blocks at + b * (256 >> k))
__device__ __forceinline__ long long slot_region(int k, int nb) { return (long long)nb * (512 - (512 >> k)); }

// Tracked-chunk schedule (one thread).  Far chunks start at the end of the
// band passes' coverage and double (at least enough bands to fill one wave of
// the scan grid); when they reach the last diagonal, the near chunk
// [m, kend) follows, for the rows still undecided; then done.
__device__ void track_schedule(TryCtl* ctl, int N, int m, int G, int scan_slots) {
    const long long k_max = (long long)N - 1;
    if (G == 0) {
        ctl->tphase = 2;
        return;
    }
    if (ctl->tphase == 0 && (long long)ctl->tK0 <= k_max) {
        const long long left = (k_max - ctl->tK0 + kW) / kW;
        long long nb = 2ll * ctl->tnb;
        const long long fill = (scan_slots + 2ll * G - 1) / (2ll * G);
        if (fill > nb) nb = fill;
        if (nb < 1) nb = 1;
        ctl->tnb = (int)(nb < left ? nb : left);
        return;
    }
    if (ctl->tphase == 0 && ctl->kend > m) {
        ctl->tphase = 1;
        ctl->tK0 = m;
        ctl->tnb = (int)(((long long)ctl->kend - m + kW - 1) / kW);
        return;
    }
    ctl->tphase = 2;
}

// after the chunk that just ran: advance, then schedule the next one
__device__ void track_next(TryCtl* ctl, int N, int m, int G, int scan_slots) {
    ctl->tpasses += 1;
    if (ctl->tphase == 1) {
        ctl->tphase = 2;
        return;
    }
    ctl->tK0 += ctl->tnb * kW;
    track_schedule(ctl, N, m, G, scan_slots);
}

__global__ void k_track_init(TryCtl* ctl, int N, int m, int bands_ran, int scan_slots) {
    pdl_enter();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ctl->kend = bands_ran ? ctl->bK0 : m;
    ctl->tK0 = ctl->kend;
    ctl->tnb = 0;
    ctl->tphase = 0;
    ctl->tpasses = 0;
    track_schedule(ctl, N, m, ctl->alive == 0 ? 0 : ctl->G, scan_slots);
}

// Finalisation of one compaction (the last CTA of the sweep, or the single
// CTA of the list path): break rule, span choice, groups, next-pass bands.
// s_cost[0][k] holds the total grouping cost of span 16 << k; list_only forces
// the groups straight from the list (the list path fills no span-block slots).
__device__ __forceinline__ void compact_finalize(int total, TryCtl* ctl, int gate, const int* __restrict__ out,
                                                 int2* __restrict__ groups, const int2* __restrict__ slots,
                                                 int nb, int n, int m, int fixed_span, float band_keep,
                                                 int scan_slots, int band_few, double (*s_cost)[kSpans],
                                                 int* wsum, int& s_k, bool list_only) {
    if (threadIdx.x == 0) {
        ctl->cticket = 0;
        ctl->cdone = 0;
        if (gate >= 0) {
            const int prev = ctl->alive;
            ctl->prev = prev;
            ctl->passes = gate + 1;
            if (total == 0 || total <= band_few) {
                ctl->stop = gate;
                ctl->stop_why = 1;
            } else if ((double)total > (double)band_keep * (double)prev) {
                ctl->stop = gate;
                ctl->stop_why = 2;
            }
            // next band pass (gate + 1): starts where this one ended
            if (gate >= 1) ctl->bK0 += ctl->bnb * kW;
        }
        ctl->alive = total;
        int k = 5;  // dense lists (>= 1 row in 64 undecided): whole 512-row blocks
        if (fixed_span > 0) {
            k = 0;
            while (k < 5 && (16 << k) < fixed_span) ++k;
        } else if (total > 0 && (total < kDenseMin ||
                                 (long long)total * 64 < (long long)(__ldcg(&out[total - 1]) - __ldcg(&out[0]) + 1))) {
            double best = 1e300;
            for (int x = 0; x < kSpans; ++x) {
                const double v = s_cost[0][x];
                if (v < best) {
                    best = v;
                    k = x;
                }
            }
        }
        s_k = k;
        ctl->span = 16 << k;
    }
    __syncthreads();
    const int k = s_k;
    const int nslot = nb * (256 >> k);
    int carry = 0;
    if (list_only || total <= nslot) {
        // short list (the usual case after pass 0): the groups straight from the
        // list — an entry starts a group when its span-block differs from its
        // predecessor's — instead of a sweep over every span-block slot
        const int sh = 4 + k;
        for (int b0 = 0; b0 < total; b0 += blockDim.x) {
            const int e = b0 + threadIdx.x;
            int r = 0, st = 0, en = 0;
            if (e < total) {
                r = __ldcg(&out[e]);
                st = e == 0 || (__ldcg(&out[e - 1]) >> sh) != (r >> sh);
                en = e + 1 == total || (__ldcg(&out[e + 1]) >> sh) != (r >> sh);
            }
            int t2;
            const int g = carry + block_exscan(st, wsum, &t2) + st - 1;
            if (e < total) {
                if (st) groups[g].x = r;
                if (en) groups[g].y = r;
            }
            carry += t2;
        }
    } else {
        const int2* sl = slots + slot_region(k, nb);
        for (int b0 = 0; b0 < nslot; b0 += blockDim.x) {
            const int e = b0 + threadIdx.x;
            int2 v = make_int2(0, -1);
            if (e < nslot) v = __ldcg(&sl[e]);
            const int ff = v.y >= 0 ? 1 : 0;
            int t2;
            const int p2 = carry + block_exscan(ff, wsum, &t2);
            if (ff) groups[p2] = v;
            carry += t2;
        }
    }
    if (threadIdx.x == 0) {
        ctl->G = carry;
        if (gate == kGateTrack) track_next(ctl, n, m, carry, scan_slots);
        if (gate >= 0 && ctl->stop == INT_MAX) {
            // Bands of the next pass: at least 2^p (the doubling schedule), and
            // enough to fill one wave of the persistent scan grid — a pass with
            // fewer tiles than CTAs costs one tile's latency anyway, so the
            // extra bands come free and kill more rows before the full rows.
            const long long k_max = (long long)n - 1, K0 = ctl->bK0;
            const long long left = K0 <= k_max ? (k_max - K0 + kW) / kW : 0;
            if (left <= 0 || carry == 0) {
                ctl->stop = gate;
                ctl->stop_why = 1;
            } else {
                long long nb = 1ll << min(gate + 1, 5);
                const long long fill = (scan_slots + 2ll * carry - 1) / (2ll * carry);
                if (fill > nb) nb = fill;
                ctl->bnb = (int)(nb < left ? nb : left);
            }
        }
    }
}

__global__ void __launch_bounds__(1024) k_compact_group(const uint8_t* __restrict__ a, int n, int* __restrict__ out,
                                                        unsigned long long* status, unsigned epoch, TryCtl* ctl,
                                                        int gate, int2* __restrict__ groups,
                                                        int2* __restrict__ slots, int m, int fixed_span,
                                                        float band_keep, int scan_slots, int band_few,
                                                        float seed_w, double* __restrict__ bcost) {
    pdl_enter();
    if (gated_off(ctl, gate)) return;
    __shared__ int s_bid, s_excl, s_last, s_k;
    __shared__ int wsum[32];
    __shared__ int s_fa[32], s_la[32];
    __shared__ int2 s_lb[32];
    __shared__ double s_cost[32][kSpans];
    const int nb = gridDim.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // List path: after band pass >= 1 the undecided rows are a subset of the
    // previous compaction's list (rows only die within a try), so a short list
    // is filtered in one CTA instead of sweeping all n flags.  (The list size
    // only shrinks, so a CTA starting after CTA 0 finished still takes it.)
    if (gate >= 1 && ctl->alive <= kListPath) {
        if (blockIdx.x != 0) return;
        __shared__ int s_l[kListPath];
        const int prev = ctl->alive;
        int rr[kCompactItems], ff[kCompactItems], cnt = 0;
#pragma unroll
        for (int k = 0; k < kCompactItems; ++k) {
            const int e = threadIdx.x * kCompactItems + k;
            rr[k] = e < prev ? out[e] : 0;
            ff[k] = (e < prev && a[rr[k]]) ? 1 : 0;
            cnt += ff[k];
        }
        int tot;
        int pos = block_exscan(cnt, wsum, &tot);
#pragma unroll
        for (int k = 0; k < kCompactItems; ++k)
            if (ff[k]) s_l[pos++] = rr[k];
        __syncthreads();
        const double cm = (double)seed_w * (double)m + (double)(1 + kDiag);
        double c6[kSpans];
#pragma unroll
        for (int k = 0; k < kSpans; ++k) c6[k] = 0.0;
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
            const int r = s_l[e];
            out[e] = r;
            const int rp = e > 0 ? s_l[e - 1] : -1, rn = e + 1 < tot ? s_l[e + 1] : -1;
#pragma unroll
            for (int k = 0; k < kSpans; ++k) {
                const int sh = 4 + k;
                const bool st = e == 0 || (rp >> sh) != (r >> sh);
                const bool en = e + 1 == tot || (rn >> sh) != (r >> sh);
                // per span-block: cm + last - first (as the sweep's per-block costs)
                c6[k] += (st ? cm - (double)r : 0.0) + (en ? (double)r : 0.0);
            }
        }
#pragma unroll
        for (int k = 0; k < kSpans; ++k) {
            double v = c6[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) s_cost[w][k] = v;
        }
        __syncthreads();
        if (threadIdx.x < kSpans) {
            double v = 0.0;
            for (int x = 0; x < 32; ++x) v += s_cost[x][threadIdx.x];
            s_cost[0][threadIdx.x] = v;
        }
        __syncthreads();
        compact_finalize(tot, ctl, gate, out, groups, slots, nb, n, m, fixed_span, band_keep, scan_slots, band_few,
                         s_cost, wsum, s_k, true);
        return;
    }
    if (threadIdx.x == 0) s_bid = atomicAdd(&ctl->cticket, 1);
    __syncthreads();
    const int bid = s_bid;
    const int base = bid * kCompactTile;
    const int i0 = base + threadIdx.x * kCompactItems;
    int f[kCompactItems];
    int c = 0;
    if (i0 + kCompactItems <= n) {
        const uchar4 v = *reinterpret_cast<const uchar4*>(a + i0);
        f[0] = v.x != 0;
        f[1] = v.y != 0;
        f[2] = v.z != 0;
        f[3] = v.w != 0;
    } else {
#pragma unroll
        for (int k = 0; k < kCompactItems; ++k) f[k] = (i0 + k < n && a[i0 + k]) ? 1 : 0;
    }
    int fa = INT_MAX, la = -1;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        c += f[k];
        if (f[k]) {
            fa = min(fa, i0 + k);
            la = i0 + k;
        }
    }
    // ---- span-blocks: spans 16..128 within a warp, 256 / 512 across warps
    {
        const double cm = (double)seed_w * (double)m + (double)(1 + kDiag);
        int mn = fa, mx = la;
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        double cst[kSpans];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int o = 2 << k;  // lanes reduced so far: o; after this step 2*o = 4 << k = span / 4
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            cst[k] = 0.0;
            if ((lane & ((4 << k) - 1)) == 0) {
                const int j = threadIdx.x >> (2 + k);
                slots[slot_region(k, nb) + (long long)bid * (256 >> k) + j] = make_int2(mn, mx);
                if (mx >= 0) cst[k] = cm + (double)(mx - mn);
            }
        }
        if (lane == 0) {
            s_fa[w] = mn;
            s_la[w] = mx;
        }
        __syncthreads();
        cst[4] = cst[5] = 0.0;
        if (threadIdx.x < 16) {  // span 256: 2 warps each
            const int j = threadIdx.x;
            const int x = min(s_fa[2 * j], s_fa[2 * j + 1]), y = max(s_la[2 * j], s_la[2 * j + 1]);
            slots[slot_region(4, nb) + (long long)bid * 16 + j] = make_int2(x, y);
            if (y >= 0) cst[4] = cm + (double)(y - x);
        } else if (threadIdx.x >= 32 && threadIdx.x < 40) {  // span 512: 4 warps each
            const int j = threadIdx.x - 32;
            const int x = min(min(s_fa[4 * j], s_fa[4 * j + 1]), min(s_fa[4 * j + 2], s_fa[4 * j + 3]));
            const int y = max(max(s_la[4 * j], s_la[4 * j + 1]), max(s_la[4 * j + 2], s_la[4 * j + 3]));
            slots[slot_region(5, nb) + (long long)bid * 8 + j] = make_int2(x, y);
            if (y >= 0) cst[5] = cm + (double)(y - x);
        }
#pragma unroll
        for (int k = 0; k < kSpans; ++k) {
            double v = cst[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) s_cost[w][k] = v;
        }
        __syncthreads();
        if (threadIdx.x < kSpans) {  // per-CTA partials: no atomic contention on 6 words
            double v = 0.0;
            for (int x = 0; x < 32; ++x) v += s_cost[x][threadIdx.x];
            bcost[bid * kSpans + threadIdx.x] = v;
        }
    }
    // ---- compaction (decoupled look-back).  Every thread examines one
    // predecessor (thread i: CTA bid-1-i), so one round of loads covers 1024
    // predecessors; each warp sums its values up to its nearest inclusive
    // prefix, and the warps combine in order.  The words carry only counts:
    // relaxed GPU-scope stores and loads suffice.
    int tot;
    const int ex = block_exscan(c, wsum, &tot);
    if (threadIdx.x == 0) {
        st_relaxed_u64(&status[bid], lb_word(epoch, bid == 0 ? 2u : 1u, (unsigned)tot));
        if (bid == 0) s_excl = 0;
    }
    if (bid > 0) {
        int excl = 0;
        for (int j0 = bid - 1;; j0 -= (int)blockDim.x) {
            const int idx = j0 - (int)threadIdx.x;
            unsigned state = 2u, val = 0u;  // before CTA 0: an inclusive zero
            if (idx >= 0) {
                unsigned long long wv;
                do {
                    wv = ld_relaxed_u64(&status[idx]);
                } while ((unsigned)(wv >> 34) != (epoch & 0x3fffffffu) || ((wv >> 32) & 3u) == 0u);
                state = (unsigned)(wv >> 32) & 3u;
                val = (unsigned)wv;
            }
            const unsigned incl = __ballot_sync(0xffffffffu, state == 2u);
            const int L = incl ? __ffs(incl) - 1 : 31;
            const unsigned part = __reduce_add_sync(0xffffffffu, lane <= L ? val : 0u);
            if (lane == 0) s_lb[w] = make_int2(incl != 0u, (int)part);
            __syncthreads();
            bool found = false;
            for (int x = 0; x < (int)(blockDim.x >> 5); ++x) {
                const int2 v = s_lb[x];
                excl += v.y;
                if (v.x) {
                    found = true;
                    break;
                }
            }
            if (found) break;
            __syncthreads();  // s_lb is rewritten by the next window
        }
        if (threadIdx.x == 0) {
            st_relaxed_u64(&status[bid], lb_word(epoch, 2u, (unsigned)(excl + tot)));
            s_excl = excl;
        }
    }
    __syncthreads();
    int pos = s_excl + ex;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        if (f[k]) out[pos++] = i0 + k;
    }
    if (bid == nb - 1 && threadIdx.x == 0) ctl->ctotal = s_excl + tot;
    // ---- the last CTA to finish sees every scatter, slot and cost: it finalises
    __syncthreads();
    if (threadIdx.x == 0) s_last = atom_add_acq_rel(&ctl->cdone, 1) == nb - 1;
    __syncthreads();
    if (!s_last) return;
    const int total = *(volatile int*)&ctl->ctotal;
    {  // span costs: sum of the per-CTA partials
        double c6[kSpans];
#pragma unroll
        for (int k = 0; k < kSpans; ++k) c6[k] = 0.0;
        for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
            for (int k = 0; k < kSpans; ++k) c6[k] += __ldcg(&bcost[b * kSpans + k]);
#pragma unroll
        for (int k = 0; k < kSpans; ++k) {
            double v = c6[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) s_cost[w][k] = v;
        }
        __syncthreads();
        if (threadIdx.x < kSpans) {
            double v = 0.0;
            for (int x = 0; x < 32; ++x) v += s_cost[x][threadIdx.x];
            s_cost[0][threadIdx.x] = v;  // row 0 read by thread 0 below (after its own partial)
        }
        __syncthreads();
    }
    compact_finalize(total, ctl, gate, out, groups, slots, nb, n, m, fixed_span, band_keep, scan_slots, band_few,
                     s_cost, wsum, s_k, false);
}

// per-survivor interval [lo, hi] of the exact nn^2 from the tracked route maxima
// (constant rows: the exact convention value)
__device__ __forceinline__ void nn_interval(int c, const unsigned* ymax, const unsigned* emax, const float* nrm,
                                            const int* const_range, int N, int m, double& l, double& h) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const double two_m = 2.0 * (double)m;
    const float cn = nrm[c];
    l = 0.0;
    h = inf;
    if (cn == 0.f) {
        const int a = const_range[0], b = const_range[1];
        double d = inf;
        if (c - a >= m || b - c >= m) d = 0.0;
        else if (c - m >= 0 || c + m <= N - 1) d = two_m;
        l = h = d;
    } else if (ymax[c] > 1u) {
        const double x = (double)key2f(ymax[c]);
        const double ee = (double)__uint_as_float(emax[c]);
        const double slack = 1e-6 + 1e-9;
        l = two_m * (1.0 - ((x + ee) * (double)cn + slack));
        h = two_m * (1.0 - ((x - ee) * (double)cn - slack));
        if (l < 0.0) l = 0.0;
    }
}

__device__ __forceinline__ unsigned long long dkey(double d) {  // order-preserving
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Decodes the per-length constant-row range written by k_derive
// (cr[0] = max(N - i), cr[1] = max(i + 1) over constant rows i; 0 = none).
__device__ __forceinline__ void crange_decode(const int* cr, int N, int out[2]) {
    out[0] = N - cr[0];
    out[1] = cr[1] - 1;
}

// The survivors stage of a try in one CTA (1024 threads):
//   1. survivors = the listed rows still alive after full rows + knife edges
//      (order-preserving filter of the pre-full-rows list) -> ctl->sc;
//   2. MERLIN (need > 0): keep the rows whose nn interval reaches the need-th
//      largest lower bound (rank count for small lists, MSB radix select
//      otherwise) -> ctl->ec;
//   3. reset their exact-nn keys (constant rows: the convention value) and
//      collection thresholds;
//   4. group them for the collection scan.
__global__ void __launch_bounds__(1024) k_survivors(const int* __restrict__ list, const uint8_t* __restrict__ alive,
                                                    TryCtl* ctl, const unsigned* __restrict__ ymax,
                                                    const unsigned* __restrict__ emax,
                                                    const float* __restrict__ nrm, const int* __restrict__ cr_raw,
                                                    int N, int m, int need, double* __restrict__ lo,
                                                    double* __restrict__ hi, int* __restrict__ cand,
                                                    float* __restrict__ ythr, unsigned long long* __restrict__ nnkey,
                                                    int2* __restrict__ groups, int fixed_span, float seed_w,
                                                    int* __restrict__ exli, int* __restrict__ surv) {
    pdl_enter();
    __shared__ int wsum[32];
    __shared__ int hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ int s_rem;
    __shared__ double s_lk;
    int cr[2];
    crange_decode(cr_raw, N, cr);
    const int cnt = ctl->alive;
    // 1. survivors
    int sc = 0;
    for (int base = 0; base < cnt; base += blockDim.x) {
        const int e = base + threadIdx.x;
        const int r = e < cnt ? list[e] : 0;
        const int f = (e < cnt && alive[r]) ? 1 : 0;
        int tot;
        const int pos = sc + block_exscan(f, wsum, &tot);
        if (f) {
            cand[pos] = r;
            if (surv) surv[pos] = r;  // every survivor (the row cache's anchors)
            if (exli) exli[r] = e;  // list index: the collection's per-(row, band) bounds
        }
        sc += tot;
    }
    __syncthreads();
    int ec = sc;
    // 2. top-k filter (the nn intervals come from the FP32 route maxima over
    // regular q only: with degenerate rows present every survivor gets exact nn)
    if (need > 0 && sc > need && cr_raw[2] == 0) {
        for (int e = threadIdx.x; e < sc; e += blockDim.x) {
            double l, h;
            nn_interval(cand[e], ymax, emax, nrm, cr, N, m, l, h);
            lo[e] = l;
            hi[e] = h;
        }
        __syncthreads();
        if (sc <= (int)blockDim.x) {
            const int e = threadIdx.x;
            if (e < sc) {
                const double v = lo[e];
                int gt = 0, ge = 0;
                for (int x = 0; x < sc; ++x) {
                    const double u = lo[x];
                    gt += u > v;
                    ge += u >= v;
                }
                if (gt < need && need <= ge) s_lk = v;  // every writer holds the same value
            }
        } else {
            if (threadIdx.x == 0) {
                s_prefix = 0ull;
                s_rem = need;
            }
            __syncthreads();
            for (int shift = 56; shift >= 0; shift -= 8) {
                for (int x = threadIdx.x; x < 256; x += blockDim.x) hist[x] = 0;
                __syncthreads();
                const unsigned long long pre = s_prefix;
                const unsigned long long hmask = shift == 56 ? 0ull : (~0ull << (shift + 8));
                for (int e = threadIdx.x; e < sc; e += blockDim.x) {
                    const unsigned long long k = dkey(lo[e]);
                    if ((k & hmask) == pre) atomicAdd(&hist[(k >> shift) & 255], 1);
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    int rem = s_rem, d = 255;
                    for (; d > 0; --d) {
                        if (hist[d] >= rem) break;
                        rem -= hist[d];
                    }
                    s_rem = rem;
                    s_prefix = pre | ((unsigned long long)d << shift);
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                const unsigned long long kk = s_prefix;
                s_lk = __longlong_as_double((long long)((kk >> 63) ? (kk & 0x7fffffffffffffffull) : ~kk));
            }
        }
        __syncthreads();
        const double lk = s_lk;
        // in-place order-preserving filter (an entry moves only to a lower index)
        ec = 0;
        for (int base = 0; base < sc; base += blockDim.x) {
            const int e = base + threadIdx.x;
            const int r = e < sc ? cand[e] : 0;
            const int f = (e < sc && hi[e] >= lk) ? 1 : 0;
            int tot;
            const int pos = ec + block_exscan(f, wsum, &tot);  // syncs: every read precedes the writes
            if (f) cand[pos] = r;
            ec += tot;
        }
        if (threadIdx.x == 0) ctl->lk = lk;
    }
    __syncthreads();
    // 3. exact-nn keys and collection thresholds.  The tracked max route value
    // x* and the row's largest tile error term e give a lower bound x* - e of
    // the row's true best corr / cn; every q whose upper bound x + E*qn reaches
    // it may be the reference's minimiser.
    for (int e = threadIdx.x; e < ec; e += blockDim.x) {
        const int c = cand[e];
        if (nrm[c] == 0.f) continue;  // degenerate: exact nn from k_recheck, never collected
        const unsigned k = ymax[c];
        float th = -FLT_MAX;  // no tracked data: collect everything
        if (k > 1u) {
            const float l = key2f(k) - __uint_as_float(emax[c]);
            // two ulps down: FP64 rounding of near-ties can never exclude the minimiser
            th = nextafterf(nextafterf(l - fabsf(l) * 2.4e-7f, -FLT_MAX), -FLT_MAX);
        }
        ythr[c] = th;
    }
    if (threadIdx.x == 0) {
        ctl->sc = sc;
        ctl->ec = ec;
    }
    // 4. groups of the rows that get exact distances
    group_body(cand, ec, groups, ctl, m, fixed_span, seed_w);
}

__global__ void k_gather_nn(const int* __restrict__ list, const int* __restrict__ cnt_p,
                            const unsigned long long* __restrict__ nnkey, double* __restrict__ out) {
    pdl_enter();
    const int cnt = *cnt_p;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x)
        out[e] = __longlong_as_double((long long)nnkey[list[e]]);
}

// ---------------------------------------------------------------------------
// Resident band-0 seed rows (north_star (a)): tile b = 2*j + side holds the raw
// dot products QT(i, i+k) of row i = j*L (side 0, k = kA + u) or i = j*L + L - 1
// (side 1, k = -kA - u), u in [0, kW).  Initialised once at the first length,
// then carried m -> m+1 with QT_{m+1}(i,q) = QT_m(i,q) + t[i+m] t[q+m].
__device__ __forceinline__ bool seed_pair(int b, int u, int L, int kA, int N, int& i, int& q) {
    const int j = b >> 1;
    i = (b & 1) ? j * L + L - 1 : j * L;
    q = (b & 1) ? i - kA - u : i + kA + u;
    return i < N && q >= 0 && q < N;
}

__global__ void k_seed_init(const double* __restrict__ t, int n, int m, int L, int kA, int nb, int bstep, int ustep,
                            double* __restrict__ qt) {
    const int N = n - m + 1;
    const long long total = (long long)nb * kW;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(e / kW);
        if (b % bstep) continue;  // rows the pair-kill walk never reads
        int i, q;
        double s = 0.0;
        if ((int)(e % kW) % ustep == 0 && seed_pair(b, (int)(e % kW), L, kA, N, i, q))  // ... and entries
            for (int k = 0; k < m; ++k) s = fma(t[i + k], t[q + k], s);
        qt[e] = s;
    }
}

__global__ void k_seed_advance(const double* __restrict__ t, int n, int m, int L, int kA, int nb, int bstep,
                               int ustep, double* __restrict__ qt) {
    pdl_enter();
    const int N1 = n - m;  // subsequence count of length m+1
    const long long total = (long long)nb * kW;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(e / kW);
        if (b % bstep || (int)(e % kW) % ustep) continue;
        int i, q;
        if (seed_pair(b, (int)(e % kW), L, kA, N1, i, q)) qt[e] = fma(t[i + m], t[q + m], qt[e]);
    }
}

// Row cache: QT(a, q) = sum_{p<m} t[a+p] t[q+p] for every q < N (FP64, m FMA
// each; 9 consecutive q per thread slide through registers over windows
// staged in shared memory, as in seed_fp64), and its length
// recurrence QT_{m+1}(a, q) = QT_m(a, q) + t[a+m] t[q+m] for every valid slot.
__global__ void __launch_bounds__(kThreads) k_rc_fill(const double* __restrict__ t, int n, int m, int a,
                                                     double* __restrict__ qt) {
    pdl_enter();
    __shared__ double sa[kSeedChunk];
    __shared__ double sw[kW + kSeedChunk];
    const int tid = threadIdx.x;
    const int N = n - m + 1;
    const int o_t = tid * kDiag;  // this thread's 9 q of the tile (odd stride: conflict-free)
    for (int q_lo = blockIdx.x * kW; q_lo < N; q_lo += gridDim.x * kW) {
        double acc[kDiag];
#pragma unroll
        for (int i = 0; i < kDiag; ++i) acc[i] = 0.0;
        for (int pc = 0; pc < m; pc += kSeedChunk) {
            const int len = min(kSeedChunk, m - pc);
            __syncthreads();
            for (int x = tid; x < len; x += kThreads) sa[x] = t[a + pc + x];
            for (int x = tid; x < kW + len - 1; x += kThreads) {
                const int g = q_lo + pc + x;
                sw[x] = g < n ? t[g] : 0.0;
            }
            __syncthreads();
            double w[kDiag];
#pragma unroll
            for (int i = 0; i < kDiag - 1; ++i) w[i] = sw[o_t + i];
            int pp = 0;
            for (; pp + kDiag <= len; pp += kDiag) {
#pragma unroll
                for (int uu = 0; uu < kDiag; ++uu) {
                    w[(uu + kDiag - 1) % kDiag] = sw[o_t + pp + uu + kDiag - 1];
                    const double av = sa[pp + uu];
#pragma unroll
                    for (int i = 0; i < kDiag; ++i) acc[i] = fma(av, w[(uu + i) % kDiag], acc[i]);
                }
            }
            for (; pp < len; ++pp) {
                const double av = sa[pp];
#pragma unroll
                for (int i = 0; i < kDiag; ++i) acc[i] = fma(av, sw[o_t + pp + i], acc[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < kDiag; ++i)
            if (q_lo + o_t + i < N) qt[q_lo + o_t + i] = acc[i];
    }
}

__global__ void k_rc_advance(const double* __restrict__ t, int n, int m, RcRows rows, long long stride,
                             double* __restrict__ qt) {
    pdl_enter();
    const int N1 = n - m;  // subsequence count of length m+1
    for (int sl = blockIdx.y; sl < rows.n; sl += gridDim.y) {
        const int a = rows.row[sl];
        if (a < 0 || a >= N1) continue;
        const double x = t[a + m];
        double* q = qt + (size_t)sl * (size_t)stride;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N1; i += gridDim.x * blockDim.x)
            q[i] = fma(x, t[i + m], q[i]);
    }
}

void launch_rc_fill(const double* t, int n, int m, int a, double* qt, cudaStream_t st) {
    launch_pdl(k_rc_fill, std::max(1, std::min((n + kW - 1) / kW, 148 * 6)), kThreads, st, t, n, m, a, qt);
}

void launch_rc_advance(const double* t, int n, int m, const RcRows& rows, long long stride, double* qt,
                       cudaStream_t st) {
    launch_pdl(k_rc_advance, dim3(148 * 2, rows.n > 0 ? rows.n : 1), 256, st, t, n, m, rows, stride, qt);
}

void launch_seed_init(const double* t, int n, int m, int L, int kA, int nb, int bstep, int ustep, double* qt, cudaStream_t st) {
    k_seed_init<<<148 * 8, 256, 0, st>>>(t, n, m, L, kA, nb, bstep, ustep, qt);
}

void launch_seed_advance(const double* t, int n, int m, int L, int kA, int nb, int bstep, int ustep, double* qt,
                         cudaStream_t st) {
    launch_pdl(k_seed_advance, 148 * 8, 256, st, t, n, m, L, kA, nb, bstep, ustep, qt);
}

static int grid_for(long long work, int threads) {
    long long b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

size_t scan_smem_bytes() { return sizeof(ScanSmem<kPruneTrack>); }

void scan_configure() {
    // the walk kernels want the largest shared-memory carveout (6 CTAs x 33 KB)
    cudaFuncSetAttribute(k_scan<kPrune>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_scan<kPruneTrack>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_scan<kCollect>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

// persistent scan: one CTA per resident slot (occupancy of each mode)
static int g_scan_grid[3] = {0, 0, 0};

template <int MODE>
static int scan_grid() {
    if (g_scan_grid[MODE] == 0) {
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scan<MODE>, kThreads, 0);
        if (const char* e = std::getenv("TSD_SCAN_CTAS")) per = std::min(per, std::max(1, std::atoi(e)));
        g_scan_grid[MODE] = sms * (per > 0 ? per : 1);
    }
    return g_scan_grid[MODE];
}

static int g_pair_grid = 0;

int band0_pair_slots() {
    if (g_pair_grid == 0) {
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int bytes = (int)sizeof(PairSmem);
        cudaFuncSetAttribute(k_band0_pair<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pair<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pair<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pair<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pair<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pair<3>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_band0_pair<3>, kThreads, bytes);
        if (const char* e = std::getenv("TSD_SCAN_CTAS")) per = std::min(per, std::max(1, std::atoi(e)));
        g_pair_grid = sms * (per > 0 ? per : 1);
    }
    return g_pair_grid;
}

static int g_pk_grid = 0;

int band0_pk_slots() {
    if (g_pk_grid == 0) {
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int bytes = (int)sizeof(PkSmem);
        cudaFuncSetAttribute(k_band0_pk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pk<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pk<3>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pk<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<6>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pk<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<9>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pk<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<12>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pk<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<20>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(k_band0_pk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_band0_pk<16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_band0_pk<3>, kThreads, bytes);
        if (const char* e = std::getenv("TSD_SCAN_CTAS")) per = std::min(per, std::max(1, std::atoi(e)));
        g_pk_grid = sms * (per > 0 ? per : 1);
    }
    return g_pk_grid;
}

static void launch_band0_pk(const ScanParams& p, cudaStream_t st) {
    const int grid = band0_pk_slots();
    const size_t bytes = sizeof(PkSmem);
    if (p.half == 2) launch_pdl_smem(k_band0_pk<2>, grid, kThreads, bytes, st, p);
    else if (p.half == 12) launch_pdl_smem(k_band0_pk<12>, grid, kThreads, bytes, st, p);
    else if (p.half == 20) launch_pdl_smem(k_band0_pk<20>, grid, kThreads, bytes, st, p);
    else if (p.half == 16) launch_pdl_smem(k_band0_pk<16>, grid, kThreads, bytes, st, p);
    else if (p.half >= 9) launch_pdl_smem(k_band0_pk<9>, grid, kThreads, bytes, st, p);
    else if (p.half >= 6) launch_pdl_smem(k_band0_pk<6>, grid, kThreads, bytes, st, p);
    else if (p.half >= 3) launch_pdl_smem(k_band0_pk<3>, grid, kThreads, bytes, st, p);
    else launch_pdl_smem(k_band0_pk<1>, grid, kThreads, bytes, st, p);
}

static void launch_band0_pair(const ScanParams& p, cudaStream_t st) {
    const int grid = band0_pair_slots();
    const size_t bytes = sizeof(PairSmem);
    if (p.half == 2) launch_pdl_smem(k_band0_pair<2>, grid, kThreads, bytes, st, p);
    else if (p.half >= 3) launch_pdl_smem(k_band0_pair<3>, grid, kThreads, bytes, st, p);
    else launch_pdl_smem(k_band0_pair<1>, grid, kThreads, bytes, st, p);
}

void launch_scan(int mode, const ScanParams& p, cudaStream_t st) {
    switch (mode) {
        case kPrune:
            if (p.space == kSpaceSeed && p.pair == 2) {  // every pair of band 0 once, both ends killed
                launch_band0_pk(p, st);
                break;
            }
            if (p.space == kSpaceSeed && p.pair) {  // both sides of band 0 in one walk
                launch_band0_pair(p, st);
                break;
            }
            if (p.half == 20) launch_pdl(k_scan<kPrune, 20>, scan_grid<kPrune>(), kThreads, st, p);
            else if (p.half == 2) launch_pdl(k_scan<kPrune, 2>, scan_grid<kPrune>(), kThreads, st, p);
            else if (p.half >= 6) launch_pdl(k_scan<kPrune, 6>, scan_grid<kPrune>(), kThreads, st, p);
            else if (p.half >= 3) launch_pdl(k_scan<kPrune, 3>, scan_grid<kPrune>(), kThreads, st, p);
            else launch_pdl(k_scan<kPrune>, scan_grid<kPrune>(), kThreads, st, p);
            break;
        case kPruneTrack: launch_pdl(k_scan<kPruneTrack>, scan_grid<kPruneTrack>(), kThreads, st, p); break;
        default: launch_pdl(k_scan<kCollect>, scan_grid<kCollect>(), kThreads, st, p); break;
    }
}

void launch_exact_rows(const double* t, int m, int N, const int* list, const TryCtl* ctl, double r_sq,
                       uint8_t* alive, unsigned long long* nnkey, int rank, int world, const Peers& peers,
                       cudaStream_t st) {
    launch_pdl(k_exact_rows, 148 * 4, kPairWarps * 32, st, t, m, N, list, ctl, r_sq, alive, nnkey, rank, world,
               peers);
}

void launch_ref_pairs(int mode, const double* t, int m, const int2* pairs, const int* count, int cap,
                      double r_sq, uint8_t* alive, unsigned long long* nnkey, TryCtl* ctl, const int* ex,
                      double* nnout, const Peers& peers, cudaStream_t st) {
    const int blocks = 148 * 4;  // grid-stride over the device-side pair count
    if (mode == 0)
        launch_pdl(k_ref_pairs<0>, blocks, kPairWarps * 32, st, t, m, pairs, count, cap, r_sq, alive, nnkey, ctl,
                   (const int*)nullptr, (double*)nullptr, peers);
    else
        launch_pdl(k_ref_pairs<1>, blocks, kPairWarps * 32, st, t, m, pairs, count, cap, r_sq, alive, nnkey, ctl, ex,
                   nnout, peers);
}

void launch_recheck(const double* t, int m, int N, const int2* pairs, const int* count, int cap, const int* list,
                    const TryCtl* ctl, const int* crange, const int* degc, const int* deg2, const float* nrm,
                    double r_sq, uint8_t* alive, unsigned long long* nnkey, int rank, int world, const Peers& peers,
                    int* wit, cudaStream_t st) {
    launch_pdl(k_recheck, 148 * 4, kPairWarps * 32, st, t, m, N, pairs, count, cap, list, ctl, crange, degc, deg2,
               nrm, r_sq, alive, nnkey, rank, world, peers, wit);
}

void launch_survivors(const int* list, const uint8_t* alive, TryCtl* ctl, const unsigned* ymax,
                      const unsigned* emax, const float* nrm, const int* crange, int N, int m, int need,
                      double* lo, double* hi, int* cand, float* ythr, unsigned long long* nnkey, int2* groups,
                      int fixed_span, float seed_w, int* exli, int* surv, cudaStream_t st) {
    launch_pdl(k_survivors, 1, 1024, st, list, alive, ctl, ymax, emax, nrm, crange, N, m, need, lo, hi, cand, ythr,
               nnkey, groups, fixed_span, seed_w, exli, surv);
}

void launch_try_init(uint8_t* alive, unsigned* ymax, unsigned* emax, float* ythr, unsigned long long* nnkey, int N,
                     TryCtl* ctl, unsigned long long* acc, int band_k0, cudaStream_t st) {
    launch_pdl(k_try_init, grid_for(N, 256), 256, st, alive, ymax, emax, ythr, nnkey, N, ctl, acc, band_k0);
}

int compact_blocks(int n) { return (n + kCompactTile - 1) / kCompactTile; }

int scan_slots_prune() { return scan_grid<kPrune>(); }

void launch_track_init(TryCtl* ctl, int N, int m, bool bands_ran, cudaStream_t st) {
    launch_pdl(k_track_init, 1, 32, st, ctl, N, m, bands_ran ? 1 : 0, scan_grid<kPruneTrack>());
}

void launch_compact_group(const uint8_t* a, int n, int* out, unsigned long long* status, unsigned epoch,
                          TryCtl* ctl, int gate, int2* groups, int2* slots, int m, int fixed_span, float band_keep,
                          int band_few, float seed_w, double* bcost, int band_slots, cudaStream_t st) {
    launch_pdl(k_compact_group, compact_blocks(n), kCompactBlock, st, a, n, out, status, epoch, ctl, gate, groups, slots,
                                                               m, fixed_span, band_keep,
                                                               gate == kGateTrack ? scan_grid<kPruneTrack>()
                                                                                  : band_slots,
                                                               band_few, seed_w, bcost);
}

int group_slots(int n) { return compact_blocks(n) * 504; }

void launch_gather_nn(const int* list, const int* cnt, const unsigned long long* nnkey, double* out,
                      cudaStream_t st) {
    launch_pdl(k_gather_nn, kSmallGrid, 256, st, list, cnt, nnkey, out);
}

}  // namespace tsd
