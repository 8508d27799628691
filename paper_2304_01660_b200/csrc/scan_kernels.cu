// PD3 scan kernels for sm_100a (north_star (b), (c)).
//
// k_scan<MODE> is the hot path: one CTA per parallelogram tile of the distance
// matrix (TileDesc).  It replaces the reference's per-segment scan_chunk loop
// (src/pardrag.cpp:157-282) with a B200 layout:
//   * seeds: the tile's first row of covariances is computed directly in FP64
//     from the series staged in shared memory (the reference seeds row+column
//     per chunk, pardrag.cpp:162-182; a parallelogram needs only the row);
//   * walk: every thread advances kDiag adjacent diagonals with the FP32
//     centered-covariance recurrence cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i
//     (2 FFMA per cell; the q-side operands slide through registers, the
//     c-side operand is a shared-memory broadcast);
//   * decision: corr = cov * nrm_c * nrm_q is compared with 1 - r^2/(2m) in a
//     branch-free fast path (one FMUL + FMNMX per cell); a cell that may be
//     within the proven FP32 error band of the threshold falls into the slow
//     path, which kills certain pairs (both ends, like cand/neighbor clearing,
//     pardrag.cpp:256-259) and queues knife-edge pairs for the exact FP64
//     recheck (the analogue of pardrag.cpp:255).
// Kills are monotone byte stores, so the final state is schedule-independent.
//
// k_ref_pairs evaluates reference_sq_dist (pardrag.cpp:57-69 -> znormalize +
// sq_ed, distance.cpp:8-33) bit-exactly, one warp per pair: the reference's
// sequential sums stay sequential (lane 0), only the element-wise z-normalised
// terms are computed in parallel.
#include <float.h>

#include "common.cuh"
#include "engine_internal.h"

namespace tsd {

constexpr float kEps32 = 5.9604645e-08f;  // 2^-24
constexpr double kSlack = 1e-9;           // absolute corr slack around the threshold

// rows are padded to a multiple of kDiag (+1 for the one-step prefetch); padded
// rows carry zero operands (exact no-op increments) and are never evaluated
constexpr int kRowsPad = kMaxRows + kDiag + 1;
constexpr int kQPad = kMaxRows + kDiag + kW + kDiag;

struct __align__(16) ScanSmem {
    float4 crow[kRowsPad];  // per row: {cdf, cdg, tc, cn}
    float cy[kRowsPad];     // kCollect: per-row collection threshold
    unsigned ykey[kRowsPad];
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
    float red[3][kThreads / 32];
    int flag;
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 6) k_scan(const ScanParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScanSmem& S = *reinterpret_cast<ScanSmem*>(smem_raw);

    const TileDesc td = p.tiles[blockIdx.x];
    const int tid = threadIdx.x;
    const int rows = td.rows;
    const int dir = td.dir;
    const int N = p.N;
    const int m = p.m;
    const int r_end = td.r0 + rows - 1;
    const int c_first = dir > 0 ? td.r0 : r_end;
    // local q coordinate u: step s, slot j of thread t sits at u = s + t*kDiag + j
    const int qbase = dir > 0 ? td.r0 + td.k0 : r_end + td.k0 + kW - 1;
    const int nq = rows - 1 + kW;

    // ---- 0. skip tiles whose rows are all decided -------------------------
    {
        int any = 0;
        for (int s = tid; s < rows; s += kThreads) any |= p.alive[td.r0 + s];
        if (!__syncthreads_or(any)) return;
    }

    // ---- 1. seeds: cov(c_first, q) for this thread's kDiag diagonals --------
    float cov[kDiag];
    double e_seed = 0.0;  // absolute error bound of FP32 seeds (0 for FP64 / resident seeds)
    if (td.seed >= 0) {
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
    } else if (MODE == kPrune) {
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
        float delta = 0.f, wmax = 0.f;
        for (int pc = 0; pc < m; pc += kSeedChunk) {
            const int len = min(kSeedChunk, m - pc);
            __syncthreads();
            for (int x = tid; x < len; x += kThreads) S.u.seed32.a[x] = (float)(p.t[c_first + pc + x] - mu_c);
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
            for (; pp + kDiag <= len; pp += kDiag) {
#pragma unroll
                for (int uu = 0; uu < kDiag; ++uu) {
                    w[(uu + kDiag - 1) % kDiag] = S.u.seed32.win[o_t + pp + uu + kDiag - 1];
                    const float av = S.u.seed32.a[pp + uu];
                    delta += av;
#pragma unroll
                    for (int i = 0; i < kDiag; ++i) acc[i] = fmaf(av, w[(uu + i) % kDiag], acc[i]);
                }
            }
            for (; pp < len; ++pp) {
                const float av = S.u.seed32.a[pp];
                delta += av;
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
            seedv[i] = (q >= 0 && q < N) ? (double)acc[i] - (p.mu[q] - anchor) * (double)delta : 0.0;
        }
        if (dir > 0) {
#pragma unroll
            for (int j = 0; j < kDiag; ++j) cov[j] = (float)seedv[j];
        } else {
#pragma unroll
            for (int j = 0; j < kDiag; ++j) cov[j] = (float)seedv[kDiag - 1 - j];
        }
    } else {
    // cov = sum_p (t[c+p]-mu_c) t[q+p] - mu_q * sum_p (t[c+p]-mu_c)
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
        for (int x = tid; x < len; x += kThreads) S.u.seed.a[x] = p.t[c_first + pc + x] - mu_c;
        for (int x = tid; x < kW + len - 1; x += kThreads) {
            const int g = qlo + pc + x;
            S.u.seed.win[x] = (g >= 0 && g < p.n) ? p.t[g] : 0.0;
        }
        __syncthreads();
        double w[kDiag];
#pragma unroll
        for (int i = 0; i < kDiag - 1; ++i) w[i] = S.u.seed.win[o_t + i];
        int pp = 0;
        for (; pp + kDiag <= len; pp += kDiag) {
#pragma unroll
            for (int uu = 0; uu < kDiag; ++uu) {
                // ring: window value for offset o_t + pp + uu + i lives in w[(uu + i) % kDiag]
                w[(uu + kDiag - 1) % kDiag] = S.u.seed.win[o_t + pp + uu + kDiag - 1];
                const double av = S.u.seed.a[pp + uu];
                delta += av;
#pragma unroll
                for (int i = 0; i < kDiag; ++i) acc[i] = fma(av, w[(uu + i) % kDiag], acc[i]);
            }
        }
        for (; pp < len; ++pp) {
            const double av = S.u.seed.a[pp];
            delta += av;
#pragma unroll
            for (int i = 0; i < kDiag; ++i) acc[i] = fma(av, S.u.seed.win[o_t + pp + i], acc[i]);
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
    __syncthreads();  // seed buffers are reused below

    // ---- 2. stage the walk operands ---------------------------------------
    float smax_c = 0.f, smax_q = 0.f, qn_max = 0.f;
    for (int s = tid; s < rows; s += kThreads) {
        const int c = dir > 0 ? td.r0 + s : r_end - s;
        float4 v;
        if (s == 0) {
            v.x = 0.f;
            v.y = 0.f;
        } else if (dir > 0) {
            v.x = p.df[c];
            v.y = p.dg[c];
        } else {
            v.x = -p.df[c + 1];
            v.y = -p.dg[c + 1];
        }
        v.w = p.nrm[c];
        v.z = 0.f;
        if (v.w != 0.f) smax_c = fmaxf(smax_c, (float)p.sig[c]);
        S.crow[s] = v;
    }
    const int rows_p = (rows + kDiag - 1) / kDiag * kDiag;
    for (int s = rows + tid; s <= rows_p; s += kThreads) S.crow[s] = make_float4(0.f, 0.f, FLT_MAX, 0.f);
    for (int u = tid; u < rows_p + kW + kDiag; u += kThreads) {
        const int q = dir > 0 ? qbase + u : qbase - u;
        float a = 0.f, b = 0.f, nn = 0.f;
        if (u < nq && q >= 0 && q < N) {
            const int qi = dir > 0 ? q : q + 1;
            if (qi < N) {
                a = p.df[qi];
                b = p.dg[qi];
            }
            nn = p.nrm[q];
            if (nn != 0.f) {
                smax_q = fmaxf(smax_q, (float)p.sig[q]);
                qn_max = fmaxf(qn_max, nn);
            }
        }
        S.u.walk.qd[u] = make_float2(a, b);
        // an invalid q gets a NaN norm: its x = cov*qn is NaN, which never passes a
        // threshold test and is ignored by fmaxf (a constant q keeps qn = 0, x = 0)
        S.u.walk.qn[u] = (u < nq && q >= 0 && q < N) ? nn : __int_as_float(0x7fffffff);
    }
    smax_c = warp_max(smax_c);
    smax_q = warp_max(smax_q);
    qn_max = warp_max(qn_max);
    if ((tid & 31) == 0) {
        S.red[0][tid >> 5] = smax_c;
        S.red[1][tid >> 5] = smax_q;
        S.red[2][tid >> 5] = qn_max;
    }
    __syncthreads();
    smax_c = 0.f;
    smax_q = 0.f;
    qn_max = 0.f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        smax_c = fmaxf(smax_c, S.red[0][w]);
        smax_q = fmaxf(smax_q, S.red[1][w]);
        qn_max = fmaxf(qn_max, S.red[2][w]);
    }
    // absolute FP32 covariance error bound for every cell of this tile
    const double E = p.err_k * (double)kEps32 * (double)m * (double)smax_c * (double)smax_q *
                         (double)(rows + 8) +
                     e_seed;
    const float Ef = (float)E;
    // Row thresholds.  crow.z = tc: a live row's cells with x = cov*qn > tc may be
    // within the error band of d^2 = r^2 (slow path); kNoEval marks rows whose
    // cells are only walked (already decided, or not a survivor in kCollect).
    constexpr float kNoEval = FLT_MAX;
    int evals = 0;
    for (int s = tid; s < rows; s += kThreads) {
        const int c = dir > 0 ? td.r0 + s : r_end - s;
        const float cn = S.crow[s].w;
        const bool live = p.alive[c] != 0;
        float tc;
        if (MODE == kCollect) {
            S.cy[s] = (live && cn != 0.f) ? p.ythr[c] : FLT_MAX;
            tc = S.cy[s] < FLT_MAX ? 0.f : kNoEval;
        } else if (!live) {
            tc = kNoEval;
        } else if (cn == 0.f) {
            tc = -FLT_MAX;  // constant row: always take the exact-convention slow path
        } else if (MODE == kPrune) {
            // band passes only make certain kills: every cell with x > tk has
            // corr - eps_cell > thr0 (eps_cell <= eps_row); knife edges are left
            // to the full-row pass
            const double eps_row = E * (double)cn * (double)qn_max + kSlack + 8.0 * (double)kEps32;
            const double tk = (p.thr0 + eps_row) / (double)cn;
            tc = (float)tk;
            tc = tc + fabsf(tc) * 2.4e-7f;  // round toward +inf (conservative)
        } else {
            const double eps_row = E * (double)cn * (double)qn_max + kSlack + 8.0 * (double)kEps32;
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
            if (cr.z != kNoEval) {  // CTA-uniform branch: the row is undecided
                float x[kDiag];
                float mx = -FLT_MAX;
#pragma unroll
                for (int j = 0; j < kDiag; ++j) {
                    x[j] = cov[j] * rn[(j + uu) % kDiag];
                    mx = fmaxf(mx, x[j]);
                }
                if (MODE == kPrune && mx > cr.z && cr.w != 0.f) {
                    // certain kill of the row candidate (FP32 only)
                    p.alive[dir > 0 ? td.r0 + ss : r_end - ss] = 0;
                } else if (MODE != kCollect && mx > cr.z) {
                    // ---- slow path: exact conventions, certain kill, knife edges.
                    // Only the row candidate is killed (the pair's other end is
                    // decided by its own row), so a decided row never re-enters.
                    const int c = dir > 0 ? td.r0 + ss : r_end - ss;
#pragma unroll
                    for (int j = 0; j < kDiag; ++j) {
                        if (!(x[j] > cr.z)) continue;
                        const int u = ss + ub + j;
                        const int q = dir > 0 ? qbase + u : qbase - u;
                        if (q < 0 || q >= N) continue;
                        const float qn = rn[(j + uu) % kDiag];
                        if (cr.w == 0.f || qn == 0.f) {
                            const double d = (cr.w == 0.f && qn == 0.f) ? 0.0 : 2.0 * (double)m;
                            if (d < p.r_sq) p.alive[c] = 0;
                            continue;
                        }
                        const double corr = (double)x[j] * (double)cr.w;
                        const double ec = E * (double)cr.w * (double)qn + kSlack;
                        if (corr - ec > p.thr0) {
                            p.alive[c] = 0;
                        } else if (MODE == kPruneTrack && corr + ec >= p.thr0) {
                            const int at = atomicAdd(p.queue_count, 1);
                            if (at < p.queue_cap) p.queue[at] = make_int2(c, q);
                        }
                    }
                }
                if (MODE == kPruneTrack && S.ykey[ss] != 0u) {
                    // row max of the FP32 route value x = cov*qn over valid q (NaN for
                    // invalid q is ignored by fmaxf; a constant q contributes exactly
                    // 0); the tile's error term E*qn_max is folded in at the end
                    float y = -FLT_MAX;
#pragma unroll
                    for (int j = 0; j < kDiag; ++j) y = fmaxf(y, x[j]);
                    y = warp_max(y);
                    if (lane == 0 && y > -FLT_MAX) atomicMax(&S.ykey[ss], f2key(y));
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
    }

    if (MODE == kPruneTrack) {
        __syncthreads();
        const unsigned ekey = __float_as_uint(Ef * qn_max * (1.f + 4.8e-7f));  // >= 0: bit order
        for (int s = tid; s < rows; s += kThreads) {
            const unsigned k = S.ykey[s];
            if (k > 1u) {
                const int c = dir > 0 ? td.r0 + s : r_end - s;
                atomicMax(&p.ymax[c], k);
                atomicMax(&p.emax[c], ekey);
            }
        }
    }
    if (tid == 0) {
        atomicAdd(&p.acc[0], (unsigned long long)rows * (unsigned long long)kW);
        atomicAdd(&p.acc[1], (unsigned long long)evals * (unsigned long long)kW);
        if (td.seed < 0) atomicAdd(&p.acc[2], (unsigned long long)kW);
    }
}

// ---------------------------------------------------------------------------
// reference_sq_dist, bit-exact, one warp per pair.  buf: 256 doubles per warp.
__device__ double ref_dist_warp(const double* __restrict__ t, int m, int i, int j, double* buf) {
    const int lane = threadIdx.x & 31;
    double mean = 0.0, sg = 0.0;
    if (lane < 2) {
        const double* x = t + (lane == 0 ? i : j);
        double s = 0.0, q = 0.0;
        for (int k = 0; k < m; ++k) {
            const double v = x[k];
            s = __dadd_rn(s, v);
            q = __dadd_rn(q, __dmul_rn(v, v));
        }
        const double md = (double)m;
        mean = __ddiv_rn(s, md);
        const double var = __dsub_rn(__ddiv_rn(q, md), __dmul_rn(mean, mean));
        sg = __dsqrt_rn(var > 0.0 ? var : 0.0);
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
                                                               unsigned long long* nnkey) {
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
                    alive[pr.x] = 0;
                    alive[pr.y] = 0;
                }
            } else {
                atomicMin(&nnkey[pr.x], (unsigned long long)__double_as_longlong(d));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// flags / compaction helpers
__global__ void k_fill_u8(uint8_t* a, int n, uint8_t v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = v;
}

constexpr int kCompactBlock = 1024;
constexpr int kCompactItems = 4;  // flags per thread
constexpr int kCompactTile = kCompactBlock * kCompactItems;

__global__ void k_compact_count(const uint8_t* __restrict__ a, int n, int* __restrict__ blk) {
    __shared__ int ws[kCompactBlock / 32];
    const int base = blockIdx.x * kCompactTile;
    int c = 0;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        const int i = base + threadIdx.x * kCompactItems + k;
        c += (i < n && a[i]) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kCompactBlock / 32; ++w) t += ws[w];
        blk[blockIdx.x] = t;
    }
}

// single CTA exclusive scan over block counts; total -> out[nb]
__global__ void k_compact_scan(int* blk, int nb) {
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? blk[i] : 0;
        // inclusive warp scan
        int x = v;
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __shared__ int wsum[32];
        if (lane == 31) wsum[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            int z = threadIdx.x < (int)(blockDim.x >> 5) ? wsum[threadIdx.x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, z, o);
                if ((int)threadIdx.x >= o) z += y;
            }
            wsum[threadIdx.x] = z;
        }
        __syncthreads();
        const int woff = (threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0;
        if (i < nb) blk[i] = carry + woff + x - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += woff + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) blk[nb] = carry;
}

__global__ void k_compact_scatter(const uint8_t* __restrict__ a, int n, const int* __restrict__ blk,
                                  int* __restrict__ out) {
    __shared__ int ws[kCompactBlock / 32];
    const int base = blockIdx.x * kCompactTile;
    int f[kCompactItems];
    int c = 0;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        const int i = base + threadIdx.x * kCompactItems + k;
        f[k] = (i < n && a[i]) ? 1 : 0;
        c += f[k];
    }
    const int lane = threadIdx.x & 31;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        int z = ws[threadIdx.x];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, z, o);
            if ((int)threadIdx.x >= o) z += y;
        }
        ws[threadIdx.x] = z;
    }
    __syncthreads();
    int pos = blk[blockIdx.x] + ((threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0) + x - c;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        if (f[k]) out[pos++] = base + threadIdx.x * kCompactItems + k;
    }
}

// survivors: reset exact-nn keys and decode collection thresholds.  The
// tracked max route value x* and the row's largest tile error term e give a
// lower bound x* - e of the row's true best corr / cn; every q whose upper
// bound x + E*qn reaches it may be the reference's minimiser.
__global__ void k_prep_survivors(const int* __restrict__ list, int cnt, const unsigned* __restrict__ ymax,
                                 const unsigned* __restrict__ emax, float* __restrict__ ythr,
                                 unsigned long long* __restrict__ nnkey) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
        const int c = list[e];
        const unsigned k = ymax[c];
        float th = -FLT_MAX;  // no tracked data: collect everything
        if (k > 1u) {
            const float lo = key2f(k) - __uint_as_float(emax[c]);
            // two ulps down: FP64 rounding of near-ties can never exclude the minimiser
            th = nextafterf(nextafterf(lo - fabsf(lo) * 2.4e-7f, -FLT_MAX), -FLT_MAX);
        }
        ythr[c] = th;
        nnkey[c] = 0x7ff0000000000000ull;  // +inf
    }
}

// per-survivor interval [lo, hi] of the exact nn^2 from the tracked route maxima
// (constant rows: the exact convention value)
__global__ void k_nn_bounds(const int* __restrict__ list, int cnt, const unsigned* __restrict__ ymax,
                            const unsigned* __restrict__ emax, const float* __restrict__ nrm,
                            const int* __restrict__ const_range, int N, int m, double* __restrict__ lo,
                            double* __restrict__ hi) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const double two_m = 2.0 * (double)m;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
        const int c = list[e];
        const float cn = nrm[c];
        double l = 0.0, h = inf;
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
        lo[e] = l;
        hi[e] = h;
    }
}

// constant survivors (stats sigma < eps): nn by the conventions of
// reference_sq_dist — 0 with an admissible constant partner, else 2m, else inf.
__global__ void k_const_nn(const int* __restrict__ list, int cnt, const float* __restrict__ nrm,
                           const int* __restrict__ const_range, int N, int m,
                           unsigned long long* __restrict__ nnkey) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
        const int c = list[e];
        if (nrm[c] != 0.f) continue;
        const int lo = const_range[0], hi = const_range[1];
        double d = __longlong_as_double(0x7ff0000000000000ll);
        if (c - lo >= m || hi - c >= m) d = 0.0;
        else if (c - m >= 0 || c + m <= N - 1) d = 2.0 * (double)m;
        nnkey[c] = (unsigned long long)__double_as_longlong(d);
    }
}

__global__ void k_const_range(const float* __restrict__ nrm, int N, int* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        if (nrm[i] == 0.f) {
            atomicMin(&out[0], i);
            atomicMax(&out[1], i);
        }
    }
}

__global__ void k_gather_nn(const int* __restrict__ list, int cnt,
                            const unsigned long long* __restrict__ nnkey, double* __restrict__ out) {
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

__global__ void k_seed_init(const double* __restrict__ t, int n, int m, int L, int kA, int nb,
                            double* __restrict__ qt) {
    const int N = n - m + 1;
    const long long total = (long long)nb * kW;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        int i, q;
        double s = 0.0;
        if (seed_pair((int)(e / kW), (int)(e % kW), L, kA, N, i, q))
            for (int k = 0; k < m; ++k) s = fma(t[i + k], t[q + k], s);
        qt[e] = s;
    }
}

__global__ void k_seed_advance(const double* __restrict__ t, int n, int m, int L, int kA, int nb,
                               double* __restrict__ qt) {
    const int N1 = n - m;  // subsequence count of length m+1
    const long long total = (long long)nb * kW;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        int i, q;
        if (seed_pair((int)(e / kW), (int)(e % kW), L, kA, N1, i, q)) qt[e] = fma(t[i + m], t[q + m], qt[e]);
    }
}

void launch_seed_init(const double* t, int n, int m, int L, int kA, int nb, double* qt, cudaStream_t st) {
    k_seed_init<<<148 * 8, 256, 0, st>>>(t, n, m, L, kA, nb, qt);
}

void launch_seed_advance(const double* t, int n, int m, int L, int kA, int nb, double* qt, cudaStream_t st) {
    k_seed_advance<<<148 * 8, 256, 0, st>>>(t, n, m, L, kA, nb, qt);
}

static int grid_for(long long work, int threads) {
    long long b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

size_t scan_smem_bytes() { return sizeof(ScanSmem); }

void scan_configure() {
    const int bytes = (int)sizeof(ScanSmem);
    cudaFuncSetAttribute(k_scan<kPrune>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan<kPruneTrack>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan<kCollect>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

void launch_scan(int mode, int ntiles, const ScanParams& p, cudaStream_t st) {
    const size_t sm = sizeof(ScanSmem);
    if (ntiles <= 0) return;
    switch (mode) {
        case kPrune: k_scan<kPrune><<<ntiles, kThreads, sm, st>>>(p); break;
        case kPruneTrack: k_scan<kPruneTrack><<<ntiles, kThreads, sm, st>>>(p); break;
        default: k_scan<kCollect><<<ntiles, kThreads, sm, st>>>(p); break;
    }
}

void launch_ref_pairs(int mode, const double* t, int m, const int2* pairs, const int* count, int cap,
                      double r_sq, uint8_t* alive, unsigned long long* nnkey, int max_pairs,
                      cudaStream_t st) {
    if (max_pairs <= 0) return;
    const int blocks = grid_for(max_pairs, kPairWarps);
    if (mode == 0)
        k_ref_pairs<0><<<blocks, kPairWarps * 32, 0, st>>>(t, m, pairs, count, cap, r_sq, alive, nnkey);
    else
        k_ref_pairs<1><<<blocks, kPairWarps * 32, 0, st>>>(t, m, pairs, count, cap, r_sq, alive, nnkey);
}

void launch_fill_u8(uint8_t* a, int n, uint8_t v, cudaStream_t st) {
    k_fill_u8<<<grid_for(n, 256), 256, 0, st>>>(a, n, v);
}

int compact_blocks(int n) { return (n + kCompactTile - 1) / kCompactTile; }

void launch_compact(const uint8_t* a, int n, int* blk, int* out, cudaStream_t st) {
    const int nb = compact_blocks(n);
    k_compact_count<<<nb, kCompactBlock, 0, st>>>(a, n, blk);
    k_compact_scan<<<1, 1024, 0, st>>>(blk, nb);
    k_compact_scatter<<<nb, kCompactBlock, 0, st>>>(a, n, blk, out);
}

void launch_prep_survivors(const int* list, int cnt, const unsigned* ymax, const unsigned* emax, float* ythr,
                           unsigned long long* nnkey, cudaStream_t st) {
    k_prep_survivors<<<grid_for(cnt, 256), 256, 0, st>>>(list, cnt, ymax, emax, ythr, nnkey);
}

void launch_nn_bounds(const int* list, int cnt, const unsigned* ymax, const unsigned* emax, const float* nrm,
                      const int* const_range, int N, int m, double* lo, double* hi, cudaStream_t st) {
    k_nn_bounds<<<grid_for(cnt, 256), 256, 0, st>>>(list, cnt, ymax, emax, nrm, const_range, N, m, lo, hi);
}

void launch_const_range(const float* nrm, int N, int* out, cudaStream_t st) {
    k_const_range<<<grid_for(N, 256), 256, 0, st>>>(nrm, N, out);
}

void launch_const_nn(const int* list, int cnt, const float* nrm, const int* const_range, int N, int m,
                     unsigned long long* nnkey, cudaStream_t st) {
    k_const_nn<<<grid_for(cnt, 256), 256, 0, st>>>(list, cnt, nrm, const_range, N, m, nnkey);
}

void launch_gather_nn(const int* list, int cnt, const unsigned long long* nnkey, double* out,
                      cudaStream_t st) {
    k_gather_nn<<<grid_for(cnt, 256), 256, 0, st>>>(list, cnt, nnkey, out);
}

}  // namespace tsd
