// Per-length subsequence statistics on the device (north_star (a)).
//
// K1  init:    Eq. 4 running sums, src/stats.cpp:7-36.  The reference's running
//              sum is a sequential FP64 recurrence, so the prefix sums are
//              produced by one thread in exactly the reference's operation
//              order (no FMA contraction) and the per-index mean/sigma by a
//              parallel pass: bit-identical to init_stats.
// K2  advance: Eq. 7-8, src/stats.cpp:38-58, one thread per index, in place,
//              bit-identical to advance_stats.
// K2b derive:  the FP32 arrays the tile scan walks (df, dg, 1/(sqrt(m) sigma)),
//              computed in FP64 and rounded once (HBM-bound, fused per length).
#include <algorithm>

#include "common.cuh"
#include "engine_internal.h"

namespace tsd {

// One CTA: the whole block stages the series through shared memory in
// coalesced chunks; thread 0 runs the reference's sequential recurrence out of
// shared memory (the only serial part), and the block writes the prefix
// values back coalesced.
constexpr int kPrefixChunk = 2048;  // 2 x 16 KB static shared memory

__global__ void __launch_bounds__(1024) k_init_prefix(const double* __restrict__ t, int n, int m,
                                                      double* __restrict__ sum,
                                                      double* __restrict__ sum_sq) {
    // ds/dq hold the per-step increments, then are overwritten in place by the
    // running sums (each position is read before it is written)
    __shared__ double ds[kPrefixChunk], dq[kPrefixChunk];
    const int cnt = n - m + 1;
    double s = 0.0, q = 0.0;
    if (threadIdx.x == 0 || threadIdx.x == 32) {
        for (int k = 0; k < m; ++k) {
            const double v = t[k];
            s = __dadd_rn(s, v);
            q = __dadd_rn(q, __dmul_rn(v, v));
        }
    }
    // index i >= 1 adds in - out and in*in - out*out with out = t[i-1], in = t[i-1+m]
    for (int base = 0; base < cnt; base += kPrefixChunk) {
        const int len = min(kPrefixChunk, cnt - base);
        __syncthreads();
        for (int x = threadIdx.x; x < len; x += blockDim.x) {
            const int i = base + x;
            if (i > 0) {
                const double out = t[i - 1], in = t[i - 1 + m];
                ds[x] = __dsub_rn(in, out);
                dq[x] = __dsub_rn(__dmul_rn(in, in), __dmul_rn(out, out));
            }
        }
        __syncthreads();
        // the two sequential chains run concurrently on two warps
        if (threadIdx.x == 0 || threadIdx.x == 32) {
            double* d = threadIdx.x == 0 ? ds : dq;
            double acc = threadIdx.x == 0 ? s : q;
            int x = 0;
            if (base == 0) {
                d[0] = acc;  // index 0: the initial window sums
                x = 1;
            }
            for (; x + 16 <= len; x += 16) {
                double v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = d[x + u];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    acc = __dadd_rn(acc, v[u]);
                    d[x + u] = acc;
                }
            }
            for (; x < len; ++x) {
                acc = __dadd_rn(acc, d[x]);
                d[x] = acc;
            }
            if (threadIdx.x == 0) s = acc;
            else q = acc;
        }
        __syncthreads();
        for (int x = threadIdx.x; x < len; x += blockDim.x) {
            sum[base + x] = ds[x];
            sum_sq[base + x] = dq[x];
        }
    }
}

__global__ void k_init_finish(const double* __restrict__ sum, const double* __restrict__ sum_sq,
                              int cnt, int m, double* __restrict__ mu, double* __restrict__ sig) {
    const double md = (double)m;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const double mean = __ddiv_rn(sum[i], md);
        const double var = __dsub_rn(__ddiv_rn(sum_sq[i], md), __dmul_rn(mean, mean));
        mu[i] = mean;
        sig[i] = __dsqrt_rn(var > 0.0 ? var : 0.0);
    }
}

// ---- statistics error (common.cuh) --------------------------
// Double-double prefix sums of the series and of its squares (P[k] = sum of
// the first k values), built once per series (tsd_series_set): three
// launches, chunk totals -> exclusive scan of the totals -> chunk scans.
constexpr int kPfxThreads = 512;

__device__ __forceinline__ dd warp_incl_scan_dd(dd v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double h = __shfl_up_sync(0xffffffffu, v.hi, o);
        const double l = __shfl_up_sync(0xffffffffu, v.lo, o);
        if (lane >= o) v = dd_add(dd{h, l}, v);
    }
    return v;
}

__global__ void __launch_bounds__(kPfxThreads) k_dd_chunk_sums(const double* __restrict__ t, int n, int chunk,
                                                                 double2* __restrict__ tot1,
                                                                 double2* __restrict__ tot2) {
    __shared__ dd r1[kPfxThreads / 32], r2[kPfxThreads / 32];
    const int b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    dd s1{0.0, 0.0}, s2{0.0, 0.0};
    for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        const double v = t[i];
        s1 = dd_add(s1, dd{v, 0.0});
        s2 = dd_add(s2, dd_sq(v));
    }
    s1 = warp_incl_scan_dd(s1);  // lane 31 holds the warp total
    s2 = warp_incl_scan_dd(s2);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 31) {
        r1[w] = s1;
        r2[w] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        dd a{0.0, 0.0}, q{0.0, 0.0};
        for (int k = 0; k < kPfxThreads / 32; ++k) {
            a = dd_add(a, r1[k]);
            q = dd_add(q, r2[k]);
        }
        tot1[blockIdx.x] = make_double2(a.hi, a.lo);
        tot2[blockIdx.x] = make_double2(q.hi, q.lo);
    }
}

__global__ void k_dd_scan_totals(double2* __restrict__ tot1, double2* __restrict__ tot2, int nb) {
    dd a{0.0, 0.0}, q{0.0, 0.0};  // exclusive, in place (one thread: nb <= a few thousand)
    for (int b = 0; b < nb; ++b) {
        const double2 x = tot1[b], y = tot2[b];
        tot1[b] = make_double2(a.hi, a.lo);
        tot2[b] = make_double2(q.hi, q.lo);
        a = dd_add(a, dd{x.x, x.y});
        q = dd_add(q, dd{y.x, y.y});
    }
}

__global__ void __launch_bounds__(kPfxThreads) k_dd_chunk_scan(const double* __restrict__ t, int n, int chunk,
                                                                 const double2* __restrict__ tot1,
                                                                 const double2* __restrict__ tot2,
                                                                 double2* __restrict__ P1, double2* __restrict__ P2) {
    __shared__ dd w1[kPfxThreads / 32], w2[kPfxThreads / 32];
    const int b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    dd c1{tot1[blockIdx.x].x, tot1[blockIdx.x].y}, c2{tot2[blockIdx.x].x, tot2[blockIdx.x].y};
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P1[0] = make_double2(0.0, 0.0);
        P2[0] = make_double2(0.0, 0.0);
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int base = b0; base < b1; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const double v = i < b1 ? t[i] : 0.0;
        dd s1 = warp_incl_scan_dd(dd{v, 0.0});
        dd s2 = warp_incl_scan_dd(i < b1 ? dd_sq(v) : dd{0.0, 0.0});
        if (lane == 31) {
            w1[w] = s1;
            w2[w] = s2;
        }
        __syncthreads();
        dd o1 = c1, o2 = c2;  // carry + totals of the earlier warps of this tile
        for (int k = 0; k < w; ++k) {
            o1 = dd_add(o1, w1[k]);
            o2 = dd_add(o2, w2[k]);
        }
        if (i < b1) {
            const dd p1 = dd_add(o1, s1), p2 = dd_add(o2, s2);
            P1[i + 1] = make_double2(p1.hi, p1.lo);
            P2[i + 1] = make_double2(p2.hi, p2.lo);
        }
        for (int k = 0; k < kPfxThreads / 32; ++k) {  // the tile total joins the carry
            c1 = dd_add(c1, w1[k]);
            c2 = dd_add(c2, w2[k]);
        }
        __syncthreads();
    }
}

// Statistics error a_i of window i (correlation units) and 1 + mu^2 / sigma^2:
//   ev  = |sigma_r^2 - var| / var  (rolling variance against the window's true
//         variance from the double-double prefix sums; >= the relative sigma
//         error, since |sqrt(a) - sqrt(b)| / sqrt(b) <= |a - b| / b),
//   gam = |mu_r - mu| / sigma,
//   eta = 3 (m + 1) u (1 + Om + sqrt(Om)), Om = mu^2 / sigma^2: the one-pass
//         variance error of the exact distance's znormalize (sequential sums of
//         m terms), relative;
//   a   = 2 ev + 2 eta + kStatsRows gam  (+inf when the window has no variance).
// Only the prefix differences and the cancelling m var = S2 - mu S1 need the
// double-double; the bound itself is formed in FP32 (its 1e-7 relative
// rounding is covered by the 1e-5 factor).
__device__ __forceinline__ float stats_err(const double2* __restrict__ P1, const double2* __restrict__ P2, int i,
                                           int m, double inv_m, double mu_r, double sg_r, float& b2) {
    const double2 x0 = P1[i], x1 = P1[i + m], y0 = P2[i], y1 = P2[i + m];
    const dd S1 = dd_add(dd{x1.x, x1.y}, dd_neg(dd{x0.x, x0.y}));
    const dd S2 = dd_add(dd{y1.x, y1.y}, dd_neg(dd{y0.x, y0.y}));
    const double md = (double)m;
    const double q1 = S1.hi * inv_m;  // mu = S1 / m as a double-double, without a division
    const dd mu = dd_fast(q1, __dadd_rn(fma(-q1, md, S1.hi), S1.lo) * inv_m);
    const dd v = dd_add(S2, dd_neg(dd_mul(mu, S1)));  // m var
    const double var = (v.hi + v.lo) * inv_m;
    b2 = 0.f;
    if (!(var > 1e-30)) return __int_as_float(0x7f800000);
    const double mua = mu.hi + mu.lo;
    const float ivar = 1.f / (float)var;
    const float ev = (float)fabs(fma(sg_r, sg_r, -var)) * ivar;
    const float gam = (float)fabs(mu_r - mua) * rsqrtf((float)var);
    const float om = (float)(mua * mua) * ivar;
    const float eta = 3.f * (float)(m + 1) * 1.1102230e-16f * (1.f + om + sqrtf(om));
    b2 = (1.f + om) * (1.f + 1e-5f);
    return (2.f * ev + 2.f * eta + (float)kStatsRows * gam) * (1.f + 1e-5f) + 1e-30f;
}

// A degenerate window (sigma < eps, or statistics too unreliable for the FP32
// filter): listed for the exact stage, split by the reference's own one-pass
// test -- all-zero z windows get the 0 / 2m conventions in O(1) per row,
// the others are evaluated exactly (scan_kernels.cu degenerate_body).  The
// regular-window threshold carries a 1% margin over kSigmaEps so that no
// regular window can be one-pass constant.
__device__ __forceinline__ void degenerate_row(const double* __restrict__ t, int i, int m, int cnt, int* cr,
                                               int* deg, int* degc, int* deg2) {
    atomicMax(&cr[0], cnt - i);
    atomicMax(&cr[1], i + 1);
    deg[atomicAdd(&cr[2], 1)] = i;
    if (onepass_const(t + i, m)) {
        atomicMax(&cr[5], cnt - i);
        atomicMax(&cr[6], i + 1);
        degc[atomicAdd(&cr[7], 1)] = i;
    } else {
        deg2[atomicAdd(&cr[8], 1)] = i;
    }
}

// block max of two non-negative floats (as int bits) into cr[3], cr[4]
__device__ __forceinline__ void stats_max_commit(float a, float b2, int* cr) {
    __shared__ int sa[32], sb[32];
    int ia = __reduce_max_sync(0xffffffffu, __float_as_int(a));
    int ib = __reduce_max_sync(0xffffffffu, __float_as_int(b2));
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sa[w] = ia;
        sb[w] = ib;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            ia = max(ia, sa[k]);
            ib = max(ib, sb[k]);
        }
        if (ia > 0) atomicMax(&cr[3], ia);
        if (ib > 0) atomicMax(&cr[4], ib);
    }
}

// stats (length m, n-m+1 valid) -> length m+1 (n-m valid), in place.
__global__ void k_advance(const double* __restrict__ t, int n, int m, double* __restrict__ mu,
                          double* __restrict__ sig) {
    pdl_enter();
    const int cnt = n - m;  // next valid_count
    const double md = (double)m;
    const double md1 = md + 1.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const double u = mu[i];
        const double sg = sig[i];
        const double in = t[i + m];
        const double delta = __dsub_rn(u, in);
        mu[i] = __ddiv_rn(__dadd_rn(__dmul_rn(md, u), in), md1);
        const double var = __dmul_rn(__ddiv_rn(md, md1),
                                     __dadd_rn(__dmul_rn(sg, sg), __ddiv_rn(__dmul_rn(delta, delta), md1)));
        sig[i] = __dsqrt_rn(var > 0.0 ? var : 0.0);
    }
}

// df[i] = (t[i+m-1] - t[i-1]) / 2, dg[i] = (t[i+m-1] - mu_i) + (t[i-1] - mu_{i-1})
// (centered-covariance diagonal step: cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i)
// nrm[i] = 1 / (sqrt(m) sigma_i), 0 for a constant subsequence.
// Per-length FP32 walk operands and the constant-row range
// (cr[0] = max(N - i), cr[1] = max(i + 1) over rows with sigma < eps, cr[2] their
// count, listed in deg; cleared
// to 0 before the launch, 0 meaning none).
__global__ void k_derive(const double* __restrict__ t, int m, int cnt, const double* __restrict__ mu,
                         const double* __restrict__ sig, float* __restrict__ df,
                         float* __restrict__ dg, float* __restrict__ nrm, int* __restrict__ cr,
                         int* __restrict__ deg, const double2* __restrict__ P1, const double2* __restrict__ P2,
                         int* __restrict__ degc, int* __restrict__ deg2) {
    pdl_enter();
    const double sqm = sqrt((double)m), inv_m = 1.0 / (double)m;
    float amax = 0.f, bmax = 0.f;
    const int cnt_w = (cnt + 31) & ~31;  // warp-uniform bound (the commit reduces over warps)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt_w; i += gridDim.x * blockDim.x) {
        if (i >= cnt) continue;
        const double s = sig[i];
        float b2 = 0.f;
        const float a = stats_err(P1, P2, i, m, inv_m, mu[i], s, b2);
        const bool dgn = s < 1.01 * kSigmaEps || !(a <= (float)kStatsUnreliable);
        nrm[i] = dgn ? 0.f : (float)(1.0 / (sqm * s));
        if (dgn) {
            degenerate_row(t, i, m, cnt, cr, deg, degc, deg2);
        } else {
            amax = fmaxf(amax, a);
            bmax = fmaxf(bmax, b2);
        }
        if (i == 0) {
            df[0] = 0.f;
            dg[0] = 0.f;
        } else {
            const double a2 = t[i + m - 1], b = t[i - 1];
            df[i] = (float)((a2 - b) * 0.5);
            dg[i] = (float)((a2 - mu[i]) + (b - mu[i - 1]));
        }
    }
    stats_max_commit(amax, bmax, cr);
}

// One MERLIN length step in one launch (north_star (a)): Eq. 7-8 advance of
// mu/sigma from length m to m+1 (ping-pong buffers, the same rounding as
// k_advance), the derived FP32 walk operands and constant-row range of length
// m+1 (as k_derive), and the resident seed rows' length recurrence
// QT_{m+1}(i,q) = QT_m(i,q) + t[i+m] t[q+m] (as k_seed_advance).  cr must be
// zero on entry; cr_next (the other parity) is cleared for the next step.
__device__ __forceinline__ void advance1(const double* __restrict__ t, int m, int i, const double* __restrict__ mu,
                                         const double* __restrict__ sig, double& mu1, double& sg1) {
    const double md = (double)m;
    const double md1 = md + 1.0;
    const double u = mu[i];
    const double sg = sig[i];
    const double in = t[i + m];
    const double delta = __dsub_rn(u, in);
    mu1 = __ddiv_rn(__dadd_rn(__dmul_rn(md, u), in), md1);
    const double var =
        __dmul_rn(__ddiv_rn(md, md1), __dadd_rn(__dmul_rn(sg, sg), __ddiv_rn(__dmul_rn(delta, delta), md1)));
    sg1 = __dsqrt_rn(var > 0.0 ? var : 0.0);
}

__global__ void __launch_bounds__(256, 6) k_next_length(const double* __restrict__ t, int n, int m, const double* __restrict__ mu_in,
                              const double* __restrict__ sig_in, double* __restrict__ mu_out,
                              double* __restrict__ sig_out, float* __restrict__ df, float* __restrict__ dg,
                              float* __restrict__ nrm, int* __restrict__ cr, int* __restrict__ cr_next, int L, int kA,
                              int nb, int bstep, int ustep, double* __restrict__ qt, int* __restrict__ deg,
                              const double2* __restrict__ P1, const double2* __restrict__ P2,
                              int* __restrict__ degc, int* __restrict__ deg2, int qblocks) {
    pdl_enter();
    const int m1 = m + 1, cnt = n - m;
    if (blockIdx.x == 0 && threadIdx.x < kCrInts) cr_next[threadIdx.x] = 0;
    if ((int)blockIdx.x < qblocks) {
        // the first qblocks blocks advance the resident seed rows, the rest the
        // statistics: two independent load chains side by side instead of one
        // after the other in every block.  One row per block iteration: no
        // 64-bit index division, the row value t[i+m] is a broadcast, qt and
        // t[q+m] are coalesced.
        for (int b = blockIdx.x * bstep; b < nb; b += qblocks * bstep) {  // bstep 2: positive sides only
            const int j = b >> 1;
            const int i = (b & 1) ? j * L + L - 1 : j * L;
            if (i >= cnt) continue;
            const double ti = t[i + m];
            double* row = qt + (size_t)b * kW;
            // every load of the row slice first (5 entries per thread in flight);
            // ustep > 1: only the entries the pass-0 walk reads (every ustep-th)
            constexpr int kPer = (kW + 255) / 256;
            double rv[kPer], tv[kPer];
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int u = (threadIdx.x + k * 256) * ustep;
                const int q = (b & 1) ? i - kA - u : i + kA + u;
                const bool ok = u < kW && q >= 0 && q < cnt;
                rv[k] = ok ? row[u] : 0.0;
                tv[k] = ok ? t[q + m] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int u = (threadIdx.x + k * 256) * ustep;
                const int q = (b & 1) ? i - kA - u : i + kA + u;
                if (u < kW && q >= 0 && q < cnt) row[u] = fma(ti, tv[k], rv[k]);
            }
        }
        return;
    }
    float amax = 0.f, bmax = 0.f;
    const double sqm = sqrt((double)m1), inv_m1 = 1.0 / (double)m1;
    const int lane = threadIdx.x & 31;
    // each warp advances 32 consecutive windows and stores the last 31: lane 0's
    // window is the halo whose new mean the next lane needs for dg (every lane
    // runs exactly one advance; no lane recomputes a neighbour's)
    const int gw = ((blockIdx.x - qblocks) * blockDim.x + threadIdx.x) >> 5,
              nw = ((gridDim.x - qblocks) * blockDim.x) >> 5;
    for (int base = gw * 31; base < cnt; base += nw * 31) {  // warp-uniform
        const int i = base + lane - 1;
        double u = 0.0, s = 0.0;
        if (i >= 0 && i < cnt) advance1(t, m, i, mu_in, sig_in, u, s);
        const double up = __shfl_up_sync(0xffffffffu, u, 1);
        if (lane == 0 || i >= cnt) continue;
        mu_out[i] = u;
        sig_out[i] = s;
        float b2 = 0.f;
        const float ae = stats_err(P1, P2, i, m1, inv_m1, u, s, b2);
        const bool dgn = s < 1.01 * kSigmaEps || !(ae <= (float)kStatsUnreliable);
        nrm[i] = dgn ? 0.f : (float)(1.0 / (sqm * s));
        if (dgn) {
            degenerate_row(t, i, m1, cnt, cr, deg, degc, deg2);
        } else {
            amax = fmaxf(amax, ae);
            bmax = fmaxf(bmax, b2);
        }
        if (i == 0) {
            df[0] = 0.f;
            dg[0] = 0.f;
        } else {
            const double a = t[i + m1 - 1], b = t[i - 1];
            df[i] = (float)((a - b) * 0.5);
            dg[i] = (float)((a - u) + (b - up));
        }
    }
    stats_max_commit(amax, bmax, cr);
}

static int grid_for(long long work, int threads) {
    long long b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

void launch_init_stats(const double* t, int n, int m, double* mu, double* sig, double* scratch_a,
                       double* scratch_b, cudaStream_t st) {
    const int cnt = n - m + 1;
    k_init_prefix<<<1, 1024, 0, st>>>(t, n, m, scratch_a, scratch_b);
    k_init_finish<<<grid_for(cnt, 256), 256, 0, st>>>(scratch_a, scratch_b, cnt, m, mu, sig);
}

void launch_advance_stats(const double* t, int n, int m, double* mu, double* sig, cudaStream_t st) {
    launch_pdl(k_advance, grid_for(n - m, 256), 256, st, t, n, m, mu, sig);
}

void launch_derive(const double* t, int m, int cnt, const double* mu, const double* sig, float* df,
                   float* dg, float* nrm, int* crange, int* deg, const double2* P1, const double2* P2,
                   int* degc, int* deg2, cudaStream_t st) {
    launch_pdl(k_derive, grid_for(cnt, 256), 256, st, t, m, cnt, mu, sig, df, dg, nrm, crange, deg, P1, P2, degc,
               deg2);
}

int dd_prefix_blocks(int n) { return std::max(1, std::min(148 * 4, (n + 4095) / 4096)); }

void launch_dd_prefix(const double* t, int n, double2* tot1, double2* tot2, double2* P1, double2* P2,
                      cudaStream_t st) {
    const int nb = dd_prefix_blocks(n);
    const int chunk = (n + nb - 1) / nb;
    k_dd_chunk_sums<<<nb, kPfxThreads, 0, st>>>(t, n, chunk, tot1, tot2);
    k_dd_scan_totals<<<1, 1, 0, st>>>(tot1, tot2, nb);
    k_dd_chunk_scan<<<nb, kPfxThreads, 0, st>>>(t, n, chunk, tot1, tot2, P1, P2);
}

void launch_next_length(const double* t, int n, int m, const double* mu_in, const double* sig_in, double* mu_out,
                        double* sig_out, float* df, float* dg, float* nrm, int* cr, int* cr_next, int L, int kA,
                        int nb, int bstep, int ustep, double* qt, int* deg, const double2* P1, const double2* P2,
                        int* degc, int* deg2, cudaStream_t st) {
    const int rows = qt != nullptr ? (nb + bstep - 1) / bstep : 0;
    const int qblocks = std::min(rows, 148 * 4);
    launch_pdl(k_next_length, grid_for(n - m, 256) + qblocks, 256, st, t, n, m, mu_in, sig_in, mu_out, sig_out, df, dg,
               nrm, cr, cr_next, L, kA, nb, bstep, ustep, qt, deg, P1, P2, degc, deg2, qblocks);
}

}  // namespace tsd
