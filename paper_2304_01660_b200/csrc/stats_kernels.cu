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
                         int* __restrict__ deg) {
    pdl_enter();
    const double sqm = sqrt((double)m);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const double s = sig[i];
        nrm[i] = s < kSigmaEps ? 0.f : (float)(1.0 / (sqm * s));
        if (s < kSigmaEps) {
            atomicMax(&cr[0], cnt - i);
            atomicMax(&cr[1], i + 1);
            deg[atomicAdd(&cr[2], 1)] = i;  // decided exactly, against every q
        }
        if (i == 0) {
            df[0] = 0.f;
            dg[0] = 0.f;
        } else {
            const double a = t[i + m - 1], b = t[i - 1];
            df[i] = (float)((a - b) * 0.5);
            dg[i] = (float)((a - mu[i]) + (b - mu[i - 1]));
        }
    }
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

__global__ void k_next_length(const double* __restrict__ t, int n, int m, const double* __restrict__ mu_in,
                              const double* __restrict__ sig_in, double* __restrict__ mu_out,
                              double* __restrict__ sig_out, float* __restrict__ df, float* __restrict__ dg,
                              float* __restrict__ nrm, int* __restrict__ cr, int* __restrict__ cr_next, int L, int kA,
                              int nb, double* __restrict__ qt, int* __restrict__ deg) {
    pdl_enter();
    const int m1 = m + 1, cnt = n - m;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        cr_next[0] = 0;
        cr_next[1] = 0;
        cr_next[2] = 0;
    }
    const double sqm = sqrt((double)m1);
    const int lane = threadIdx.x & 31;
    // the loop bound is warp-uniform (the shuffle below needs every lane)
    const int cnt_w = (cnt + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt_w; i += gridDim.x * blockDim.x) {
        double u = 0.0, s = 0.0;
        if (i < cnt) advance1(t, m, i, mu_in, sig_in, u, s);
        // mu_{i-1} of length m+1 from the neighbouring lane (lane 0 recomputes it)
        double up = __shfl_up_sync(0xffffffffu, u, 1);
        if (i >= cnt) continue;
        mu_out[i] = u;
        sig_out[i] = s;
        nrm[i] = s < kSigmaEps ? 0.f : (float)(1.0 / (sqm * s));
        if (s < kSigmaEps) {
            atomicMax(&cr[0], cnt - i);
            atomicMax(&cr[1], i + 1);
            deg[atomicAdd(&cr[2], 1)] = i;  // decided exactly, against every q
        }
        if (i == 0) {
            df[0] = 0.f;
            dg[0] = 0.f;
        } else {
            if (lane == 0) {
                double sp;
                advance1(t, m, i - 1, mu_in, sig_in, up, sp);  // same rounding as the neighbour's
            }
            const double a = t[i + m1 - 1], b = t[i - 1];
            df[i] = (float)((a - b) * 0.5);
            dg[i] = (float)((a - u) + (b - up));
        }
    }
    if (qt != nullptr) {
        // one seed row per block iteration: no 64-bit index division, the row
        // value t[i+m] is a broadcast, qt and t[q+m] are coalesced
        for (int b = blockIdx.x; b < nb; b += gridDim.x) {
            const int j = b >> 1;
            const int i = (b & 1) ? j * L + L - 1 : j * L;
            if (i >= cnt) continue;
            const double ti = t[i + m];
            double* row = qt + (size_t)b * kW;
            for (int u = threadIdx.x; u < kW; u += blockDim.x) {
                const int q = (b & 1) ? i - kA - u : i + kA + u;
                if (q >= 0 && q < cnt) row[u] = fma(ti, t[q + m], row[u]);
            }
        }
    }
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
                   float* dg, float* nrm, int* crange, int* deg, cudaStream_t st) {
    launch_pdl(k_derive, grid_for(cnt, 256), 256, st, t, m, cnt, mu, sig, df, dg, nrm, crange, deg);
}

void launch_next_length(const double* t, int n, int m, const double* mu_in, const double* sig_in, double* mu_out,
                        double* sig_out, float* df, float* dg, float* nrm, int* cr, int* cr_next, int L, int kA,
                        int nb, double* qt, int* deg, cudaStream_t st) {
    launch_pdl(k_next_length, grid_for(n - m, 256), 256, st, t, n, m, mu_in, sig_in, mu_out, sig_out, df, dg, nrm, cr,
               cr_next, L, kA, nb, qt, deg);
}

}  // namespace tsd
