// Independent FP64 matrix profile on the device (a
// brute-force checker for C4/C5 sizes, where the reference's brute_force_nn
// (src/drag.cpp:137-149, O(N^2 m)) and the CPU reference (~1 h) are out of
// reach).  Different algorithm and arithmetic from the product path: the
// STOMP diagonal recurrence QT(i+1,j+1) = QT(i,j) - t_i t_j + t_{i+m} t_{j+m}
// in FP64 on a mean-centred copy of the series, re-seeded by a direct dot
// product every kRowsMP rows, with every cell's correlation evaluated (no
// pruning).  It agrees with the reference's exact distances to ~1e-10
// relative, which is what the tests allow.
//
// Layout: thread = one diagonal k >= m, CTA = 128 consecutive diagonals x a
// row chunk.  Only column maxima of the correlation are kept: a column's
// running max moves one lane down per step (__shfl_down), lane 0 retires it
// into a shared-memory column array, and the CTA flushes that array with one
// global atomicMax per column.  Cells below the diagonal come from the same
// kernel on the reversed series (a reversal maps subsequence i to N-1-i and
// preserves z-normalised distances).
#include <float.h>
#include <math.h>
#include <stdint.h>

#include "engine_internal.h"

namespace tsd {

constexpr int kRowsMP = 2048;  // rows per CTA (one direct seed per thread each)
constexpr int kDiagMP = 128;   // diagonals per CTA

__device__ __forceinline__ unsigned long long okey(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// best[c] (ordered key) = max over rows r <= c - m of corr(r, c)
__global__ void __launch_bounds__(kDiagMP) k_mp_cols(const double* __restrict__ tc, int N, int m,
                                                     const double* __restrict__ mu,
                                                     const double* __restrict__ isg,
                                                     unsigned long long* __restrict__ best) {
    __shared__ unsigned long long colbest[kRowsMP + kDiagMP];
    const int lane = threadIdx.x & 31;
    const long long k0 = (long long)m + (long long)blockIdx.x * kDiagMP;  // CTA's first diagonal
    const long long k = k0 + threadIdx.x;
    const int i0 = blockIdx.y * kRowsMP;
    if (k0 >= N || i0 + k0 >= N) return;  // no valid cell (uniform)
    const int rows = min(kRowsMP, N - i0);
    for (int x = threadIdx.x; x < kRowsMP + kDiagMP; x += blockDim.x) colbest[x] = 0ull;
    __syncthreads();
    const double inv_m = 1.0 / (double)m;
    // direct seed QT(i0, i0 + k)
    double qt = 0.0;
    if (i0 + k < N)
        for (int p = 0; p < m; ++p) qt = fma(tc[i0 + p], tc[i0 + k + p], qt);
    double cm = -DBL_MAX;  // running max of the column this lane holds
    const long long c0 = (long long)i0 + k0;  // CTA's first column
    for (int s = 0; s < rows; ++s) {
        const int i = i0 + s;
        const long long j = (long long)i + k;
        double corr = -DBL_MAX;
        if (j < N) {
            if (s > 0) qt = fma(tc[i + m - 1], tc[j + m - 1], fma(-tc[i - 1], tc[j - 1], qt));
            const double si = isg[i], sj = isg[j];
            if (si == 0.0 && sj == 0.0) corr = 1.0;  // both constant: d = 0
            else corr = (qt - (double)m * mu[i] * mu[j]) * si * sj * inv_m;  // one constant: 0 (d = 2m)
        }
        cm = fmax(cm, corr);
        if (lane == 0 && cm > -DBL_MAX) atomicMax(&colbest[s + (threadIdx.x >> 5) * 32], okey(cm));
        cm = __shfl_down_sync(0xffffffffu, cm, 1);
        if (lane == 31) cm = -DBL_MAX;
    }
    // columns still held: lane l holds column i0 + rows + k0 + l (offset rows + tid)
    if (cm > -DBL_MAX) atomicMax(&colbest[rows + threadIdx.x], okey(cm));
    __syncthreads();
    for (int x = threadIdx.x; x < rows + kDiagMP; x += blockDim.x) {
        const long long c = c0 + x;
        if (c < N && colbest[x] != 0ull) atomicMax(&best[c], colbest[x]);
    }
}

// centred copy of the series (and its reversal)
__global__ void k_mp_center(const double* __restrict__ t, int n, double gmean, double* __restrict__ tc,
                            double* __restrict__ tr) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const double v = t[p] - gmean;
        tc[p] = v;
        tr[n - 1 - p] = v;
    }
}

// per-window mean and 1/sigma by two passes over the centred window (not the
// rolling Eq. 4/7-8 statistics: at n=1M their sigma carries ~1e-9 relative
// error, which the exact distance of the reference does not have)
__global__ void k_mp_stats(const double* __restrict__ tc, int N, int m, double* __restrict__ muc,
                           double* __restrict__ mur, double* __restrict__ isg, double* __restrict__ isr) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < m; ++p) s += tc[i + p];
        const double mean = s / (double)m;
        double q = 0.0;
        for (int p = 0; p < m; ++p) {
            const double d = tc[i + p] - mean;
            q = fma(d, d, q);
        }
        const double sg = sqrt(q / (double)m);
        const double is = sg < kSigmaEps ? 0.0 : 1.0 / sg;
        muc[i] = mean;
        mur[N - 1 - i] = mean;
        isg[i] = is;
        isr[N - 1 - i] = is;
    }
}

__global__ void k_mp_finish(const unsigned long long* __restrict__ fwd, const unsigned long long* __restrict__ rev,
                            int N, int m, double* __restrict__ out) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
        const unsigned long long a = fwd[c], b = rev[N - 1 - c];
        const unsigned long long k = a > b ? a : b;
        out[c] = k == 0ull ? __longlong_as_double(0x7ff0000000000000ll)  // no non-self match: +inf
                           : 2.0 * (double)m * (1.0 - okey_inv(k));
    }
}

void mp_fp64(const double* t, int n, int m, double gmean, double* scratch,
             unsigned long long* keys, double* out, cudaStream_t st) {
    const int N = n - m + 1;
    double* tc = scratch;
    double* tr = tc + n;
    double* muc = tr + n;
    double* mur = muc + N;
    double* isg = mur + N;
    double* isr = isg + N;
    k_mp_center<<<148 * 4, 256, 0, st>>>(t, n, gmean, tc, tr);
    k_mp_stats<<<148 * 4, 256, 0, st>>>(tc, N, m, muc, mur, isg, isr);
    cudaMemsetAsync(keys, 0, 2 * (size_t)N * sizeof(unsigned long long), st);
    const long long ndiag = (long long)N - m;  // diagonals k in [m, N-1]
    if (ndiag > 0) {
        dim3 grid((unsigned)((ndiag + kDiagMP - 1) / kDiagMP), (unsigned)((N + kRowsMP - 1) / kRowsMP));
        k_mp_cols<<<grid, kDiagMP, 0, st>>>(tc, N, m, muc, isg, keys);
        k_mp_cols<<<grid, kDiagMP, 0, st>>>(tr, N, m, mur, isr, keys + N);
    }
    k_mp_finish<<<148 * 4, 256, 0, st>>>(keys, keys + N, N, m, out);
}

}  // namespace tsd
