// Heatmap / ranking of a multi-length discord set on the device (SURVEY §8f
// rank 2; reference src/heatmap.cpp:18-57, PAPER Eq. 10/11).
//
// The score matrix is rows = lengths minL..maxL x cols = start indices
// 1..n-minL, row-major FP64 (C4: 513 x 999,488 = 4.1 GB, resident in HBM).
// Building it is a scatter of the (few) records into a zeroed matrix; the
// ranking needs every column's maximum over the lengths, one HBM-bound pass
// over the whole matrix (k_hm_colmax), followed by a host sort of the
// non-zero columns (at most one per record).
#include <stdint.h>

#include "engine_internal.h"

namespace tsd {

__global__ void k_hm_scatter(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols_idx,
                             const double* __restrict__ vals, int64_t count, int64_t ncols,
                             double* __restrict__ hm) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x)
        hm[rows[e] * ncols + cols_idx[e]] = vals[e];
}

// Per column: the largest score and the first (smallest) length reaching it
// (heatmap.cpp:37-45 keeps the first strict maximum over ascending lengths).
// Thread per column; a warp reads 32 consecutive doubles of a row, the row
// loop is unrolled for memory-level parallelism.
__global__ void __launch_bounds__(256) k_hm_colmax(const double* __restrict__ hm, int64_t nrows, int64_t ncols,
                                                   int64_t min_len, HmCol* __restrict__ out,
                                                   unsigned long long* __restrict__ count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncols;
         i += (int64_t)gridDim.x * blockDim.x) {
        double best = 0.0;
        int64_t len = 0;
        int64_t r = 0;
        for (; r + 8 <= nrows; r += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(&hm[(r + u) * ncols + i]);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (v[u] > best) {
                    best = v[u];
                    len = min_len + r + u;
                }
        }
        for (; r < nrows; ++r) {
            const double v = __ldcs(&hm[r * ncols + i]);
            if (v > best) {
                best = v;
                len = min_len + r;
            }
        }
        if (best > 0.0) {
            const unsigned long long at = atomicAdd(count, 1ull);
            out[at] = HmCol{i + 1, len, best};
        }
    }
}

void launch_hm_scatter(const int64_t* rows, const int64_t* cols_idx, const double* vals, int64_t count,
                       int64_t ncols, double* hm, cudaStream_t st) {
    if (count <= 0) return;
    const int64_t b = (count + 255) / 256;
    k_hm_scatter<<<(int)(b < 4096 ? b : 4096), 256, 0, st>>>(rows, cols_idx, vals, count, ncols, hm);
}

void launch_hm_colmax(const double* hm, int64_t nrows, int64_t ncols, int64_t min_len, HmCol* out,
                      unsigned long long* count, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = (ncols + 255) / 256;
    const int64_t grid = need < (int64_t)sms * 8 ? need : (int64_t)sms * 8;
    k_hm_colmax<<<(int)(grid > 0 ? grid : 1), 256, 0, st>>>(hm, nrows, ncols, min_len, out, count);
}

}  // namespace tsd

// ---------------------------------------------------------------------------
// peer all-reduce (peer_group.cuh): every rank reads all ranks' buffers
#include "peer_group.cuh"

namespace tsd {

template <typename T, int KIND>
__global__ void k_peer_reduce(PeerPtrs in, int nranks, T* __restrict__ out, size_t cnt) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < cnt; i += (size_t)gridDim.x * blockDim.x) {
        T v = static_cast<const T*>(in.p[0])[i];
        for (int r = 1; r < nranks; ++r) {
            const T w = static_cast<const T*>(in.p[r])[i];
            v = KIND == 1 ? (w > v ? w : v) : (w < v ? w : v);
        }
        out[i] = v;
    }
}

// Device-side barrier of a rank group over peer memory (no host round trip):
// one thread fences the rank's preceding work (its peer stores included)
// system-wide, publishes `epoch` in its slot of every rank's flag array, and
// spins until every rank's slot in its own array has reached `epoch`.  Epochs
// only grow, so the flags never need resetting.  A rank that never arrives
// makes the kernel trap after ~10 s (a loud error instead of a hang).
__global__ void k_flag_barrier(FlagPtrs f, int world, int rank, unsigned long long epoch) {
    // no early launch of the dependents: their CTAs would occupy the SMs while
    // this kernel spins, and ranks sharing a device need them to arrive
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x != 0) return;
    __threadfence_system();
    for (int r = 0; r < world; ++r)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f.p[r] + rank), "l"(epoch) : "memory");
    unsigned long long spins = 0;
    for (int r = 0; r < world; ++r) {
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f.p[rank] + r) : "memory");
            if (v >= epoch) break;
            __nanosleep(64);
            if (++spins > (1ull << 27)) __trap();
        }
    }
    __threadfence_system();
}

void launch_flag_barrier(const FlagPtrs& f, int world, int rank, unsigned long long epoch, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_flag_barrier, f, world, rank, epoch);
}

void launch_peer_reduce(int kind, PeerPtrs in, int nranks, void* out, size_t cnt, cudaStream_t st) {
    if (cnt == 0) return;
    size_t b = (cnt + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    if (kind == 0) k_peer_reduce<uint8_t, 0><<<(int)b, 256, 0, st>>>(in, nranks, (uint8_t*)out, cnt);
    else if (kind == 1) k_peer_reduce<unsigned, 1><<<(int)b, 256, 0, st>>>(in, nranks, (unsigned*)out, cnt);
    else k_peer_reduce<unsigned long long, 2><<<(int)b, 256, 0, st>>>(in, nranks, (unsigned long long*)out, cnt);
}

}  // namespace tsd
