// Launch wrappers shared between the kernel translation units and the host engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tsd {

// Launch with programmatic stream serialization (kernels call pdl_enter()).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// the same with dynamic shared memory
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_smem(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                   Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

void launch_init_stats(const double* t, int n, int m, double* mu, double* sig, double* scratch_a,
                       double* scratch_b, cudaStream_t st);
void launch_advance_stats(const double* t, int n, int m, double* mu, double* sig, cudaStream_t st);
void launch_derive(const double* t, int m, int cnt, const double* mu, const double* sig, float* df,
                   float* dg, float* nrm, int* crange, int* deg, const double2* P1, const double2* P2,
                   int* degc, int* deg2, cudaStream_t st);
// double-double prefix sums of t and t^2 (n + 1 entries each; tot: dd_prefix_blocks(n) scratch)
int dd_prefix_blocks(int n);
void launch_dd_prefix(const double* t, int n, double2* tot1, double2* tot2, double2* P1, double2* P2,
                      cudaStream_t st);

// advance + derive (+ seed rows when qt != nullptr) of one MERLIN length step
void launch_next_length(const double* t, int n, int m, const double* mu_in, const double* sig_in, double* mu_out,
                        double* sig_out, float* df, float* dg, float* nrm, int* cr, int* cr_next, int L, int kA,
                        int nb, int bstep, int ustep, double* qt, int* deg, const double2* P1, const double2* P2,
                        int* degc, int* deg2, cudaStream_t st);

size_t scan_smem_bytes();
void scan_configure();
// persistent tile scan over the launch's tile space (ScanParams::space)
void launch_scan(int mode, const ScanParams& p, cudaStream_t st);
// mode 0: knife-edge recheck; mode 1: exact nn (ex != nullptr: the last CTA also
// gathers nnout[e] = nn(ex[e]) for e < ctl->ec — single rank only)
void launch_ref_pairs(int mode, const double* t, int m, const int2* pairs, const int* count, int cap,
                      double r_sq, uint8_t* alive, unsigned long long* nnkey, TryCtl* ctl, const int* ex,
                      double* nnout, const Peers& peers, cudaStream_t st);
void launch_survivors(const int* list, const uint8_t* alive, TryCtl* ctl, const unsigned* ymax,
                      const unsigned* emax, const float* nrm, const int* crange, int N, int m, int need,
                      double* lo, double* hi, int* cand, float* ythr, unsigned long long* nnkey, int2* groups,
                      int fixed_span, float seed_w, int* exli, int* surv, cudaStream_t st);
// degenerate rows (sigma < eps): every (alive row, degenerate row) and
// (degenerate row, any q) pair by the exact distance — kills and exact-nn keys
// knife-edge recheck + degenerate pairs in one launch
void launch_recheck(const double* t, int m, int N, const int2* pairs, const int* count, int cap, const int* list,
                    const TryCtl* ctl, const int* crange, const int* degc, const int* deg2, const float* nrm,
                    double r_sq, uint8_t* alive,
                    unsigned long long* nnkey, int rank, int world, const Peers& peers, int* wit, cudaStream_t st);
// overflow fallback: every listed row (ctl->alive of them) still alive x every
// admissible q by the exact routine (kills + exact-nn keys)
void launch_exact_rows(const double* t, int m, int N, const int* list, const TryCtl* ctl, double r_sq,
                       uint8_t* alive, unsigned long long* nnkey, int rank, int world, const Peers& peers,
                       cudaStream_t st);
// kill witnesses of earlier tries tested before band pass 0 (ScanParams::wit)
void launch_witness(const ScanParams& p, int4* wl, int2* wl2, cudaStream_t st);  // wl, wl2: N entries of scratch
void launch_try_init(uint8_t* alive, unsigned* ymax, unsigned* emax, float* ythr, unsigned long long* nnkey, int N,
                     TryCtl* ctl, unsigned long long* acc, int band_k0, cudaStream_t st);
int compact_blocks(int n);
// gate: band pass index (>= 0), kGateNone or kGateTrack (common.cuh)
// compaction + break rule + grouping in one kernel (status: >= compact_blocks(n)
// words; slots: group_slots(n) entries)
void launch_compact_group(const uint8_t* a, int n, int* out, unsigned long long* status, unsigned epoch,
                          TryCtl* ctl, int gate, int2* groups, int2* slots, int m, int fixed_span, float band_keep,
                          int band_few, float seed_w, double* bcost, int band_slots, cudaStream_t st);
int group_slots(int n);
int scan_slots_prune();
int band0_pk_slots();    // persistent grid of the pair-kill band-0 walk (k_band0_pk)
int band0_pair_slots();  // persistent grid of the paired band-0 walk (k_band0_pair)  // persistent grid of the band-pass scan (SMs x resident CTAs)
// tracked full-row chunks: schedule of the first chunk (after the band passes)
void launch_track_init(TryCtl* ctl, int N, int m, bool bands_ran, cudaStream_t st);
// row cache (ScanParams::rcqt): fill one slot at length m / advance every slot m -> m+1
void launch_rc_fill(const double* t, int n, int m, int a, double* qt, cudaStream_t st);
void launch_rc_advance(const double* t, int n, int m, const RcRows& rows, long long stride, double* qt,
                       cudaStream_t st);
// bstep 2: the positive-side rows only (even indices; the pair-kill band 0)
void launch_seed_init(const double* t, int n, int m, int L, int kA, int nb, int bstep, int ustep, double* qt,
                      cudaStream_t st);
void launch_seed_advance(const double* t, int n, int m, int L, int kA, int nb, int bstep, int ustep, double* qt,
                         cudaStream_t st);
void launch_gather_nn(const int* list, const int* cnt, const unsigned long long* nnkey, double* out,
                      cudaStream_t st);

// independent FP64 matrix profile (mp_fp64.cu); scratch: 2n + 4N doubles, keys: 2N
void mp_fp64(const double* t, int n, int m, double gmean, double* scratch,
             unsigned long long* keys, double* out, cudaStream_t st);

// heatmap (heatmap_kernels.cu)
struct HmCol {
    int64_t index;   // 1-based start index
    int64_t length;  // first length reaching the column maximum
    double score;    // column maximum
};
void launch_hm_scatter(const int64_t* rows, const int64_t* cols_idx, const double* vals, int64_t count,
                       int64_t ncols, double* hm, cudaStream_t st);
void launch_hm_colmax(const double* hm, int64_t nrows, int64_t ncols, int64_t min_len, HmCol* out,
                      unsigned long long* count, cudaStream_t st);

}  // namespace tsd
