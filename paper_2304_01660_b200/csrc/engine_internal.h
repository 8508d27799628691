// Launch wrappers shared between the kernel translation units and the host engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tsd {

void launch_init_stats(const double* t, int n, int m, double* mu, double* sig, double* scratch_a,
                       double* scratch_b, cudaStream_t st);
void launch_advance_stats(const double* t, int n, int m, double* mu, double* sig, cudaStream_t st);
void launch_derive(const double* t, int m, int cnt, const double* mu, const double* sig, float* df,
                   float* dg, float* nrm, cudaStream_t st);

size_t scan_smem_bytes();
void scan_configure();
void launch_scan(int mode, int ntiles, const ScanParams& p, cudaStream_t st);
void launch_ref_pairs(int mode, const double* t, int m, const int2* pairs, const int* count, int cap,
                      double r_sq, uint8_t* alive, unsigned long long* nnkey, int max_pairs,
                      cudaStream_t st);
void launch_fill_u8(uint8_t* a, int n, uint8_t v, cudaStream_t st);
int compact_blocks(int n);
void launch_compact(const uint8_t* a, int n, int* blk, int* out, cudaStream_t st);
void launch_prep_survivors(const int* list, int cnt, const unsigned* ymax, const unsigned* emax, float* ythr,
                           unsigned long long* nnkey, cudaStream_t st);
void launch_nn_bounds(const int* list, int cnt, const unsigned* ymax, const unsigned* emax, const float* nrm,
                      const int* const_range, int N, int m, double* lo, double* hi, cudaStream_t st);
void launch_seed_init(const double* t, int n, int m, int L, int kA, int nb, double* qt, cudaStream_t st);
void launch_seed_advance(const double* t, int n, int m, int L, int kA, int nb, double* qt, cudaStream_t st);
void launch_const_range(const float* nrm, int N, int* out, cudaStream_t st);
void launch_const_nn(const int* list, int cnt, const float* nrm, const int* const_range, int N, int m,
                     unsigned long long* nnkey, cudaStream_t st);
void launch_gather_nn(const int* list, int cnt, const unsigned long long* nnkey, double* out,
                      cudaStream_t st);

}  // namespace tsd
