// FP32 FFMA throughput probe (diagnostic; gives the roofline denominator for the
// FP32-bound scan kernel, since MEASURED_PEAKS.json carries only HBM and bf16).
#include <cuda_runtime.h>

#include "../../include/tsdiscord_b200.h"

namespace {

// 8 independent chains per thread, 3-register FFMA form (like the scan's cell update).
__global__ void k_ffma(float* out, float b, int iters) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
          a6 = a0 + 6, a7 = a0 + 7;
    const float c = b * 0.5f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fmaf(a0, b, c);
            a1 = fmaf(a1, b, c);
            a2 = fmaf(a2, b, c);
            a3 = fmaf(a3, b, c);
            a4 = fmaf(a4, b, c);
            a5 = fmaf(a5, b, c);
            a6 = fmaf(a6, b, c);
            a7 = fmaf(a7, b, c);
        }
    }
    const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1234.5f) out[blockIdx.x] = s;  // keep the work alive
}

}  // namespace

extern "C" int tsd_fp32_peak_probe(int device, double* tflops) {
    if (!tflops) return TSD_EINVAL;
    *tflops = 0.0;
    if (cudaSetDevice(device) != cudaSuccess) return TSD_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, 4096 * sizeof(float)) != cudaSuccess) return TSD_ECUDA;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    k_ffma<<<blocks, threads>>>(out, 0.999f, 64);  // warm-up
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_ffma<<<blocks, threads>>>(out, 0.999f, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double flops = 2.0 * 16.0 * 8.0 * (double)iters * threads * (double)blocks;
        if (ms > 0) best = flops / (ms * 1e-3) / 1e12 > best ? flops / (ms * 1e-3) / 1e12 : best;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return TSD_ECUDA;
    *tflops = best;
    return TSD_OK;
}
