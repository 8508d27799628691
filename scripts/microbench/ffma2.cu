#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, float a, float b, int iters) {
    float c[16];
    float2 c2[8];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = threadIdx.x * 0.001f + i;
#pragma unroll
    for (int i = 0; i < 8; ++i) c2[i] = make_float2(c[2 * i], c[2 * i + 1]);
    const float2 a2 = make_float2(a, b), b2 = make_float2(b, a);
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) c[i] = fmaf(c[i], a, b);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) c2[i] = __ffma2_rn(c2[i], a2, b2);
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c2[i].x + c2[i].y;
    if (s == 1234.5f) out[0] = s;
}
int main() {
    float* o; cudaMalloc(&o, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) for (int rep = 0; rep < 2; ++rep) {
        const int iters = 20000, blocks = 148 * 8, threads = 256;
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<blocks, threads>>>(o, 0.999f, 0.001f, iters);
        else k<1><<<blocks, threads>>>(o, 0.999f, 0.001f, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * iters * (double)blocks * threads;
        printf("mode %s: %.3f ms  %.1f TFLOP/s\n", mode ? "FFMA2" : "FFMA ", ms, flops / ms / 1e9);
    }
}
