// k_probe.cu — FP32 FFMA throughput probe (roofline denominator for the
// FFMA-bound kernels; MEASURED_PEAKS.json carries HBM and bf16 peaks only).
#include <algorithm>

#include "erx_common.cuh"

namespace erxk {
namespace {

__global__ void __launch_bounds__(256) ffma_probe_kernel(int iters, float x, float y, float* sink) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = float(threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], x, y);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 123.456f) sink[0] = s;
}

}  // namespace

double probe_ffma_tflops(cudaStream_t st) {
    float* sink = nullptr;
    cudaMalloc(&sink, sizeof(float));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256, iters = 8192;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a, st);
        ffma_probe_kernel<<<blocks, threads, 0, st>>>(iters, 0.999f, 1e-3f, sink);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0) best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    const double flops = 2.0 * 8.0 * double(iters) * blocks * threads;
    return flops / (double(best) * 1e-3) / 1e12;
}

}  // namespace erxk
