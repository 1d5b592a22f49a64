// Micro-benchmark: per-SM issue rates of DFMA, F2F.F64.F32 / F2F.F32.F64 and the dependent DFMA latency
// on this GPU (design evidence for the fp64 kernels: k_small.cu, k_scan.cu, k_fixup.cu).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_rate fp64_rate.cu && ./fp64_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, float* outf, int iters, double a, float fa) {
    double x[8];
    float f[8];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-3 + i; f[i] = float(threadIdx.x) + i; }
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // independent DFMAs
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, 1.0);
        } else if (MODE == 1) {  // one dependent chain
#pragma unroll
            for (int i = 0; i < 8; ++i) x[0] = fma(x[0], a, 1.0);
        } else if (MODE == 2) {  // fp32 -> fp64 -> add -> fp32 round trips (2 conversions + 1 DADD each)
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = float(double(f[i]) + a);
        } else if (MODE == 3) {  // independent FFMAs for comparison
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], fa, 1.0f);
        }
    }
    double s = 0; float sf = 0;
    for (int i = 0; i < 8; ++i) { s += x[i]; sf += f[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    outf[blockIdx.x * blockDim.x + threadIdx.x] = sf;
}

template <int MODE>
void run(const char* name, int warps_per_sm, double ops_per_iter) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = warps_per_sm * 32, iters = 20000;
    double* out; float* outf;
    cudaMalloc(&out, sizeof(double) * sms * threads); cudaMalloc(&outf, sizeof(float) * sms * threads);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<sms, threads>>>(out, outf, 100, 1.0000001, 1.0000001f);
    cudaEventRecord(e0);
    k<MODE><<<sms, threads>>>(out, outf, iters, 1.0000001, 1.0000001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cycles = ms * 1e-3 * clk * 1e3;
    const double lane_ops = double(threads) * iters * ops_per_iter;  // per SM
    printf("%-28s %2d warps/SM: %.2f lane-ops/clk/SM, %.1f cycles per warp-iteration (8 ops)\n", name, warps_per_sm,
           lane_ops / cycles, cycles / iters);
    cudaFree(out); cudaFree(outf);
}

int main() {
    for (int w : {1, 4, 8, 16, 32}) run<0>("DFMA independent", w, 8);
    for (int w : {1, 4}) run<1>("DFMA dependent chain", w, 8);
    for (int w : {1, 4, 8, 16, 32}) run<2>("F2D + DADD + D2F", w, 8);
    for (int w : {4, 16}) run<3>("FFMA independent", w, 8);
    return 0;
}
