// probe_api.cu — C ABI of liberx_probe.so (include/erx_probe.h): the device
// probes and tcgen05 self-tests, kept out of the product library.
#include <cuda_runtime.h>

#include "../../include/erx_probe.h"
#include "erx_common.cuh"

namespace erxk {
// k_probe.cu, k_stream_probe.cu, k_tc_selftest.cu
void probe_ffma_tflops(cudaStream_t st, double* reg_form, double* const_form);
double probe_ffma2_tflops(cudaStream_t st);
double probe_stream_gbs(cudaStream_t st, int mode, int chunk_bytes, int stages, int ctas_per_sm, size_t bytes);
int tc_selftest(const float* dA, const float* dB, int K, int split, float* dD, cudaStream_t st);
int tc_selftest_i8(const int8_t* dA, const int8_t* dB, int K, int N, int a_mn, int ms, int ks, int lbo, int sbo,
                   int* dD, cudaStream_t st);
}  // namespace erxk

namespace {
constexpr int kOk = 0, kBad = 2, kCuda = 16;
int enter(int device) { return cudaSetDevice(device) == cudaSuccess ? kOk : kCuda; }
int leave() { return cudaGetLastError() == cudaSuccess ? kOk : kCuda; }
}  // namespace

extern "C" {

int erx_probe_fp32_tflops(int device, void* stream, double* reg_form, double* const_form) {
    if (enter(device)) return kCuda;
    double r = 0, c = 0;
    erxk::probe_ffma_tflops(static_cast<cudaStream_t>(stream), &r, &c);
    if (reg_form) *reg_form = r;
    if (const_form) *const_form = c;
    return leave();
}

int erx_probe_ffma2_tflops(int device, void* stream, double* tflops) {
    if (enter(device)) return kCuda;
    *tflops = erxk::probe_ffma2_tflops(static_cast<cudaStream_t>(stream));
    return leave();
}

int erx_probe_stream(int device, void* stream, int mode, uint32_t chunk_bytes, int stages, int ctas_per_sm,
                     uint64_t bytes, double* gbs) {
    if (mode < 0 || mode > 2 || stages < 1 || stages > 8 || chunk_bytes % 1024 || ctas_per_sm < 1) return kBad;
    if (enter(device)) return kCuda;
    *gbs = erxk::probe_stream_gbs(static_cast<cudaStream_t>(stream), mode, int(chunk_bytes), stages, ctas_per_sm,
                                  size_t(bytes));
    return leave();
}

int erx_tc_selftest(int device, void* stream, const float* dA, const float* dB, int K, int split, float* dD) {
    if (K % 16 || K < 16 || K > 256) return kBad;
    if (enter(device)) return kCuda;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (erxk::tc_selftest(dA, dB, K, split, dD, st) != 0) return kCuda;
    if (cudaStreamSynchronize(st) != cudaSuccess) return kCuda;
    return leave();
}

int erx_tc_selftest_i8(int device, void* stream, const int8_t* dA, const int8_t* dB, int K, int N, int a_mn,
                       int ms, int ks, int lbo, int sbo, int* dD) {
    if (K < 32 || K % 32 || K > 128 || N < 16 || N > 128 || N % 16) return kBad;
    if (enter(device)) return kCuda;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (erxk::tc_selftest_i8(dA, dB, K, N, a_mn, ms, ks, lbo, sbo, dD, st) != 0) return kCuda;
    if (cudaStreamSynchronize(st) != cudaSuccess) return kCuda;
    return leave();
}

}  // extern "C"
