// erx_common.cuh — device helpers shared by the ERX kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "erx_kernels.cuh"

namespace erxk {

__host__ __device__ __forceinline__ size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Line l = s * n + t of a window whose input buffer holds in_stride lines per stream.
__device__ __forceinline__ const float* line_ptr(const float* x, int line, int n, int in_stride, const Geometry& g) {
    const int s = line / n, t = line - s * n;
    return x + (size_t(s) * in_stride + t) * size_t(g.P) * g.B;
}

// Sparse random projection of one pixel row onto output dim j (project_line,
// projection.hpp:31-34): z_j = |w| * sum_k sign_k x[band_k], summed in fp64 —
// an fp32 radiance times +-1 is exact and the sum keeps fp64 precision, so z
// matches the reference's fp64 Z = X W to rounding.
__device__ __forceinline__ double srp_z(const Geometry& g, const float* __restrict__ row, int j) {
    double z = 0.0;
    for (int k = g.srp_ptr[j]; k < g.srp_ptr[j + 1]; ++k) z += double(__ldg(row + g.srp_band[k])) * double(g.srp_w[k]);
    return z * g.srp_scale;
}

// Projected value of dim j of a pixel row (identity or SRP), fp64.
__device__ __forceinline__ double proj(const Geometry& g, const float* __restrict__ row, int j) {
    return g.srp ? srp_z(g, row, j) : double(__ldg(row + j));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Conditioning bound of the fp32 factor: a line whose Cholesky pivot L_ii^2 falls below
// (K + eps I)_ii / kCondTau is factored again in fp64 (k_fixup.cu).  Emulated fp32 factor +
// whitening against fp64: median raw-score error ~2e-9 x max_i A_ii / L_ii^2, so
// 1e3 keeps the fp32 lines ~5x inside the 1e-5 median gate; every BASELINE config stays below ~500.
constexpr float kCondTau = 1000.f;

// Put a line the fp32 factor gave up on onto the fp64 rescue list ([0] count, [2..] lines).
__device__ __forceinline__ void list_for_fixup(int* fixlist, int* status, int line) {
    status[line] = -2;  // pending: the rescue writes the final status
    const int pos = atomicAdd(fixlist, 1);
    fixlist[2 + pos] = line;
}

// A line whose scores spread less than kFlatRel of their mean (e.g. a two-pixel line scored
// against its own statistics: both deltas are equal, std = 0 in fp64) is normalised from fp32
// deltas whose own rounding is then comparable to that spread; the fp64 rescue redoes it, so the
// zero-variance rule (std < 1e-12 -> 0) is applied to fp64 deltas as the reference
// does.  Real lines spread by tens of percent (delta ~ chi with D degrees of freedom).
constexpr double kFlatRel = 1e-2;
__device__ __forceinline__ bool flat_line(double mean, double sd) { return mean > 0.0 && sd < kFlatRel * mean; }

// Per-device launch helpers.  Function attributes and SM counts are per device, so engines on
// several GPUs in one process (or host threads) each get them set; the calls are idempotent.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev);
}
// (Always set: a per-type cache would be shared by kernels with the same signature; the call is
// cheap next to the kernels it precedes.)
template <typename Kernel>
inline void ensure_smem(Kernel kernel, size_t bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}
inline int sm_count() {
    static std::atomic<int> cache[kMaxDevices];
    const int dev = current_device();
    int n = cache[dev].load(std::memory_order_relaxed);
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

}  // namespace erxk
