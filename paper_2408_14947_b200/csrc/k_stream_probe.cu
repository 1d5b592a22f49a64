// k_stream_probe.cu — measured streaming throughput of the two global->shared
// paths a memory-bound kernel can use on this GPU (design input for the
// tensor-core stats / score kernels, tools/probe.py):
//   mode 0  cp.async.bulk ring: one thread issues chunk copies into an
//           NS-deep shared-memory ring (mbarrier tx counts), 8 warps release
//   mode 1  LDG.128 by 256 threads (register sink), the plain-load reference
//   mode 2  cp.async 16-byte copies by all 256 threads into the ring
// Each persistent CTA streams its own contiguous share of the buffer.
#include "erx_common.cuh"
#include "tc_common.cuh"

namespace erxk {
namespace {

__global__ void __launch_bounds__(288) stream_probe_kernel(const float* __restrict__ src, size_t n_floats,
                                                           int chunk_floats, int NS, int mode, float* sink) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[8], empty[8];
    float* ring = reinterpret_cast<float*>(smem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t per = (n_floats / gridDim.x) / chunk_floats * chunk_floats;
    const float* base = src + per * blockIdx.x;
    const int nchunks = int(per / chunk_floats);
    if (mode == 1) {
        if (warp >= 8) return;
        float acc = 0.f;
        const float4* p = reinterpret_cast<const float4*>(base);
        const size_t n4 = per / 4;
#pragma unroll 8
        for (size_t i = tid; i < n4; i += 256) {
            const float4 v = __ldcs(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
        if (acc == 12345.f) sink[0] = acc;
        return;
    }
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            tc::mbar_init(&full[s], mode == 0 ? 1 : 256);
            tc::mbar_init(&empty[s], 8);
        }
        tc::fence_barrier_init();
    }
    __syncthreads();
    if (mode == 0) {
        if (warp == 8) {
            if (lane == 0)
                for (int j = 0; j < nchunks; ++j) {
                    const int st = j % NS;
                    if (j >= NS) tc::mbar_wait(&empty[st], uint32_t((j / NS) - 1) & 1u);
                    tc::mbar_expect_tx(&full[st], uint32_t(chunk_floats) * 4);
                    tc::bulk_g2s(ring + size_t(st) * chunk_floats, base + size_t(j) * chunk_floats,
                                 uint32_t(chunk_floats) * 4, &full[st]);
                }
            return;
        }
        float acc = 0.f;
        for (int j = 0; j < nchunks; ++j) {
            const int st = j % NS;
            tc::mbar_wait(&full[st], uint32_t(j / NS) & 1u);
            acc += ring[size_t(st) * chunk_floats + tid];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&empty[st])) : "memory");
        }
        if (acc == 12345.f) sink[0] = acc;
        return;
    }
    // mode 2: every thread copies, multistage cp.async with per-thread mbarrier arrival
    if (warp >= 8) return;
    float acc = 0.f;
    auto issue = [&](int j) {
        const int st = j % NS;
        float* dst = ring + size_t(st) * chunk_floats;
        const float* s = base + size_t(j) * chunk_floats;
        for (int q = tid; q < chunk_floats / 4; q += 256) cp_async16(dst + 4 * q, s + 4 * q);
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[st])) : "memory");
    };
    for (int j = 0; j < NS - 1 && j < nchunks; ++j) issue(j);
    for (int j = 0; j < nchunks; ++j) {
        if (j + NS - 1 < nchunks) {
            if (j >= 1) {
                // stage (j + NS - 1) % NS was consumed at visit j - 1 by every warp
                const int st2 = (j + NS - 1) % NS;
                tc::mbar_wait(&empty[st2], uint32_t((j - 1) / NS) & 1u);
            }
            issue(j + NS - 1);
        }
        const int st = j % NS;
        tc::mbar_wait(&full[st], uint32_t(j / NS) & 1u);
        acc += ring[size_t(st) * chunk_floats + tid];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&empty[st])) : "memory");
    }
    if (acc == 12345.f) sink[0] = acc;
}

}  // namespace

double probe_stream_gbs(cudaStream_t st, int mode, int chunk_bytes, int stages, int ctas_per_sm, size_t bytes) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* buf = nullptr;
    if (cudaMalloc(&buf, bytes + 64) != cudaSuccess) return -1.0;
    cudaMemsetAsync(buf, 0, bytes + 64, st);
    const size_t smem = size_t(chunk_bytes) * stages;
    cudaFuncSetAttribute(stream_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    const int grid = sms * ctas_per_sm;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a, st);
        stream_probe_kernel<<<grid, 288, smem, st>>>(buf, bytes / 4, chunk_bytes / 4, stages, mode, buf + bytes / 4);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    const size_t per = (bytes / 4 / grid) / (chunk_bytes / 4) * (chunk_bytes / 4);
    return double(per) * 4 * grid / (double(best) * 1e-3) / 1e9;
}

}  // namespace erxk
