// k_tc_selftest.cu — hardware check of the hand-written tcgen05 path
// (tc_common.cuh): D[128][128] = A[128][K] . B[128][K]^T with A, B given in
// fp32, computed either from single bf16 planes (split = 0) or with the
// 3-way bf16 split and 6 MMA products (split = 1).  Exposed through the
// C ABI (erx_tc_selftest) so tests can compare with a host reference.
#include "erx_common.cuh"
#include "tc_common.cuh"

namespace erxk {
namespace {

__global__ void __launch_bounds__(128) tc_selftest_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                          int K, int split, float* __restrict__ D) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t plane = uint32_t(K / 16) * tc::kSliceBytes;  // bytes per operand plane
    unsigned char* pa = smem;              // A planes: hi, mid, lo
    unsigned char* pb = smem + 3 * plane;  // B planes
    // thread = row m; 8 consecutive k per 16-byte store
    for (int k0 = 0; k0 < K; k0 += 8) {
        uint32_t ah[4], am[4], al[4], bh[4], bm[4], bl[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            tc::split3_bf16x2(A[tid * K + k0 + 2 * j], A[tid * K + k0 + 2 * j + 1], ah[j], am[j], al[j]);
            tc::split3_bf16x2(B[tid * K + k0 + 2 * j], B[tid * K + k0 + 2 * j + 1], bh[j], bm[j], bl[j]);
        }
        const uint32_t off = tc::kmajor_off(tid, k0);
        *reinterpret_cast<uint4*>(pa + off) = make_uint4(ah[0], ah[1], ah[2], ah[3]);
        *reinterpret_cast<uint4*>(pa + plane + off) = make_uint4(am[0], am[1], am[2], am[3]);
        *reinterpret_cast<uint4*>(pa + 2 * plane + off) = make_uint4(al[0], al[1], al[2], al[3]);
        *reinterpret_cast<uint4*>(pb + off) = make_uint4(bh[0], bh[1], bh[2], bh[3]);
        *reinterpret_cast<uint4*>(pb + plane + off) = make_uint4(bm[0], bm[1], bm[2], bm[3]);
        *reinterpret_cast<uint4*>(pb + 2 * plane + off) = make_uint4(bl[0], bl[1], bl[2], bl[3]);
    }
    if (warp == 0) tc::tmem_alloc<128>(&tmem_slot);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_barrier_init();
    }
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_bf16_f32(128, 128);
        const uint32_t a0 = tc::smem_u32(pa), b0 = tc::smem_u32(pb);
        // products: (hi,hi) then, when split, (hi,mid) (mid,hi) (hi,lo) (lo,hi) (mid,mid)
        const int pairs[6][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {2, 0}, {1, 1}};
        const int np = split ? 6 : 1;
        uint32_t acc = 0;
        for (int s = 0; s < K / 16; ++s)
            for (int q = 0; q < np; ++q) {
                const uint64_t ad = tc::smem_desc(a0 + pairs[q][0] * plane + s * tc::kSliceBytes);
                const uint64_t bd = tc::smem_desc(b0 + pairs[q][1] * plane + s * tc::kSliceBytes);
                tc::mma_bf16(tmem, ad, bd, idesc, acc);
                acc = 1;
            }
        tc::mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::tc_fence_after();
    // warp w reads TMEM lanes 32w..32w+31 (rows), 128 columns
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) D[row * 128 + c0 + i] = v[i];
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<128>(tmem);
}

// int8 check: D[128][N] (s32) = A[128][K] . B[N][K]^T, K = 32 * ksteps.  A is laid out either
// K-major (kmajor_off_s8) or MN-major: K-step s, 16-row M group mg, 8-row K group kg at
// s * 4096 + mg * ms + kg * ks (+ row * 16 + m % 16), described with (lbo, sbo).
__global__ void __launch_bounds__(128) tc_selftest_i8_kernel(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                             int K, int N, int a_mn, int ms, int ks, int lbo, int sbo,
                                                             int* __restrict__ D) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int ksteps = K / 32;
    unsigned char* pa = smem;
    unsigned char* pb = smem + ksteps * 4096;
    for (int m = tid; m < 128; m += 128)
        for (int k = 0; k < K; ++k) {
            uint32_t off;
            if (a_mn) {
                const int s = k >> 5, kg = (k & 31) >> 3, r = k & 7, mg = m >> 4;
                off = uint32_t(s * 4096 + mg * ms + kg * ks + r * 16 + (m & 15));
            } else {
                off = tc::kmajor_off_s8(m, k);
            }
            pa[off] = uint8_t(A[m * K + k]);
        }
    for (int n = tid; n < N; n += 128)
        for (int k = 0; k < K; ++k) pb[tc::kmajor_off_s8(n, k)] = uint8_t(B[n * K + k]);
    if (warp == 0) tc::tmem_alloc<256>(&tmem_slot);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_barrier_init();
    }
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_s8_s32(128, N, a_mn != 0, false);
        for (int s = 0; s < ksteps; ++s) {
            const uint64_t ad = a_mn ? tc::smem_desc_ls(tc::smem_u32(pa) + s * 4096, uint32_t(lbo), uint32_t(sbo))
                                     : tc::smem_desc(tc::smem_u32(pa) + s * 4096);
            const uint64_t bd = tc::smem_desc(tc::smem_u32(pb) + s * 4096);
            tc::mma_s8(tmem, ad, bd, idesc, s > 0 ? 1u : 0u);
        }
        tc::mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::tc_fence_after();
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
#pragma unroll
        for (int i = 0; i < 16; ++i) D[row * N + c0 + i] = __float_as_int(v[i]);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(tmem);
}

}  // namespace

int tc_selftest_i8(const int8_t* dA, const int8_t* dB, int K, int N, int a_mn, int ms, int ks, int lbo, int sbo,
                   int* dD, cudaStream_t st) {
    const size_t smem = 2 * size_t(K / 32) * 4096;
    cudaFuncSetAttribute(tc_selftest_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    tc_selftest_i8_kernel<<<1, 128, smem, st>>>(dA, dB, K, N, a_mn, ms, ks, lbo, sbo, dD);
    return int(cudaGetLastError());
}

int tc_selftest(const float* dA, const float* dB, int K, int split, float* dD, cudaStream_t st) {
    const size_t smem = 6 * size_t(K / 16) * tc::kSliceBytes;
    cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    tc_selftest_kernel<<<1, 128, smem, st>>>(dA, dB, K, split, dD);
    return int(cudaGetLastError());
}

}  // namespace erxk
