// k_stats_tc.cu — line_stats (erx.hpp:38-40) on the 5th-generation tensor
// cores: the rank-P update S = sum_p v_p v_p^T of one line is one
// 128 x 128 x P tcgen05 GEMM (A = B = V^T, K = pixels), fp32 accumulators in
// TMEM.  Used for the full-covariance path with 32 < D <= 128.
//
// Precision: v (fp32, centred on the line's first-32-pixel mean) is split
// into three bf16 planes, v = h + m + l to ~2^-24, and six products
// (hh, hm, mh, hl, lh, mm) accumulate into the same TMEM accumulator, which
// reproduces fp32-product accuracy (emulated median 2.5e-7 vs
// 1.9e-6 for 3xTF32).  Two accumulators each take half the pixels and are
// summed in fp64 at the end (a 2-level accumulation like the FFMA kernel).
//
// Pipeline per 32-pixel chunk (double-buffered): cp.async raw fp32 rows ->
// all 4 warps centre + split + write the K-major operand planes -> one
// thread issues 2 K-slices x 6 MMAs and commits to the chunk buffer's
// mbarrier, which gates the buffer's reuse two chunks later.
//
// Output slot per line: [c (D) | s = sum(v) (D) | S packed lower], fp64 —
// the same contract as k_stats.cu, finished by the scan kernel.
#include "erx_common.cuh"
#include "tc_common.cuh"

namespace erxk {
namespace {

constexpr int kChunk = 32;                                   // pixels per chunk (2 K-slices)
constexpr uint32_t kPlaneBytes = (kChunk / 16) * tc::kSliceBytes;  // 8 KB per bf16 plane
constexpr uint32_t kOpBytes = 3 * kPlaneBytes;                // hi, mid, lo

struct StatsTcArgs {
    Geometry g;
    const float* x;
    int n;
    int in_stride;
    double* stats;
};

__global__ void __launch_bounds__(128) stats_tc_kernel(StatsTcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t mbar[2];
    const Geometry& g = a.g;
    const int line = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5;
    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);

    unsigned char* ops = smem;                                        // [2][3 planes]
    float* stage = reinterpret_cast<float*>(smem + 2 * kOpBytes);     // [2][kChunk][B]
    double* colsum = reinterpret_cast<double*>(stage + 2 * kChunk * g.B);
    float* cen = reinterpret_cast<float*>(colsum + 128);

    const int nchunks = (g.P + kChunk - 1) / kChunk;
    auto issue_raw = [&](int c) {
        const int c0 = c * kChunk, n = min(kChunk, g.P - c0);
        float* dst = stage + (c & 1) * kChunk * g.B;
        const float* src = xl + size_t(c0) * g.B;
        for (int i = tid; i < n * g.B / 4; i += 128) cp_async16(dst + 4 * i, src + 4 * i);
        cp_async_commit();
    };
    issue_raw(0);
    if (nchunks > 1) issue_raw(1);

    if (warp == 0) tc::tmem_alloc<256>(&tmem_slot);
    if (tid == 0) {
        tc::mbar_init(&mbar[0], 1);
        tc::mbar_init(&mbar[1], 1);
        tc::fence_barrier_init();
    }
    // centre: fp64 mean of the first min(32, P) pixels, rounded to fp32
    {
        const int n0 = min(32, g.P);
        double s = 0.0;
        if (tid < g.D)
            for (int pp = 0; pp < n0; ++pp) s += double(__ldg(xl + size_t(pp) * g.B + tid));
        cen[tid] = (tid < g.D) ? float(s / double(n0)) : 0.f;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t idesc = tc::idesc_bf16_f32(128, 128);
    const float cd = cen[tid];
    const bool live = tid < g.D;
    double cs = 0.0;
    const int half = (nchunks + 1) / 2;

    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        const int n = min(kChunk, g.P - c * kChunk);
        if (c + 1 < nchunks)
            cp_async_wait<1>();
        else
            cp_async_wait<0>();
        __syncthreads();
        if (c >= 2) tc::mbar_wait(&mbar[buf], ((c - 2) >> 1) & 1);  // MMAs of chunk c-2 released the planes
        // thread = dim; 8 pixels per 16-byte K run; padded dims / pixels are zero
        unsigned char* op = ops + buf * kOpBytes;
        const float* st = stage + buf * kChunk * g.B;
        float s = 0.f;
#pragma unroll
        for (int k0 = 0; k0 < kChunk; k0 += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int pp = k0 + j;
                v[j] = (live && pp < n) ? st[pp * g.B + tid] - cd : 0.f;
                s += v[j];
            }
            uint32_t h[4], m[4], l[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) tc::split3_bf16x2(v[2 * j], v[2 * j + 1], h[j], m[j], l[j]);
            const uint32_t off = tc::kmajor_off(tid, k0);
            *reinterpret_cast<uint4*>(op + off) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(op + kPlaneBytes + off) = make_uint4(m[0], m[1], m[2], m[3]);
            *reinterpret_cast<uint4*>(op + 2 * kPlaneBytes + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        cs += double(s);
        tc::fence_proxy_async();
        tc::tc_fence_before();
        __syncthreads();  // planes written; raw stage buffer free
        if (c + 2 < nchunks) issue_raw(c + 2);
        if (tid == 0) {
            tc::tc_fence_after();
            const uint32_t base = tc::smem_u32(op);
            const uint32_t dacc = tmem + (c < half ? 0u : 128u);
            const int pairs[6][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {2, 0}, {1, 1}};
#pragma unroll
            for (int sl = 0; sl < kChunk / 16; ++sl)
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const uint64_t ad = tc::smem_desc(base + pairs[q][0] * kPlaneBytes + sl * tc::kSliceBytes);
                    const uint64_t bd = tc::smem_desc(base + pairs[q][1] * kPlaneBytes + sl * tc::kSliceBytes);
                    const uint32_t accum = (c == 0 || c == half) && sl == 0 && q == 0 ? 0u : 1u;
                    tc::mma_bf16(dacc, ad, bd, idesc, accum);
                }
            tc::mma_commit(&mbar[buf]);
        }
    }
    // the last commit covers every MMA issued before it
    tc::mbar_wait(&mbar[(nchunks - 1) & 1], ((nchunks - 1) >> 1) & 1);
    tc::tc_fence_after();

    double* out = a.stats + size_t(line) * (g.SE + g.D);
    if (live) {
        out[tid] = double(cd);
        out[g.D + tid] = cs;
    }
    // epilogue: row d = tid of both accumulators, summed in fp64, lower triangle
    double* S = out + 2 * g.D;
    const int d = tid;
    const bool two = nchunks > half;  // accumulator 1 holds the second half of the pixels
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    for (int c0 = 0; c0 < 128; c0 += 16) {
        float v0[16], v1[16];
        tc::tmem_ld16(tmem + lane_base + uint32_t(c0), v0);
        tc::tmem_ld16(tmem + lane_base + 128u + uint32_t(c0), v1);
        if (live && c0 <= d) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int e = c0 + i;
                if (e <= d) S[tri(d, e)] = double(v0[i]) + (two ? double(v1[i]) : 0.0);
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(tmem);
}

}  // namespace

bool stats_tc_eligible(const Geometry& g) { return !g.srp && g.D > 32 && g.D <= 128 && (g.B % 4) == 0; }

size_t stats_tc_smem(const Geometry& g) {
    return 2 * size_t(kOpBytes) + 2 * size_t(kChunk) * g.B * 4 + 128 * 8 + 128 * 4;
}

void launch_stats_tc(const Geometry& g, const float* x, int n_per_stream, int in_stride, int n_lines_total,
                     double* stats, cudaStream_t st) {
    const size_t sm = stats_tc_smem(g);
    ensure_smem(stats_tc_kernel, 200 * 1024);
    StatsTcArgs a{g, x, n_per_stream, in_stride, stats};
    stats_tc_kernel<<<n_lines_total, 128, sm, st>>>(a);
}

}  // namespace erxk
