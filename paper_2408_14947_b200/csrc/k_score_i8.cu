// k_score_i8.cu — per-pixel Mahalanobis distance (SPEC.md:305,
// forward_substitute as a whitening multiply, linalg.hpp:21) on the
// 5th-generation tensor cores with EXACT integer accumulation (kind::i8),
// the companion of k_stats_i8.cu.
//
// For one line, delta_p = ||m_p||, m_p = W (z_p - mu_{t-1}), W = L^{-1}.  The
// stats kernel has already quantised the centred line v = x - c per dim
// (vq = rint(v s), s_j = R / max_p |v_j|) into three int8 digit planes laid
// out as this kernel's MN-major A operand (i8_common.cuh: vplane_off), and
// the factor kernel writes W'_ij = W_ij / s_j per-row quantised (r_i) as the
// K-major B operand plus (W (mu - c))_i (k_factor.cu: write_wplanes).  So
//   m_i = (sum_j vq_pj Wq_ij) / r_i - (W (mu - c))_i
// and this kernel does no quantisation at all: per 128-pixel tile it streams
// 48 KB of digit planes, issues 4 K-steps x 8 digit pairs of M=128,
// N=roundup16(D), K=32 MMAs (classes i + j >= 1, four exact s32 TMEM
// accumulators; class 0 is 2^-30 relative and dropped) and reduces the
// accumulators to delta.  Emulated raw-score error vs fp64 on configs[3]:
// max 3.3e-6 / median 4.4e-7 (tools/emulate_i8.py, "score from stats' v planes").
//
// Warp roles (persistent CTA per SM, whole lines): warps 0-15 epilogue
// (TMEM -> m_i -> delta), warp 16 producer (bulk copies: per line the W block
// into a double buffer, per tile the v planes into a 2-deep ring), warp 17
// MMA issuer.  All hand-offs are mbarriers.
#include "erx_common.cuh"
#include "i8_common.cuh"

namespace erxk {
namespace {

constexpr int kTile = 128;                          // pixels per tile (MMA M)
constexpr int kKSteps = 4;                          // K = 128 dims
constexpr int kThreads = 512;                       // epilogue threads (16 warps)
constexpr int kEW = kThreads / 32;
constexpr int kStages = 3;                          // v-plane tile ring
constexpr uint32_t kVSlack = 2048;                  // the K-step-3 reads of the last plane run past its used head

// Shared-memory images, compacted from the global layouts (i8_common.cuh):
//  * v tile: the three planes' used heads vb = vplane_used_bytes(D) back to back (the MMA of K-step 3
//    reads dims >= the used head from the next plane's bytes, against W's zero columns);
//  * W planes: K-step s only reaches output rows >= 32 s (W lower triangular) and < N, so slice s keeps
//    rows [32 s, N): (N - 32 s) x 32 B, whole 8-row core-matrix groups.
struct SmemPlan {
    uint32_t vb;       // bytes per v plane head
    uint32_t wpb;      // bytes per compact W plane
    uint32_t so[4];    // compact offset of W slice s (rows from 32 s)
    uint32_t sl[4];    // its bytes (0: the slice reaches no row)
};
__host__ __device__ inline SmemPlan smem_plan(int D) {
    SmemPlan sp{};
    const int N = (D + 15) / 16 * 16;
    sp.vb = i8::vplane_used_bytes(D);
    uint32_t off = 0;
    for (int s = 0; s < 4; ++s) {
        const int rows = N - 32 * s;
        sp.so[s] = off;
        sp.sl[s] = rows > 0 ? uint32_t(rows) * 32u : 0u;
        off += sp.sl[s];
    }
    sp.wpb = off;
    return sp;
}
__host__ __device__ inline size_t score_i8_smem_bytes(int D) {
    const SmemPlan sp = smem_plan(D);
    return 2 * 3 * size_t(sp.wpb) + kStages * 3 * size_t(sp.vb) + kVSlack;
}
static_assert(i8::kVPlane == kKSteps * tc::kSliceBytes, "v plane layout");

struct ScoreI8Args {
    Geometry g;
    int n_lines;
    const unsigned char* vplanes;   // [line][tile][i8::kTileBytes]  (k_stats_i8)
    const unsigned char* wplanes;   // [line][i8::kWBytes]           (k_factor write_wplanes)
    float* raw;
    int N;                          // MMA N = roundup16(D)
};

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(m)) : "memory");
}

__global__ void __launch_bounds__(kThreads + 64, 1) score_i8_kernel(ScoreI8Args a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t wfull[2], wempty[2], tfull[kStages], tempty[kStages], accfull[2], accempty[2];
    __shared__ __align__(16) float aux_s[2][2 * 128];  // per line parity: 256 / r_i, then (W (mu - c))_i
    __shared__ float red_s[2][3][128];

    const Geometry& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int P = g.P;
    const SmemPlan sp = smem_plan(g.D);
    unsigned char* wops = smem;                            // [2][3][wpb] compact W' digit planes
    unsigned char* vops = smem + 2 * 3 * sp.wpb;           // [kStages][3][vb] v digit plane heads
    const int ntile = (P + kTile - 1) / kTile;
    const int my_lines = blockIdx.x < a.n_lines ? (a.n_lines - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&wfull[b], 1);
            tc::mbar_init(&wempty[b], 1);
        }
        for (int b = 0; b < kStages; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 1);
        }
        for (int h = 0; h < 2; ++h) {
            tc::mbar_init(&accfull[h], 1);
            tc::mbar_init(&accempty[h], kEW);  // one arrival per epilogue warp
        }
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(&tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == kEW) {
        // ---------------- producer: W block of line k (double-buffered), then its tiles
        if (lane == 0) {
            int j = 0;
            for (int k = 0; k < my_lines; ++k) {
                const int line = blockIdx.x + k * gridDim.x;
                const int wb = k & 1;
                if (k >= 2) tc::mbar_wait(&wempty[wb], uint32_t((k - 2) >> 1) & 1u);  // MMAs of line k-2 done
                const unsigned char* wsrc = a.wplanes + size_t(line) * i8::kWBytes;
                tc::mbar_expect_tx(&wfull[wb], 3 * sp.wpb + i8::kWAux);
                for (int pl = 0; pl < 3; ++pl)
                    for (int s = 0; s < kKSteps; ++s)
                        if (sp.sl[s])
                            tc::bulk_g2s(wops + (wb * 3 + pl) * sp.wpb + sp.so[s],
                                         wsrc + pl * i8::kWPlane + s * tc::kSliceBytes + uint32_t(32 * s) * 32u,
                                         sp.sl[s], &wfull[wb]);
                tc::bulk_g2s(aux_s[wb], wsrc + 3 * i8::kWPlane, i8::kWAux, &wfull[wb]);
                for (int t = 0; t < ntile; ++t, ++j) {
                    const int st = j % kStages;
                    if (j >= kStages) tc::mbar_wait(&tempty[st], uint32_t((j / kStages) - 1) & 1u);
                    // only the planes' used head (dims 0 .. D); the MMA reads the stale tail against W's
                    // zero columns
                    const uint32_t vb = i8::vplane_used_bytes(a.g.D);
                    tc::mbar_expect_tx(&tfull[st], 3 * vb);
                    const unsigned char* src = a.vplanes + (size_t(line) * ntile + t) * i8::kTileBytes;
                    for (int pl = 0; pl < 3; ++pl)
                        tc::bulk_g2s(vops + (st * 3 + pl) * vb, src + pl * i8::kVPlane, vb,
                                     &tfull[st]);
                }
            }
        }
        return;
    }
    if (warp == kEW + 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            // (v digit, W digit, class - 1), v digit + W digit >= 1
            const int pr[8][3] = {{0, 1, 0}, {1, 0, 0}, {0, 2, 1}, {1, 1, 1}, {2, 0, 1}, {1, 2, 2}, {2, 1, 2}, {2, 2, 3}};
            // W is lower triangular: K-step s (input dims 32s .. 32s + 31) only reaches output rows
            // >= 32s, so it runs at N_s = a.N - 32s into accumulator columns 32s.. with the B operand
            // from W row 32s (4s core-matrix groups of 256 B on): 256 instead of 448 MMA columns at
            // D = 108
            uint32_t idesc_s[kKSteps];
#pragma unroll
            for (int s = 0; s < kKSteps; ++s) {
                const int ns = a.N - 32 * s;
                idesc_s[s] = tc::idesc_s8_s32(128, ns > 0 ? ns : 16, /*a_mn=*/true, /*b_mn=*/false);
            }
            int j = 0;
            for (int k = 0; k < my_lines; ++k) {
                const int wb = k & 1;
                tc::mbar_wait(&wfull[wb], uint32_t(k >> 1) & 1u);
                const uint32_t wbase = tc::smem_u32(wops + wb * 3 * sp.wpb);
                for (int t = 0; t < ntile; ++t, ++j) {
                    const int st = j % kStages;
                    tc::mbar_wait(&tfull[st], uint32_t(j / kStages) & 1u);
                    const uint32_t vbase = tc::smem_u32(vops + st * 3 * sp.vb);
                    // classes 1-2 (pairs 0-4, TMEM columns 0-255) then classes 3-4 (pairs 5-7, columns
                    // 256-511), each half with its own full / empty barriers: the epilogue reads one half
                    // while the tensor core fills the other
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (j >= 1) tc::mbar_wait(&accempty[h], uint32_t(j - 1) & 1u);
                        tc::tc_fence_after();
#pragma unroll
                        for (int s = 0; s < kKSteps; ++s) {
                            if (a.N - 32 * s <= 0) break;  // no output row reaches these dims
#pragma unroll
                            for (int q = h ? 5 : 0; q < (h ? 8 : 5); ++q) {
                                const uint64_t ad = tc::smem_desc_ls(vbase + pr[q][0] * sp.vb + s * tc::kSliceBytes,
                                                                     i8::kVLbo, i8::kVSbo);
                                const uint64_t bd = tc::smem_desc(wbase + pr[q][1] * sp.wpb + sp.so[s]);
                                const bool first = s == 0 && (q == 0 || q == 2 || q == 5 || q == 7);
                                tc::mma_s8(tmem + uint32_t(pr[q][2]) * 128u + uint32_t(32 * s), ad, bd, idesc_s[s],
                                           first ? 0u : 1u);
                            }
                        }
                        if (h) tc::mma_commit(&tempty[st]);
                        tc::mma_commit(&accfull[h]);
                    }
                }
                tc::mma_commit(&wempty[wb]);
            }
        }
        return;
    }

    // ---------------- epilogue warps 0-15: thread = (pixel row of the tile, column quarter)
    const int row = (warp & 3) * 32 + lane;
    const uint32_t taddr = tmem + (uint32_t((warp & 3) * 32) << 16);
    const int colq = warp >> 2;
    const int ngrp = a.N / 16;
    const int g0 = colq * ngrp / 4, g1 = (colq + 1) * ngrp / 4;
    int j = 0;
    for (int k = 0; k < my_lines; ++k) {
        const int line = blockIdx.x + k * gridDim.x;
        const int wb = k & 1;
        tc::mbar_wait(&wfull[wb], uint32_t(k >> 1) & 1u);  // the line's row factors / offsets
        const float* invr = aux_s[wb];
        const float* wdc = aux_s[wb] + 128;
        for (int t = 0; t < ntile; ++t, ++j) {
            // half 0: classes 1-2 -> lo = a1 + 2^8 a2 (exact int32), released before half 1 is waited for
            int lo[2][16];
            tc::mbar_wait(&accfull[0], uint32_t(j) & 1u);
            tc::tc_fence_after();
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (g0 + u < g1) {
                    uint32_t v[2][16];
                    tc::tmem_ld16x2(taddr + uint32_t((g0 + u) * 16), 128u, v);
#pragma unroll
                    for (int ii = 0; ii < 16; ++ii) lo[u][ii] = int(v[0][ii]) + int(v[1][ii]) * 256;
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[0]);
            // half 1: classes 3-4 -> hi = a3 + 2^8 a4; m_int = lo + 2^16 hi (every class sum is below 2^22
            // for D <= 127, so both halves are exact in int32); invr = 256 / r_i (0 for padding rows)
            tc::mbar_wait(&accfull[1], uint32_t(j) & 1u);
            tc::tc_fence_after();
            // column pairs (i, i + 1) as paired FMAs (fma.rn.f32x2); invr / wdc pairs are one 8-byte load each
            float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (g0 + u < g1) {
                    uint32_t v[2][16];
                    tc::tmem_ld16x2(taddr + 256u + uint32_t((g0 + u) * 16), 128u, v);
                    if (u == 1 || g0 + 1 >= g1) {  // the last load of this warp: release the half
                        tc::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&accempty[1]);
                    }
#pragma unroll
                    for (int ii = 0; ii < 16; ii += 2) {
                        const int i = (g0 + u) * 16 + ii;
                        const float2 hi = make_float2(float(int(v[0][ii]) + int(v[1][ii]) * 256),
                                                      float(int(v[0][ii + 1]) + int(v[1][ii + 1]) * 256));
                        const float2 lo2 = make_float2(float(lo[u][ii]), float(lo[u][ii + 1]));
                        const float2 r2 = *reinterpret_cast<const float2*>(invr + i);
                        const float2 w2 = *reinterpret_cast<const float2*>(wdc + i);
                        float2 m = __ffma2_rn(hi, make_float2(65536.f, 65536.f), lo2);
                        m = __ffma2_rn(m, r2, make_float2(-w2.x, -w2.y));
                        acc2 = __ffma2_rn(m, m, acc2);
                    }
                }
            }
            const float acc = acc2.x + acc2.y;
            if (g0 >= g1) {  // no columns for this warp
                __syncwarp();
                if (lane == 0) mbar_arrive(&accempty[1]);
            }
            if (colq) red_s[j & 1][colq - 1][row] = acc;
            bar_compute();
            const int p = t * kTile + row;
            if (!colq && p < P)
                a.raw[size_t(line) * P + p] = sqrtf(acc + red_s[j & 1][0][row] + red_s[j & 1][1][row] + red_s[j & 1][2][row]);
        }
    }
    tc::tc_fence_before();
    bar_compute();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

}  // namespace

size_t wplanes_bytes_per_line() { return i8::kWBytes; }
size_t vplanes_bytes_per_line(const Geometry& g) { return size_t((g.P + kTile - 1) / kTile) * i8::kTileBytes; }

bool score_i8_eligible(const Geometry& g) { return !g.srp && g.D > 16 && g.D <= 127 && (g.B % 4) == 0; }

void launch_score_i8(const Geometry& g, const unsigned char* vplanes, const unsigned char* wplanes, int n_lines_total,
                     float* raw, cudaStream_t st) {
    const size_t smem = score_i8_smem_bytes(g.D);
    const int sms = sm_count();
    ensure_smem(score_i8_kernel, smem);
    ScoreI8Args a{g, n_lines_total, vplanes, wplanes, raw, (g.D + 15) / 16 * 16};
    const int grid = n_lines_total < sms ? n_lines_total : sms;
    score_i8_kernel<<<grid, kThreads + 64, smem, st>>>(a);
}

}  // namespace erxk
