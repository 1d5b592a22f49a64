// k_score_i8.cu — per-pixel Mahalanobis distance (SPEC.md:305,
// forward_substitute as a whitening multiply, linalg.hpp:21) on the
// 5th-generation tensor cores with EXACT integer accumulation (kind::i8),
// the companion of k_stats_i8.cu.
//
// For one line, m = W y_p with W = L^{-1} and y_p = z_p - mu_{t-1};
// delta_p = ||m||.  As one GEMM per 128-pixel tile:
// D[p][i] = sum_j yq[p][j] * Wq[i][j] with
//   y_pd  = fl32(fl32(x_pd - c_d) - fl32(mu_d - c_d))    (c: the stats centre)
//   s_d   = R / bound_d,  bound_d = (max_p |x_pd - c_d| + |mu_d - c_d|)(1 + 2^-20)
//           (max from k_stats_i8, so |y s| <= R without another pass)
//   yq    = rint(y s),                 |yq| <= R = 4194000 < 2^22
//   W'_ij = fl32(W_ij * fl32(1 / s_j)),  r_i = R / max_j |W'_ij|,  Wq_ij = rint(W'_ij r_i)
//   m_i   = (sum_j yq_pj Wq_ij) / r_i
// (i8_common.cuh: y_scale; the factor kernel writes Wq as int8 digit planes,
// k_factor.cu: write_wplanes).  Both operands are three balanced signed int8
// digits; digit-pair products with weight class i + j >= 1 accumulate exactly
// in four s32 TMEM accumulators (class 0 is 2^-30 relative and dropped).
// Emulated raw-score error vs fp64 on configs[3]: max 3.4e-6 / median 4.0e-7
// (tools/emulate_i8.py; classes >= 2 alone would give 2.3e-6 median).
//
// Pipeline: one persistent CTA per SM walks whole lines.  Per line one bulk
// copy brings the line's W planes (48 KB + row factors) into shared memory.
// Warps 0-7 stage x with cp.async one tile ahead (64 dims of one pixel per
// thread, private shared slots), quantise into double-buffered y digit planes
// and run the epilogue (TMEM -> m_i -> delta); warp 8 issues 4 K-steps x 8
// digit pairs of M=128, N=roundup16(D), K=32 MMAs per tile.  The epilogue of
// tile t-1 runs after the quantisation of tile t.
#include "erx_common.cuh"
#include "i8_common.cuh"

namespace erxk {
namespace {

constexpr int kTile = 128;                          // pixels per tile (MMA M)
constexpr int kKSteps = 4;                          // K = 128 dims
constexpr uint32_t kPlane = kKSteps * tc::kSliceBytes;  // 16 KB: 128 rows x 128 int8
constexpr uint32_t kOps = 3 * kPlane;               // three digit planes
constexpr int kThreads = 256;
static_assert(kPlane == i8::kWPlane, "W plane layout");

struct ScoreI8Args {
    Geometry g;
    const float* x;
    int n;
    int in_stride;
    int n_lines;
    const double* stats;            // [c | s | S] per line (c = the centre used by k_stats_i8)
    const float* vmax;              // [line][D] max_p |fl32(x - c)|
    const double* prior;            // [line][SE]: mu_{t-1}, K_{t-1}
    const unsigned char* wplanes;   // [line][i8::kWBytes]
    float* raw;
    int N;                          // MMA N = roundup16(D)
};

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(m)) : "memory");
}

// Epilogue of one tile: wait for its MMAs, m_i = m_int * (256 / r_i) from the four class
// accumulators of this thread's column half, partial ||m||^2 combined across the two halves.
__device__ __noinline__ void score_epilogue(uint32_t taddr, int g0, int g1, int colh, int row, int tid, int tall,
                                            uint64_t* accfull, uint64_t* accempty, const float* invr, float* red,
                                            float* out) {
    tc::mbar_wait(accfull, uint32_t(tall) & 1u);
    tc::tc_fence_after();
    float acc = 0.f;
    for (int gi = g0; gi < g1; ++gi) {
        uint32_t v[4][16];
        tc::tmem_ld16x4(taddr + uint32_t(gi * 16), 128u, v);
#pragma unroll
        for (int ii = 0; ii < 16; ++ii) {
            // m_int = 256 (a1 + 256 (a2 + 256 (a3 + 256 a4))); invr holds 256 / r_i (0 for padding)
            float m = fmaf(float(int(v[3][ii])), 256.f, float(int(v[2][ii])));
            m = fmaf(m, 256.f, float(int(v[1][ii])));
            m = fmaf(m, 256.f, float(int(v[0][ii])));
            m *= invr[gi * 16 + ii];
            acc = fmaf(m, m, acc);
        }
    }
    tc::tc_fence_before();
    if (colh) red[row] = acc;
    bar_compute();
    if (tid == 0) mbar_arrive(accempty);
    if (!colh && out) *out = sqrtf(acc + red[row]);
}

__global__ void __launch_bounds__(kThreads + 32, 1) score_i8_kernel(ScoreI8Args a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t wfull, pfull[2], pempty[2], accfull, accempty;
    __shared__ __align__(16) float cen_s[128], dc_s[128], sc_s[128];
    __shared__ __align__(16) float invr_s[128];
    __shared__ float red_s[2][128];

    const Geometry& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int B = g.B, D = g.D, P = g.P;
    unsigned char* wops = smem;                 // W digit planes [3][128 rows x 128 K]
    unsigned char* yops = smem + kOps;          // y digit planes [2][3][128 x 128]
    const int ntile = (P + kTile - 1) / kTile;
    const int my_lines = blockIdx.x < a.n_lines ? (a.n_lines - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (tid == 0) {
        tc::mbar_init(&wfull, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&pfull[b], 8);
            tc::mbar_init(&pempty[b], 1);
        }
        tc::mbar_init(&accfull, 1);
        tc::mbar_init(&accempty, 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(&tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 8) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_s8_s32(128, a.N);
            // (y digit, W digit, class - 1), y digit + W digit >= 1
            const int pr[8][3] = {{0, 1, 0}, {1, 0, 0}, {0, 2, 1}, {1, 1, 1}, {2, 0, 1}, {1, 2, 2}, {2, 1, 2}, {2, 2, 3}};
            const uint32_t wbase = tc::smem_u32(wops);
            int t_all = 0;
            for (int k = 0; k < my_lines; ++k) {
                tc::mbar_wait(&wfull, uint32_t(k) & 1u);
                for (int t = 0; t < ntile; ++t, ++t_all) {
                    const int buf = t_all & 1;
                    tc::mbar_wait(&pfull[buf], uint32_t(t_all >> 1) & 1u);
                    if (t_all >= 1) tc::mbar_wait(&accempty, uint32_t(t_all - 1) & 1u);
                    tc::tc_fence_after();
                    const uint32_t ybase = tc::smem_u32(yops + buf * kOps);
#pragma unroll
                    for (int s = 0; s < kKSteps; ++s)
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const uint64_t ad = tc::smem_desc(ybase + pr[q][0] * kPlane + s * tc::kSliceBytes);
                            const uint64_t bd = tc::smem_desc(wbase + pr[q][1] * kPlane + s * tc::kSliceBytes);
                            const bool first = s == 0 && (q == 0 || q == 2 || q == 5 || q == 7);
                            tc::mma_s8(tmem + uint32_t(pr[q][2]) * 128u, ad, bd, idesc, first ? 0u : 1u);
                        }
                    tc::mma_commit(&pempty[buf]);
                    tc::mma_commit(&accfull);
                }
            }
        }
        return;
    }

    // ---------------- compute warps 0-7
    const int row = (warp & 3) * 32 + lane;  // TMEM lane = pixel of the tile (epilogue)
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const int colh = warp >> 2;
    const int ngrp = a.N / 16;
    const int g0 = colh ? (ngrp + 1) / 2 : 0, g1 = colh ? ngrp : (ngrp + 1) / 2;
    const int qp = tid & 127, qh = tid >> 7;  // quantisation: pixel, 64-dim half
    int t_all = 0;

    auto epilogue = [&](int kk, int t, int tall) {
        const int line = blockIdx.x + kk * int(gridDim.x);
        if (t == 0) tc::mbar_wait(&wfull, uint32_t(kk) & 1u);  // the line's row factors have landed
        score_epilogue(tmem + lane_base, g0, g1, colh, row, tid, tall, &accfull, &accempty, invr_s, red_s[tall & 1],
                       t * kTile + row < P ? a.raw + size_t(line) * P + t * kTile + row : nullptr);
    };

    // x staging: thread-private 16-byte slots laid out [float4 r4][thread] (conflict-free), filled with
    // cp.async one tile ahead by the thread that later quantises them (no barrier needed)
    float4* stage = reinterpret_cast<float4*>(smem + 3 * size_t(kOps));
    auto issue_x = [&](int ln, int tn) {
        const int pp = tn * kTile + qp;
        if (pp < P) {
            const float* src = line_ptr(a.x, ln, a.n, a.in_stride, g) + size_t(pp) * B + qh * 64;
#pragma unroll
            for (int r4 = 0; r4 < 16; ++r4)
                if (qh * 64 + r4 * 4 < B) cp_async16(stage + r4 * kThreads + tid, src + r4 * 4);
        }
        cp_async_commit();
    };
    if (my_lines > 0) issue_x(blockIdx.x, 0);
    for (int k = 0; k < my_lines; ++k) {
        const int line = blockIdx.x + k * gridDim.x;
        // ---- the previous line's last epilogue drains its MMAs; then the W planes may be replaced
        if (k > 0) epilogue(k - 1, ntile - 1, t_all - 1);
        if (tid == 0) {
            const unsigned char* src = a.wplanes + size_t(line) * i8::kWBytes;
            tc::mbar_expect_tx(&wfull, i8::kWBytes);
            tc::bulk_g2s(wops, src, 3 * i8::kWPlane, &wfull);
            tc::bulk_g2s(invr_s, src + 3 * i8::kWPlane, 128 * 4, &wfull);
        }
        if (tid < 128) {
            const int d = tid;
            i8::YScale ys{0.f, 0.f, 0.f};
            if (d < D)
                ys = i8::y_scale(a.stats + size_t(line) * (g.SE + g.D), a.prior + size_t(line) * g.SE,
                                 a.vmax + size_t(line) * D, d);
            cen_s[d] = ys.c;
            dc_s[d] = ys.dc;
            sc_s[d] = ys.s;
        }
        bar_compute();
        // ---- pixel tiles
        for (int t = 0; t < ntile; ++t, ++t_all) {
            const int buf = t_all & 1;
            const int p = t * kTile + qp;
            const bool pv = p < P;
            cp_async_wait<0>();  // this thread's 64 dims of pixel p (issued one tile ahead)
            if (t_all >= 2) tc::mbar_wait(&pempty[buf], uint32_t((t_all - 2) >> 1) & 1u);
            unsigned char* op = yops + buf * kOps;
#pragma unroll 1
            for (int run = 0; run < 4; ++run) {
                uint32_t w[3][4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const float4 x4 = stage[(run * 4 + q4) * kThreads + tid];
                    const int d0 = qh * 64 + run * 16 + q4 * 4;
                    const float4 c4 = *reinterpret_cast<const float4*>(&cen_s[d0]);
                    const float4 e4 = *reinterpret_cast<const float4*>(&dc_s[d0]);
                    const float4 s4 = *reinterpret_cast<const float4*>(&sc_s[d0]);
                    uint32_t u[4];
                    u[0] = i8::quant_u((x4.x - c4.x) - e4.x, s4.x);
                    u[1] = i8::quant_u((x4.y - c4.y) - e4.y, s4.y);
                    u[2] = i8::quant_u((x4.z - c4.z) - e4.z, s4.z);
                    u[3] = i8::quant_u((x4.w - c4.w) - e4.w, s4.w);
                    if (!pv) u[0] = u[1] = u[2] = u[3] = 0x808080u;
                    i8::pack_digits(u, w[0][q4], w[1][q4], w[2][q4]);
                }
                const uint32_t off = tc::kmajor_off_s8(qp, qh * 64 + run * 16);
#pragma unroll
                for (int pl = 0; pl < 3; ++pl)
                    *reinterpret_cast<uint4*>(op + pl * kPlane + off) = make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]);
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[buf]);
            // prefetch the next tile (of this line or the next one) into the same private slots; issued
            // after the proxy fence, which would otherwise wait for these copies to land
            {
                const int tn = t + 1 < ntile ? t + 1 : 0;
                const int ln = t + 1 < ntile ? line : line + int(gridDim.x);
                if (t + 1 < ntile || k + 1 < my_lines) issue_x(ln, tn);
            }
            if (t > 0) epilogue(k, t - 1, t_all - 1);
        }
    }
    if (my_lines > 0) epilogue(my_lines - 1, ntile - 1, t_all - 1);
    tc::tc_fence_before();
    bar_compute();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

}  // namespace

size_t wplanes_bytes_per_line() { return i8::kWBytes; }

bool score_i8_eligible(const Geometry& g) { return !g.srp && g.D > 16 && g.D <= 127 && (g.B % 4) == 0; }

void launch_score_i8(const Geometry& g, const float* x, int n_per_stream, int in_stride, const double* stats,
                     const float* vmax, const double* prior, const unsigned char* wplanes, int n_lines_total,
                     float* raw, cudaStream_t st) {
    static int sms = 0;
    const size_t smem = 3 * size_t(kOps) + 16 * size_t(kThreads) * 16;  // W + 2 y plane sets + x staging
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(score_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    }
    ScoreI8Args a{g, x, n_per_stream, in_stride, n_lines_total, stats, vmax, prior, wplanes, raw, (g.D + 15) / 16 * 16};
    const int grid = n_lines_total < sms ? n_lines_total : sms;
    score_i8_kernel<<<grid, kThreads + 32, smem, st>>>(a);
}

}  // namespace erxk
