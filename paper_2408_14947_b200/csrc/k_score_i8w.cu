// k_score_i8w.cu — the exact-integer tensor-core score for WIDE lines
// (127 < D <= 512), the companion of k_stats_i8t.cu, and the conversion of
// the factor's fp32 W = L^{-1} blocks into its int8 operand.
//
// delta_p = ||m_p||, m_p = W (z_p - mu_{t-1})  (forward_substitute
// as a whitening multiply, linalg.hpp:21).  As in k_score_i8.cu the statistics
// kernel leaves v = x - c quantised per dim (vq = rint(v s_j)) as int8 digit
// planes, so  m_i = (sum_j vq_pj Wq_ij) / r_i - (W (mu - c))_i  with
// W'_ij = W_ij / s_j quantised per row (r_i = R / max_j |W'_ij|).  At D > 128 the
// product is tiled: output rows in 128-row tiles nt (one TMEM block of four s32
// class accumulators, 4 x 128 columns), input dims in 128-dim tiles kt <= nt (W
// is lower triangular): per 128-pixel tile and row tile, sum over kt of
// 4 K-steps x 8 digit-pair MMAs (M = 128 pixels, MN-major A = the v planes of
// (pixel tile, kt); N = rows of nt, K-major B = the W planes of (nt, kt)); the
// epilogue turns the row tile's accumulators into m_i and adds m_i^2 to the
// pixel's running delta^2.
//
//   wplanes_w_kernel   fp32 W blocks (k_factor.cu: write_wblocks, any factor kernel)
//                      -> [line][pair (nt, kt)][3 digit planes][128 rows x 128 K] int8
//                         + 256 / r_i and (W (mu - c))_i per row
//   score_i8w_kernel   persistent CTA per SM over (line, pixel tile) items: warps 0-15
//                      epilogue, warp 16 producer (bulk copies of A / B tile pairs into a
//                      2-deep ring), warp 17 MMA issuer; hand-offs through mbarriers.
#include "erx_common.cuh"
#include "i8_common.cuh"

namespace erxk {
namespace {

constexpr int kT = 128;                             // pixels per tile / dims per tile / rows per tile
constexpr uint32_t kPl = 16384;                     // one 128 x 128 int8 digit plane
constexpr uint32_t kPair = 3 * kPl;                 // three planes
constexpr int kThreads = 512;                       // epilogue threads
constexpr int kEW = kThreads / 32;
constexpr int kStages = 2;

__host__ __device__ inline int n_tiles(int D) { return (D + kT - 1) / kT; }
__host__ __device__ inline size_t wplw_bytes(int D) {
    const int nt = n_tiles(D);
    return size_t(nt) * (nt + 1) / 2 * kPair + 2 * size_t(nt) * kT * 4;
}

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(m)) : "memory");
}

// ---------------------------------------------------------------------------
// W planes: one CTA per (line, 128-row tile), a thread per output row.  The row tile's W blocks are
// staged 128 x 128 at a time (one dim tile kt) into a dense shared-memory tile with coalesced 16-byte
// loads of the packed column-major 8x8 blocks: pass A over every kt gives each row's scale r_i and
// (W dc)_i, pass B stages the tiles again and writes the int8 digit planes.
// ---------------------------------------------------------------------------
constexpr int kWLd = kT + 1;  // staged tile row stride (floats): row-wise reads by 32 rows hit 32 banks

__global__ void __launch_bounds__(kT) wplanes_w_kernel(Geometry g, const float* __restrict__ whiten,
                                                       const double* __restrict__ stats,
                                                       const double* __restrict__ prior,
                                                       const float* __restrict__ vmax,
                                                       unsigned char* __restrict__ wpl) {
    extern __shared__ __align__(16) unsigned char smem[];
    float* Wt = reinterpret_cast<float*>(smem);  // [128][kWLd] W[ti rows][kt cols], zero past the diagonal / D
    __shared__ float isc[kT];
    __shared__ double dcs[kT];
    const int D = g.D, nt = n_tiles(D), Dt = nt * kT;
    const int line = blockIdx.x / nt, ti = blockIdx.x - line * nt, tid = threadIdx.x;
    const int nblk = g.nb * (g.nb + 1) / 2;
    const float* W = whiten + size_t(line) * nblk * 64;
    const int i = ti * kT + tid;  // this thread's row
    auto stage = [&](int kt) {   // W[ti tile][kt tile] -> Wt (+ the kt tile's column scales)
        __syncthreads();
        // 16 x 16 blocks of 64 floats; block (bi, bj) valid when J <= I and the block exists (I < nb)
        // batches of kLB loads per thread in flight before any is scattered (the kernel waits on L2: ncu
        // 49 % long-scoreboard at one load per iteration); blocks that do not exist read block 0 and are
        // zeroed by the (gi, gj) test
        constexpr int kLB = 8;
        for (int q0 = tid; q0 < 16 * 16 * 16; q0 += kLB * kT) {
            float4 v[kLB];
#pragma unroll
            for (int b = 0; b < kLB; ++b) {
                const int q = q0 + b * kT;
                const int blk = q >> 4, part = q & 15;  // 16 float4 per block
                const int I = ti * 16 + (blk >> 4), J = kt * 16 + (blk & 15);
                const bool ok = J <= I && I < g.nb;
                v[b] = __ldg(reinterpret_cast<const float4*>(W + size_t(ok ? tri(I, J) : 0) * 64) + part);
                if (!ok) v[b] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int b = 0; b < kLB; ++b) {
                const int q = q0 + b * kT;
                const int blk = q >> 4, part = q & 15;
                const int bi = blk >> 4, bj = blk & 15;
                // element e = c * 8 + r (column-major inside the block); part covers e = 4 part .. 4 part + 3
                const float vv[4] = {v[b].x, v[b].y, v[b].z, v[b].w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = 4 * part + u, c = e >> 3, r = e & 7;
                    const int row = bi * 8 + r, col = bj * 8 + c;
                    const int gi = ti * kT + row, gj = kt * kT + col;
                    Wt[row * kWLd + col] = (gi < D && gj <= gi) ? vv[u] : 0.f;
                }
            }
        }
        for (int d = tid; d < kT; d += kT) {
            const int gd = kt * kT + d;
            float v = 0.f;
            double dc = 0.0;
            if (gd < D) {
                const float sc = i8::v_scale(vmax[size_t(line) * D + gd]);
                v = sc > 0.f ? 1.f / sc : 0.f;
                dc = prior[size_t(line) * g.SE + gd] - stats[size_t(line) * (g.SE + D) + gd];
            }
            isc[d] = v;
            dcs[d] = dc;
        }
        __syncthreads();
    };
    // ---- pass A: the row's scale and offset over every dim tile
    float mx = 0.f;
    double cr[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kt = 0; kt <= ti; ++kt) {
        stage(kt);
        const float* wr = Wt + tid * kWLd;
#pragma unroll 4
        for (int c = 0; c < kT; ++c) {
            const float wv = wr[c];
            mx = fmaxf(mx, fabsf(wv * isc[c]));
            cr[c & 3] += double(wv) * dcs[c];
        }
    }
    const float r = (mx > 0.f && mx <= 3.402823466e38f) ? i8::kR / mx : 0.f;
    unsigned char* out = wpl + size_t(line) * wplw_bytes(D);
    float* invr = reinterpret_cast<float*>(out + size_t(nt) * (nt + 1) / 2 * kPair);
    float* wdc = invr + Dt;
    invr[i] = r > 0.f ? 256.f / r : 0.f;
    wdc[i] = float((cr[0] + cr[1]) + (cr[2] + cr[3]));
    // ---- pass B: the digit planes, one dim tile at a time
    for (int kt = 0; kt <= ti; ++kt) {
        if (kt < ti || ti > 0) stage(kt);  // (the last staged tile is still there when ti == 0)
        unsigned char* blk = out + size_t(ti * (ti + 1) / 2 + kt) * kPair;
        const float* wr = Wt + tid * kWLd;
        for (int run = 0; run < kT / 16; ++run) {
            uint32_t wd[3][4];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                uint32_t u[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = run * 16 + q4 * 4 + e;
                    u[e] = i8::quant_u(wr[c] * isc[c], r);
                }
                i8::pack_digits(u, wd[0][q4], wd[1][q4], wd[2][q4]);
            }
            const uint32_t off = tc::kmajor_off_s8(tid, run * 16);
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
                *reinterpret_cast<uint4*>(blk + pl * kPl + off) = make_uint4(wd[pl][0], wd[pl][1], wd[pl][2], wd[pl][3]);
        }
    }
}

// ---------------------------------------------------------------------------
// the score
// ---------------------------------------------------------------------------
struct ScoreI8WArgs {
    Geometry g;
    int n_lines;
    int ntile;     // dim / row tiles
    int nptile;    // pixel tiles per line
    const unsigned char* vplanes;   // [line][pixel tile][dim tile][3][16 KB]  (k_stats_i8t)
    const unsigned char* wplanes;   // [line][wplw_bytes]                     (wplanes_w_kernel)
    float* raw;
};

__global__ void __launch_bounds__(kThreads + 64, 1) score_i8w_kernel(ScoreI8WArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], accfull, accempty;
    __shared__ float red_s[3][128];
    __shared__ float aux_s[2 * 512];  // the item's line: 256 / r_i, then (W (mu - c))_i

    const Geometry& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int P = g.P, D = g.D, NT = a.ntile;
    const int n_items = a.n_lines * a.nptile;
    const int my_items = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const size_t wpl_line = wplw_bytes(D);
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
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

    if (warp == kEW) {
        // ---------------- producer: per item, per row tile nt, per dim tile kt <= nt: A (v) + B (W) planes
        if (lane == 0) {
            int j = 0;
            for (int k = 0; k < my_items; ++k) {
                const int it = blockIdx.x + k * gridDim.x;
                const int line = it / a.nptile, t = it - line * a.nptile;
                for (int nt = 0; nt < NT; ++nt)
                    for (int kt = 0; kt <= nt; ++kt, ++j) {
                        const int st = j % kStages;
                        if (j >= kStages) tc::mbar_wait(&empty[st], uint32_t(j / kStages - 1) & 1u);
                        tc::mbar_expect_tx(&full[st], 2 * kPair);
                        unsigned char* dst = smem + size_t(st) * 2 * kPair;
                        const unsigned char* va = a.vplanes + ((size_t(line) * a.nptile + t) * NT + kt) * kPair;
                        const unsigned char* wb = a.wplanes + size_t(line) * wpl_line +
                                                  size_t(nt * (nt + 1) / 2 + kt) * kPair;
                        tc::bulk_g2s(dst, va, kPair, &full[st]);
                        tc::bulk_g2s(dst + kPair, wb, kPair, &full[st]);
                    }
            }
        }
        return;
    }
    if (warp == kEW + 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const int pr[8][3] = {{0, 1, 0}, {1, 0, 0}, {0, 2, 1}, {1, 1, 1}, {2, 0, 1}, {1, 2, 2}, {2, 1, 2}, {2, 2, 3}};
            int j = 0, acc_i = 0;
            for (int k = 0; k < my_items; ++k) {
                for (int nt = 0; nt < NT; ++nt, ++acc_i) {
                    const int N = (min(kT, D - nt * kT) + 15) / 16 * 16;  // rows of this tile
                    if (acc_i >= 1) tc::mbar_wait(&accempty, uint32_t(acc_i - 1) & 1u);
                    for (int kt = 0; kt <= nt; ++kt, ++j) {
                        const int st = j % kStages;
                        tc::mbar_wait(&full[st], uint32_t(j / kStages) & 1u);
                        tc::tc_fence_after();
                        const uint32_t vbase = tc::smem_u32(smem + size_t(st) * 2 * kPair);
                        const uint32_t wbase = vbase + kPair;
                        const bool diag = kt == nt;
#pragma unroll
                        for (int s = 0; s < 4; ++s) {
                            // diagonal block: K-step s (dims 32s..) only reaches rows >= 32s of the tile
                            const int c0 = diag ? 32 * s : 0;
                            const int ns = N - c0;
                            if (ns <= 0) break;
                            const uint32_t idesc = tc::idesc_s8_s32(128, ns, /*a_mn=*/true, /*b_mn=*/false);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const uint64_t ad = tc::smem_desc_ls(vbase + pr[q][0] * kPl + s * tc::kSliceBytes,
                                                                     i8::kVLbo, i8::kVSbo);
                                const uint64_t bd = tc::smem_desc(wbase + pr[q][1] * kPl + s * tc::kSliceBytes +
                                                                  uint32_t(c0 / 8) * 256u);
                                const bool first = kt == 0 && s == 0 && (q == 0 || q == 2 || q == 5 || q == 7);
                                tc::mma_s8(tmem + uint32_t(pr[q][2]) * 128u + uint32_t(c0), ad, bd, idesc,
                                           first ? 0u : 1u);
                            }
                        }
                        tc::mma_commit(&empty[st]);
                    }
                    tc::mma_commit(&accfull);
                }
            }
        }
        return;
    }

    // ---------------- epilogue warps 0-15: thread = (pixel row of the tile, column quarter)
    const int row = (warp & 3) * 32 + lane;
    const uint32_t taddr = tmem + (uint32_t((warp & 3) * 32) << 16);
    const int colq = warp >> 2;
    int acc_i = 0;
    for (int k = 0; k < my_items; ++k) {
        const int it = blockIdx.x + k * gridDim.x;
        const int line = it / a.nptile, t = it - line * a.nptile;
        {  // the line's row factors / offsets into shared memory (read 16 per accumulator group below)
            const float* src = reinterpret_cast<const float*>(a.wplanes + size_t(line) * wpl_line +
                                                              size_t(NT) * (NT + 1) / 2 * kPair);
            for (int q = tid; q < 2 * NT * kT; q += kThreads) aux_s[q] = __ldg(src + q);
            bar_compute();
        }
        const float* invr = aux_s;
        const float* wdc = aux_s + NT * kT;
        float d2 = 0.f;
        for (int nt = 0; nt < NT; ++nt, ++acc_i) {
            const int N = (min(kT, D - nt * kT) + 15) / 16 * 16;
            const int ngrp = N / 16;
            const int g0 = colq * ngrp / 4, g1 = (colq + 1) * ngrp / 4;
            tc::mbar_wait(&accfull, uint32_t(acc_i) & 1u);
            tc::tc_fence_after();
            for (int gi = g0; gi < g1; ++gi) {
                uint32_t v[4][16];
                tc::tmem_ld16x4(taddr + uint32_t(gi * 16), 128u, v);
#pragma unroll
                for (int ii = 0; ii < 16; ++ii) {
                    const int i = nt * kT + gi * 16 + ii;
                    float m = fmaf(float(int(v[3][ii])), 256.f, float(int(v[2][ii])));
                    m = fmaf(m, 256.f, float(int(v[1][ii])));
                    m = fmaf(m, 256.f, float(int(v[0][ii])));
                    m = fmaf(m, invr[i], -wdc[i]);
                    d2 = fmaf(m, m, d2);
                }
            }
            tc::tc_fence_before();
            bar_compute();  // every quarter has read the accumulators
            if (tid == 0) mbar_arrive(&accempty);
        }
        if (colq) red_s[colq - 1][row] = d2;
        bar_compute();
        const int p = t * kT + row;
        if (!colq && p < P) a.raw[size_t(line) * P + p] = sqrtf(d2 + red_s[0][row] + red_s[1][row] + red_s[2][row]);
        bar_compute();  // red_s is rewritten by the next item
    }
    tc::tc_fence_before();
    bar_compute();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

}  // namespace

size_t wplanes_w_bytes_per_line(const Geometry& g) { return wplw_bytes(g.D); }
size_t vplanes_w_bytes_per_line(const Geometry& g) {
    return size_t((g.P + kT - 1) / kT) * n_tiles(g.D) * kPair;
}
bool score_i8w_eligible(const Geometry& g) { return !g.srp && g.D > 127 && g.D <= 512 && (g.B % 4) == 0; }

void launch_wplanes_w(const Geometry& g, const float* whiten, const double* stats, const double* prior,
                      const float* vmax, int n_lines_total, unsigned char* wpl, cudaStream_t st) {
    const size_t sm = size_t(kT) * kWLd * 4;
    ensure_smem(wplanes_w_kernel, sm);
    wplanes_w_kernel<<<n_lines_total * n_tiles(g.D), kT, sm, st>>>(g, whiten, stats, prior, vmax, wpl);
}

void launch_score_i8w(const Geometry& g, const unsigned char* vplanes, const unsigned char* wplanes, int n_lines_total,
                      float* raw, cudaStream_t st) {
    const size_t smem = size_t(kStages) * 2 * kPair + 1024;
    ensure_smem(score_i8w_kernel, smem);
    ScoreI8WArgs a{g, n_lines_total, n_tiles(g.D), (g.P + kT - 1) / kT, vplanes, wplanes, raw};
    const int items = n_lines_total * a.nptile;
    const int grid = items < sm_count() ? items : sm_count();
    score_i8w_kernel<<<grid, kThreads + 64, smem, st>>>(a);
}

}  // namespace erxk
