// k_stats_i8.cu — line_stats (erx.hpp:38-40) on the
// 5th-generation tensor cores with EXACT integer accumulation (kind::i8).
//
// The second moment S = sum_p v_p v_p^T of one line is a D x D x P GEMM.
// Tensor-core fp32 accumulation truncates (tools/tc_bias.py), which biases K
// in its small-eigenvalue directions, so this kernel never lets the tensor
// core round: v is turned into integers and the products are summed in s32.
//
//   pass 1  stream the line once: per-dim min / max of x, the centre
//           c = fp32(mean of the first min(32, P) pixels) (k_stats.cu's rule)
//   scale   s_d = R / max_p |fl32(x_pd - c_d)|,  R = 4194000 < 2^22
//   pass 2  stream the line again (L2): q_pd = rint(v_pd * s_d) with
//           v = fl32(x - c), rounded ONCE by fma(v, s, 1.5 * 2^23) (the
//           integer lands in the low mantissa bits), |q| <= 2^22, split
//           into three balanced signed int8 digits
//           q = d0 + 2^8 d1 + 2^16 d2  ((q + 0x808080) ^ 0x808080, bytewise)
//           and accumulate digit-plane products (i, j) with i + j >= 1 in
//           four s32 TMEM accumulators, one per weight class 2^(8(i+j)).
//
// Every s32 sum is exact (|class sum| <= 3 * 2^14 * P < 2^31 for P < 43690);
// the class-0 products d0 d0 are summed exactly on the diagonal by the
// quantiser (int32) and dropped off it; the only approximations are the
// quantisation of v (2^-23 of the per-dim range) and the dropped off-diagonal
// class-0 products (zero-mean, 2^-30 relative): emulated
// max / median raw-score error vs fp64 on configs[3] (tools/emulate_i8.py)
// well inside the fp32 FFMA kernel's 2.5e-6 / 1.2e-7.
// An extra operand row D holds q = 256 (digit d1 = 1) on real pixels, so
// column D of the product is 256 * sum_p q_a: the sums s come out of the same
// exact MMAs.
//
// Output slot per line: [c (D) | s = sum v (D) | S = sum v v^T packed lower],
// fp64 — the k_stats.cu contract, finished by the scan kernel.
//
// Pipeline: a persistent CTA (256 compute threads + a producer warp + an MMA
// warp, 512 TMEM columns) per SM walks its lines.  Step k interleaves, chunk
// by chunk, pass 1 of line k (HBM) with pass 2 of line k-1 (the same chunks
// again, from L2), so the range pass streams under the quantise / MMA work of
// the previous line.  Thread 0 of the producer warp issues 64-pixel
// cp.async.bulk copies into a 5-deep ring (mbarrier tx counts); pass-2 chunks
// are quantised into double-buffered digit planes (K-major, 128 rows x 64 K
// per plane); the MMA warp issues 2 K-steps x 8 MMAs (M = 128 dims,
// N = roundup16(D + 1)) per chunk; the epilogue stages S over the idle plane
// buffers.  With the score kernel in use, pass 2 also writes its digits to
// global memory as that kernel's MN-major A operand (i8_common.cuh).
#include <cstdlib>

#include "erx_common.cuh"
#include "i8_common.cuh"
#include "tc_common.cuh"

namespace erxk {
namespace {

constexpr int kCh = 64;                                   // pixels per chunk (2 K-steps)
constexpr int kMaxStages = 8;                             // bulk-copy ring depth (upper bound)
constexpr uint32_t kPlane = (kCh / 32) * tc::kSliceBytes;  // 8 KB: 128 rows x 64 int8
constexpr uint32_t kOps = 3 * kPlane;                     // d0, d1, d2 planes
constexpr float kMagic = 12582912.f;                      // 1.5 * 2^23
constexpr int kThreads = 256;
// Digit planes of one chunk in shared memory: per 32-pixel K-slice the three planes d0, d1, d2 one after
// the other (128 rows x 32 B each, canonical K-major), so a B descriptor that starts at plane i and runs
// past its 128 rows continues into plane i + 1: one MMA of N = 128 + N' multiplies an A plane with TWO
// B planes and lands in two neighbouring class accumulators (128 TMEM columns apart).
constexpr uint32_t kSliceOps = 3 * tc::kSliceBytes;
__device__ __forceinline__ uint32_t plane_off(int m, int k) {  // int8 element (row m, pixel k) of plane 0
    return uint32_t(k >> 5) * kSliceOps + uint32_t(m >> 3) * 256u + uint32_t((k >> 4) & 1) * 128u +
           uint32_t(m & 7) * 16u + uint32_t(k & 15);
}
// The 8 digit-plane pairs (i, j), i + j >= 1, of one chunk (2 K-slices) as 5 MMAs per slice; class
// i + j - 1 accumulates at TMEM column 128 (i + j - 1).  first: the line's first chunk (accumulators
// are overwritten by the first MMA that reaches them).  Integer sums: any order gives the same bits.
__device__ __forceinline__ void issue_chunk_mmas(uint32_t tmem, uint32_t base, int Nn, bool first) {
    const uint32_t id_cat = tc::idesc_s8_s32(128, 128 + Nn), id_one = tc::idesc_s8_s32(128, Nn);
#pragma unroll
    for (int s = 0; s < kCh / 32; ++s) {
        const uint32_t sb = base + s * kSliceOps;
        const uint64_t d0 = tc::smem_desc(sb), d1 = tc::smem_desc(sb + tc::kSliceBytes),
                       d2 = tc::smem_desc(sb + 2 * tc::kSliceBytes);
        const uint32_t acc = (first && s == 0) ? 0u : 1u;
        tc::mma_s8(tmem, d0, d1, id_cat, acc);         // (0,1) -> class 0, (0,2) -> class 1
        tc::mma_s8(tmem, d1, d0, id_cat, 1u);          // (1,0) -> class 0, (1,1) -> class 1
        tc::mma_s8(tmem + 256u, d1, d2, id_one, acc);  // (1,2) -> class 2
        tc::mma_s8(tmem + 128u, d2, d0, id_cat, 1u);   // (2,0) -> class 1, (2,1) -> class 2
        tc::mma_s8(tmem + 384u, d2, d2, id_one, acc);  // (2,2) -> class 3
    }
}
constexpr size_t kSmemCap = 232448;  // 227 KB per CTA

struct StatsI8Args {
    Geometry g;
    const float* x;
    int n;
    int in_stride;
    int n_lines;
    double* stats;
    float* vmax;  // [line][D] max_p |fl32(x - c)| (the score kernel's y range), may be null
    unsigned char* vplanes;  // [line][tile][3][i8::kTileBytes / 3]: v digit planes for k_score_i8, may be null
    int* c0;     // [line][4][D] class-0 diagonal partials sum_p d0^2 (q units), per pixel group
    int N;       // MMA N = roundup16(D + 1)
    int stages;  // ring depth
    int ring1;   // stats_i8_ws: stages of the pass-1 ring (the rest: pass 2)
    // one-pass statistics (stats_i8_op_kernel): lines whose values leave the predicted range are listed
    // here ([0] count of this launch, [1] running total, [2..] line ids) and redone by stats_i8_kernel,
    // which then walks the list instead of the line range
    int* redo;
    float headroom;  // one-pass: range = headroom x the range of the line's first chunk (a power of two)
};

// line handled at step k of this CTA: the k-th of its share of the range, or of the redo list
__device__ __forceinline__ int line_at(const StatsI8Args& a, bool listed, int k) {
    const int i = blockIdx.x + k * gridDim.x;
    return listed ? a.redo[2 + i] : i;
}

__device__ __forceinline__ void pack_digits(const uint32_t (&u)[4], uint32_t& w0, uint32_t& w1, uint32_t& w2) {
    const uint32_t t01 = __byte_perm(u[0], u[1], 0x5140), t23 = __byte_perm(u[2], u[3], 0x5140);
    w0 = __byte_perm(t01, t23, 0x5410) ^ 0x80808080u;
    w1 = __byte_perm(t01, t23, 0x7632) ^ 0x80808080u;
    const uint32_t r01 = __byte_perm(u[0], u[1], 0x0062), r23 = __byte_perm(u[2], u[3], 0x0062);
    w2 = __byte_perm(r01, r23, 0x5410) ^ 0x80808080u;
}

__device__ __forceinline__ float fmin_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(m)) : "memory");
}

// Warp roles: warps 0-7 compute (range pass, quantisation, epilogue), warp 8
// streams chunks (TMA bulk copies), warp 9 issues the MMAs.  No CTA-wide
// barrier inside the chunk loop: stages and plane buffers hand over through
// mbarriers (full / empty, pfull / pempty), the accumulator through
// accfull / accempty, so copies, quantisation and MMAs of different chunks
// overlap.  The epilogue of line k-1 runs after pass 1 of line k, when the
// MMAs of line k-1 have long finished.
// kBT > 0: the band count as a compile-time constant (the pixel stride of every shared-memory chunk
// access folds into immediate offsets); 0: runtime g.B
template <int kBT, bool kListed = false>
__global__ void __launch_bounds__(kThreads + 64, 1) stats_i8_kernel(StatsI8Args a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
    __shared__ __align__(8) uint64_t pfull[2], pempty[2], accfull, accempty;
    __shared__ __align__(16) float red_mn[8][128];
    __shared__ __align__(16) float red_mx[8][128];

    __shared__ double red_cs[4][128];
    __shared__ float cen_s[128], scale_s[128], add_s[128];
    __shared__ double inv_s[128];
    __shared__ double sum_s[128];
    __shared__ int bad_s[8];

    const Geometry& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int B = kBT > 0 ? kBT : g.B, D = g.D, P = g.P;
    const int NS = a.stages;

    unsigned char* ops = smem;                                   // [2][kOps]
    float* ring = reinterpret_cast<float*>(smem + 2 * kOps);     // [NS][kCh * B]
    // S staging: over the plane buffers when it fits (the epilogue runs while they are idle)
    const size_t tri_bytes = size_t(D) * (D + 1) / 2 * 8;
    double* S = reinterpret_cast<double*>(tri_bytes <= 2 * kOps ? smem : smem + 2 * kOps + size_t(NS) * kCh * B * 4);
    const int nch = (P + kCh - 1) / kCh;
    const int ntile_v = (P + 127) / 128;  // score tiles per line (v planes)
    const bool listed = kListed;  // redo pass of the one-pass statistics: the lines of a.redo
    const int n_lines = listed ? min(a.redo[0], a.n_lines) : a.n_lines;
    const int my_lines = blockIdx.x < n_lines ? (n_lines - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (listed && my_lines == 0) return;  // (the usual case: nothing listed)

    // Ring: chunk loads in one sequence, slot j % NS.  Step k interleaves pass 1 (range) of line k
    // with pass 2 (quantise + MMA) of line k-1, chunk by chunk, so the HBM stream of one line runs
    // under the tensor-core work of the previous one; pass-2 chunks are re-read from L2.
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 8);
        }
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
        // ---------------- producer: the interleaved chunk sequence of the compute warps
        if (lane == 0) {
            int st = 0;
            uint32_t rnd = 0;  // ring slot and round of the next chunk (no integer division per chunk)
            // pass-1 chunks are read again one line later (pass 2): keep them in L2
            const uint64_t keep = tc::policy_evict_last(), drop = tc::policy_evict_first();
            auto load = [&](int k, int c, bool again) {
                if (rnd >= 1) tc::mbar_wait(&empty[st], (rnd - 1) & 1u);
                const int line = line_at(a, listed, k);
                const int n = min(kCh, P - c * kCh);
                const uint32_t bytes = uint32_t(n) * B * 4;
                const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
                tc::mbar_expect_tx(&full[st], bytes);
                tc::bulk_g2s_hint(ring + size_t(st) * kCh * B, xl + size_t(c) * kCh * B, bytes, &full[st],
                                  again ? keep : drop);
                if (++st == NS) {
                    st = 0;
                    ++rnd;
                }
            };
            for (int k = 0; k <= my_lines; ++k)
                for (int c = 0; c < nch; ++c) {
                    if (k < my_lines) load(k, c, true);
                    if (k >= 1) load(k - 1, c, false);
                }
        }
        return;
    }
    if (warp == 9) {
        // ---------------- MMA issuer: 2 K-steps x 8 digit-plane pairs per chunk
        if (lane == 0) {
            for (int k = 0; k < my_lines; ++k) {
                if (k >= 1) tc::mbar_wait(&accempty, uint32_t(k - 1) & 1u);
                for (int c = 0; c < nch; ++c) {
                    const int k2 = k * nch + c, buf = k2 & 1;
                    tc::mbar_wait(&pfull[buf], uint32_t(k2 >> 1) & 1u);
                    tc::tc_fence_after();
                    const uint32_t base = tc::smem_u32(ops + buf * kOps);
                    issue_chunk_mmas(tmem, base, a.N, c == 0);
                    tc::mma_commit(&pempty[buf]);
                }
                tc::mma_commit(&accfull);
            }
        }
        return;
    }

    // ---------------- compute warps 0-7
    const int lane_grp = warp & 3, colh = warp >> 2;
    const int row = lane_grp * 32 + lane;
    const uint32_t lane_base = uint32_t(lane_grp * 32) << 16;
    const int ngrp = a.N / 16;
    const int g0 = colh ? (ngrp + 1) / 2 : 0, g1 = colh ? ngrp : (ngrp + 1) / 2;
    // pass 1 mapping: warp = 8-pixel group, lane = 4 consecutive dims (one 16-byte load per pixel)
    const bool quad_live = 4 * lane < B;
    // pass 2 mapping: warp = (16-pixel group, dim half), lane -> dims lane + 32k + 64 * half (conflict-free
    // 16-byte plane stores: 8 consecutive rows per quarter warp); loads clamp to a real band, the scale 0
    // of padded rows makes their value irrelevant
    const int pg2 = warp & 3, dh = warp >> 2;
    const int dd0 = lane + 64 * dh, dd1 = dd0 + 32;
    const int ld0 = min(dd0, B - 1), ld1 = min(dd1, B - 1);

    // epilogue of line kk: S_int = sum_c 2^(8c) acc_c scaled by 1 / (s_a s_b), staged in smem, then stored
    auto epilogue = [&](int kk) {
        const int line = line_at(a, listed, kk);
        tc::mbar_wait(&accfull, uint32_t(kk) & 1u);
        tc::tc_fence_after();
        for (int gi = g0; gi < g1; ++gi) {
            uint32_t v[4][16];
            tc::tmem_ld16x4(tmem + lane_base + uint32_t(gi * 16), 128u, v);
            if (row < D) {
                const double ia = inv_s[row];
#pragma unroll
                for (int ii = 0; ii < 16; ++ii) {
                    const int e = gi * 16 + ii;
                    // S_int = 2^8 a1 + 2^16 a2 + 2^24 a3 + 2^32 a4, exact in int64, one conversion
                    const long long si_i = (static_cast<long long>(int(v[3][ii])) << 32) +
                                           (static_cast<long long>(int(v[2][ii])) << 24) +
                                           (static_cast<long long>(int(v[1][ii])) << 16) +
                                           (static_cast<long long>(int(v[0][ii])) << 8);
                    const double si = double(si_i);  // (the ones column: no class-0 term)
                    if (e <= row) S[tri(row, e)] = si * ia * inv_s[e];
                    if (e == D) sum_s[row] = si * (1.0 / 256.0) * ia;
                }
            }
        }
        tc::tc_fence_before();
        bar_compute();
        if (tid == 0) mbar_arrive(&accempty);  // TMEM free for the next line's MMAs
        double* out = a.stats + size_t(line) * (g.SE + g.D);
        const bool bad = bad_s[0] | bad_s[1] | bad_s[2] | bad_s[3] | bad_s[4] | bad_s[5] | bad_s[6] | bad_s[7];
        const double poison = bad ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
        for (int i = tid; i < D; i += kThreads) {
            out[i] = double(cen_s[i]) + poison;
            out[D + i] = sum_s[i] + poison;
        }
        const int ntri = D * (D + 1) / 2;
        for (int i = tid; i < ntri; i += kThreads) out[2 * D + i] = S[i] + poison;
        bar_compute();  // S / sum_s / cen_s / bad_s are rewritten for the next line
    };

    float cdk[2] = {0.f, 0.f}, sdk[2] = {0.f, 0.f}, adk[2] = {kMagic, kMagic};
    // class-0 products (d0 d0, weight 1) are not accumulated by the MMAs; on the diagonal they are a
    // systematic + sum_p d0^2 (~P 2^14 / 3 in q^2 units), which biases K's small eigenvalues when the
    // background is ill-conditioned, so the quantiser sums them exactly here (one dp4a per 4 digits)
    // and leaves the four pixel-group partials per dim in c0 [line][4][D]; c0_fold_kernel adds them to
    // the diagonal of the stats slot.  Off the diagonal they are zero-mean and stay dropped (2^-30
    // relative).
    int c0a = 0, c0b = 0;
    int jst = 0;       // ring slot of the next chunk in the sequence (as the producer's)
    uint32_t jph = 0;  // its full-barrier phase
    auto next_slot = [&]() {
        if (++jst == NS) {
            jst = 0;
            jph ^= 1u;
        }
    };
    for (int k = 0; k <= my_lines; ++k) {
        const bool do1 = k < my_lines, do2 = k >= 1;
        float4 mn = make_float4(3.402823466e38f, 3.402823466e38f, 3.402823466e38f, 3.402823466e38f);
        float4 mx = make_float4(-3.402823466e38f, -3.402823466e38f, -3.402823466e38f, -3.402823466e38f);
        for (int c = 0; c < nch; ++c) {
            const int n = min(kCh, P - c * kCh);
            if (do1) {
                // ---- pass 1 of line k: range of x per dim (min propagates NaN, max sees +inf); centre
                const int st = jst;
                tc::mbar_wait(&full[st], jph);
                next_slot();
                const float* sb = ring + size_t(st) * kCh * B;
                if (quad_live) {
                    const int p0 = warp * 8;
                    const float* xp = sb + p0 * B + 4 * lane;
                    if (n >= p0 + 8) {
#pragma unroll
                        for (int pp = 0; pp < 8; ++pp) {
                            const float4 x = *reinterpret_cast<const float4*>(xp + pp * B);
                            mn.x = fmin_nan(mn.x, x.x); mn.y = fmin_nan(mn.y, x.y);
                            mn.z = fmin_nan(mn.z, x.z); mn.w = fmin_nan(mn.w, x.w);
                            mx.x = fmaxf(mx.x, x.x); mx.y = fmaxf(mx.y, x.y); mx.z = fmaxf(mx.z, x.z); mx.w = fmaxf(mx.w, x.w);
                        }
                    } else {
                        for (int pp = 0; pp < n - p0; ++pp) {
                            const float4 x = *reinterpret_cast<const float4*>(xp + pp * B);
                            mn.x = fmin_nan(mn.x, x.x); mn.y = fmin_nan(mn.y, x.y);
                            mn.z = fmin_nan(mn.z, x.z); mn.w = fmin_nan(mn.w, x.w);
                            mx.x = fmaxf(mx.x, x.x); mx.y = fmaxf(mx.y, x.y); mx.z = fmaxf(mx.z, x.z); mx.w = fmaxf(mx.w, x.w);
                        }
                    }
                    if (c == 0 && warp < 4) {
                        double4 cs = make_double4(0.0, 0.0, 0.0, 0.0);
                        for (int pp = 0; pp < min(8, n - p0); ++pp) {
                            const float4 x = *reinterpret_cast<const float4*>(xp + pp * B);
                            cs.x += double(x.x); cs.y += double(x.y); cs.z += double(x.z); cs.w += double(x.w);
                        }
                        red_cs[warp][4 * lane] = cs.x; red_cs[warp][4 * lane + 1] = cs.y;
                        red_cs[warp][4 * lane + 2] = cs.z; red_cs[warp][4 * lane + 3] = cs.w;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
            }
            if (do2) {
                // ---- pass 2 of line k-1: quantise the chunk into digit planes:
                // y = fma(x - c, s, 1.5 * 2^23) rounds v * s to an integer in the low mantissa bits
                // (|v s| <= 2^22), u = q + 0x808080 = bits(y) - 0x4B400000 + 0x808080
                const int st = jst;
                const int k2 = (k - 1) * nch + c, buf = k2 & 1;
                tc::mbar_wait(&full[st], jph);
                next_slot();
                if (k2 >= 2) tc::mbar_wait(&pempty[buf], uint32_t((k2 - 2) >> 1) & 1u);
                const float* sb = ring + size_t(st) * kCh * B + (pg2 * 16) * B;
                unsigned char* op = ops + buf * kOps;
                uint32_t w[2][3][4];
                if (n == kCh) {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        uint32_t u0[4], u1[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float* xp = sb + (jj * 4 + e) * B;
                            u0[e] = __float_as_uint(fmaf(xp[ld0] - cdk[0], sdk[0], adk[0])) + (0x808080u - 0x4B400000u);
                            u1[e] = __float_as_uint(fmaf(xp[ld1] - cdk[1], sdk[1], adk[1])) + (0x808080u - 0x4B400000u);
                        }
                        pack_digits(u0, w[0][0][jj], w[0][1][jj], w[0][2][jj]);
                        pack_digits(u1, w[1][0][jj], w[1][1][jj], w[1][2][jj]);
                        // d0 plane words hold 4 signed digits: one dp4a sums their squares
                        c0a = __dp4a(int(w[0][0][jj]), int(w[0][0][jj]), c0a);
                        c0b = __dp4a(int(w[1][0][jj]), int(w[1][0][jj]), c0b);
                    }
                } else {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        uint32_t u0[4], u1[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int p = pg2 * 16 + jj * 4 + e;
                            const float* xp = sb + (jj * 4 + e) * B;
                            u0[e] = __float_as_uint(fmaf(xp[ld0] - cdk[0], sdk[0], adk[0])) + (0x808080u - 0x4B400000u);
                            u1[e] = __float_as_uint(fmaf(xp[ld1] - cdk[1], sdk[1], adk[1])) + (0x808080u - 0x4B400000u);
                            if (p >= n) u0[e] = u1[e] = 0x808080u;
                        }
                        pack_digits(u0, w[0][0][jj], w[0][1][jj], w[0][2][jj]);
                        pack_digits(u1, w[1][0][jj], w[1][1][jj], w[1][2][jj]);
                        c0a = __dp4a(int(w[0][0][jj]), int(w[0][0][jj]), c0a);
                        c0b = __dp4a(int(w[1][0][jj]), int(w[1][0][jj]), c0b);
                    }
                }
                const uint32_t off0 = plane_off(dd0, pg2 * 16), off1 = plane_off(dd1, pg2 * 16);
#pragma unroll
                for (int pl = 0; pl < 3; ++pl) {
                    *reinterpret_cast<uint4*>(op + pl * tc::kSliceBytes + off0) = make_uint4(w[0][pl][0], w[0][pl][1], w[0][pl][2], w[0][pl][3]);
                    *reinterpret_cast<uint4*>(op + pl * tc::kSliceBytes + off1) = make_uint4(w[1][pl][0], w[1][pl][1], w[1][pl][2], w[1][pl][3]);
                }
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty[st]);
                    mbar_arrive(&pfull[buf]);
                }
                if (c == nch - 1) {  // the line's class-0 diagonal partials (consumed by the scan)
                    int* c0l = a.c0 + size_t(line_at(a, listed, k - 1)) * 4 * D + pg2 * D;
                    if (dd0 < D) c0l[dd0] = c0a;
                    if (dd1 < D) c0l[dd1] = c0b;
                    c0a = c0b = 0;
                }
                if (a.vplanes) {
                    // the same digits, as the score kernel's MN-major A operand (i8::vplane_off): one warp
                    // writes 2 x 512 contiguous bytes per plane
                    const int line = line_at(a, listed, k - 1);
                    const int gp = c * kCh + pg2 * 16;
                    unsigned char* vt = a.vplanes + (size_t(line) * ntile_v + (gp >> 7)) * i8::kTileBytes;
                    const uint64_t stream_out = tc::policy_evict_first();  // do not push x out of L2
                    const int used = i8::vplane_used_dims(D);  // the score never reads dims beyond
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl) {
                        if (dd0 < used)
                            tc::st16_hint(vt + i8::vplane_off(pl, dd0, gp & 127),
                                          make_uint4(w[0][pl][0], w[0][pl][1], w[0][pl][2], w[0][pl][3]), stream_out);
                        if (dd1 < used)
                            tc::st16_hint(vt + i8::vplane_off(pl, dd1, gp & 127),
                                          make_uint4(w[1][pl][0], w[1][pl][1], w[1][pl][2], w[1][pl][3]), stream_out);
                    }
                }
            }
        }
        // ---- line k-1 is complete: its epilogue (reads bad_s / cen_s / inv_s / c0_s of line k-1)
        if (do2) {
            epilogue(k - 1);
        }
        if (!do1) break;
        // ---- ranges of all pixel groups -> centre and per-dim scale of line k
        const bool bad_mine = quad_live && !(isfinite(mn.x) && isfinite(mn.y) && isfinite(mn.z) && isfinite(mn.w) &&
                                             isfinite(mx.x) && isfinite(mx.y) && isfinite(mx.z) && isfinite(mx.w));
        if (quad_live) {
            *reinterpret_cast<float4*>(&red_mn[warp][4 * lane]) = mn;
            *reinterpret_cast<float4*>(&red_mx[warp][4 * lane]) = mx;
        }
        const unsigned bw = __ballot_sync(0xffffffffu, bad_mine);
        if (lane == 0) bad_s[warp] = bw != 0;
        bar_compute();
        if (tid < 128) {
            const int d = tid;
            float cd = 0.f, sd = 0.f;
            const float ad = kMagic + (d == D ? 256.f : 0.f);  // ones row: q = 256
            if (d < D) {
                const int n0 = min(32, P);
                const double c0 = red_cs[0][d] + red_cs[1][d] + red_cs[2][d] + red_cs[3][d];
                cd = float(c0 / double(n0));
                float lo = red_mn[0][d], hi = red_mx[0][d];
                for (int w = 1; w < 8; ++w) {
                    lo = fminf(lo, red_mn[w][d]);
                    hi = fmaxf(hi, red_mx[w][d]);
                }
                const float m = fmaxf(hi - cd, cd - lo);
                sd = i8::v_scale(m);
                if (a.vmax) a.vmax[size_t(line_at(a, listed, k)) * D + d] = m;
            }
            cen_s[d] = cd;
            scale_s[d] = sd;
            add_s[d] = ad;
            inv_s[d] = sd > 0.f ? 1.0 / double(sd) : 0.0;
        }
        bar_compute();
        cdk[0] = cen_s[dd0 & 127]; sdk[0] = scale_s[dd0 & 127]; adk[0] = add_s[dd0 & 127];
        cdk[1] = cen_s[dd1 & 127]; sdk[1] = scale_s[dd1 & 127]; adk[1] = add_s[dd1 & 127];
    }
    if (warp == 0) tc::tmem_free<512>(tmem);
}

#ifdef ERX_X_TRACE  // A/B timeline instrumentation of CTA 0 (tools/stats_trace.py)
__device__ unsigned long long g_trace[1 << 16];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace_ev(int id, int k, int c) {
    if (blockIdx.x == 0) {
        const unsigned i = atomicAdd(&g_trace_n, 1u);
        if (i < (1u << 15)) {
            g_trace[2 * i] = clock64();
            g_trace[2 * i + 1] = (unsigned long long)((id << 24) | (k << 12) | c);
        }
    }
}
#define TR(id, k, c) trace_ev(id, k, c)
#else
#define TR(id, k, c)
#endif
// ---------------------------------------------------------------------------
// stats_i8_op: the same statistics in ONE pass over the line.  The two-pass kernels read every line
// twice (range, then quantise) because the quantisation scale is the line's exact per-dim range; both
// reads cross the L2 fabric, and with the digit planes written for the score kernel that traffic (not
// the tensor core, not the quantiser) bounds them.  Here the scale is PREDICTED from the
// line's first chunk: range_d = headroom x max over the first 64 pixels of |x_d - c_d| (headroom a
// power of two, 8 by default; a line of one chunk gets its exact range, i.e. the two-pass result).  The
// quantiser then runs straight off the HBM stream, every ring stage feeding it, and checks every
// rounded value against the digit range [-2^22, 2^22] (two min / max per element on the fma result,
// which also catches NaN and +-inf).  A line with any value outside is appended to a.redo and redone,
// exactly, by stats_i8_kernel<., true> (the next launch on the stream); its outputs here are
// overwritten.  A dim that is constant over the first chunk gets a huge quantiser scale (any later
// deviation overflows and lists the line) while its statistics scale stays 0 as in the two-pass kernels.
// Per line the result depends on that line only, so re-cutting the windows does not change a bit.
// Cost: the predicted range is ~headroom / 1.3 wider than the exact one on a clean line, i.e. ~2.6 bits
// of the 22 (tools/emulate_onepass.py; the parity gates hold with the margin recorded in DESIGN.md).
// Warps: 0-7 range of chunk 0, quantise, epilogue; 8 producer; 9 MMA issuer (as stats_i8_kernel).
// ---------------------------------------------------------------------------
constexpr float kYLo = 8388608.f, kYHi = 16777216.f;  // kMagic -+ 2^22: the fma results of in-range values

template <int kBT>
__global__ void __launch_bounds__(kThreads + 64, 1) stats_i8_op_kernel(StatsI8Args a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
    __shared__ __align__(8) uint64_t pfull[2], pempty[2], accfull, accempty;
    __shared__ __align__(16) float red_mn[8][128];
    __shared__ __align__(16) float red_mx[8][128];
    __shared__ double red_cs[4][128];
    __shared__ float cen_s[128], scale_s[128], add_s[128];
    __shared__ double inv_s[128];
    __shared__ double sum_s[128];
    __shared__ int bad_s[8];

    const Geometry& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int B = kBT > 0 ? kBT : g.B, D = g.D, P = g.P;
    const int NS = a.stages;

    unsigned char* ops = smem;                                   // [2][kOps]
    float* ring = reinterpret_cast<float*>(smem + 2 * kOps);     // [NS][kCh * B]
    const size_t tri_bytes = size_t(D) * (D + 1) / 2 * 8;
    double* S = reinterpret_cast<double*>(tri_bytes <= 2 * kOps ? smem : smem + 2 * kOps + size_t(NS) * kCh * B * 4);
    const int nch = (P + kCh - 1) / kCh;
    const int ntile_v = (P + 127) / 128;
    const int my_lines = blockIdx.x < a.n_lines ? (a.n_lines - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 8);
        }
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
        // ---------------- producer: every chunk once, straight from HBM (nothing is read again)
        if (lane == 0) {
            int st = 0;
            uint32_t rnd = 0;
            const uint64_t drop = tc::policy_evict_first();
            for (int k = 0; k < my_lines; ++k) {
                const float* xl = line_ptr(a.x, blockIdx.x + k * gridDim.x, a.n, a.in_stride, g);
                for (int c = 0; c < nch; ++c) {
                    if (rnd >= 1) tc::mbar_wait(&empty[st], (rnd - 1) & 1u);
                    TR(30, k, c);
                    const uint32_t bytes = uint32_t(min(kCh, P - c * kCh)) * B * 4;
                    tc::mbar_expect_tx(&full[st], bytes);
                    tc::bulk_g2s_hint(ring + size_t(st) * kCh * B, xl + size_t(c) * kCh * B, bytes, &full[st], drop);
                    if (++st == NS) {
                        st = 0;
                        ++rnd;
                    }
                }
            }
        }
        return;
    }
    if (warp == 9) {
        // ---------------- MMA issuer: 2 K-steps x 8 digit-plane pairs per chunk (as stats_i8_kernel)
        if (lane == 0) {
            for (int k = 0; k < my_lines; ++k) {
                if (k >= 1) tc::mbar_wait(&accempty, uint32_t(k - 1) & 1u);
                for (int c = 0; c < nch; ++c) {
                    const int k2 = k * nch + c, buf = k2 & 1;
                    tc::mbar_wait(&pfull[buf], uint32_t(k2 >> 1) & 1u);
                    tc::tc_fence_after();
                    const uint32_t base = tc::smem_u32(ops + buf * kOps);
                    issue_chunk_mmas(tmem, base, a.N, c == 0);
                    tc::mma_commit(&pempty[buf]);
                }
                tc::mma_commit(&accfull);
            }
        }
        return;
    }

    // ---------------- compute warps 0-7
    const int lane_grp = warp & 3, colh = warp >> 2;
    const int row = lane_grp * 32 + lane;
    const uint32_t lane_base = uint32_t(lane_grp * 32) << 16;
    const int ngrp = a.N / 16;
    const int g0 = colh ? (ngrp + 1) / 2 : 0, g1 = colh ? ngrp : (ngrp + 1) / 2;
    const bool quad_live = 4 * lane < B;  // range mapping: warp = 8-pixel group, lane = 4 consecutive dims
    const int pg2 = warp & 3, dh = warp >> 2;  // quantise mapping (stats_i8_kernel's)
    const int dd0 = lane + 64 * dh, dd1 = dd0 + 32;
    const int ld0 = min(dd0, B - 1), ld1 = min(dd1, B - 1);
    const float head = nch > 1 ? a.headroom : 1.f;

    int jst = 0;
    uint32_t jph = 0;
    int c0a = 0, c0b = 0;
    for (int k = 0; k < my_lines; ++k) {
        const int line = blockIdx.x + k * gridDim.x;
        float cdk0 = 0.f, sdk0 = 0.f, adk0 = kMagic, cdk1 = 0.f, sdk1 = 0.f, adk1 = kMagic;
        float ylo = kMagic, yhi = kMagic;
        for (int c = 0; c < nch; ++c) {
            const int n = min(kCh, P - c * kCh);
            const int st = jst;
            const int k2 = k * nch + c, buf = k2 & 1;
            tc::mbar_wait(&full[st], jph);
            if (tid == 0) TR(1, k, c);
            if (++jst == NS) {
                jst = 0;
                jph ^= 1u;
            }
            if (c == 0) {
                // ---- the line's centre and predicted range, from the chunk just landed
                float4 mn = make_float4(3.402823466e38f, 3.402823466e38f, 3.402823466e38f, 3.402823466e38f);
                float4 mx = make_float4(-3.402823466e38f, -3.402823466e38f, -3.402823466e38f, -3.402823466e38f);
                if (quad_live) {
                    const int p0 = warp * 8;
                    const float* xp = ring + size_t(st) * kCh * B + p0 * B + 4 * lane;
                    const int np = min(8, n - p0);
                    for (int pp = 0; pp < np; ++pp) {
                        const float4 x = *reinterpret_cast<const float4*>(xp + pp * B);
                        mn.x = fmin_nan(mn.x, x.x); mn.y = fmin_nan(mn.y, x.y);
                        mn.z = fmin_nan(mn.z, x.z); mn.w = fmin_nan(mn.w, x.w);
                        mx.x = fmaxf(mx.x, x.x); mx.y = fmaxf(mx.y, x.y); mx.z = fmaxf(mx.z, x.z); mx.w = fmaxf(mx.w, x.w);
                    }
                    if (warp < 4) {  // centre: the first 32 pixels, per 8-pixel group (k_stats.cu's rule)
                        double4 cs = make_double4(0.0, 0.0, 0.0, 0.0);
                        for (int pp = 0; pp < np; ++pp) {
                            const float4 x = *reinterpret_cast<const float4*>(xp + pp * B);
                            cs.x += double(x.x); cs.y += double(x.y); cs.z += double(x.z); cs.w += double(x.w);
                        }
                        red_cs[warp][4 * lane] = cs.x; red_cs[warp][4 * lane + 1] = cs.y;
                        red_cs[warp][4 * lane + 2] = cs.z; red_cs[warp][4 * lane + 3] = cs.w;
                    }
                    *reinterpret_cast<float4*>(&red_mn[warp][4 * lane]) = mn;
                    *reinterpret_cast<float4*>(&red_mx[warp][4 * lane]) = mx;
                }
                bar_compute();
                if (tid < 128) {
                    const int d = tid;
                    float cd = 0.f, sd = 0.f, sq = 0.f;
                    const float ad = kMagic + (d == D ? 256.f : 0.f);  // ones row: q = 256
                    if (d < D) {
                        const int n0 = min(32, P);
                        const double c0 = red_cs[0][d] + red_cs[1][d] + red_cs[2][d] + red_cs[3][d];
                        cd = float(c0 / double(n0));
                        float lo = red_mn[0][d], hi = red_mx[0][d];
                        for (int w = 1; w < 8; ++w) {  // (groups past the line's end hold the neutral +-FLT_MAX)
                            lo = fminf(lo, red_mn[w][d]);
                            hi = fmaxf(hi, red_mx[w][d]);
                        }
                        const float m = head * fmaxf(hi - cd, cd - lo);
                        sd = i8::v_scale(m);
                        // a dim with no range in the first chunk: any later deviation must overflow
                        sq = sd > 0.f ? sd : (nch > 1 ? 3.0e38f : 0.f);
                        if (a.vmax) a.vmax[size_t(line) * D + d] = (m <= 3.402823466e38f) ? m : 0.f;
                    }
                    cen_s[d] = cd;
                    scale_s[d] = sq;
                    add_s[d] = ad;
                    inv_s[d] = sd > 0.f ? 1.0 / double(sd) : 0.0;
                }
                bar_compute();
                cdk0 = cen_s[dd0 & 127]; sdk0 = scale_s[dd0 & 127]; adk0 = add_s[dd0 & 127];
                cdk1 = cen_s[dd1 & 127]; sdk1 = scale_s[dd1 & 127]; adk1 = add_s[dd1 & 127];
                if (tid == 0) TR(6, k, c);
            }
            // ---- quantise the chunk into digit planes (stats_i8_kernel's arithmetic) and check the range
            if (k2 >= 2) tc::mbar_wait(&pempty[buf], uint32_t((k2 - 2) >> 1) & 1u);
            if (tid == 0) TR(2, k, c);
            const float* sb = ring + size_t(st) * kCh * B + (pg2 * 16) * B;
            unsigned char* op = ops + buf * kOps;
            uint32_t w[2][3][4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                uint32_t u0[4], u1[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float* xp = sb + (jj * 4 + e) * B;
                    float y0 = fmaf(xp[ld0] - cdk0, sdk0, adk0), y1 = fmaf(xp[ld1] - cdk1, sdk1, adk1);
                    if (n != kCh && pg2 * 16 + jj * 4 + e >= n) y0 = y1 = kMagic;  // past the line's end
                    ylo = fmin_nan(fmin_nan(ylo, y0), y1);
                    yhi = fmaxf(fmaxf(yhi, y0), y1);
                    u0[e] = __float_as_uint(y0) + (0x808080u - 0x4B400000u);
                    u1[e] = __float_as_uint(y1) + (0x808080u - 0x4B400000u);
                }
                pack_digits(u0, w[0][0][jj], w[0][1][jj], w[0][2][jj]);
                pack_digits(u1, w[1][0][jj], w[1][1][jj], w[1][2][jj]);
                c0a = __dp4a(int(w[0][0][jj]), int(w[0][0][jj]), c0a);
                c0b = __dp4a(int(w[1][0][jj]), int(w[1][0][jj]), c0b);
            }
            const uint32_t off0 = plane_off(dd0, pg2 * 16), off1 = plane_off(dd1, pg2 * 16);
#pragma unroll
            for (int pl = 0; pl < 3; ++pl) {
                *reinterpret_cast<uint4*>(op + pl * tc::kSliceBytes + off0) = make_uint4(w[0][pl][0], w[0][pl][1], w[0][pl][2], w[0][pl][3]);
                *reinterpret_cast<uint4*>(op + pl * tc::kSliceBytes + off1) = make_uint4(w[1][pl][0], w[1][pl][1], w[1][pl][2], w[1][pl][3]);
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[st]);
                mbar_arrive(&pfull[buf]);
            }
            if (tid == 0) TR(3, k, c);
            if (c == nch - 1) {  // the line's class-0 diagonal partials (folded by c0_fold_kernel)
                int* c0l = a.c0 + size_t(line) * 4 * D + pg2 * D;
                if (dd0 < D) c0l[dd0] = c0a;
                if (dd1 < D) c0l[dd1] = c0b;
                c0a = c0b = 0;
            }
            if (a.vplanes) {
                const int gp = c * kCh + pg2 * 16;
                unsigned char* vt = a.vplanes + (size_t(line) * ntile_v + (gp >> 7)) * i8::kTileBytes;
                const uint64_t stream_out = tc::policy_evict_first();
                const int used = i8::vplane_used_dims(D);
#pragma unroll
                for (int pl = 0; pl < 3; ++pl) {
                    if (dd0 < used)
                        tc::st16_hint(vt + i8::vplane_off(pl, dd0, gp & 127),
                                      make_uint4(w[0][pl][0], w[0][pl][1], w[0][pl][2], w[0][pl][3]), stream_out);
                    if (dd1 < used)
                        tc::st16_hint(vt + i8::vplane_off(pl, dd1, gp & 127),
                                      make_uint4(w[1][pl][0], w[1][pl][1], w[1][pl][2], w[1][pl][3]), stream_out);
                }
            }
        }
        // ---- every rounded value inside the digit range?  (false for NaN / inf as well)
        const bool bad_mine = !(ylo >= kYLo && yhi <= kYHi);
        const unsigned bw = __ballot_sync(0xffffffffu, bad_mine);
        if (lane == 0) bad_s[warp] = bw != 0;
        // ---- epilogue (stats_i8_kernel's); a line out of range is listed for the redo pass instead
        if (tid == 0) TR(7, k, 0);
        tc::mbar_wait(&accfull, uint32_t(k) & 1u);
        if (tid == 0) TR(4, k, 0);
        tc::tc_fence_after();
        for (int gi = g0; gi < g1; ++gi) {
            uint32_t v[4][16];
            tc::tmem_ld16x4(tmem + lane_base + uint32_t(gi * 16), 128u, v);
            if (row < D) {
                const double ia = inv_s[row];
#pragma unroll
                for (int ii = 0; ii < 16; ++ii) {
                    const int e = gi * 16 + ii;
                    const long long si_i = (static_cast<long long>(int(v[3][ii])) << 32) +
                                           (static_cast<long long>(int(v[2][ii])) << 24) +
                                           (static_cast<long long>(int(v[1][ii])) << 16) +
                                           (static_cast<long long>(int(v[0][ii])) << 8);
                    const double si = double(si_i);
                    if (e <= row) S[tri(row, e)] = si * ia * inv_s[e];
                    if (e == D) sum_s[row] = si * (1.0 / 256.0) * ia;
                }
            }
        }
        tc::tc_fence_before();
        bar_compute();
        if (tid == 0) TR(8, k, 0);
        if (tid == 0) mbar_arrive(&accempty);  // TMEM free for the next line's MMAs
        const bool bad = bad_s[0] | bad_s[1] | bad_s[2] | bad_s[3] | bad_s[4] | bad_s[5] | bad_s[6] | bad_s[7];
        if (bad) {
            if (tid == 0) a.redo[2 + atomicAdd(&a.redo[0], 1)] = line;
        } else {
            double* out = a.stats + size_t(line) * (g.SE + g.D);
            for (int i = tid; i < D; i += kThreads) {
                out[i] = double(cen_s[i]);
                out[D + i] = sum_s[i];
            }
            const int ntri = D * (D + 1) / 2;
            for (int i = tid; i < ntri; i += kThreads) out[2 * D + i] = S[i];
        }
        bar_compute();  // S / sum_s / cen_s / bad_s are rewritten for the next line
        if (tid == 0) TR(5, k, 0);
    }
    if (warp == 0) tc::tmem_free<512>(tmem);
}

// ---------------------------------------------------------------------------
// stats_i8_ws: the same statistics with the range pass on its own warps.  In stats_i8_kernel the
// eight compute warps run the range pass of line k, the quantise pass of line k-1, its epilogue and
// the range step one after the other; measured, that chain (not the loads) bounds the kernel
// (DESIGN.md §6).  Here warps 8-11 stream pass 1 (range of line k, its own ring, HBM, evict_last)
// and hand each line's centre / scale to the quantise warps through per-parity shared arrays
// (sready / sfree mbarriers), so the range pass runs beside the quantise / MMA / epilogue chain of
// warps 0-7.  The pass-2 producer re-reads a chunk from L2 only once the range warps have passed it
// (a monotonic chunk count).  Arithmetic per line is the stats_i8_kernel's (bit-identical output).
// Warps: 0-7 quantise + epilogue, 8-11 range, 12 pass-1 producer, 13 pass-2 producer, 14 MMA issuer.
// ---------------------------------------------------------------------------
constexpr int kWsThreads = 480;

__device__ __forceinline__ void bar_range() { asm volatile("bar.sync 2, 128;" ::); }

template <int kBT>
__global__ void __launch_bounds__(kWsThreads, 1) stats_i8_ws_kernel(StatsI8Args a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t full1[kMaxStages], empty1[kMaxStages], full2[kMaxStages], empty2[kMaxStages];
    __shared__ __align__(8) uint64_t pfull[2], pempty[2], accfull, accempty, sready[2], sfree[2];
    __shared__ __align__(16) float red_mn[4][128];
    __shared__ __align__(16) float red_mx[4][128];
    __shared__ double red_cs[4][128];
    __shared__ float cen_s[2][128], scale_s[2][128], add_s[2][128];  // per line parity
    __shared__ double inv_s[2][128];
    __shared__ double sum_s[128];
    __shared__ int bad_s[2][4];
    __shared__ int p1_count;  // pass-1 chunks finished by the range warps, x 4 (monotonic)

    const Geometry& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int B = kBT > 0 ? kBT : g.B, D = g.D, P = g.P;
    const int NS1 = a.ring1, NS2 = a.stages - a.ring1;

    unsigned char* ops = smem;                                          // [2][kOps]
    float* ring1 = reinterpret_cast<float*>(smem + 2 * kOps);           // [NS1][kCh * B]
    float* ring2 = ring1 + size_t(NS1) * kCh * B;                       // [NS2][kCh * B]
    const size_t tri_bytes = size_t(D) * (D + 1) / 2 * 8;
    double* S = reinterpret_cast<double*>(tri_bytes <= 2 * kOps ? smem : smem + 2 * kOps + size_t(a.stages) * kCh * B * 4);
    const int nch = (P + kCh - 1) / kCh;
    const int ntile_v = (P + 127) / 128;
    const int my_lines = blockIdx.x < a.n_lines ? (a.n_lines - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (tid == 0) {
        for (int s = 0; s < NS1; ++s) {
            tc::mbar_init(&full1[s], 1);
            tc::mbar_init(&empty1[s], 4);
        }
        for (int s = 0; s < NS2; ++s) {
            tc::mbar_init(&full2[s], 1);
            tc::mbar_init(&empty2[s], 8);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&pfull[b], 8);
            tc::mbar_init(&pempty[b], 1);
            tc::mbar_init(&sready[b], 4);
            tc::mbar_init(&sfree[b], 8);
        }
        tc::mbar_init(&accfull, 1);
        tc::mbar_init(&accempty, 1);
        p1_count = 0;
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(&tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 12 || warp == 13) {
        // ---------------- producers: warp 12 pass 1 (HBM, kept in L2), warp 13 pass 2 (the L2 re-read)
        if (lane == 0) {
            const bool p1 = warp == 12;
            const int NSx = p1 ? NS1 : NS2;
            float* ring = p1 ? ring1 : ring2;
            uint64_t* fullx = p1 ? full1 : full2;
            uint64_t* emptyx = p1 ? empty1 : empty2;
            const uint64_t pol = p1 ? tc::policy_evict_last() : tc::policy_evict_first();
            int st = 0;
            uint32_t rnd = 0;
            for (int k = 0; k < my_lines; ++k)
                for (int c = 0; c < nch; ++c) {
                    if (!p1)  // the range warps have read this chunk (it is in L2 now)
                        while (*reinterpret_cast<volatile int*>(&p1_count) < 4 * (k * nch + c + 1)) __nanosleep(64);
                    if (rnd >= 1) tc::mbar_wait(&emptyx[st], (rnd - 1) & 1u);
                    TR(p1 ? 30 : 31, k, c);
                    const int line = blockIdx.x + k * gridDim.x;
                    const int n = min(kCh, P - c * kCh);
                    const uint32_t bytes = uint32_t(n) * B * 4;
                    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
                    tc::mbar_expect_tx(&fullx[st], bytes);
                    tc::bulk_g2s_hint(ring + size_t(st) * kCh * B, xl + size_t(c) * kCh * B, bytes, &fullx[st], pol);
                    if (++st == NSx) {
                        st = 0;
                        ++rnd;
                    }
                }
        }
        return;
    }
    if (warp == 14) {
        // ---------------- MMA issuer: 2 K-steps x 8 digit-plane pairs per chunk (as stats_i8_kernel)
        if (lane == 0) {
            for (int k = 0; k < my_lines; ++k) {
                if (k >= 1) tc::mbar_wait(&accempty, uint32_t(k - 1) & 1u);
                for (int c = 0; c < nch; ++c) {
                    const int k2 = k * nch + c, buf = k2 & 1;
                    tc::mbar_wait(&pfull[buf], uint32_t(k2 >> 1) & 1u);
                    TR(20, k, c);
                    tc::tc_fence_after();
                    const uint32_t base = tc::smem_u32(ops + buf * kOps);
                    issue_chunk_mmas(tmem, base, a.N, c == 0);
                    tc::mma_commit(&pempty[buf]);
                    TR(21, k, c);
                }
                tc::mma_commit(&accfull);
            }
        }
        return;
    }
    if (warp >= 8) {
        // ---------------- range warps 8-11: pass 1 of every line and its range step
        const int wr = warp - 8, t2 = tid - 256;
        const bool quad_live = 4 * lane < B;
        int st = 0;
        uint32_t ph = 0;
        for (int k = 0; k < my_lines; ++k) {
            float4 mn = make_float4(3.402823466e38f, 3.402823466e38f, 3.402823466e38f, 3.402823466e38f);
            float4 mx = make_float4(-3.402823466e38f, -3.402823466e38f, -3.402823466e38f, -3.402823466e38f);
            for (int c = 0; c < nch; ++c) {
                const int n = min(kCh, P - c * kCh);
                tc::mbar_wait(&full1[st], ph);
                if (lane == 0 && wr == 0) TR(10, k, c);
                const float* sb = ring1 + size_t(st) * kCh * B;
                if (quad_live) {
                    // 8-pixel groups wr and wr + 4 (stats_i8_kernel's groups, two per warp here)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int p0 = (wr + 4 * h) * 8;
                        const float* xp = sb + p0 * B + 4 * lane;
                        const int np = min(8, n - p0);
#pragma unroll
                        for (int pp = 0; pp < 8; ++pp) {
                            if (pp < np) {
                                const float4 x = *reinterpret_cast<const float4*>(xp + pp * B);
                                mn.x = fmin_nan(mn.x, x.x); mn.y = fmin_nan(mn.y, x.y);
                                mn.z = fmin_nan(mn.z, x.z); mn.w = fmin_nan(mn.w, x.w);
                                mx.x = fmaxf(mx.x, x.x); mx.y = fmaxf(mx.y, x.y); mx.z = fmaxf(mx.z, x.z); mx.w = fmaxf(mx.w, x.w);
                            }
                        }
                        if (c == 0 && h == 0) {  // centre: the first 32 pixels, per 8-pixel group as stats_i8_kernel
                            double4 cs = make_double4(0.0, 0.0, 0.0, 0.0);
                            for (int pp = 0; pp < np; ++pp) {
                                const float4 x = *reinterpret_cast<const float4*>(xp + pp * B);
                                cs.x += double(x.x); cs.y += double(x.y); cs.z += double(x.z); cs.w += double(x.w);
                            }
                            red_cs[wr][4 * lane] = cs.x; red_cs[wr][4 * lane + 1] = cs.y;
                            red_cs[wr][4 * lane + 2] = cs.z; red_cs[wr][4 * lane + 3] = cs.w;
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty1[st]);
                    atomicAdd(&p1_count, 1);
                }
                if (++st == NS1) {
                    st = 0;
                    ph ^= 1u;
                }
            }
            // ---- range step of line k: centre and per-dim scale into the line's parity slot
            const bool bad_mine = quad_live && !(isfinite(mn.x) && isfinite(mn.y) && isfinite(mn.z) && isfinite(mn.w) &&
                                                 isfinite(mx.x) && isfinite(mx.y) && isfinite(mx.z) && isfinite(mx.w));
            if (quad_live) {
                *reinterpret_cast<float4*>(&red_mn[wr][4 * lane]) = mn;
                *reinterpret_cast<float4*>(&red_mx[wr][4 * lane]) = mx;
            }
            const unsigned bw = __ballot_sync(0xffffffffu, bad_mine);
            bar_range();
            const int par = k & 1;
            if (k >= 2) tc::mbar_wait(&sfree[par], uint32_t((k - 2) >> 1) & 1u);  // line k-2 done with the slot
            if (lane == 0) bad_s[par][wr] = bw != 0;
            {
                const int d = t2;
                float cd = 0.f, sd = 0.f;
                const float ad = kMagic + (d == D ? 256.f : 0.f);  // ones row: q = 256
                if (d < D) {
                    const int n0 = min(32, P);
                    const double c0 = red_cs[0][d] + red_cs[1][d] + red_cs[2][d] + red_cs[3][d];
                    cd = float(c0 / double(n0));
                    float lo = red_mn[0][d], hi = red_mx[0][d];
                    for (int w = 1; w < 4; ++w) {
                        lo = fminf(lo, red_mn[w][d]);
                        hi = fmaxf(hi, red_mx[w][d]);
                    }
                    const float m = fmaxf(hi - cd, cd - lo);
                    sd = i8::v_scale(m);
                    if (a.vmax) a.vmax[size_t(blockIdx.x + k * gridDim.x) * D + d] = m;
                }
                cen_s[par][d] = cd;
                scale_s[par][d] = sd;
                add_s[par][d] = ad;
                inv_s[par][d] = sd > 0.f ? 1.0 / double(sd) : 0.0;
            }
            bar_range();  // (red_* are rewritten by the next line's pass 1 only after every thread read them)
            if (lane == 0) mbar_arrive(&sready[par]);
            if (lane == 0 && wr == 0) TR(11, k, 0);
        }
        return;
    }

    // ---------------- warps 0-7: quantise (pass 2) and the epilogue of every line
    const int lane_grp = warp & 3, colh = warp >> 2;
    const int row = lane_grp * 32 + lane;
    const uint32_t lane_base = uint32_t(lane_grp * 32) << 16;
    const int ngrp = a.N / 16;
    const int g0 = colh ? (ngrp + 1) / 2 : 0, g1 = colh ? ngrp : (ngrp + 1) / 2;
    const int pg2 = warp & 3, dh = warp >> 2;
    const int dd0 = lane + 64 * dh, dd1 = dd0 + 32;
    const int ld0 = min(dd0, B - 1), ld1 = min(dd1, B - 1);
    int st = 0;
    uint32_t ph = 0;
    int c0a = 0, c0b = 0;
    for (int k = 0; k < my_lines; ++k) {
        const int par = k & 1;
        const int line = blockIdx.x + k * gridDim.x;
        tc::mbar_wait(&sready[par], uint32_t(k >> 1) & 1u);
        if (tid == 0) TR(0, k, 0);
        const float cdk0 = cen_s[par][dd0 & 127], sdk0 = scale_s[par][dd0 & 127], adk0 = add_s[par][dd0 & 127];
        const float cdk1 = cen_s[par][dd1 & 127], sdk1 = scale_s[par][dd1 & 127], adk1 = add_s[par][dd1 & 127];
        for (int c = 0; c < nch; ++c) {
            const int n = min(kCh, P - c * kCh);
            const int k2 = k * nch + c, buf = k2 & 1;
            tc::mbar_wait(&full2[st], ph);
            if (tid == 0) TR(1, k, c);
            if (k2 >= 2) tc::mbar_wait(&pempty[buf], uint32_t((k2 - 2) >> 1) & 1u);
            if (tid == 0) TR(2, k, c);
            const float* sb = ring2 + size_t(st) * kCh * B + (pg2 * 16) * B;
            unsigned char* op = ops + buf * kOps;
            uint32_t w[2][3][4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                uint32_t u0[4], u1[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float* xp = sb + (jj * 4 + e) * B;
                    u0[e] = __float_as_uint(fmaf(xp[ld0] - cdk0, sdk0, adk0)) + (0x808080u - 0x4B400000u);
                    u1[e] = __float_as_uint(fmaf(xp[ld1] - cdk1, sdk1, adk1)) + (0x808080u - 0x4B400000u);
                    if (n != kCh && pg2 * 16 + jj * 4 + e >= n) u0[e] = u1[e] = 0x808080u;
                }
                pack_digits(u0, w[0][0][jj], w[0][1][jj], w[0][2][jj]);
                pack_digits(u1, w[1][0][jj], w[1][1][jj], w[1][2][jj]);
                c0a = __dp4a(int(w[0][0][jj]), int(w[0][0][jj]), c0a);
                c0b = __dp4a(int(w[1][0][jj]), int(w[1][0][jj]), c0b);
            }
            const uint32_t off0 = plane_off(dd0, pg2 * 16), off1 = plane_off(dd1, pg2 * 16);
#pragma unroll
            for (int pl = 0; pl < 3; ++pl) {
                *reinterpret_cast<uint4*>(op + pl * tc::kSliceBytes + off0) = make_uint4(w[0][pl][0], w[0][pl][1], w[0][pl][2], w[0][pl][3]);
                *reinterpret_cast<uint4*>(op + pl * tc::kSliceBytes + off1) = make_uint4(w[1][pl][0], w[1][pl][1], w[1][pl][2], w[1][pl][3]);
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty2[st]);
                mbar_arrive(&pfull[buf]);
            }
            if (tid == 0) TR(3, k, c);
            if (++st == NS2) {
                st = 0;
                ph ^= 1u;
            }
            if (c == nch - 1) {  // the line's class-0 diagonal partials (folded by c0_fold_kernel)
                int* c0l = a.c0 + size_t(line) * 4 * D + pg2 * D;
                if (dd0 < D) c0l[dd0] = c0a;
                if (dd1 < D) c0l[dd1] = c0b;
                c0a = c0b = 0;
            }
            if (a.vplanes) {
                const int gp = c * kCh + pg2 * 16;
                unsigned char* vt = a.vplanes + (size_t(line) * ntile_v + (gp >> 7)) * i8::kTileBytes;
                const uint64_t stream_out = tc::policy_evict_first();
                const int used = i8::vplane_used_dims(D);
#pragma unroll
                for (int pl = 0; pl < 3; ++pl) {
                    if (dd0 < used)
                        tc::st16_hint(vt + i8::vplane_off(pl, dd0, gp & 127),
                                      make_uint4(w[0][pl][0], w[0][pl][1], w[0][pl][2], w[0][pl][3]), stream_out);
                    if (dd1 < used)
                        tc::st16_hint(vt + i8::vplane_off(pl, dd1, gp & 127),
                                      make_uint4(w[1][pl][0], w[1][pl][1], w[1][pl][2], w[1][pl][3]), stream_out);
                }
            }
        }
        // ---- epilogue of line k (stats_i8_kernel's, with the line's parity slot)
        tc::mbar_wait(&accfull, uint32_t(k) & 1u);
        if (tid == 0) TR(4, k, 0);
        tc::tc_fence_after();
        for (int gi = g0; gi < g1; ++gi) {
            uint32_t v[4][16];
            tc::tmem_ld16x4(tmem + lane_base + uint32_t(gi * 16), 128u, v);
            if (row < D) {
                const double ia = inv_s[par][row];
#pragma unroll
                for (int ii = 0; ii < 16; ++ii) {
                    const int e = gi * 16 + ii;
                    const long long si_i = (static_cast<long long>(int(v[3][ii])) << 32) +
                                           (static_cast<long long>(int(v[2][ii])) << 24) +
                                           (static_cast<long long>(int(v[1][ii])) << 16) +
                                           (static_cast<long long>(int(v[0][ii])) << 8);
                    const double si = double(si_i);
                    if (e <= row) S[tri(row, e)] = si * ia * inv_s[par][e];
                    if (e == D) sum_s[row] = si * (1.0 / 256.0) * ia;
                }
            }
        }
        tc::tc_fence_before();
        bar_compute();
        if (tid == 0) mbar_arrive(&accempty);
        double* out = a.stats + size_t(line) * (g.SE + g.D);
        const bool bad = bad_s[par][0] | bad_s[par][1] | bad_s[par][2] | bad_s[par][3];
        const double poison = bad ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
        for (int i = tid; i < D; i += kThreads) {
            out[i] = double(cen_s[par][i]) + poison;
            out[D + i] = sum_s[i] + poison;
        }
        const int ntri = D * (D + 1) / 2;
        for (int i = tid; i < ntri; i += kThreads) out[2 * D + i] = S[i] + poison;
        bar_compute();  // S / sum_s rewritten by the next line; the parity slot is free for line k + 2
        if (lane == 0) mbar_arrive(&sfree[par]);
        if (tid == 0) TR(5, k, 0);
    }
    tc::tc_fence_before();
    bar_compute();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

// S_aa += sum_p d0_a^2 / s_a^2 for every (line, dim): the class-0 diagonal the MMAs leave out, from the
// quantiser's four pixel-group partials (exact int32 sums), scaled exactly as the epilogue scales S.
__global__ void __launch_bounds__(256) c0_fold_kernel(int D, int SS, int n_lines, const int* __restrict__ c0,
                                                      const float* __restrict__ vmax, double* __restrict__ stats,
                                                      int* redo) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && redo) {  // the one-pass statistics' redo list: consumed by the launch before this one
        redo[1] += redo[0];
        redo[0] = 0;
    }
    if (i >= n_lines * D) return;
    const int line = i / D, a = i - line * D;
    const float s = i8::v_scale(vmax[i]);
    if (!(s > 0.f)) return;
    const int* p = c0 + size_t(line) * 4 * D + a;
    const long long q = (long long)(p[0]) + p[D] + p[2 * D] + p[3 * D];
    const double inv = 1.0 / double(s);
    stats[size_t(line) * SS + 2 * D + tri(a, a)] += double(q) * inv * inv;
}

constexpr size_t kStaticSmem = 17 * 1024;  // static shared arrays of the kernel (ptxas: 16.0 KB)

size_t i8_tri_extra(const Geometry& g) {  // S staging beyond the plane buffers it aliases when it fits
    const size_t tri = size_t(g.D) * (g.D + 1) / 2 * 8;
    return tri <= 2 * size_t(kOps) ? 0 : tri;
}

int i8_stages(const Geometry& g) {
    const size_t fixed = 2 * size_t(kOps) + i8_tri_extra(g) + kStaticSmem;
    const size_t chunk = size_t(kCh) * g.B * 4;
    const int st = int((kSmemCap - fixed) / chunk);
    return st < kMaxStages ? st : kMaxStages;
}

size_t stats_i8_smem(const Geometry& g) {
    return 2 * size_t(kOps) + size_t(i8_stages(g)) * kCh * g.B * 4 + i8_tri_extra(g);
}

}  // namespace

bool stats_i8_eligible(const Geometry& g) {
    // P < 43690: every s32 class sum (<= 3 digit pairs x 2^14 x P) stays exact
    return !g.srp && g.D > 16 && g.D <= 127 && (g.B % 4) == 0 && g.P < 43690 && i8_stages(g) >= 2;
}

void launch_stats_i8(const Geometry& g, const float* x, int n_per_stream, int in_stride, int n_lines_total,
                     double* stats, float* vmax, unsigned char* vplanes, int* c0, cudaStream_t st, int ring1,
                     int* redo, int headroom) {
    const int sms = sm_count();
    ensure_smem(stats_i8_kernel<0>, kSmemCap - kStaticSmem);
    ensure_smem(stats_i8_kernel<108>, kSmemCap - kStaticSmem);
    StatsI8Args a{g, x, n_per_stream, in_stride, n_lines_total, stats, vmax, vplanes, c0, (g.D + 1 + 15) / 16 * 16,
                  i8_stages(g), 0, redo, float(headroom)};
    const int grid = n_lines_total < sms ? n_lines_total : sms;
    if (redo && headroom > 0) {
        // one pass with the predicted range, then the exact two-pass kernel over the lines it listed
        ensure_smem(stats_i8_op_kernel<0>, kSmemCap - kStaticSmem);
        ensure_smem(stats_i8_op_kernel<108>, kSmemCap - kStaticSmem);
        ensure_smem(stats_i8_kernel<0, true>, kSmemCap - kStaticSmem);
        ensure_smem(stats_i8_kernel<108, true>, kSmemCap - kStaticSmem);
        if (g.B == 108) {
            stats_i8_op_kernel<108><<<grid, kThreads + 64, stats_i8_smem(g), st>>>(a);
            stats_i8_kernel<108, true><<<grid, kThreads + 64, stats_i8_smem(g), st>>>(a);
        } else {
            stats_i8_op_kernel<0><<<grid, kThreads + 64, stats_i8_smem(g), st>>>(a);
            stats_i8_kernel<0, true><<<grid, kThreads + 64, stats_i8_smem(g), st>>>(a);
        }
        const int items = n_lines_total * g.D;
        c0_fold_kernel<<<(items + 255) / 256, 256, 0, st>>>(g.D, g.SE + g.D, n_lines_total, c0, vmax, stats, redo);
        return;
    }
    a.redo = nullptr;
    // ring1 > 0: the range pass on its own warps (stats_i8_ws_kernel) with ring1 pass-1 stages, where
    // the ring holds at least ring1 + 2 (ERX_OPT_STATS_SPLIT); 0: the single-role kernel
    const int ws = (ring1 > 0 && a.stages >= ring1 + 2) ? ring1 : 0;
    a.ring1 = ws;
    if (ws) {  // range pass on its own warps
        ensure_smem(stats_i8_ws_kernel<0>, kSmemCap - kStaticSmem);
        ensure_smem(stats_i8_ws_kernel<108>, kSmemCap - kStaticSmem);
        if (g.B == 108)
            stats_i8_ws_kernel<108><<<grid, kWsThreads, stats_i8_smem(g), st>>>(a);
        else
            stats_i8_ws_kernel<0><<<grid, kWsThreads, stats_i8_smem(g), st>>>(a);
    } else if (g.B == 108)  // configs[0] / configs[3]
        stats_i8_kernel<108><<<grid, kThreads + 64, stats_i8_smem(g), st>>>(a);
    else
        stats_i8_kernel<0><<<grid, kThreads + 64, stats_i8_smem(g), st>>>(a);
    const int items = n_lines_total * g.D;
    c0_fold_kernel<<<(items + 255) / 256, 256, 0, st>>>(g.D, g.SE + g.D, n_lines_total, c0, vmax, stats, nullptr);
}

}  // namespace erxk

#ifdef ERX_X_TRACE
extern "C" int erx_x_trace(unsigned long long* out, int n_pairs) {
    unsigned int cnt = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&cnt, erxk::g_trace_n, sizeof(cnt));
    const int m = int(cnt) < n_pairs ? int(cnt) : n_pairs;
    cudaMemcpyFromSymbol(out, erxk::g_trace, size_t(m) * 2 * sizeof(unsigned long long));
    const unsigned int zero = 0;
    cudaMemcpyToSymbol(erxk::g_trace_n, &zero, sizeof(zero));
    return m;
}
#endif
