// k_factor.cu — per-line factorisation of the pre-update background:
// L = cholesky_lower(K_{t-1} + eps I) (linalg.hpp:12-15) with the eps x10
// escalation up to 1e-1, then W = L^{-1} written as fp32 for
// the whitening multiply of the score kernel.  A failing pivot is reported
// per line (status) and latched for the device-resident path (latch).
//
// Three kernels, one CTA per line (ERX_OPT_FACTOR_PRECISION picks):
//   factor_blk_kernel (32, default while it fits: D <= 233)  fp32, whole
//       matrix in shared memory, 8x8 register-tiled blocked Cholesky and
//       in-place blocked inverse;
//   factor_smem_kernel<double> (64, D <= 165)  fp64 scalar right-looking
//       Cholesky + in-place inverse in shared memory;
//   factor_global_kernel (1, and any D beyond the above)  blocked (panel 32)
//       fp64 over an L2-resident global workspace.
#include <algorithm>
#include <cstdlib>

#ifndef FACTOR_MB128
#define FACTOR_MB128 7  // resident 128-thread lines per SM the register budget allows (A/B: 5, 6)
#endif

#include "tc_common.cuh"

#include "erx_common.cuh"
#include "f64_factor.cuh"
#include "i8_common.cuh"

namespace erxk {
namespace {

// W = L^{-1} leaves the factor kernels as the lower-triangular 8x8 blocks of
// one line, packed in row-major block order (block (I, J), J <= I, at
// tri(I, J)), each block column-major (element (r, c) at c * 8 + r) so the
// score kernel reads row pairs of a column as one float2.  Entries above the
// diagonal or in the padding are zero.
template <typename Get>
__device__ __forceinline__ void write_wblocks(float* __restrict__ whiten, int line, const Geometry& g, Get get) {
    const int nblk = g.nb * (g.nb + 1) / 2;
    float* Wp = whiten + size_t(line) * nblk * 64;
    if (nblk * 64 < 8 * int(blockDim.x)) {  // small matrices: one value per thread and pass
        for (int idx = threadIdx.x; idx < nblk * 64; idx += blockDim.x) {
            const int bq = idx >> 6, e = idx & 63, c = e >> 3, r = e & 7;
            int I = int((sqrtf(8.f * bq + 1.f) - 1.f) * 0.5f);
            while (I * (I + 1) / 2 > bq) --I;
            while ((I + 1) * (I + 2) / 2 <= bq) ++I;
            const int J = bq - I * (I + 1) / 2;
            const int i = I * kBlk + r, j = J * kBlk + c;
            Wp[idx] = (i < g.D && j <= i) ? get(i, j) : 0.f;
        }
        return;
    }
    constexpr int kLB = 4;  // values per thread fetched before the stores (get() may read an L2 workspace)
    for (int i0 = threadIdx.x; i0 < nblk * 64; i0 += kLB * blockDim.x) {
        float v[kLB];
#pragma unroll
        for (int b = 0; b < kLB; ++b) {
            const int idx = min(i0 + b * int(blockDim.x), nblk * 64 - 1);
            const int bq = idx >> 6, e = idx & 63, c = e >> 3, r = e & 7;
            int I = int((sqrtf(8.f * bq + 1.f) - 1.f) * 0.5f);
            while (I * (I + 1) / 2 > bq) --I;
            while ((I + 1) * (I + 2) / 2 <= bq) ++I;
            const int J = bq - I * (I + 1) / 2;
            const int i = I * kBlk + r, j = J * kBlk + c;
            v[b] = (i < g.D && j <= i) ? get(i, j) : 0.f;
        }
#pragma unroll
        for (int b = 0; b < kLB; ++b) {
            const int idx = i0 + b * int(blockDim.x);
            if (idx < nblk * 64) Wp[idx] = v[b];
        }
    }
}

// The tensor path's whitening operand (k_score_i8.cu), written instead of the fp32 blocks.  The
// score multiplies the STATS' quantised v = x - c (per-dim scale s_j = i8::v_scale(vmax_j)), so
//   m_i = sum_j W_ij (v_j - dc_j) = sum_j W'_ij (v_j s_j) - (W dc)_i,  W'_ij = W_ij / s_j,
// dc = mu_{t-1} - c.  Each row of W' is scaled by r_i = R / max_j |W'_ij| and rounded once to three
// int8 digit planes laid out as the score kernel's K-major MMA B operand; the block ends with
// 256 / r_i and (W dc)_i (fp64 sum) per row (i8::kWBytes per line).
template <typename ElPtr>
__device__ void write_wplanes(unsigned char* __restrict__ planes, int line, const Geometry& g, ElPtr el,
                              const double* __restrict__ stats, const double* __restrict__ prior,
                              const float* __restrict__ vmax, float* isc, double* dcs) {
    // isc / dcs: 128 floats / 128 doubles of the caller's shared memory
    const int tid = threadIdx.x, nt = blockDim.x, D = g.D;
    for (int d = tid; d < 128; d += nt) {
        float v = 0.f;
        double dc = 0.0;
        if (d < D) {
            const float s = i8::v_scale(vmax[size_t(line) * D + d]);
            v = s > 0.f ? 1.f / s : 0.f;
            dc = prior[size_t(line) * g.SE + d] - stats[size_t(line) * (g.SE + g.D) + d];
        }
        isc[d] = v;
        dcs[d] = dc;
    }
    __syncthreads();
    unsigned char* out = planes + size_t(line) * i8::kWBytes;
    float* invr = reinterpret_cast<float*>(out + 3 * i8::kWPlane);
    float* wdc = invr + 128;
    for (int i = tid; i < 128; i += nt) {
        float mx = 0.f;
        double cr[4] = {0.0, 0.0, 0.0, 0.0};  // four partial sums: no 108-long dependent DFMA chain
        if (i < D) {
            for (int j0 = 0; j0 <= i; j0 += 4) {  // 4 consecutive j of one block row: 16-byte aligned
                const float4 w4 = *reinterpret_cast<const float4*>(el(i, j0));
                const float w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = j0 + e;
                    const float wv = j <= i ? w[e] : 0.f;
                    mx = fmaxf(mx, fabsf(wv * isc[j]));
                    cr[e] += double(wv) * dcs[j];
                }
            }
        }
        const float r = (mx > 0.f && mx <= 3.402823466e38f) ? i8::kR / mx : 0.f;
        invr[i] = r > 0.f ? 256.f / r : 0.f;
        wdc[i] = float((cr[0] + cr[1]) + (cr[2] + cr[3]));
        const int nrun = i < D ? i / 16 + 1 : 0;  // runs past the diagonal (or padding rows) are all-zero digits
        for (int run = 0; run < 8; ++run) {
            uint32_t w[3][4] = {{0u, 0u, 0u, 0u}, {0u, 0u, 0u, 0u}, {0u, 0u, 0u, 0u}};
            if (run < nrun) {
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const int j0 = run * 16 + q4 * 4;
                    float4 w4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (j0 <= i) w4 = *reinterpret_cast<const float4*>(el(i, j0));
                    const float wr[4] = {w4.x, w4.y, w4.z, w4.w};
                    uint32_t u[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int j = j0 + e;
                        const float wv = j <= i ? wr[e] * isc[j] : 0.f;
                        u[e] = i8::quant_u(wv, r);
                    }
                    i8::pack_digits(u, w[0][q4], w[1][q4], w[2][q4]);
                }
            }
            const uint32_t off = tc::kmajor_off_s8(i, run * 16);
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
                *reinterpret_cast<uint4*>(out + pl * i8::kWPlane + off) = make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]);
        }
    }
}

__global__ void __launch_bounds__(256) factor_global_kernel(Geometry g, const double* __restrict__ prior, double eps0,
                                                     double* __restrict__ work, float* __restrict__ whiten,
                                                     int* __restrict__ status, unsigned long long* __restrict__ latch,
                                                     const WinMeta* __restrict__ meta, long long line_mult,
                                                     long long line_off) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_fail;
    const int line = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int D = g.D, Dp = g.Dp;
    double* A = work + size_t(line) * 2 * Dp * Dp;
    double* X = A + size_t(Dp) * Dp;
    const double* K = prior + size_t(line) * g.SE + D;
    double* Lkk = reinterpret_cast<double*>(smem);
    double* pnl = Lkk + kNB * (kNB + 1);
    double eps = eps0;
    int fail = -1;
    while (true) {
        for (int idx = tid; idx < D * D; idx += nt) {
            int i = idx / D, j = idx - i * D;
            if (j <= i) A[size_t(i) * Dp + j] = K[tri(i, j)] + (i == j ? eps : 0.0);
        }
        __syncthreads();
        fail = chol_blocked(A, D, Dp, Lkk, pnl, &s_fail);
        __syncthreads();
        if (fail < 0) break;
        const double next = eps * 10.0;
        if (!(next <= 1e-1 * (1.0 + 1e-9))) break;
        eps = next;
    }
    if (fail >= 0) {
        if (tid == 0) {
            status[line] = fail;
            if (atomicCAS(latch, 0ull, 1ull) == 0ull) {
                latch[1] = static_cast<unsigned long long>(meta->lines_seen * line_mult + line_off + line);
                latch[2] = static_cast<unsigned long long>(fail);
            }
        }
        return;
    }
    tri_inverse_blocked(A, X, D, Dp, reinterpret_cast<double*>(smem));
    write_wblocks(whiten, line, g, [&](int i, int j) { return float(X[size_t(i) * Dp + j]); });
    if (tid == 0) status[line] = -1;
}

// ---------------------------------------------------------------------------
// factor_big: fp32 blocked Cholesky and triangular inverse for D > 233 (the
// matrix does not fit in shared memory): A and X live in the global (L2)
// workspace, 256 threads per line, panel width 32.  Cholesky step k: the
// diagonal block is factored by one warp with the rows in registers (shuffles
// for the column broadcasts) and inverted by the same warp (Di = L_kk^{-1},
// which is also X's diagonal block); the panel rows become A_ik Di^T, one row
// per thread, kept transposed in shared memory; the trailing update runs 8x8
// register tiles (two 16-byte shared loads per 64 FMAs) with one
// read-modify-write of the tile in L2.  The inverse is right-looking by block
// rows with the same tiles: step k finishes X_kJ = Di T_kJ and pushes
// T_IJ -= L_Ik X_kJ into every block row below.
// ---------------------------------------------------------------------------
constexpr int kBB = 32;
constexpr int kLD = kBB + 1;

__device__ __forceinline__ float rsqrt_nr(float d) {
    float rs = rsqrtf(d);
    return rs * fmaf(-0.5f * d * rs, rs, 1.5f);
}

// Di = Lkk^{-1} for one 32x32 lower block (rows/cols past the block size are identity in Lkk and
// come out identity): lane c computes column c by forward substitution, four partial sums per row
// split the FMA chains.  Entries above the diagonal come out exactly 0.
__device__ __forceinline__ void tri_inv32_warp(const float* __restrict__ Lkk, float* __restrict__ Di, int lane) {
    float col[kBB];
#pragma unroll
    for (int r = 0; r < kBB; ++r) {
        float s[4] = {r == lane ? 1.f : 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int l = 0; l < r; ++l) s[l & 3] = fmaf(-Lkk[r * kLD + l], col[l], s[l & 3]);
        col[r] = ((s[0] + s[1]) + (s[2] + s[3])) / Lkk[r * kLD + r];
    }
#pragma unroll
    for (int r = 0; r < kBB; ++r) Di[r * kLD + lane] = col[r];
}

// Fire-and-forget fp32 adds at L2 (REDG.ADD.F32x4): the trailing updates of factor_big subtract their tile
// from the L2 workspace without reading it first -- each element gets exactly one update per step, from one
// thread, so the result is the plain fp32 subtraction's (denormals flush).  The read-modify-write form left
// two loads in flight per thread and the kernel on the long scoreboard (ncu: 39 % of its stalls).  The
// workspace is then always READ with ld.global.cg (L2): the L1 does not see the reductions.
__device__ __forceinline__ void red_add4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void red_add1(float* p, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}

// C[rows r0.., cols 0..ncol) op= Pt^T Bk over l < 32 as 8x8 register tiles: Pt is [32][LDT]
// (row l holds the 32-column factor block transposed), Bk is [32][ldb] (row l of the right-hand
// block row).  A warp takes 8 row tiles x 4 column tiles: the B reads of a warp are one 128-byte
// wavefront and the A reads two.  init_from: columns >= init_from are written (-acc), the rest
// read-modify-written (-= acc); lower: only entries on or below the diagonal (trailing update).
__device__ __forceinline__ void tile_update(const float* __restrict__ Pt, int LDT, const float* __restrict__ Bk,
                                            int ldb, float* __restrict__ C, int ldc, int nr, int ncol, int init_from,
                                            bool lower, int warp, int lane, int nwarps) {
    const int nR = (nr + 7) / 8, nC = ncol / 8;
    const int wR = (nR + 7) / 8, wC = (nC + 3) / 4;
    for (int wb = warp; wb < wR * wC; wb += nwarps) {
        const int wr = wb / wC, wc = wb - wr * wC;
        const int R = wr * 8 + (lane >> 2), Cc = wc * 4 + (lane & 3);
        if (R >= nR || Cc >= nC || (lower && Cc > R)) continue;
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int jx = 0; jx < 8; ++jx) acc[i][jx] = 0.f;
#pragma unroll 4
        for (int l = 0; l < kBB; ++l) {
            const float4 a0 = *reinterpret_cast<const float4*>(Pt + l * LDT + R * 8);
            const float4 a1 = *reinterpret_cast<const float4*>(Pt + l * LDT + R * 8 + 4);
            const float4 b0 = *reinterpret_cast<const float4*>(Bk + l * ldb + Cc * 8);
            const float4 b1 = *reinterpret_cast<const float4*>(Bk + l * ldb + Cc * 8 + 4);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int jx = 0; jx < 8; ++jx) acc[i][jx] = fmaf(av[i], bv[jx], acc[i][jx]);
        }
        const bool init = Cc * 8 >= init_from;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int ri = R * 8 + i;
            if (ri >= nr) continue;
            float4* crow = reinterpret_cast<float4*>(C + size_t(ri) * ldc + Cc * 8);
            if (lower && Cc == R) {  // diagonal tile: lower triangle only
                float* cr = C + size_t(ri) * ldc + Cc * 8;
#pragma unroll
                for (int jx = 0; jx < 8; ++jx)
                    if (jx <= i) red_add1(cr + jx, -acc[i][jx]);
                continue;
            }
            if (init) {
                crow[0] = make_float4(-acc[i][0], -acc[i][1], -acc[i][2], -acc[i][3]);
                crow[1] = make_float4(-acc[i][4], -acc[i][5], -acc[i][6], -acc[i][7]);
            } else {
                red_add4(reinterpret_cast<float*>(crow), -acc[i][0], -acc[i][1], -acc[i][2], -acc[i][3]);
                red_add4(reinterpret_cast<float*>(crow + 1), -acc[i][4], -acc[i][5], -acc[i][6], -acc[i][7]);
            }
        }
    }
}

// Load the 32-column block of rows r0..r0+nr of M (cols k0..k0+31) transposed into Pt[c][rr]
// (rows up to roundup8(nr) zero-padded).  Lanes take 4 rows x 8 columns: 32-byte row segments
// from L2 and conflict-free shared stores for any LDT = 4 (mod 8).
__device__ __forceinline__ void load_panel_t(float* __restrict__ Pt, int LDT, const float* __restrict__ M, int ldm,
                                             int r0, int k0, int nr, int tid, int nt) {
    const int nr8 = (nr + 7) & ~7;
    constexpr int kLB = 4;  // loads per thread in flight before the shared stores
    for (int i0 = tid; i0 < nr8 * kBB; i0 += kLB * nt) {
        float v[kLB];
#pragma unroll
        for (int b = 0; b < kLB; ++b) {
            const int idx = i0 + b * nt;
            const int q = idx >> 5, ln = idx & 31;
            const int c = (q & 3) * 8 + (ln & 7), rr = (q >> 2) * 4 + (ln >> 3);
            v[b] = (idx < nr8 * kBB && rr < nr) ? __ldcg(M + size_t(r0 + rr) * ldm + k0 + c) : 0.f;
        }
#pragma unroll
        for (int b = 0; b < kLB; ++b) {
            const int idx = i0 + b * nt;
            const int q = idx >> 5, ln = idx & 31;
            const int c = (q & 3) * 8 + (ln & 7), rr = (q >> 2) * 4 + (ln >> 3);
            if (idx < nr8 * kBB) Pt[c * LDT + rr] = v[b];
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(NT) factor_big_kernel(Geometry g, const double* __restrict__ prior, double eps0,
                                                         float* __restrict__ work, float* __restrict__ whiten,
                                                         int* __restrict__ status, int* __restrict__ fixlist,
                                                         bool xk_smem) {
    extern __shared__ __align__(16) float fsm[];
    __shared__ int s_fail;
    const int line = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int D = g.D, Dp = g.Dp;
    const int LDT = Dp + 4;                  // row stride of the transposed panels / staged block rows
    float* A = work + size_t(line) * 2 * Dp * Dp;
    float* X = A + size_t(Dp) * Dp;
    float* Lkk = fsm;                        // [32][33]
    float* Di = Lkk + kBB * kLD;             // [32][33] L_kk^{-1}
    float* Pt = Di + kBB * kLD;              // [32][LDT]: panel / L column block (transposed), T_k staging
    float* Xk = Pt + kBB * LDT;              // [32][LDT]: finished X block row (xk_smem)
    float* dg = Xk + (xk_smem ? kBB * LDT : 0);  // [Dp]: diagonal of K + eps I (the conditioning test)
    const double* K = prior + size_t(line) * g.SE + D;
    const int ntri = D * (D + 1) / 2;
    const double eps = eps0;
    int fail = -1;
    {
        {   // fill the lower triangle (packed fp64 K -> fp32 A), 8 loads in flight per thread
            int i = int((sqrtf(8.f * tid + 1.f) - 1.f) * 0.5f), j;
            while (i * (i + 1) / 2 > tid) --i;
            while ((i + 1) * (i + 2) / 2 <= tid) ++i;
            j = tid - i * (i + 1) / 2;
            for (int idx = tid; idx < ntri; idx += 8 * nt) {
                double kv[8];
                int iu[8], ju[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    iu[u] = i;
                    ju[u] = j;
                    kv[u] = idx + u * nt < ntri ? __ldg(K + idx + u * nt) : 0.0;
                    j += nt;
                    while (j > i) {
                        j -= i + 1;
                        ++i;
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (idx + u * nt < ntri) {
                        const float v = float(kv[u] + (iu[u] == ju[u] ? eps : 0.0));
                        A[size_t(iu[u]) * Dp + ju[u]] = v;
                        if (iu[u] == ju[u]) dg[iu[u]] = v;
                    }
            }
        }
        __syncthreads();
        fail = -1;
        for (int k0 = 0; k0 < D; k0 += kBB) {
            const int kb = min(kBB, D - k0);
            for (int idx = tid; idx < kBB * kBB; idx += nt) {
                const int r = idx >> 5, c = idx & 31;
                Lkk[r * kLD + c] = r < kb ? (c <= r ? __ldcg(A + size_t(k0 + r) * Dp + k0 + c) : 0.f) : (r == c ? 1.f : 0.f);
            }
            if (tid == 0) s_fail = -1;
            __syncthreads();
            if (warp == 0) {
                // lane r holds row r; column j: broadcast the diagonal, scale the column, then update
                // the trailing entries of every row with the column's values from their lanes
                float row[kBB];
#pragma unroll
                for (int c = 0; c < kBB; ++c) row[c] = Lkk[lane * kLD + c];
                int f = -1;
#pragma unroll
                for (int jj = 0; jj < kBB; ++jj) {
                    if (jj < kb && f < 0) {
                        const float d = __shfl_sync(0xffffffffu, row[jj], jj);
                        if (!(d > 0.f) || d * kCondTau < dg[k0 + jj]) {  // failed or ill-conditioned: fp64
                            f = k0 + jj;
                        } else {
                            const float rs = rsqrt_nr(d);
                            if (lane == jj) {
                                row[jj] = d * rs;
                            } else if (lane > jj) {
                                row[jj] *= rs;
                            }
#pragma unroll
                            for (int c = jj + 1; c < kBB; ++c) {
                                const float lcj = __shfl_sync(0xffffffffu, row[jj], c);
                                if (lane >= c) row[c] = fmaf(-row[jj], lcj, row[c]);
                            }
                        }
                    }
                }
                if (lane == 0) s_fail = f;
                if (f < 0) {  // f is warp-uniform (the pivot is broadcast)
                    if (lane < kb) {
#pragma unroll
                        for (int c = 0; c < kBB; ++c) {
                            const float v = c <= lane ? row[c] : 0.f;
                            Lkk[lane * kLD + c] = v;
                            if (c <= lane) A[size_t(k0 + lane) * Dp + k0 + c] = v;
                        }
                    }
                    __syncwarp();
                    tri_inv32_warp(Lkk, Di, lane);
                    __syncwarp();
                    if (lane < kb)  // X_kk = Di (zeros above the diagonal)
                        for (int r = 0; r < kb; ++r) X[size_t(k0 + r) * Dp + k0 + lane] = Di[r * kLD + lane];
                }
            }
            __syncthreads();
            fail = s_fail;
            if (fail >= 0) break;
            // panel: L_ik = A_ik L_kk^{-T} = A_ik Di^T, one row per thread, kept transposed in shared memory
            const int r0 = k0 + kb, nr = D - r0;  // nr > 0 implies kb == 32
            for (int rr = tid; rr < nr; rr += nt) {
                float4* arow = reinterpret_cast<float4*>(A + size_t(r0 + rr) * Dp + k0);
                float av[kBB], x[kBB];
#pragma unroll
                for (int q = 0; q < kBB / 4; ++q) {
                    const float4 v = __ldcg(arow + q);
                    av[4 * q] = v.x, av[4 * q + 1] = v.y, av[4 * q + 2] = v.z, av[4 * q + 3] = v.w;
                }
#pragma unroll
                for (int c = 0; c < kBB; ++c) {
                    float s0 = 0.f, s1 = 0.f;
#pragma unroll
                    for (int l = 0; l <= c; ++l) {
                        if (l & 1) s1 = fmaf(av[l], Di[c * kLD + l], s1);
                        else s0 = fmaf(av[l], Di[c * kLD + l], s0);
                    }
                    x[c] = s0 + s1;
                    Pt[c * LDT + rr] = x[c];
                }
#pragma unroll
                for (int q = 0; q < kBB / 4; ++q) arow[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
            }
            // zero the transposed panel's padding rows so 8-row tiles read zeros
            for (int idx = tid; idx < kBB * 8; idx += nt) Pt[(idx >> 3) * LDT + nr + (idx & 7)] = 0.f;
            __syncthreads();
            // trailing update A22 -= P P^T over the lower triangle
            if (nr > 0)
                tile_update(Pt, LDT, Pt, LDT, A + size_t(r0) * Dp + r0, Dp, nr, (nr + 7) & ~7, 1 << 30, true, warp,
                            lane, nw);
            __syncthreads();
        }
    }
    if (fail >= 0) {  // the fp64 rescue (k_fixup.cu) redoes this line, escalation included
        if (tid == 0) list_for_fixup(fixlist, status, line);
        return;
    }
    // X = L^{-1}, right-looking by block rows.  Before step k, X's block row k holds
    // T_kJ = -sum_{m<k} L_km X_mJ (J < k) and X_kk = Di (written by the factor); step k finishes
    // X_kJ = Di T_kJ and pushes T_IJ -= L_Ik X_kJ into every block row I > k.
    for (int k0 = 0; k0 < D; k0 += kBB) {
        const int kb = min(kBB, D - k0), r0 = k0 + kb, nr = D - r0;
        __syncthreads();
        for (int idx = tid; idx < kBB * kBB; idx += nt) {
            const int r = idx >> 5, c = idx & 31;
            Di[r * kLD + c] = (r < kb && c < kb) ? __ldcg(X + size_t(k0 + r) * Dp + k0 + c) : 0.f;
        }
        for (int r = warp; r < kBB; r += nw)
            for (int j = lane; j < k0; j += 32) Pt[r * LDT + j] = r < kb ? __ldcg(X + size_t(k0 + r) * Dp + j) : 0.f;
        __syncthreads();
        float* xk = xk_smem ? Xk : X + size_t(k0) * Dp;
        const int ldx = xk_smem ? LDT : Dp;
        for (int j = tid; j < k0; j += nt) {  // X_kJ = Di T_kJ, one column per thread
            float t[kBB];
#pragma unroll
            for (int l = 0; l < kBB; ++l) t[l] = Pt[l * LDT + j];
#pragma unroll
            for (int r = 0; r < kBB; ++r) {
                float s0 = 0.f, s1 = 0.f;
#pragma unroll
                for (int l = 0; l <= r; ++l) {
                    if (l & 1) s1 = fmaf(Di[r * kLD + l], t[l], s1);
                    else s0 = fmaf(Di[r * kLD + l], t[l], s0);
                }
                if (r < kb) {
                    if (xk_smem) Xk[r * LDT + j] = s0 + s1;
                    X[size_t(k0 + r) * Dp + j] = s0 + s1;
                }
            }
        }
        if (xk_smem)
            for (int idx = tid; idx < kBB * kBB; idx += nt) {
                const int r = idx >> 5, c = idx & 31;
                Xk[r * LDT + k0 + c] = Di[r * kLD + c];
            }
        if (nr > 0) {
            __syncthreads();  // T_k staging read out of Pt
            load_panel_t(Pt, LDT, A, Dp, r0, k0, nr, tid, nt);
            __syncthreads();
            tile_update(Pt, LDT, xk, ldx, X + size_t(r0) * Dp, Dp, nr, k0 + kb, k0, false, warp, lane, nw);
        }
    }
    __syncthreads();
    write_wblocks(whiten, line, g, [&](int i, int j) { return __ldcg(X + size_t(i) * Dp + j); });
    if (tid == 0) status[line] = -1;
}

// ---------------------------------------------------------------------------
// shared-memory resident factorisation (D <= 233)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) factor_smem_kernel(Geometry g, const double* __restrict__ prior, double eps0,
                                                          float* __restrict__ whiten, int* __restrict__ status,
                                                          unsigned long long* __restrict__ latch,
                                                          const WinMeta* __restrict__ meta, long long line_mult,
                                                          long long line_off) {
    extern __shared__ __align__(16) unsigned char smem[];
    T* A = reinterpret_cast<T*>(smem);
    const int D = g.D, LD = D + 1;  // odd leading dimension: conflict-free column walks
    const int line = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const double* K = prior + size_t(line) * g.SE + D;
    double eps = eps0;
    int fail;
    while (true) {
        for (int i = warp; i < D; i += nw)
            for (int j = lane; j <= i; j += 32) A[i * LD + j] = T(K[tri(i, j)] + (i == j ? eps : 0.0));
        __syncthreads();
        fail = -1;
        for (int j = 0; j < D; ++j) {
            const T djj = A[j * LD + j];
            if (!(djj > T(0))) {  // uniform: every thread read the same value after the last barrier
                fail = j;
                break;
            }
            const T s = sqrt(djj);
            for (int i = j + 1 + tid; i < D; i += nt) A[i * LD + j] /= s;
            __syncthreads();
            if (tid == 0) A[j * LD + j] = s;
            for (int i = j + 1 + warp; i < D; i += nw) {
                const T lij = A[i * LD + j];
                for (int k = j + 1 + lane; k <= i; k += 32) A[i * LD + k] -= lij * A[k * LD + j];
            }
            __syncthreads();
        }
        if (fail < 0) break;
        const double next = eps * 10.0;
        if (!(next <= 1e-1 * (1.0 + 1e-9))) break;
        eps = next;
        __syncthreads();
    }
    if (fail >= 0) {
        if (tid == 0) {
            status[line] = fail;
            if (atomicCAS(latch, 0ull, 1ull) == 0ull) {
                latch[1] = static_cast<unsigned long long>(meta->lines_seen * line_mult + line_off + line);
                latch[2] = static_cast<unsigned long long>(fail);
            }
        }
        return;
    }
    // In-place inverse, right-looking by rows: before step k, row i > k holds
    // T_ic = -sum_{m<k} L_im X_mc in columns c < k and L_ic in columns >= k.
    for (int k = 0; k < D; ++k) {
        const T lkk = A[k * LD + k];
        __syncthreads();
        const T inv = T(1) / lkk;
        for (int c = tid; c < k; c += nt) A[k * LD + c] *= inv;
        if (tid == 0) A[k * LD + k] = inv;
        __syncthreads();
        for (int i = k + 1 + warp; i < D; i += nw) {
            const T l = A[i * LD + k];
            __syncwarp();
            for (int c = lane; c <= k; c += 32) {
                if (c == k)
                    A[i * LD + k] = -l * A[k * LD + k];
                else
                    A[i * LD + c] -= l * A[k * LD + c];
            }
        }
        __syncthreads();
    }
    write_wblocks(whiten, line, g, [&](int i, int j) { return float(A[i * LD + j]); });
    if (tid == 0) status[line] = -1;
}

// ---------------------------------------------------------------------------
// fp32 blocked factorisation in shared memory (default for D <= 233): the
// same 8x8 block grid as the stats / score kernels, Cholesky and inverse
// merged into ONE right-looking sweep over the block columns (two barriers
// per step).  Step k, with L_kk's inverse Di already in block (k, k):
//   (b) panel rows: L_Ik = A_Ik Di^T (kept in Lc), and block (I, k) becomes
//       T_Ik = -L_Ik Di; row finalisation: X_kJ = Di T_kJ (J < k);
//   (c) Cholesky trailing update A_IJ -= L_Ik L_Jk^T (k < J <= I) and inverse
//       update T_IJ -= L_Ik X_kJ (J < k), one block row per thread, four
//       blocks of one block column per warp; the eight
//       lanes that finish block (k+1, k+1) factor and invert it in registers
//       (8-wide shuffles) for the next step.
// At the end every block (I, J) holds X_IJ, X = L^{-1}.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ld8(const float* p, float* v) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
constexpr int kLcLd = 72;  // panel block stride (floats): rows of blocks J and J + 1..3 on different banks
// Element (r, c) of a shared-memory 8x8 block lives at r * 8 + (c ^ (r & 4)): rows 4-7 keep their two
// 16-byte halves swapped, so the eight threads of a group reading eight different rows of one block
// touch 32 distinct banks (the plain row-major layout puts rows r and r + 4 on the same banks).
// Aligned groups of 4 columns stay contiguous (float4 reads of the plane writer are unaffected).
__device__ __forceinline__ int swz(int r, int c) { return r * kBlk + (c ^ (r & 4)); }
__device__ __forceinline__ void ld8r(const float* blk, int r, float* v) {  // row r, logical column order
    const float* p = blk + r * kBlk;
    const int h = r & 4;
    const float4 a = *reinterpret_cast<const float4*>(p + h);
    const float4 b = *reinterpret_cast<const float4*>(p + (h ^ 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8r(float* blk, int r, const float* v) {
    float* p = blk + r * kBlk;
    const int h = r & 4;
    *reinterpret_cast<float4*>(p + h) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + (h ^ 4)) = make_float4(v[4], v[5], v[6], v[7]);
}

// acc[c] -= sum_l a[l] b[l] for one row c of the right operand, as paired FMAs (FFMA2) over l:
// four fma.rn.f32x2 on (a[2i], a[2i+1]) and the row's (b[2i], b[2i+1]), then one add of the halves.
__device__ __forceinline__ float dot8_sub(const float2 (&na)[4], const float (&b)[kBlk], float acc) {
    float2 p = make_float2(acc, 0.f);
#pragma unroll
    for (int i = 0; i < 4; ++i) p = __ffma2_rn(na[i], make_float2(b[2 * i], b[2 * i + 1]), p);
    return p.x + p.y;
}
__device__ __forceinline__ void neg_pairs(const float (&a)[kBlk], float2 (&na)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) na[i] = make_float2(-a[2 * i], -a[2 * i + 1]);
}

// Eight lanes (one aligned 8-lane group, lane gl holding row gl of an updated diagonal block in
// row[]) factor the block (Cholesky, 1/sqrt from MUFU.RSQ + one Newton step) and invert the
// factor (lane c: column c by forward substitution); the columns of L are exchanged through dit
// (0.174 -> 0.170 ms per 2048 lines against a shuffle per entry).  Di goes to blk (swizzled rows, zeros above the
// diagonal), Di^T to dit (plain rows).  Returns the first pivot (k0 + j) that is non-positive or below
// dg / kCondTau (dg: the diagonal of K + eps I), or -1, group-uniform.
__device__ __forceinline__ int diag_factor8(float (&row)[kBlk], unsigned gmask, int gl, int k0, float* blk,
                                            float* dit, const float* dg) {
    int f = -1;
    float rd[kBlk];
    // the block's conditioning bounds up front (a shared-memory load behind each column's dit store would sit
    // on the pivot chain)
    float dgr[kBlk];
    ld8(dg + k0, dgr);
    // the columns of L go through dit (free until Di^T is written at the end): one 4-byte store per
    // lane and two 16-byte broadcast loads per column instead of a shuffle per entry; the pivot chain
    // itself stays in registers (lane j + 1 updates its own next pivot)
#pragma unroll
    for (int j = 0; j < kBlk; ++j) {
        float d = __shfl_sync(gmask, row[j], j, kBlk);
        if (!(d > 0.f) || d * kCondTau < dgr[j]) {
            if (f < 0) f = k0 + j;
            d = 1.f;
        }
        const float rs = rsqrt_nr(d);
        rd[j] = rs;
        if (gl == j) row[j] = d * rs;
        else if (gl > j) row[j] *= rs;
        dit[j * kBlk + gl] = row[j];
        __syncwarp(gmask);
        float lc[kBlk];
        ld8(dit + j * kBlk, lc);  // L[0..7][j]
#pragma unroll
        for (int c = j + 1; c < kBlk; ++c)
            if (gl >= c) row[c] = fmaf(-row[j], lc[c], row[c]);
    }
    float col[kBlk];
#pragma unroll
    for (int r = 0; r < kBlk; ++r) col[r] = 0.f;
    // forward substitution for column gl of L^{-1}, by columns of L (dit holds L column-major)
#pragma unroll
    for (int l = 0; l < kBlk; ++l) {
        float lc[kBlk];
        ld8(dit + l * kBlk, lc);
        col[l] = ((l == gl ? 1.f : 0.f) + col[l]) * rd[l];
#pragma unroll
        for (int r = l + 1; r < kBlk; ++r) col[r] = fmaf(-lc[r], col[l], col[r]);
    }
    __syncwarp(gmask);  // every lane's reads of L precede the Di^T stores over it
#pragma unroll
    for (int r = 0; r < kBlk; ++r) blk[swz(r, gl)] = col[r];
    st8(dit + gl * kBlk, col);
    return f;
}

#ifdef ERX_X_TRACE  // A/B timeline instrumentation of one CTA (tools/factor_trace.py)
__device__ unsigned long long g_ftrace[1 << 14];
__device__ unsigned int g_ftrace_n;
__device__ __forceinline__ void ftrace(int id, int k, int t) {
    if (blockIdx.x == 1000) {
        const unsigned i = atomicAdd(&g_ftrace_n, 1u);
        if (i < (1u << 13)) {
            g_ftrace[2 * i] = clock64();
            g_ftrace[2 * i + 1] = (unsigned long long)((id << 24) | (k << 12) | t);
        }
    }
}
#define FTR(id, k, t) ftrace(id, k, t)
#else
#define FTR(id, k, t)
#endif

// fp32 blocked factor, one CTA of NT threads per line.  The minimum-blocks bound keeps
// 64- and 128-thread CTAs at <= 72 registers so the seven lines that fit shared memory (configs[3]) are
// all resident.
template <int NT, int MB>
__global__ void __launch_bounds__(NT, MB) factor_blk_kernel(Geometry g, const double* __restrict__ prior,
                                                                          double eps0, float* __restrict__ whiten,
                                                                          int* __restrict__ status,
                                                                          int* __restrict__ fixlist,
                                                                          const double* __restrict__ stats,
                                                                          const float* __restrict__ vmax,
                                                                          const float* __restrict__ kblk) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_fail;
    const int D = g.D, Dp = g.Dp, nb = g.nb;
    // packed lower 8x8 blocks, swizzled rows (swz): block (I, J) at tri(I, J) * 64; padding dims carry
    // an identity block
    float* A = reinterpret_cast<float*>(smem);
    auto BP = [&](int I, int J) { return A + (I * (I + 1) / 2 + J) * 64; };
    auto EL = [&](int i, int j) { return BP(i >> 3, j >> 3) + swz(i & 7, j & 7); };
    float* Lc = A + size_t(nb * (nb + 1) / 2) * 64;  // [nb][kLcLd]: the current panel L_Ik (swizzled rows)
    float* DiT = Lc + size_t(nb) * kLcLd;       // [64]: Di^T of the current diagonal block (plain rows)
    // [Dp]: diagonal of K + eps I for the conditioning test (past the plane writer's scratch, which reuses
    // Lc + DiT after the factorisation)
    float* dg = Lc + (size_t(nb) * kLcLd + 64 > 384 ? size_t(nb) * kLcLd + 64 : 384);
    const int line = blockIdx.x, tid = threadIdx.x;
    constexpr int nt = NT;
    const int lane = tid & 31, gl = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const double* K = prior + size_t(line) * g.SE + D;
    const double eps = eps0;
    int fail;
    const int ntri = D * (D + 1) / 2;
    FTR(9, 0, tid);
    {
        if (tid == 0) s_fail = -1;
        if (kblk) {
            // fill from the scan's fp32 block image (same swizzled layout): a straight 16-byte copy,
            // then + eps on the diagonal and zeros above it inside the diagonal blocks
            const int nfl = nb * (nb + 1) / 2 * 64;
            const float4* src = reinterpret_cast<const float4*>(kblk + size_t(line) * nfl);
            for (int q = tid; q < nfl / 4; q += nt) cp_async16(A + 4 * q, src + q);
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
            const float fe = float(eps);
            for (int q = tid; q < nb * 64; q += nt) {
                const int kk = q >> 6, r = (q >> 3) & 7, c = q & 7;
                float* p = BP(kk, kk) + swz(r, c);
                if (c > r) {
                    *p = 0.f;
                } else if (c == r && kk * kBlk + r < D) {
                    *p += fe;
                    dg[kk * kBlk + r] = *p;
                }
            }
        } else {
            // fill: coalesced reads of the packed fp64 K, 1024 loads in flight per line (the (i, j) of
            // idx + nt follows from (i, j) of idx incrementally)
            constexpr int kFill = 1024 / NT;
            int i = int((sqrtf(8.f * tid + 1.f) - 1.f) * 0.5f), j;
            while (i * (i + 1) / 2 > tid) --i;
            while ((i + 1) * (i + 2) / 2 <= tid) ++i;
            j = tid - i * (i + 1) / 2;
            for (int base = tid; base < ntri; base += kFill * nt) {
                double v[kFill];
                int ii[kFill], jj[kFill];
#pragma unroll
                for (int u = 0; u < kFill; ++u) {
                    const int idx = base + u * nt;
                    v[u] = idx < ntri ? __ldg(K + idx) : 0.0;
                    ii[u] = i;
                    jj[u] = j;
                    j += nt;  // advance (i, j) by nt packed positions
                    while (j > i) {
                        j -= i + 1;
                        ++i;
                    }
                }
#pragma unroll
                for (int u = 0; u < kFill; ++u)
                    if (base + u * nt < ntri) {
                        const float fv = float(v[u] + (ii[u] == jj[u] ? eps : 0.0));
                        *EL(ii[u], jj[u]) = fv;
                        if (ii[u] == jj[u]) dg[ii[u]] = fv;
                    }
            }
        }
        __syncthreads();
        for (int i = D + tid; i < Dp; i += nt) {  // padding dims: identity
            for (int j = 0; j <= i; ++j) *EL(i, j) = (i == j) ? 1.f : 0.f;
            dg[i] = 1.f;
        }
        __syncthreads();
        if (tid < kBlk) {  // block (0, 0)
            float row[kBlk];
            ld8r(BP(0, 0), gl, row);
            const int f = diag_factor8(row, gmask, gl, 0, BP(0, 0), DiT, dg);
            if (gl == 0 && f >= 0) s_fail = f;
        }
        __syncthreads();
        fail = s_fail;
        FTR(0, 0, tid);
        for (int k = 0; k < nb && fail < 0; ++k) {
            FTR(1, k, tid);
            const float* Di = BP(k, k);
            // (b) panel rows I > k (tasks 0 ..) and finalisation of block row k (J < k); Di and Di^T rows
            // are broadcasts
            const int npan = (nb - k - 1) * kBlk;
            for (int q = tid; q < npan + k * kBlk; q += nt) {
                const int r = q & 7;
                if (q < npan) {
                    const int I = k + 1 + (q >> 3);
                    float* blk = BP(I, k);
                    float a[kBlk], x[kBlk], t[kBlk];
                    ld8r(blk, r, a);
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) {
                        float d[kBlk];
                        ld8r(Di, c, d);
                        float s = 0.f;
#pragma unroll
                        for (int l = 0; l <= c; ++l) s = fmaf(a[l], d[l], s);
                        x[c] = s;
                    }
                    st8r(Lc + I * kLcLd, r, x);
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) {
                        float d[kBlk];
                        ld8(DiT + c * kBlk, d);
                        float s = 0.f;
#pragma unroll
                        for (int l = c; l < kBlk; ++l) s = fmaf(x[l], d[l], s);
                        t[c] = -s;
                    }
                    st8r(blk, r, t);
                } else {
                    const int J = (q - npan) >> 3;
                    float* blk = BP(k, J);
                    float acc[kBlk], d[kBlk];
                    ld8r(Di, r, d);
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) acc[c] = 0.f;
#pragma unroll
                    for (int l = 0; l < kBlk; ++l) {
                        float tr[kBlk];
                        ld8r(blk, l, tr);  // broadcast across the group
#pragma unroll
                        for (int c = 0; c < kBlk; ++c) acc[c] = fmaf(d[l], tr[c], acc[c]);  // d[l] = 0 for l > r
                    }
                    __syncwarp(gmask);  // the group's reads of T_kJ precede its writes
                    st8r(blk, r, acc);
                }
            }
            FTR(2, k, tid);
            __syncthreads();
            FTR(3, k, tid);
            // (c) trailing Cholesky update A_IJ -= L_Ik L_Jk^T (I >= J > k), then inverse update
            // T_IJ -= L_Ik X_kJ (I > k, J < k).  Task = (block pair, row r = tid % 8); pairs run
            // column-major (stride nt / 8, decoded incrementally), so the four lane groups of a warp
            // mostly share J and the 16 right-operand row loads are one address per warp (Lc rows
            // of neighbouring J sit on different banks: stride kLcLd)
            // Warp 0 owns pair 0 (block (k+1, k+1): update, then the 8-lane factor + inverse for the next
            // step) and nothing else: its other lanes would wait out that divergent, shuffle-bound chain
            // (measured ~6k cycles) before their own tasks and hold the step's barrier (the timeline in
            // tools/factor_trace.py); the other warps take the remaining pairs with stride (nt - 32) / 8.
            {
                constexpr int step = (nt - 32) / kBlk;
                const int r = gl;
                const int m = nb - k - 1;
                float a[kBlk], acc[kBlk];
                const bool dwarp = tid < 32;
                // trailing pair: column jr, row ir (relative to k + 1), ir >= jr; flat index 0 is pair 0
                int jr = 0, ir = dwarp ? 0 : (tid >> 3) - 3;
                if (tid < kBlk && m > 0) {
                    // pair 0 = block (k+1, k+1) first, outside the loop (keeps the loop's registers low):
                    // update, then factor + invert it for the next step
                    float* blk = BP(k + 1, k + 1);
                    const float* bj = Lc + (k + 1) * kLcLd;
                    ld8r(bj, r, a);
                    ld8r(blk, r, acc);
                    float2 na[4];
                    neg_pairs(a, na);
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) {
                        float b[kBlk];
                        ld8r(bj, c, b);
                        acc[c] = dot8_sub(na, b, acc[c]);
                    }
                    st8r(blk, r, acc);
                    FTR(5, k, tid);
                    const int f = diag_factor8(acc, gmask, gl, (k + 1) * kBlk, blk, DiT, dg);
                    FTR(6, k, tid);
                    if (gl == 0 && f >= 0) s_fail = f;
                }
                if (dwarp) jr = m;  // no trailing / inverse pairs for warp 0
                while (ir >= m && jr < m) {
                    ir = ir - m + jr + 1;
                    ++jr;
                }
                for (; jr < m;) {
                    const int I = k + 1 + ir, J = k + 1 + jr;
                    float* blk = BP(I, J);
                    const float* bj = Lc + J * kLcLd;
                    ld8r(Lc + I * kLcLd, r, a);
                    ld8r(blk, r, acc);
                    float2 na[4];
                    neg_pairs(a, na);
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) {
                        float b[kBlk];
                        ld8r(bj, c, b);
                        acc[c] = dot8_sub(na, b, acc[c]);
                    }
                    st8r(blk, r, acc);
                    ir += step;
                    while (ir >= m && jr < m) {
                        ir = ir - m + jr + 1;
                        ++jr;
                    }
                }
                // inverse pairs: the flat index continues past the m (m + 1) / 2 trailing pairs
                if (k > 0 && m > 0 && !dwarp) {
                    int J;
                    // ir - m + jr + 1 overshoots as if column m had rows from m: rebase to the inverse range
                    ir = ir - jr;  // == flat index past the trailing pairs (jr == m here)
                    J = ir / m;
                    ir -= J * m;
                    for (; J < k;) {
                        const int I = k + 1 + ir;
                        float* blk = BP(I, J);
                        const float* xk = BP(k, J);
                        ld8r(Lc + I * kLcLd, r, a);
                        float2 acc2[4];
                        {
                            float t8[kBlk];
                            ld8r(blk, r, t8);
#pragma unroll
                            for (int i = 0; i < 4; ++i) acc2[i] = make_float2(t8[2 * i], t8[2 * i + 1]);
                        }
                        // acc[c] -= a[l] X_kJ[l][c]: paired FMAs over column pairs (c, c + 1)
#pragma unroll
                        for (int l = 0; l < kBlk; ++l) {
                            float xr[kBlk];
                            ld8r(xk, l, xr);
                            const float2 nal = make_float2(-a[l], -a[l]);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                acc2[i] = __ffma2_rn(nal, make_float2(xr[2 * i], xr[2 * i + 1]), acc2[i]);
                        }
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            acc[2 * i] = acc2[i].x;
                            acc[2 * i + 1] = acc2[i].y;
                        }
                        st8r(blk, r, acc);
                        ir += step;
                        while (ir >= m) {
                            ir -= m;
                            ++J;
                        }
                    }
                }
            }
            FTR(4, k, tid);
            __syncthreads();
            fail = s_fail;
        }
    }
    FTR(7, 0, tid);
    if (fail >= 0) {  // the fp64 rescue (k_fixup.cu) redoes this line, escalation included
        if (tid == 0) list_for_fixup(fixlist, status, line);
        return;
    }
    if (vmax) {
        write_wplanes(reinterpret_cast<unsigned char*>(whiten), line, g, [&](int i, int j) { return EL(i, j); }, stats,
                      prior, vmax, Lc, reinterpret_cast<double*>(Lc + 128));
    } else {
        write_wblocks(whiten, line, g, [&](int i, int j) { return *EL(i, j); });
    }
    FTR(8, 0, tid);
    if (tid == 0) status[line] = -1;
}

// ---------------------------------------------------------------------------
// D <= 8 (the reference default d = 5): the whole matrix is ONE 8x8 block, so diag_factor8 is the whole
// factorisation.  factor_blk spends a 128-thread CTA, two CTA barriers and a block-grid walk per line on it
// (configs[3] d = 5: 0.029 ms per 8192 lines, 0.009 ms of a 0.033-ms lag-0 line); here sixteen lines share a
// CTA, eight lanes each, no CTA barrier.  Same arithmetic in the same order as factor_blk (bit-identical W).
// ---------------------------------------------------------------------------
constexpr int kTinyLines = 16;
__global__ void __launch_bounds__(kTinyLines * 8) factor_tiny_kernel(Geometry g, double eps0, float* __restrict__ whiten,
                                                                    int* __restrict__ status, int* __restrict__ fixlist,
                                                                    const float* __restrict__ kblk, int n_lines) {
    __shared__ __align__(16) float blk_s[kTinyLines][64], dit_s[kTinyLines][64], dg_s[kTinyLines][kBlk];
    const int tid = threadIdx.x, grp = tid >> 3, gl = tid & 7, lane = tid & 31;
    const unsigned gmask = 0xffu << (lane & 24);
    const int line = blockIdx.x * kTinyLines + grp;
    if (line >= n_lines) return;  // (whole 8-lane groups leave together; only group-wide syncs below)
    const int D = g.D;
    float row[kBlk];
    ld8r(kblk + size_t(line) * 64, gl, row);  // the scan's fp32 block image (swizzled rows), row gl
    const float fe = float(eps0);
    float dgv = 1.f;
#pragma unroll
    for (int c = 0; c < kBlk; ++c) {
        if (gl >= D) row[c] = (c == gl) ? 1.f : 0.f;  // padding dims: identity
        else if (c > gl) row[c] = 0.f;
        else if (c == gl) {
            row[c] += fe;
            dgv = row[c];
        }
    }
    dg_s[grp][gl] = dgv;
    __syncwarp(gmask);
    const int f = diag_factor8(row, gmask, gl, 0, blk_s[grp], dit_s[grp], dg_s[grp]);
    if (f >= 0) {  // the fp64 rescue (k_fixup.cu) redoes this line, escalation included
        if (gl == 0) list_for_fixup(fixlist, status, line);
        return;
    }
    __syncwarp(gmask);
    // dit holds Di^T in plain rows: dit[c * 8 + r] = Di[r][c], the W block's own column-major layout
    float w[kBlk];
    ld8(dit_s[grp] + gl * kBlk, w);
#pragma unroll
    for (int r = 0; r < kBlk; ++r) w[r] = (r < D && gl <= r) ? w[r] : 0.f;
    st8(whiten + size_t(line) * 64 + gl * kBlk, w);
    if (gl == 0) status[line] = -1;
}

// ---------------------------------------------------------------------------
// factor_cl (fp32, default for D > 233: configs[4]'s 448 bands): factor_blk's merged Cholesky +
// inverse sweep over a THREAD-BLOCK CLUSTER of CL CTAs (one SM each), the packed lower 8x8 blocks
// distributed block-row-cyclically (CTA c owns block rows I = c mod CL) so the whole factor lives in
// the cluster's shared memory (448 bands: 402 KB over 4 x ~100 KB) instead of an L2 workspace.
// Step k, two cluster barriers (barrier.cluster):
//   1  owners of block rows I > k form the panel L_Ik = A_Ik Di^T and push it into EVERY CTA's
//      panel buffer Lc (st.shared::cluster to mapa-translated addresses), keeping T_Ik = -L_Ik Di;
//      the owner of block row k finalises X_kJ = Di T_kJ (J < k) and pushes it to every CTA's Xr;
//   2  every CTA updates its own block rows from its local copies: A_IJ -= L_Ik L_Jk^T (J > k) and
//      T_IJ -= L_Ik X_kJ (J < k); the owner of block row k + 1 updates the diagonal block first,
//      factors and inverts it (8 lanes, shuffles, the conditioning test) and pushes Di / Di^T and a
//      failure flag to every CTA for step k + 1.
// Lines that fail or are ill-conditioned go to the fp64 rescue like factor_blk's.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cl_map(const void* local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tc::smem_u32(local)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_st4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void cl_st1i(uint32_t addr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// row r of a swizzled 8x8 block at `blk` (logical column order v) into the same block of every CTA
template <int CL>
__device__ __forceinline__ void cl_st8r_all(float* blk, int r, const float* v) {
    float* p = blk + r * kBlk;
    const int h = r & 4;
#pragma unroll
    for (int q = 0; q < CL; ++q) {
        cl_st4(cl_map(p + h, q), v[0], v[1], v[2], v[3]);
        cl_st4(cl_map(p + (h ^ 4), q), v[4], v[5], v[6], v[7]);
    }
}
template <int CL>
__device__ __forceinline__ void cl_st8_all(float* row, const float* v) {  // plain 8-float row
#pragma unroll
    for (int q = 0; q < CL; ++q) {
        cl_st4(cl_map(row, q), v[0], v[1], v[2], v[3]);
        cl_st4(cl_map(row + 4, q), v[4], v[5], v[6], v[7]);
    }
}

constexpr int kCb = 68;  // factor_cl block stride (floats): consecutive blocks on distinct banks



template <int CL>
__global__ void __launch_bounds__(256, 1) factor_cl_kernel(Geometry g, const double* __restrict__ prior, double eps0,
                                                            float* __restrict__ whiten, int* __restrict__ status,
                                                            int* __restrict__ fixlist) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_fail;
    constexpr int NT = 256;
    const int D = g.D, Dp = g.Dp, nb = g.nb;
    const int c = int(cl_rank());
    const int line = blockIdx.x / CL, tid = threadIdx.x;
    const int lane = tid & 31, gl = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const int nown = (nb - c + CL - 1) / CL;  // block rows owned by this CTA
    // the buffers other CTAs write into sit at the same offset in every CTA (mapa keeps the offset)
    // blocks are kCb = 68 floats apart: a warp's threads working on consecutive blocks (one 8x8 task
    // each) then hit 32 distinct banks per 16-byte load instead of all the same four
    float* LcT = reinterpret_cast<float*>(smem);  // [nb][8 cols l][8 rows r]: the step's panel, transposed
    float* Xr = LcT + size_t(nb) * kCb;           // [nb] X_kJ of the step's block row (swizzled rows)
    float* DiS = Xr + size_t(nb) * kCb;           // [64] Di (swizzled rows)
    float* DiT = DiS + 64;                        // [64] Di^T (plain rows)
    float* dg = DiT + 64;                         // [Dp] diagonal of K + eps I
    float* A = dg + Dp;                           // owned block rows, packed (per CTA)
    auto LB = [&](int I, int J) {  // owned block row I = c + CL li starts at li (c + 1) + CL li (li - 1) / 2
        const int li = I / CL;
        return A + (size_t(li) * (c + 1) + size_t(CL) * li * (li - 1) / 2 + J) * kCb;
    };
    const double* K = prior + size_t(line) * g.SE + D;
    // ---- load the owned block rows (fp64 packed K -> fp32, + eps; identity padding) and the diagonal
    for (int li = 0; li < nown; ++li) {
        const int I = c + CL * li;
        for (int q = tid; q < (I + 1) * 64; q += NT) {
            const int J = q >> 6, r = (q >> 3) & 7, cc = q & 7;
            const int i = I * kBlk + r, j = J * kBlk + cc;
            float v;
            if (i >= D) v = (i == j) ? 1.f : 0.f;
            else if (j > i) v = 0.f;
            else v = float(K[tri(i, j)] + (i == j ? eps0 : 0.0));
            LB(I, J)[swz(r, cc)] = v;
        }
    }
    for (int i = tid; i < Dp; i += NT) dg[i] = i < D ? float(K[tri(i, i)] + eps0) : 1.f;
    if (tid == 0) s_fail = -1;
    __syncthreads();
    // the 8 lanes of a group push a freshly factored Di / Di^T (and a failure) to every CTA
    auto push_di = [&](int f) {
        __syncwarp(0xffu);  // every lane wrote a column of Di
        float dl[kBlk], dt[kBlk];
        ld8r(DiS, gl, dl);
        ld8(DiT + gl * kBlk, dt);
        cl_st8r_all<CL>(DiS, gl, dl);
        cl_st8_all<CL>(DiT + gl * kBlk, dt);
        if (gl == 0 && f >= 0)
            for (int q = 0; q < CL; ++q) cl_st1i(cl_map(&s_fail, q), f);
    };
    if (c == 0 && tid < kBlk) {  // Di of block 0 (owner: CTA 0)
        float row[kBlk];
        ld8r(LB(0, 0), gl, row);
        push_di(diag_factor8(row, gmask, gl, 0, DiS, DiT, dg));
    }
    cl_sync();
    int fail = s_fail;
    for (int k = 0; k < nb && fail < 0; ++k) {
        const int li0 = (k + 1 - c + CL - 1) / CL;  // first owned block row past k
        const int npb = nown - li0;                 // owned panel blocks
        const bool own_k = (k % CL) == c;
        // ---- 1a: panel columns L_Ik[:, l] = A_Ik Di^T[:, l] -> every CTA's LcT[I][l] (one task per
        // (block, column)); the owner of block row k finalises X_kJ = Di T_kJ -> every CTA's Xr[J]
        {
            const int ncol = npb * kBlk, nfin = own_k ? k * kBlk : 0;
            for (int q = tid; q < ncol + nfin; q += NT) {
                if (q < ncol) {
                    const int I = c + CL * (li0 + (q >> 3)), l = q & 7;
                    const float* blk = LB(I, k);
                    float d[kBlk], x[kBlk];
                    ld8r(DiS, l, d);  // Di row l: L[r][l] = sum_{m <= l} A[r][m] Di[l][m]
#pragma unroll
                    for (int r = 0; r < kBlk; ++r) {
                        float ar[kBlk];
                        ld8r(blk, r, ar);
                        float sacc = 0.f;
#pragma unroll
                        for (int m = 0; m < kBlk; ++m)
                            if (m <= l) sacc = fmaf(ar[m], d[m], sacc);
                        x[r] = sacc;
                    }
                    cl_st8_all<CL>(LcT + I * kCb + l * kBlk, x);
                } else {
                    const int J = (q - ncol) >> 3, r = (q - ncol) & 7;
                    float* blk = LB(k, J);
                    float acc[kBlk], d[kBlk];
                    ld8r(DiS, r, d);
#pragma unroll
                    for (int cc = 0; cc < kBlk; ++cc) acc[cc] = 0.f;
#pragma unroll
                    for (int l = 0; l < kBlk; ++l) {
                        float tr[kBlk];
                        ld8r(blk, l, tr);
#pragma unroll
                        for (int cc = 0; cc < kBlk; ++cc) acc[cc] = fmaf(d[l], tr[cc], acc[cc]);
                    }
                    __syncwarp(gmask);  // the group's reads of T_kJ precede its writes
                    st8r(blk, r, acc);
                    cl_st8r_all<CL>(Xr + J * kCb, r, acc);
                }
            }
            if (own_k && tid < kBlk) {  // X_kk = Di into the owner's diagonal block
                float dl[kBlk];
                ld8r(DiS, tid, dl);
                st8r(LB(k, k), tid, dl);
            }
        }
        __syncthreads();  // this CTA's own panel columns are in its LcT
        // ---- 1b: T_Ik = -L_Ik Di into the owned panel blocks (row tasks; L from the local LcT)
        for (int q = tid; q < npb * kBlk; q += NT) {
            const int I = c + CL * (li0 + (q >> 3)), r = q & 7;
            const float* lt = LcT + I * kCb;
            float x[kBlk], t[kBlk];
#pragma unroll
            for (int l = 0; l < kBlk; ++l) x[l] = lt[l * kBlk + r];
#pragma unroll
            for (int cc = 0; cc < kBlk; ++cc) {
                float d[kBlk];
                ld8(DiT + cc * kBlk, d);
                float sacc = 0.f;
#pragma unroll
                for (int l = 0; l < kBlk; ++l)
                    if (l >= cc) sacc = fmaf(x[l], d[l], sacc);
                t[cc] = -sacc;
            }
            st8r(LB(I, k), r, t);
        }
        cl_sync();
        // ---- 2: block tasks over the owned block rows I > k (8x8 accumulators per thread):
        //      A_IJ -= L_Ik L_Jk^T (J > k) and T_IJ -= L_Ik X_kJ (J < k); the owner of block row k + 1
        //      first updates and factors the diagonal block (8 lanes) for the next step
        {
            const bool own_next = (k + 1 < nb) && ((k + 1) % CL) == c;
            if (own_next && tid < kBlk) {
                float* blk = LB(k + 1, k + 1);
                const float* lt = LcT + (k + 1) * kCb;
                float acc[kBlk];
                ld8r(blk, gl, acc);
#pragma unroll
                for (int l = 0; l < kBlk; ++l) {
                    float b[kBlk];
                    ld8(lt + l * kBlk, b);
                    const float ar = b[gl];
#pragma unroll
                    for (int cc = 0; cc < kBlk; ++cc) acc[cc] = fmaf(-ar, b[cc], acc[cc]);
                }
                st8r(blk, gl, acc);
                push_di(diag_factor8(acc, gmask, gl, (k + 1) * kBlk, DiS, DiT, dg));
            }
            // flat tasks (owned row li >= li0, J in [0, I]) minus J = k and the diagonal block above, dealt
            // round-robin over the threads not busy with that diagonal block
            const int t0 = own_next ? kBlk : 0, nthr = NT - t0, me = tid - t0;
            if (me >= 0) {
                int base = 0;
                for (int li = li0; li < nown; ++li) {
                    const int I = c + CL * li;
                    const int nt = I + 1;
                    for (int J = ((me - base) % nthr + nthr) % nthr; J < nt; J += nthr) {
                        if (J == k || (I == k + 1 && J == k + 1)) continue;
                        float* blk = LB(I, J);
                        float acc[kBlk][kBlk];
#pragma unroll
                        for (int r = 0; r < kBlk; ++r) ld8r(blk, r, acc[r]);
                        const float* ai = LcT + I * kCb;
                        if (J > k) {
                            const float* bj = LcT + J * kCb;
#pragma unroll
                            for (int l = 0; l < kBlk; ++l) {
                                float av[kBlk], bv[kBlk];
                                ld8(ai + l * kBlk, av);
                                ld8(bj + l * kBlk, bv);
#pragma unroll
                                for (int r = 0; r < kBlk; ++r)
#pragma unroll
                                    for (int cc = 0; cc < kBlk; ++cc) acc[r][cc] = fmaf(-av[r], bv[cc], acc[r][cc]);
                            }
                        } else {
                            const float* xj = Xr + J * kCb;
#pragma unroll
                            for (int l = 0; l < kBlk; ++l) {
                                float av[kBlk], xv[kBlk];
                                ld8(ai + l * kBlk, av);
                                ld8r(xj, l, xv);
#pragma unroll
                                for (int r = 0; r < kBlk; ++r)
#pragma unroll
                                    for (int cc = 0; cc < kBlk; ++cc) acc[r][cc] = fmaf(-av[r], xv[cc], acc[r][cc]);
                            }
                        }
#pragma unroll
                        for (int r = 0; r < kBlk; ++r) st8r(blk, r, acc[r]);
                    }
                    base += nt;
                }
            }
        }
        cl_sync();
        fail = s_fail;
    }
    if (fail >= 0) {  // the fp64 rescue (k_fixup.cu) redoes this line, escalation included
        if (c == 0 && tid == 0) list_for_fixup(fixlist, status, line);
        return;
    }
    // ---- X = L^{-1}: each CTA writes its block rows as the score's fp32 W blocks (column-major blocks)
    const int nblk = nb * (nb + 1) / 2;
    float* Wp = whiten + size_t(line) * nblk * 64;
    for (int li = 0; li < nown; ++li) {
        const int I = c + CL * li;
        for (int q = tid; q < (I + 1) * 64; q += NT) {
            const int J = q >> 6, e = q & 63, cc = e >> 3, r = e & 7;  // column-major inside the block
            const int i = I * kBlk + r, j = J * kBlk + cc;
            Wp[size_t(tri(I, J)) * 64 + e] = (i < D && j <= i) ? LB(I, J)[swz(r, cc)] : 0.f;
        }
    }
    if (c == 0 && tid == 0) status[line] = -1;
}

template <int CL>
size_t factor_cl_smem_t(const Geometry& g) {
    size_t worst = 0;
    for (int c = 0; c < CL; ++c) {
        const int nown = (g.nb - c + CL - 1) / CL;
        const size_t nloc = size_t(nown) * (c + 1) + size_t(CL) * nown * (nown - 1) / 2;
        worst = std::max(worst, nloc);
    }
    return (worst * kCb + 2 * size_t(g.nb) * kCb + 128 + g.Dp) * 4;
}

}  // namespace

size_t factor_blk_smem(const Geometry& g) {
    // packed blocks + Lc (kLcLd per block) + Di^T (the plane writer's 1.5 KB scratch reuses Lc + Di^T)
    // + the diagonal for the conditioning test
    return (size_t(g.nb) * (g.nb + 1) / 2 * 64 + std::max<size_t>(size_t(g.nb) * kLcLd + 64, 6 * 64) + g.Dp) * 4;
}

// factor_big: Lkk + Di, the transposed panel, (when it fits) the finished X block row, the diagonal
size_t factor_big_smem(const Geometry& g, bool xk) {
    return (2 * size_t(kBB) * kLD + (xk ? 2 : 1) * size_t(kBB) * (g.Dp + 4) + g.Dp) * 4;
}
bool factor_big_xk(const Geometry& g) { return factor_big_smem(g, true) <= 220 * 1024; }

// cluster size of the cluster factor for this geometry (0: does not fit 8 CTAs)
int factor_cl_size(const Geometry& g) {
    const size_t cap = 220 * 1024;
    if (factor_cl_smem_t<2>(g) <= cap) return 2;
    if (factor_cl_smem_t<4>(g) <= cap) return 4;
    if (factor_cl_smem_t<8>(g) <= cap) return 8;
    return 0;
}

size_t factor_smem(const Geometry& g, int precision) {
    if (precision == 64) return size_t(g.D) * (g.D + 1) * 8;
    if (precision == 30) {
        const int cl = factor_cl_size(g);
        return cl == 2 ? factor_cl_smem_t<2>(g) : cl == 4 ? factor_cl_smem_t<4>(g) : factor_cl_smem_t<8>(g);
    }
    if (precision == 32) return factor_blk_smem(g);
    if (precision == 31) return factor_big_smem(g, factor_big_xk(g));
    // global path: panel + diagonal block, or the inverse's row block
    size_t chol = size_t(kNB) * (kNB + 1) * 8 + size_t(std::max(g.D, 1)) * (kNB + 1) * 8;
    size_t inv = size_t(kNB) * (g.D + 1) * 8;
    return std::max(chol, inv);
}

// Auto choice for D > 233 (measured at configs[4], 448 bands, 128 lines per window: factor_big 1.42 ms,
// factor_cl 1.88 ms; one line: factor_cl ~4x shorter): the cluster kernel when one wave of clusters
// holds every line of a launch (the latency regime: lag 0, few streams), else the L2-workspace kernel.
int factor_precision(const Geometry& g, int requested, int lines_per_launch) {
    const size_t cap = 220 * 1024;
    const bool blk_fits = factor_blk_smem(g) <= cap;
    const bool f64_fits = size_t(g.D) * (g.D + 1) * 8 <= cap;
    if (requested == 64 && f64_fits) return 64;
    const bool big_fits = factor_big_smem(g, false) <= cap;
    if (requested == 31 && big_fits) return 31;
    if (requested == 30 && factor_cl_size(g)) return 30;
    if ((requested == 32 || requested == 0) && blk_fits) return 32;
    const int cl = factor_cl_size(g);
    if ((requested == 32 || requested == 0) && cl && (!big_fits || lines_per_launch * cl <= sm_count()))
        return 30;  // fp32 in a cluster's shared memory (large D, one wave)
    if ((requested == 32 || requested == 0 || requested == 31) && big_fits) return 31;  // fp32 over L2
    return 0;  // blocked fp64 over global memory
}

void launch_factor(const Geometry& g, const double* prior, int n_lines_total, double eps0, double* work,
                   float* whiten, int* status, unsigned long long* latch, const WinMeta* meta, long long line_mult,
                   long long line_off, int precision, cudaStream_t st, int* fixlist, const double* stats,
                   const float* vmax, const float* kblk, int blk_threads) {
    const size_t sm = factor_smem(g, precision);
    if (precision == 32 && g.nb == 1 && kblk && !vmax) {
        factor_tiny_kernel<<<(n_lines_total + kTinyLines - 1) / kTinyLines, kTinyLines * 8, 0, st>>>(
            g, eps0, whiten, status, fixlist, kblk, n_lines_total);
        return;
    }
    if (precision == 32) {
        ensure_smem(factor_blk_kernel<64, 7>, sm);
        ensure_smem(factor_blk_kernel<128, FACTOR_MB128>, sm);
        ensure_smem(factor_blk_kernel<256, 3>, sm);
        // 128 threads per line when the SMs hold >= 6 lines each (configs[3]: 7 per SM by shared
        // memory); with fewer resident lines (small windows, lag 0, or D > ~150 where a line's blocks
        // take 100 KB: configs[1]) 256 threads per line shorten each line's latency instead
        int dev = 0;
        cudaGetDevice(&dev);
        int smem_sm = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        const int cap = std::max(1, int(size_t(smem_sm) / (sm + 1024)));
        const int per_sm = (n_lines_total + sm_count() - 1) / sm_count();
        int threads = std::min(cap, per_sm) >= 6 ? 128 : 256;
        if (blk_threads) threads = blk_threads;  // ERX_OPT_FACTOR_THREADS
        if (threads == 64)
            factor_blk_kernel<64, 7><<<n_lines_total, 64, sm, st>>>(g, prior, eps0, whiten, status, fixlist, stats,
                                                                 vmax, kblk);
        else if (threads == 128)
            factor_blk_kernel<128, FACTOR_MB128><<<n_lines_total, 128, sm, st>>>(g, prior, eps0, whiten, status, fixlist, stats,
                                                                   vmax, kblk);
        else if (threads == 512) {
            ensure_smem(factor_blk_kernel<512, 2>, sm);
            factor_blk_kernel<512, 2><<<n_lines_total, 512, sm, st>>>(g, prior, eps0, whiten, status, fixlist, stats,
                                                                   vmax, kblk);
        } else
            factor_blk_kernel<256, 3><<<n_lines_total, 256, sm, st>>>(g, prior, eps0, whiten, status, fixlist, stats,
                                                                   vmax, kblk);
    } else if (precision == 64) {
        ensure_smem(factor_smem_kernel<double>, sm);
        factor_smem_kernel<double><<<n_lines_total, 256, sm, st>>>(g, prior, eps0, whiten, status, latch, meta,
                                                                    line_mult, line_off);
    } else if (precision == 30) {
        const int cl = factor_cl_size(g);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(n_lines_total * cl));
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(cl);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cl == 2) {
            ensure_smem(factor_cl_kernel<2>, sm);
            cudaLaunchKernelEx(&cfg, factor_cl_kernel<2>, g, prior, eps0, whiten, status, fixlist);
        } else if (cl == 4) {
            ensure_smem(factor_cl_kernel<4>, sm);
            cudaLaunchKernelEx(&cfg, factor_cl_kernel<4>, g, prior, eps0, whiten, status, fixlist);
        } else {
            ensure_smem(factor_cl_kernel<8>, sm);
            cudaLaunchKernelEx(&cfg, factor_cl_kernel<8>, g, prior, eps0, whiten, status, fixlist);
        }
    } else if (precision == 31) {
        // 512 threads per line (16 warps, 128 registers): the kernel waits on its L2 workspace (ncu at 256
        // threads: 39 % long-scoreboard, 27 % barrier stalls, 8 warps per SM); measured at 448 bands,
        // 256 / 384 / 512 / 768 threads: 1.41 / 1.20 / 1.11 / 1.78 ms per 128 lines.  ERX_FACTOR_BIG_THREADS=256
        // keeps the round-2d launch (A/B).
        static const int big_nt = [] {
            const char* e = std::getenv("ERX_FACTOR_BIG_THREADS");
            return e ? std::atoi(e) : 512;
        }();
        if (big_nt == 256) {
            ensure_smem(factor_big_kernel<256>, sm);
            factor_big_kernel<256><<<n_lines_total, 256, sm, st>>>(g, prior, eps0, reinterpret_cast<float*>(work), whiten,
                                                                   status, fixlist, factor_big_xk(g));
        } else {
            ensure_smem(factor_big_kernel<512>, sm);
            factor_big_kernel<512><<<n_lines_total, 512, sm, st>>>(g, prior, eps0, reinterpret_cast<float*>(work), whiten,
                                                                   status, fixlist, factor_big_xk(g));
        }
    } else {
        ensure_smem(factor_global_kernel, sm);
        factor_global_kernel<<<n_lines_total, 256, sm, st>>>(g, prior, eps0, work, whiten, status, latch, meta,
                                                               line_mult, line_off);
    }
}

}  // namespace erxk

#ifdef ERX_X_TRACE
extern "C" int erx_x_ftrace(unsigned long long* out, int n_pairs) {
    unsigned int cnt = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&cnt, erxk::g_ftrace_n, sizeof(cnt));
    const int m = int(cnt) < n_pairs ? int(cnt) : n_pairs;
    cudaMemcpyFromSymbol(out, erxk::g_ftrace, size_t(m) * 2 * sizeof(unsigned long long));
    const unsigned int zero = 0;
    cudaMemcpyToSymbol(erxk::g_ftrace_n, &zero, sizeof(zero));
    return m;
}
#endif
