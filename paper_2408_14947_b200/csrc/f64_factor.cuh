// f64_factor.cuh — fp64 blocked Cholesky (cholesky_lower, linalg.hpp:12-15)
// and triangular inverse over a global (L2-resident) workspace, one CTA per
// line: the on-request fp64 factor (k_factor.cu: factor_global_kernel) and
// the fp64 rescue of lines the fp32 factor cannot take (k_fixup.cu).
#pragma once

#include "erx_common.cuh"

namespace erxk {

// ---------------------------------------------------------------------------
// factor: L = chol(K_{t-1} + eps I) with eps escalation x10 up to 1e-1
// (SPEC.md:306), then X = L^{-1}, written as fp32 W (Dp x Dp, zeros above the
// diagonal and in the padding).  One CTA per line; fp64; blocked with panel
// width kNB over a global (L2-resident) workspace; the diagonal block is
// factored by one warp in shared memory.
// ---------------------------------------------------------------------------
__device__ inline int chol_blocked(double* __restrict__ A, int D, int Dp, double* Lkk, double* pnl, int* s_fail) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int LD = kNB + 1;
    for (int k0 = 0; k0 < D; k0 += kNB) {
        const int kb = min(kNB, D - k0);
        for (int idx = tid; idx < kb * kb; idx += nt) {
            int r = idx / kb, c = idx - r * kb;
            if (c <= r) Lkk[r * LD + c] = A[size_t(k0 + r) * Dp + k0 + c];
        }
        if (tid == 0) *s_fail = -1;
        __syncthreads();
        if (warp == 0) {
            for (int j = 0; j < kb; ++j) {
                __syncwarp();
                const double djj = Lkk[j * LD + j];
                if (!(djj > 0.0)) {
                    if (lane == 0) *s_fail = k0 + j;
                    break;
                }
                const double sq = sqrt(djj);
                __syncwarp();
                if (lane > j && lane < kb) Lkk[lane * LD + j] /= sq;
                __syncwarp();
                if (lane == j) Lkk[j * LD + j] = sq;
                if (lane > j && lane < kb) {
                    const double lij = Lkk[lane * LD + j];
                    for (int c = j + 1; c <= lane; ++c) Lkk[lane * LD + c] -= lij * Lkk[c * LD + j];
                }
            }
        }
        __syncthreads();
        if (*s_fail >= 0) return *s_fail;
        for (int idx = tid; idx < kb * kb; idx += nt) {
            int r = idx / kb, c = idx - r * kb;
            if (c <= r) A[size_t(k0 + r) * Dp + k0 + c] = Lkk[r * LD + c];
        }
        // panel: rows below the diagonal block, L_ik = A_ik L_kk^{-T}
        const int r0 = k0 + kb;
        const int nr = D - r0;
        for (int r = tid; r < nr; r += nt) {
            double* prow = pnl + size_t(r) * LD;
            const double* arow = A + size_t(r0 + r) * Dp + k0;
            for (int c = 0; c < kb; ++c) {
                double s = arow[c];
                for (int l = 0; l < c; ++l) s -= prow[l] * Lkk[c * LD + l];
                prow[c] = s / Lkk[c * LD + c];
            }
            double* w = A + size_t(r0 + r) * Dp + k0;
            for (int c = 0; c < kb; ++c) w[c] = prow[c];
        }
        __syncthreads();
        // trailing update A22 -= P P^T, 4x4 register tiles over the lower triangle
        const int nt4 = (nr + 3) / 4;
        const int ntile = nt4 * (nt4 + 1) / 2;
        for (int tix = tid; tix < ntile; tix += nt) {
            int R = int((sqrt(8.0 * tix + 1.0) - 1.0) * 0.5);
            while (R * (R + 1) / 2 > tix) --R;
            while ((R + 1) * (R + 2) / 2 <= tix) ++R;
            const int C = tix - R * (R + 1) / 2;
            double acc[4][4] = {};
            for (int l = 0; l < kb; ++l) {
                double av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    int ri = R * 4 + i, ci = C * 4 + i;
                    av[i] = (ri < nr) ? pnl[size_t(ri) * LD + l] : 0.0;
                    bv[i] = (ci < nr) ? pnl[size_t(ci) * LD + l] : 0.0;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    int ri = R * 4 + i, ci = C * 4 + j;
                    if (ri < nr && ci <= ri) A[size_t(r0 + ri) * Dp + r0 + ci] -= acc[i][j];
                }
        }
        __syncthreads();
    }
    return -1;
}

// X = L^{-1} by block rows: X_I = L_II^{-1} (E_I - sum_{J<I} L_IJ X_J).
__device__ inline void tri_inverse_blocked(const double* __restrict__ A, double* __restrict__ X, int D, int Dp,
                                    double* Lrow) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int LDR = D + 1;
    for (int i0 = 0; i0 < D; i0 += kNB) {
        const int ib = min(kNB, D - i0);
        const int ncol = i0 + ib;
        for (int idx = tid; idx < ib * ncol; idx += nt) {
            int r = idx / ncol, c = idx - r * ncol;
            Lrow[r * LDR + c] = (c <= i0 + r) ? A[size_t(i0 + r) * Dp + c] : 0.0;
        }
        __syncthreads();
        for (int c = tid; c < ncol; c += nt) {
            double t[kNB];
#pragma unroll
            for (int r = 0; r < kNB; ++r) t[r] = (r < ib && i0 + r == c) ? 1.0 : 0.0;
            const int jstart = c & ~31;  // warp-uniform start: row-wise (coalesced) loads of X
            for (int j = jstart; j < i0; ++j) {
                const double xj = (j >= c) ? X[size_t(j) * Dp + c] : 0.0;
#pragma unroll
                for (int r = 0; r < kNB; ++r)
                    if (r < ib) t[r] = fma(-Lrow[r * LDR + j], xj, t[r]);
            }
#pragma unroll
            for (int r = 0; r < kNB; ++r) {
                if (r < ib) {
                    double s = t[r];
#pragma unroll
                    for (int j = 0; j < r; ++j) s = fma(-Lrow[r * LDR + i0 + j], t[j], s);
                    t[r] = s / Lrow[r * LDR + i0 + r];
                    if (i0 + r < c) t[r] = 0.0;
                }
            }
#pragma unroll
            for (int r = 0; r < kNB; ++r)
                if (r < ib) X[size_t(i0 + r) * Dp + c] = t[r];
        }
        __syncthreads();
    }
}

}  // namespace erxk
