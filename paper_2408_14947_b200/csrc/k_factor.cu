// k_factor.cu — per-line factorisation of the pre-update background:
// L = cholesky_lower(K_{t-1} + eps I) (linalg.hpp:12-15) with the eps x10
// escalation up to 1e-1, then W = L^{-1} written as fp32 for
// the whitening multiply of the score kernel.  A failing pivot is reported
// per line (status) and latched for the device-resident path (latch).
//
// Two kernels, one CTA per line, chosen by the matrix size:
//   factor_smem_kernel<T>   the whole matrix in shared memory (T = double
//                            while D(D+1)*8 fits, float up to D = 233):
//                            right-looking Cholesky then an in-place
//                            right-looking triangular inverse;
//   factor_global_kernel     blocked (panel 32) fp64 over an L2-resident
//                            global workspace for larger D.
#include <algorithm>

#include "erx_common.cuh"

namespace erxk {
namespace {

// ---------------------------------------------------------------------------
// factor: L = chol(K_{t-1} + eps I) with eps escalation x10 up to 1e-1
// (SPEC.md:306), then X = L^{-1}, written as fp32 W (Dp x Dp, zeros above the
// diagonal and in the padding).  One CTA per line; fp64; blocked with panel
// width kNB over a global (L2-resident) workspace; the diagonal block is
// factored by one warp in shared memory.
// ---------------------------------------------------------------------------
__device__ int chol_blocked(double* __restrict__ A, int D, int Dp, double* Lkk, double* pnl, int* s_fail) {
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
__device__ void tri_inverse_blocked(const double* __restrict__ A, double* __restrict__ X, int D, int Dp,
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

__global__ void __launch_bounds__(256) factor_global_kernel(Geometry g, const double* __restrict__ prior, double eps0,
                                                     double* __restrict__ work, float* __restrict__ whiten,
                                                     int* __restrict__ status, int* __restrict__ latch,
                                                     int line_base) {
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
            if (atomicCAS(latch, 0, 1) == 0) {
                latch[1] = line_base + line;
                latch[2] = fail;
            }
        }
        return;
    }
    tri_inverse_blocked(A, X, D, Dp, reinterpret_cast<double*>(smem));
    float* W = whiten + size_t(line) * Dp * Dp;
    for (int idx = tid; idx < Dp * Dp; idx += nt) {
        int i = idx / Dp, j = idx - i * Dp;
        W[idx] = (i < D && j <= i) ? float(X[size_t(i) * Dp + j]) : 0.f;
    }
    if (tid == 0) status[line] = -1;
}

// ---------------------------------------------------------------------------
// shared-memory resident factorisation (D <= 233)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) factor_smem_kernel(Geometry g, const double* __restrict__ prior, double eps0,
                                                          float* __restrict__ whiten, int* __restrict__ status,
                                                          int* __restrict__ latch, int line_base) {
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
            if (atomicCAS(latch, 0, 1) == 0) {
                latch[1] = line_base + line;
                latch[2] = fail;
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
    float* W = whiten + size_t(line) * g.Dp * g.Dp;
    for (int idx = tid; idx < g.Dp * g.Dp; idx += nt) {
        const int i = idx / g.Dp, j = idx - i * g.Dp;
        W[idx] = (i < D && j <= i) ? float(A[i * LD + j]) : 0.f;
    }
    if (tid == 0) status[line] = -1;
}

// ---------------------------------------------------------------------------
// one warp per line (D <= kWarpFactorMaxD): no block barriers at all.  Lanes
// own whole rows, so every step is __syncwarp-ordered and the inner loops run
// over independent elements (ILP); a row pair {r, 63-r} per lane and round
// balances the shrinking triangle of the Cholesky update.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(32) factor_warp_kernel(Geometry g, const double* __restrict__ prior, double eps0,
                                                         float* __restrict__ whiten, int* __restrict__ status,
                                                         int* __restrict__ latch, int line_base) {
    extern __shared__ __align__(16) unsigned char smem[];
    T* A = reinterpret_cast<T*>(smem);
    const int D = g.D, LD = D + 1;
    const int line = blockIdx.x, lane = threadIdx.x;
    const double* K = prior + size_t(line) * g.SE + D;
    double eps = eps0;
    int fail;
    while (true) {
        for (int i = 0; i < D; ++i)
            for (int j = lane; j <= i; j += 32) A[i * LD + j] = T(K[tri(i, j)] + (i == j ? eps : 0.0));
        __syncwarp();
        fail = -1;
        for (int j = 0; j < D; ++j) {
            const T djj = A[j * LD + j];
            if (!(djj > T(0))) {
                fail = j;
                break;
            }
            const T s = sqrt(djj);
            for (int i = j + 1 + lane; i < D; i += 32) A[i * LD + j] /= s;
            __syncwarp();
            if (lane == 0) A[j * LD + j] = s;
            const T* colj = A + j;
            const int n = D - j - 1;
            for (int base = 0; base < n; base += 64) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = base + (h == 0 ? lane : 63 - lane);
                    if (r >= n) continue;
                    const int i = j + 1 + r;
                    T* rowi = A + i * LD;
                    const T lij = rowi[j];
#pragma unroll 4
                    for (int k = j + 1; k <= i; ++k) rowi[k] -= lij * colj[k * LD];
                }
            }
            __syncwarp();
        }
        if (fail < 0) break;
        const double next = eps * 10.0;
        if (!(next <= 1e-1 * (1.0 + 1e-9))) break;
        eps = next;
        __syncwarp();
    }
    if (fail >= 0) {
        if (lane == 0) {
            status[line] = fail;
            if (atomicCAS(latch, 0, 1) == 0) {
                latch[1] = line_base + line;
                latch[2] = fail;
            }
        }
        return;
    }
    // in-place inverse, right-looking by rows (see factor_smem_kernel); lane = row
    for (int k = 0; k < D; ++k) {
        const T inv = T(1) / A[k * LD + k];
        __syncwarp();
        for (int c = lane; c < k; c += 32) A[k * LD + c] *= inv;
        if (lane == 0) A[k * LD + k] = inv;
        __syncwarp();
        const T* rowk = A + k * LD;
        for (int i = k + 1 + lane; i < D; i += 32) {
            T* rowi = A + i * LD;
            const T l = rowi[k];
            rowi[k] = -l * inv;
#pragma unroll 4
            for (int c = 0; c < k; ++c) rowi[c] -= l * rowk[c];
        }
        __syncwarp();
    }
    float* W = whiten + size_t(line) * g.Dp * g.Dp;
    for (int i = 0; i < g.Dp; ++i)
        for (int j = lane; j < g.Dp; j += 32) W[size_t(i) * g.Dp + j] = (i < D && j <= i) ? float(A[i * LD + j]) : 0.f;
    if (lane == 0) status[line] = -1;
}

}  // namespace

size_t factor_smem(const Geometry& g, int precision) {
    if (precision == 64) return size_t(g.D) * (g.D + 1) * 8;
    if (precision == 32) return size_t(g.D) * (g.D + 1) * 4;
    // global path: panel + diagonal block, or the inverse's row block
    size_t chol = size_t(kNB) * (kNB + 1) * 8 + size_t(std::max(g.D, 1)) * (kNB + 1) * 8;
    size_t inv = size_t(kNB) * (g.D + 1) * 8;
    return std::max(chol, inv);
}

int factor_precision(const Geometry& g, int requested) {
    const size_t cap = 220 * 1024;
    if (requested == 1) return 0;  // force the blocked global-memory path
    if (requested == 64 && size_t(g.D) * (g.D + 1) * 8 <= cap) return 64;
    if (requested == 32 && size_t(g.D) * (g.D + 1) * 4 <= cap) return 32;
    if (requested == 0) {
        if (size_t(g.D) * (g.D + 1) * 8 <= cap) return 64;
        if (size_t(g.D) * (g.D + 1) * 4 <= cap) return 32;
    }
    return 0;  // blocked fp64 over global memory
}

void launch_factor(const Geometry& g, const double* prior, int n_lines_total, double eps0, double* work,
                   float* whiten, int* status, int* latch, int line_base, int precision, cudaStream_t st) {
    const size_t sm = factor_smem(g, precision);
    if ((precision == 64 || precision == 32) && g.D <= kWarpFactorMaxD) {
        if (precision == 64) {
            cudaFuncSetAttribute(factor_warp_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            factor_warp_kernel<double><<<n_lines_total, 32, sm, st>>>(g, prior, eps0, whiten, status, latch,
                                                                       line_base);
        } else {
            cudaFuncSetAttribute(factor_warp_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            factor_warp_kernel<float><<<n_lines_total, 32, sm, st>>>(g, prior, eps0, whiten, status, latch,
                                                                      line_base);
        }
    } else if (precision == 64) {
        cudaFuncSetAttribute(factor_smem_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        factor_smem_kernel<double><<<n_lines_total, 256, sm, st>>>(g, prior, eps0, whiten, status, latch, line_base);
    } else if (precision == 32) {
        cudaFuncSetAttribute(factor_smem_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        factor_smem_kernel<float><<<n_lines_total, 256, sm, st>>>(g, prior, eps0, whiten, status, latch, line_base);
    } else {
        cudaFuncSetAttribute(factor_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        factor_global_kernel<<<n_lines_total, 256, sm, st>>>(g, prior, eps0, work, whiten, status, latch,
                                                               line_base);
    }
}

}  // namespace erxk
