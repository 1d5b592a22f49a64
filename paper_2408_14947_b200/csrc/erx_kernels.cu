// erx_kernels.cu — sm_100a kernels of the windowed ERX pipeline.
// See erx_kernels.cuh for the mapping onto the reference functions.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "erx_kernels.cuh"

namespace erxk {

namespace {

__device__ __forceinline__ size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// Line staging shared by stats and score: pixel rows [p0, p0 + n) of one
// line, projected (SRP) or copied (identity), minus a per-dim centre `cen`
// (fp64), written as fp32 into `dst(pixel, dim)`.  SRP sums run in fp64 —
// the products of an fp32 radiance and an fp32-exact weight are exact in
// fp64 — so z matches project_line's fp64 Z (projection.hpp:31-34) and the
// subtraction of the large projected mean happens before rounding to fp32.
// ---------------------------------------------------------------------------
template <typename Dst>
__device__ __forceinline__ void stage_rows(const Geometry& g, const float* __restrict__ xl, int p0, int n,
                                           float* __restrict__ xs, const double* __restrict__ cen, Dst dst) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (!g.srp) {
        const float* src = xl + size_t(p0) * g.B;
        const int total = n * g.B;
        for (int i = tid; i < total; i += nt) {
            int pp = i / g.B;
            int b = i - pp * g.B;
            dst(pp, b, float(double(__ldg(src + i)) - cen[b]));
        }
    } else {
        const float* src = xl + size_t(p0) * g.B;
        const int total = n * g.B;
        for (int i = tid; i < total; i += nt) xs[i] = __ldg(src + i);
        __syncthreads();
        const int tot2 = n * g.D;
        for (int i = tid; i < tot2; i += nt) {
            int pp = i / g.D;
            int j = i - pp * g.D;
            double z = 0.0;
            const float* row = xs + pp * g.B;
            for (int k = g.srp_ptr[j]; k < g.srp_ptr[j + 1]; ++k) z += double(row[g.srp_band[k]]) * double(g.srp_w[k]);
            dst(pp, j, float(z * g.srp_scale - cen[j]));
        }
    }
}

// ---------------------------------------------------------------------------
// stats: line_stats (erx.hpp:38-40) for every line of the window.
//
// Each thread owns one 8x8 block (I, J), I >= J, of the lower-triangular
// second-moment matrix of v = z - c, where c is the mean of the line's first
// min(32, P) pixels (a cheap centring that removes the mean before any fp32
// rounding; the exact line mean is restored in fp64 at the end:
// mu_hat = c + sum(v)/P, K_hat = (S - sum(v) sum(v)^T / P) / (P - 1)).
// Products accumulate in fp32 over one staged chunk (<= CH pixels) and the
// chunk sums in a second fp32 level; the SURVEY §7 precision study put this
// ~100x inside the 1e-5 median bar.
// ---------------------------------------------------------------------------
struct StatsArgs {
    Geometry g;
    StatsLaunch sl;
    const float* x;
    int n;          // lines per stream in this window (line id l = s * n + t)
    int in_stride;  // lines per stream in the input buffer
    double* stats;
};

__device__ __forceinline__ const float* line_ptr(const float* x, int line, int n, int in_stride, const Geometry& g) {
    const int s = line / n, t = line - s * n;
    return x + (size_t(s) * in_stride + t) * size_t(g.P) * g.B;
}

__global__ void __launch_bounds__(128) stats_kernel(StatsArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geometry& g = a.g;
    const StatsLaunch& sl = a.sl;
    const int line = blockIdx.x / sl.cpl;
    const int cta = blockIdx.x - line * sl.cpl;
    const int tid = threadIdx.x;

    // smem carve: v [CH][Dp] f32 | xs [CH][B] f32 (srp) | cen [Dp] f64 | colsum [Dp] f64 ;
    // the reduction buffer red [128][64] f64 aliases v/xs (used only after the chunk loop).
    float* v = reinterpret_cast<float*>(smem);
    float* xs = v + size_t(sl.CH) * g.Dp;
    size_t off = align_up(size_t(sl.CH) * g.Dp * 4 + (g.srp ? size_t(sl.CH) * g.B * 4 : 0), 16);
    const size_t red_bytes = (sl.G > 1) ? size_t(128) * 64 * 8 : 0;
    off = off > red_bytes ? off : red_bytes;
    double* cen = reinterpret_cast<double*>(smem + off);
    double* colsum = cen + g.Dp;
    double* red = reinterpret_cast<double*>(smem);

    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);

    // pair ownership, column-major enumeration of the lower triangle of blocks
    const int q_local = tid / sl.G;
    const int grp = tid - q_local * sl.G;
    const int q = cta * sl.npc + q_local;
    const bool active = (q_local < sl.npc) && (q < sl.n_pairs);
    int I = 0, J = 0;
    if (active) {
        int rem = q;
        while (rem >= g.nb - J) {
            rem -= g.nb - J;
            ++J;
        }
        I = J + rem;
    }

    // zero the padded columns once (identity never writes dims >= B; srp writes dims < D)
    for (int i = tid; i < sl.CH * g.Dp; i += blockDim.x) v[i] = 0.f;
    for (int j = tid; j < g.Dp; j += blockDim.x) {
        cen[j] = 0.0;
        colsum[j] = 0.0;
    }
    __syncthreads();

    float acc[kBlk][kBlk], acc2[kBlk][kBlk];
#pragma unroll
    for (int r = 0; r < kBlk; ++r)
#pragma unroll
        for (int c = 0; c < kBlk; ++c) acc2[r][c] = 0.f;
    double cs[4] = {0.0, 0.0, 0.0, 0.0};

    // centre c: fp64 mean of the first min(32, P) projected pixels (read straight from L2)
    {
        const int n0 = min(32, g.P);
        for (int j = tid; j < g.D; j += blockDim.x) {
            double s = 0.0;
            for (int pp = 0; pp < n0; ++pp) {
                const float* row = xl + size_t(pp) * g.B;
                if (!g.srp) {
                    s += double(__ldg(row + j));
                } else {
                    double z = 0.0;
                    for (int k = g.srp_ptr[j]; k < g.srp_ptr[j + 1]; ++k)
                        z += double(__ldg(row + g.srp_band[k])) * double(g.srp_w[k]);
                    s += z * g.srp_scale;
                }
            }
            cen[j] = s / double(n0);
        }
        __syncthreads();
    }

    for (int c0 = 0; c0 < g.P; c0 += sl.CH) {
        const int n = min(sl.CH, g.P - c0);
        stage_rows(g, xl, c0, n, xs, cen, [&](int pp, int j, float val) { v[pp * g.Dp + j] = val; });
        __syncthreads();
        // column sums (fp32 per chunk, fp64 across chunks)
        for (int k = 0; k < 4; ++k) {
            int j = tid + k * blockDim.x;
            if (j < g.D) {
                float s = 0.f;
                for (int pp = 0; pp < n; ++pp) s += v[pp * g.Dp + j];
                cs[k] += double(s);
            }
        }
        if (active) {
#pragma unroll
            for (int r = 0; r < kBlk; ++r)
#pragma unroll
                for (int c = 0; c < kBlk; ++c) acc[r][c] = 0.f;
            for (int pp = grp; pp < n; pp += sl.G) {
                const float4* ra = reinterpret_cast<const float4*>(v + pp * g.Dp + I * kBlk);
                const float4* rb = reinterpret_cast<const float4*>(v + pp * g.Dp + J * kBlk);
                float4 a0 = ra[0], a1 = ra[1], b0 = rb[0], b1 = rb[1];
                float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int r = 0; r < kBlk; ++r)
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
            }
#pragma unroll
            for (int r = 0; r < kBlk; ++r)
#pragma unroll
                for (int c = 0; c < kBlk; ++c) acc2[r][c] += acc[r][c];
        }
        __syncthreads();
    }

    for (int k = 0; k < 4; ++k) {
        int j = tid + k * blockDim.x;
        if (j < g.D) colsum[j] = cs[k];
    }
    if (sl.G > 1) {
        // cross-group reduction in fp64, fixed order (deterministic).
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kBlk; ++r)
#pragma unroll
            for (int c = 0; c < kBlk; ++c) red[tid * 64 + r * 8 + c] = double(acc2[r][c]);
    }
    __syncthreads();

    double* out = a.stats + size_t(line) * g.SE;
    const double P = double(g.P);
    if (cta == 0) {
        for (int j = tid; j < g.D; j += blockDim.x) out[j] = cen[j] + colsum[j] / P;
    }
    if (active && grp == 0) {
#pragma unroll
        for (int r = 0; r < kBlk; ++r) {
            const int ai = I * kBlk + r;
#pragma unroll
            for (int c = 0; c < kBlk; ++c) {
                const int bj = J * kBlk + c;
                if (ai < g.D && bj <= ai) {
                    double s;
                    if (sl.G > 1) {
                        s = 0.0;
                        for (int gg = 0; gg < sl.G; ++gg) s += red[(q_local * sl.G + gg) * 64 + r * 8 + c];
                    } else {
                        s = double(acc2[r][c]);
                    }
                    out[g.D + tri(ai, bj)] = (s - colsum[ai] * colsum[bj] / P) / (P - 1.0);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// scan: the EMA (erx.hpp:42-44) or batched-Welford (linalg.hpp:33-36)
// recurrence over the window's lines, element-wise over (mu, packed K).
// Writes, per line, the PRE-update background (score-then-update,
// SPEC.md:324).  The first line ever initialises the background with its own
// statistics (erx.hpp:54-55).  Multiplications are rounded separately
// (__dmul_rn) to reproduce the reference's (1-a)*K + a*K_hat rounding.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) scan_kernel(Geometry g, const double* __restrict__ stats,
                                                   double* __restrict__ prior, const double* __restrict__ st_in,
                                                   double* __restrict__ st_out, int n, int initialized,
                                                   double alpha, int incremental, int64_t n_seen0) {
    const int s = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.SE) return;
    const double* in = st_in + size_t(s) * g.SE;
    const size_t l0 = size_t(s) * n;
    if (!incremental) {
        const double om = 1.0 - alpha;
        double state = in[e];
        for (int t = 0; t < n; ++t) {
            const size_t l = l0 + t;
            const double stat = stats[l * g.SE + e];
            double pr;
            if (!initialized && t == 0) {
                pr = stat;
                state = stat;
            } else {
                pr = state;
                state = __dadd_rn(__dmul_rn(om, state), __dmul_rn(alpha, stat));
            }
            prior[l * g.SE + e] = pr;
        }
        st_out[size_t(s) * g.SE + e] = state;
    } else {
        int a, b;
        if (e < g.D) {
            a = b = e;
        } else {
            int k = e - g.D;
            a = int((sqrt(8.0 * k + 1.0) - 1.0) * 0.5);
            while (a * (a + 1) / 2 > k) --a;
            while ((a + 1) * (a + 2) / 2 <= k) ++a;
            b = k - a * (a + 1) / 2;
        }
        double ma = in[a], mb = in[b];
        double cov = (e >= g.D) ? in[e] : 0.0;
        double nseen = double(n_seen0);
        const double nb = double(g.P);
        for (int t = 0; t < n; ++t) {
            const size_t l = l0 + t;
            const double* st = stats + l * g.SE;
            const double mha = st[a], mhb = st[b];
            double pr;
            if (!initialized && t == 0) {
                ma = mha;
                mb = mhb;
                if (e >= g.D) cov = st[e];
                nseen = nb;
                pr = (e < g.D) ? ma : cov;
            } else {
                pr = (e < g.D) ? ma : cov;
                const double na = nseen, nn = na + nb;
                const double da = mha - ma, db = mhb - mb;
                if (e >= g.D) {
                    const double m2a = (na >= 2.0) ? cov * (na - 1.0) : 0.0;
                    const double m2b = st[e] * (nb - 1.0);
                    const double m2 = m2a + m2b + da * db * (na * nb / nn);
                    cov = (nn >= 2.0) ? m2 / (nn - 1.0) : 0.0;
                }
                ma += da * (nb / nn);
                mb += db * (nb / nn);
                nseen = nn;
            }
            prior[l * g.SE + e] = pr;
        }
        st_out[size_t(s) * g.SE + e] = (e < g.D) ? ma : cov;
    }
}

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

__global__ void __launch_bounds__(256) factor_kernel(Geometry g, const double* __restrict__ prior, double eps0,
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
// score: delta_i = || W (z_i - mu_{t-1}) ||  with W = L^{-1}
// (forward_substitute_inplace, linalg.hpp:21).  One CTA per
// (line, 64-pixel tile); v tile [Dp][64] fp32 in smem; thread = (row-block
// slot, 4-pixel group); 8x4 register accumulators; W streamed from L2 with
// warp-broadcast loads.  Partial sum-of-squares per row block are reduced in
// a fixed order (deterministic).
// ---------------------------------------------------------------------------
struct ScoreArgs {
    Geometry g;
    const float* x;
    int n;
    int in_stride;
    const double* prior;
    const float* W;
    float* raw;
    int tiles;
};

__global__ void __launch_bounds__(256) score_kernel(ScoreArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geometry& g = a.g;
    const int line = blockIdx.x / a.tiles;
    const int tile = blockIdx.x - line * a.tiles;
    const int p0 = tile * kScoreTile;
    const int np = min(kScoreTile, g.P - p0);
    const int tid = threadIdx.x;
    float* vt = reinterpret_cast<float*>(smem);                      // [Dp][kScoreStride]
    float* red = vt + size_t(g.Dp) * kScoreStride;                   // [nb][64]
    float* xs = red + size_t(g.nb) * kScoreTile;                     // [64][B] (srp)
    double* mu = reinterpret_cast<double*>(
        smem + align_up((size_t(g.Dp) * kScoreStride + size_t(g.nb) * kScoreTile +
                         (g.srp ? size_t(kScoreTile) * g.B : 0)) * 4, 16));
    const double* pr = a.prior + size_t(line) * g.SE;
    for (int j = tid; j < g.Dp; j += blockDim.x) mu[j] = (j < g.D) ? pr[j] : 0.0;
    // zero padding rows (dims >= D) and padding pixels (>= np)
    for (int i = tid; i < g.Dp * kScoreStride; i += blockDim.x) {
        int d = i / kScoreStride, pp = i - d * kScoreStride;
        if (d >= g.D || pp >= np) vt[i] = 0.f;
    }
    __syncthreads();
    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
    stage_rows(g, xl, p0, np, xs, mu, [&](int pp, int j, float val) { vt[j * kScoreStride + pp] = val; });
    __syncthreads();

    const int q = tid & 15;       // pixel group: pixels 4q .. 4q+3
    const int slot = tid >> 4;    // 0..15
    const float* Wl = a.W + size_t(line) * g.Dp * g.Dp;
    for (int I = slot; I < g.nb; I += 16) {
        float acc[kBlk][4];
#pragma unroll
        for (int r = 0; r < kBlk; ++r)
#pragma unroll
            for (int p = 0; p < 4; ++p) acc[r][p] = 0.f;
        for (int J = 0; J <= I; ++J) {
            float vb[kBlk][4];
#pragma unroll
            for (int c = 0; c < kBlk; ++c) {
                float4 t = *reinterpret_cast<const float4*>(vt + (J * kBlk + c) * kScoreStride + 4 * q);
                vb[c][0] = t.x;
                vb[c][1] = t.y;
                vb[c][2] = t.z;
                vb[c][3] = t.w;
            }
#pragma unroll
            for (int r = 0; r < kBlk; ++r) {
                const float4* wr = reinterpret_cast<const float4*>(Wl + size_t(I * kBlk + r) * g.Dp + J * kBlk);
                float4 w0 = __ldg(wr), w1 = __ldg(wr + 1);
                float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int c = 0; c < kBlk; ++c)
#pragma unroll
                    for (int p = 0; p < 4; ++p) acc[r][p] = fmaf(wv[c], vb[c][p], acc[r][p]);
            }
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            float s = 0.f;
#pragma unroll
            for (int r = 0; r < kBlk; ++r) s = fmaf(acc[r][p], acc[r][p], s);
            red[I * kScoreTile + 4 * q + p] = s;
        }
    }
    __syncthreads();
    for (int pp = tid; pp < np; pp += blockDim.x) {
        float s = 0.f;
        for (int I = 0; I < g.nb; ++I) s += red[I * kScoreTile + pp];
        a.raw[size_t(line) * g.P + p0 + pp] = sqrtf(s);
    }
}

// ---------------------------------------------------------------------------
// normalize: per-line z-score, population std, std < 1e-12 -> zeros
// (detector.hpp:29-32).  One warp per line, fp64.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) normalize_kernel(int P, const float* __restrict__ raw, int n_lines,
                                                        float* __restrict__ norm) {
    const int line = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (line >= n_lines) return;
    const float* r = raw + size_t(line) * P;
    double s = 0.0;
    for (int i = lane; i < P; i += 32) s += double(r[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double mean = s / double(P);
    double v = 0.0;
    for (int i = lane; i < P; i += 32) {
        double d = double(r[i]) - mean;
        v += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const double sd = sqrt(v / double(P));
    float* out = norm + size_t(line) * P;
    for (int i = lane; i < P; i += 32) out[i] = (sd < 1e-12) ? 0.f : float((double(r[i]) - mean) / sd);
}

// FP32 FFMA throughput probe: the roofline denominator for the FFMA-bound
// kernels (MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only).
__global__ void __launch_bounds__(256) ffma_probe_kernel(int iters, float x, float y, float* sink) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = float(threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], x, y);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 123.456f) sink[0] = s;
}

}  // namespace

double probe_ffma_tflops(cudaStream_t st) {
    float* sink = nullptr;
    cudaMalloc(&sink, sizeof(float));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256, iters = 8192;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a, st);
        ffma_probe_kernel<<<blocks, threads, 0, st>>>(iters, 0.999f, 1e-3f, sink);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0) best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    const double flops = 2.0 * 8.0 * double(iters) * blocks * threads;
    return flops / (double(best) * 1e-3) / 1e12;
}

// ---------------------------------------------------------------------------
// host-side planning and launchers
// ---------------------------------------------------------------------------
StatsLaunch plan_stats(const Geometry& g) {
    StatsLaunch sl{};
    sl.n_pairs = g.nb * (g.nb + 1) / 2;
    if (sl.n_pairs <= 64) {
        sl.G = 128 / sl.n_pairs;
        sl.npc = sl.n_pairs;
        sl.cpl = 1;
    } else {
        sl.G = 1;
        sl.npc = 128;
        sl.cpl = (sl.n_pairs + 127) / 128;
    }
    // chunk: enough pixels that every pixel group sees >= 4 pixels, capped by smem.
    const size_t per_px = size_t(g.Dp) * 4 + (g.srp ? size_t(g.B) * 4 : 0);
    int ch = std::max(32, std::min(256, 4 * sl.G));
    while (ch > 32 && size_t(ch) * per_px > 96 * 1024) ch /= 2;
    sl.CH = ch;
    size_t off = (size_t(ch) * per_px + 15) / 16 * 16;
    const size_t red_bytes = (sl.G > 1) ? size_t(128) * 64 * 8 : 0;
    off = std::max(off, red_bytes);
    sl.smem = off + 2 * size_t(g.Dp) * 8;
    return sl;
}

size_t score_smem(const Geometry& g) {
    size_t f = size_t(g.Dp) * kScoreStride + size_t(g.nb) * kScoreTile + (g.srp ? size_t(kScoreTile) * g.B : 0);
    return (f * 4 + 15) / 16 * 16 + size_t(g.Dp) * 8;
}

size_t factor_smem(const Geometry& g) {
    size_t chol = size_t(kNB) * (kNB + 1) * 8 + size_t(std::max(g.D, 1)) * (kNB + 1) * 8;
    size_t inv = size_t(kNB) * (g.D + 1) * 8;
    return std::max(chol, inv);
}

void launch_stats(const Geometry& g, const StatsLaunch& sl, const float* x, int n_per_stream, int in_stride,
                  int n_lines_total, double* stats, cudaStream_t st) {
    StatsArgs a{g, sl, x, n_per_stream, in_stride, stats};
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_done = true;
    }
    stats_kernel<<<n_lines_total * sl.cpl, 128, sl.smem, st>>>(a);
}

void launch_scan(const Geometry& g, const double* stats, double* prior, const double* state_in, double* state_out,
                 int n_streams, int n_per_stream, int initialized, double alpha, int incremental, int64_t n_seen0,
                 cudaStream_t st) {
    dim3 grid((g.SE + 127) / 128, n_streams);
    scan_kernel<<<grid, 128, 0, st>>>(g, stats, prior, state_in, state_out, n_per_stream, initialized, alpha,
                                      incremental, n_seen0);
}

void launch_factor(const Geometry& g, const double* prior, int n_lines_total, double eps0, double* work,
                   float* whiten, int* status, int* latch, int line_base, cudaStream_t st) {
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_done = true;
    }
    factor_kernel<<<n_lines_total, 256, factor_smem(g), st>>>(g, prior, eps0, work, whiten, status, latch,
                                                              line_base);
}

void launch_score(const Geometry& g, const float* x, int n_per_stream, int in_stride, const double* prior,
                  const float* whiten, int n_lines_total, float* raw, cudaStream_t st) {
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_done = true;
    }
    const int tiles = (g.P + kScoreTile - 1) / kScoreTile;
    ScoreArgs a{g, x, n_per_stream, in_stride, prior, whiten, raw, tiles};
    score_kernel<<<n_lines_total * tiles, 256, score_smem(g), st>>>(a);
}

void launch_normalize(const Geometry& g, const float* raw, int n_lines_total, float* norm, cudaStream_t st) {
    normalize_kernel<<<(n_lines_total + 3) / 4, 128, 0, st>>>(g.P, raw, n_lines_total, norm);
}

}  // namespace erxk
