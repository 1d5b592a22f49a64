// k_score.cu — per-pixel Mahalanobis distance against the pre-update
// background: delta_i = || W (z_i - mu_{t-1}) ||, W = L^{-1},
// i.e. forward_substitute_inplace (linalg.hpp:21) done as a whitening
// multiply; and normalize_scores (detector.hpp:29-32).
//
// score: one CTA per (line, pixel tile).  The tile's centred pixels sit in
// shared memory as rows [pixel][Dpad] (Dpad = 4 mod 32: consecutive pixel
// rows hit distinct banks).  The line's W arrives as packed lower 8x8 blocks,
// column-major inside a block (k_factor.cu: write_wblocks), staged into
// shared memory with cp.async when it fits.  Thread (s, q) owns the
// row-block pair {s, nb-1-s} (equal total work, nb+1 block steps) and pixels
// q + G*p, p < 4; per block column c it issues 16 paired FFMA2 (rows
// 2k, 2k+1 of W times a broadcast pixel value).  Partial sums of squares per
// row block are reduced in a fixed order (bitwise deterministic).
#include "erx_common.cuh"

namespace erxk {
namespace {

struct ScoreArgs {
    Geometry g;
    ScoreLaunch sc;
    const float* x;
    int n;
    int in_stride;
    const double* prior;
    const float* W;
    float* raw;
};

// W too large for shared memory (D > ~180: configs[1], configs[4]): group s walks its row-block pair
// {s, nb-1-s} in nb + 1 block steps, step t touching one 8x8 block W(I_s(t), J_s(t)).  The CTA stages
// the blocks of step t + 2 (one per group, 256 B each) into a 4-deep shared ring with cp.async while
// it computes step t, so the FFMA2 loop reads W from shared memory instead of waiting on L2.  One
// barrier per step: the slot refilled at step t was last read at step t - 2, which every thread
// finished before the barrier of step t - 1.
constexpr int kSlabDepth = 4;
__device__ __forceinline__ void slab_block(const Geometry& g, int s, int t, int& I, int& J) {
    if (t <= s) {
        I = s;
        J = t;
    } else {
        I = g.nb - 1 - s;
        J = t - s - 1;
    }
}
__device__ void score_slabs(const Geometry& g, const ScoreLaunch& sc, const float* vt, float* red, const float* Wl,
                            int s, int q) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int nsteps = g.nb + 1;
    float* ring = reinterpret_cast<float*>(smem + sc.slab_off);  // [kSlabDepth][npairs][64]
    const bool active = s < sc.npairs;
    const bool single = active && (g.nb - 1 - s == s);  // middle row block of an odd nb: one pass
    auto stage = [&](int t) {
        if (active && t < nsteps && !(single && t > s)) {
            int I, J;
            slab_block(g, s, t, I, J);
            const float* src = Wl + (size_t(I) * (I + 1) / 2 + J) * 64;
            float* dst = ring + (size_t(t % kSlabDepth) * sc.npairs + s) * 64;
            if (q < 16) cp_async16(dst + 4 * q, src + 4 * q);
        }
        cp_async_commit();
    };
    stage(0);
    stage(1);
    float2 acc[kBlk / 2][4];  // rows (2k, 2k+1) x pixel p
    auto flush = [&](int I) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            float ssq = 0.f;
#pragma unroll
            for (int k = 0; k < kBlk / 2; ++k) {
                ssq = fmaf(acc[k][p].x, acc[k][p].x, ssq);
                ssq = fmaf(acc[k][p].y, acc[k][p].y, ssq);
            }
            red[I * sc.PT + q + sc.G * p] = ssq;
        }
    };
    auto zero = [&]() {
#pragma unroll
        for (int k = 0; k < kBlk / 2; ++k)
#pragma unroll
            for (int p = 0; p < 4; ++p) acc[k][p] = make_float2(0.f, 0.f);
    };
    zero();
    for (int t = 0; t < nsteps; ++t) {
        stage(t + 2);
        cp_async_wait<2>();
        __syncthreads();  // step t's blocks (every group's) have landed
        if (active && !(single && t > s)) {
            int I, J;
            slab_block(g, s, t, I, J);
            float vb[kBlk][4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float* row = vt + size_t(q + sc.G * p) * sc.Dpad + J * kBlk;
                const float4 t0 = *reinterpret_cast<const float4*>(row);
                const float4 t1 = *reinterpret_cast<const float4*>(row + 4);
                vb[0][p] = t0.x;
                vb[1][p] = t0.y;
                vb[2][p] = t0.z;
                vb[3][p] = t0.w;
                vb[4][p] = t1.x;
                vb[5][p] = t1.y;
                vb[6][p] = t1.z;
                vb[7][p] = t1.w;
            }
            const float* wb = ring + (size_t(t % kSlabDepth) * sc.npairs + s) * 64;
#pragma unroll
            for (int c = 0; c < kBlk; ++c) {
                const float4 w0 = *reinterpret_cast<const float4*>(wb + c * 8);  // broadcast in the group
                const float4 w1 = *reinterpret_cast<const float4*>(wb + c * 8 + 4);
                const float2 wp[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                                      make_float2(w1.z, w1.w)};
#pragma unroll
                for (int k = 0; k < kBlk / 2; ++k)
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        acc[k][p] = __ffma2_rn(wp[k], make_float2(vb[c][p], vb[c][p]), acc[k][p]);
            }
            if (J == I) {  // row block I complete
                flush(I);
                zero();
            }
        }
    }
    cp_async_wait<0>();
}

__global__ void __launch_bounds__(512) score_kernel(ScoreArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geometry& g = a.g;
    const ScoreLaunch& sc = a.sc;
    const int line = blockIdx.x / sc.tiles;
    const int tile = blockIdx.x - line * sc.tiles;
    const int p0 = tile * sc.PT;
    const int np = min(sc.PT, g.P - p0);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nblk = g.nb * (g.nb + 1) / 2;
    float* vt = reinterpret_cast<float*>(smem);                    // [PT][Dpad]
    float* red = vt + size_t(sc.PT) * sc.Dpad;                      // [nb][PT]
    const size_t mu_off = align_up((size_t(sc.PT) * sc.Dpad + size_t(g.nb) * sc.PT) * 4, 16);
    double* mu = reinterpret_cast<double*>(smem + mu_off);
    float* Ws = reinterpret_cast<float*>(smem + mu_off + align_up(size_t(g.Dp) * 8, 16));
    const float* Wl = a.W + size_t(line) * nblk * 64;
    if (sc.wsmem) {  // the line's packed W blocks -> smem, overlapping the pixel staging
        for (int i = tid; i < nblk * 16; i += nt) cp_async16(Ws + 4 * i, Wl + 4 * i);
        cp_async_commit();
    }
    const double* pr = a.prior + size_t(line) * g.SE;
    for (int j = tid; j < g.Dp; j += nt) mu[j] = (j < g.D) ? pr[j] : 0.0;
    __syncthreads();
    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
    // stage: v = z - mu_{t-1} rounded once to fp32; padding dims / pixels are zero
    if (!g.srp) {
        const float* src = xl + size_t(p0) * g.B;
        for (int i = tid; i < np * g.B; i += nt) {
            const int pp = i / g.B, b = i - pp * g.B;
            vt[size_t(pp) * sc.Dpad + b] = float(double(__ldg(src + i)) - mu[b]);
        }
    } else {
        for (int i = tid; i < np * g.D; i += nt) {
            const int pp = i / g.D, j = i - pp * g.D;
            vt[size_t(pp) * sc.Dpad + j] = float(srp_z(g, xl + size_t(p0 + pp) * g.B, j) - mu[j]);
        }
    }
    for (int i = tid; i < sc.PT * (g.Dp - g.D); i += nt) {
        const int pp = i / (g.Dp - g.D), d = g.D + i % (g.Dp - g.D);
        vt[size_t(pp) * sc.Dpad + d] = 0.f;
    }
    for (int i = tid; i < (sc.PT - np) * g.D; i += nt) {
        const int pp = np + i / g.D, d = i % g.D;
        vt[size_t(pp) * sc.Dpad + d] = 0.f;
    }
    if (sc.wsmem) cp_async_wait<0>();
    __syncthreads();

    const int s = tid / sc.G;
    const int q = tid - s * sc.G;
    const float* Wsrc = sc.wsmem ? Ws : Wl;
    if (!sc.wsmem) {
        score_slabs(g, sc, vt, red, Wl, s, q);
    } else if (s < sc.npairs) {
        for (int h = 0; h < 2; ++h) {
            const int I = h == 0 ? s : g.nb - 1 - s;
            if (h == 1 && I == s) break;
            float2 acc[kBlk / 2][4];  // rows (2k, 2k+1) x pixel p
#pragma unroll
            for (int k = 0; k < kBlk / 2; ++k)
#pragma unroll
                for (int p = 0; p < 4; ++p) acc[k][p] = make_float2(0.f, 0.f);
            const float* wrow = Wsrc + size_t(I * (I + 1) / 2) * 64;
            for (int J = 0; J <= I; ++J) {
                float vb[kBlk][4];
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const float* row = vt + size_t(q + sc.G * p) * sc.Dpad + J * kBlk;
                    const float4 t0 = *reinterpret_cast<const float4*>(row);
                    const float4 t1 = *reinterpret_cast<const float4*>(row + 4);
                    vb[0][p] = t0.x;
                    vb[1][p] = t0.y;
                    vb[2][p] = t0.z;
                    vb[3][p] = t0.w;
                    vb[4][p] = t1.x;
                    vb[5][p] = t1.y;
                    vb[6][p] = t1.z;
                    vb[7][p] = t1.w;
                }
                const float* wb = wrow + J * 64;
#pragma unroll
                for (int c = 0; c < kBlk; ++c) {
                    float4 w0, w1;  // column c, rows 0..3 and 4..7 (warp-uniform address: broadcast)
                    if (sc.wsmem) {
                        w0 = *reinterpret_cast<const float4*>(wb + c * 8);
                        w1 = *reinterpret_cast<const float4*>(wb + c * 8 + 4);
                    } else {
                        w0 = __ldg(reinterpret_cast<const float4*>(wb + c * 8));
                        w1 = __ldg(reinterpret_cast<const float4*>(wb + c * 8 + 4));
                    }
                    const float2 wp[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                                          make_float2(w1.z, w1.w)};
#pragma unroll
                    for (int k = 0; k < kBlk / 2; ++k)
#pragma unroll
                        for (int p = 0; p < 4; ++p)
                            acc[k][p] = __ffma2_rn(wp[k], make_float2(vb[c][p], vb[c][p]), acc[k][p]);
                }
            }
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                float ssq = 0.f;
#pragma unroll
                for (int k = 0; k < kBlk / 2; ++k) {
                    ssq = fmaf(acc[k][p].x, acc[k][p].x, ssq);
                    ssq = fmaf(acc[k][p].y, acc[k][p].y, ssq);
                }
                red[I * sc.PT + q + sc.G * p] = ssq;
            }
        }
    }
    __syncthreads();
    for (int pp = tid; pp < np; pp += nt) {
        float ssq = 0.f;
        for (int I = 0; I < g.nb; ++I) ssq += red[I * sc.PT + pp];
        a.raw[size_t(line) * g.P + p0 + pp] = sqrtf(ssq);
    }
}

// normalize_scores: per-line z-score, population std, std < 1e-12 -> zeros
// (detector.hpp:29-32).  One warp per line, fp64.
__global__ void __launch_bounds__(128) normalize_kernel(int P, const float* __restrict__ raw, int n_lines,
                                                        float* __restrict__ norm, int* __restrict__ status,
                                                        int* __restrict__ fixlist) {
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
        const double d = double(r[i]) - mean;
        v += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const double sd = sqrt(v / double(P));
    if (lane == 0 && fixlist && flat_line(mean, sd) && status[line] != -2) list_for_fixup(fixlist, status, line);
    float* out = norm + size_t(line) * P;
    for (int i = lane; i < P; i += 32) out[i] = (sd < 1e-12) ? 0.f : float((double(r[i]) - mean) / sd);
}

}  // namespace

ScoreLaunch plan_score(const Geometry& g) {
    ScoreLaunch sc{};
    sc.npairs = (g.nb + 1) / 2;
    int rep = 1;
    while (sc.npairs * 16 * rep * 2 <= 256 && rep < 8) rep *= 2;
    sc.G = 16 * rep;
    sc.PT = 4 * sc.G;
    sc.threads = sc.npairs * sc.G;
    sc.threads = (sc.threads + 31) / 32 * 32;
    sc.Dpad = g.Dp + ((4 - g.Dp) % 32 + 32) % 32;  // Dpad = 4 (mod 32)
    sc.tiles = (g.P + sc.PT - 1) / sc.PT;
    sc.smem = align_up((size_t(sc.PT) * sc.Dpad + size_t(g.nb) * sc.PT) * 4, 16) + align_up(size_t(g.Dp) * 8, 16);
    const size_t wbytes = size_t(g.nb) * (g.nb + 1) / 2 * 64 * 4;
    // stage W in smem when it is small (D <= ~180); a larger W would cost the CTA its SM-mates and
    // reads better from L2 (configs[1], D = 224: 0.50 -> 0.445 ms per 256 lines)
    sc.wsmem = (sc.smem + wbytes <= 200 * 1024 && wbytes <= 64 * 1024) ? 1 : 0;
    if (sc.wsmem) {
        sc.smem += wbytes;
    } else {  // W blocks staged per step (score_slabs)
        sc.slab_off = sc.smem;
        sc.smem += size_t(kSlabDepth) * sc.npairs * 64 * 4;
    }
    return sc;
}

size_t whiten_floats_per_line(const Geometry& g) { return size_t(g.nb) * (g.nb + 1) / 2 * 64; }

void launch_score(const Geometry& g, const ScoreLaunch& sc, const float* x, int n_per_stream, int in_stride,
                  const double* prior, const float* whiten, int n_lines_total, float* raw, cudaStream_t st) {
    {
        ensure_smem(score_kernel, 220 * 1024);
    }
    ScoreArgs a{g, sc, x, n_per_stream, in_stride, prior, whiten, raw};
    score_kernel<<<n_lines_total * sc.tiles, sc.threads, sc.smem, st>>>(a);
}

void launch_normalize(const Geometry& g, const float* raw, int n_lines_total, float* norm, int* status, int* fixlist,
                      cudaStream_t st) {
    normalize_kernel<<<(n_lines_total + 3) / 4, 128, 0, st>>>(g.P, raw, n_lines_total, norm, status, fixlist);
}

}  // namespace erxk
