// k_stats.cu — line_stats (erx.hpp:38-40) for every line of
// a window, fused with project_line (projection.hpp:31-34).
//
// Output slot per line (fp64): [c (D) | s = sum(v) (D) | S = sum(v v^T) packed
// lower (D(D+1)/2)] with v = z - c.  The scan kernel turns it into
//   mu_hat = c + s/P,  K_hat = (S - s s^T / P) / (P - 1)
// so no fp64 division runs here.
//
// Work decomposition: the lower triangle of the D x D second-moment matrix is
// tiled into 8x8 blocks (I >= J); one thread owns one block for a subset of
// pixels (G pixel groups per block when the triangle is small, several CTAs
// per line when it is large).  Pixels stream through shared memory in chunks
// of CH rows, double-buffered with cp.async so the next chunk's HBM read
// overlaps this chunk's FFMA work.  Rows are stored swizzled (low halves of
// all 8-blocks, then high halves) so 16-byte reads of distinct blocks hit
// distinct banks.
//
// Precision: c = the line's first min(32, P) pixels' mean,
// rounded to fp32; v = fl32(x - c) is the correctly rounded difference (exact
// whenever x is within a factor 2 of c); products accumulate in fp32 within
// a chunk and chunk sums in a second fp32 level.
#include "erx_common.cuh"

namespace erxk {
namespace {

__device__ __forceinline__ int spos(int d, int nb) { return ((((d >> 2) & 1) * nb) + (d >> 3)) * 4 + (d & 3); }

struct StatsArgs {
    Geometry g;
    StatsLaunch sl;
    const float* x;
    int n;
    int in_stride;
    double* stats;
};

template <int kMaxThreads, int kMinBlocks>
__global__ void __launch_bounds__(kMaxThreads, kMinBlocks) stats_kernel(StatsArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geometry& g = a.g;
    const StatsLaunch& sl = a.sl;
    const int line = blockIdx.x / sl.cpl;
    const int cta = blockIdx.x - line * sl.cpl;
    const int tid = threadIdx.x;
    const int nt = blockDim.x;

    const size_t buf_floats = size_t(sl.CH) * g.Dp;
    float* vbuf0 = reinterpret_cast<float*>(smem);
    size_t off = align_up(2 * buf_floats * 4, 16);
    const size_t red_bytes = (sl.G > 1) ? size_t(128) * 64 * 8 : 0;
    off = off > red_bytes ? off : red_bytes;
    double* colsum = reinterpret_cast<double*>(smem + off);       // [Dp] fp64 column sums of v
    float* cen = reinterpret_cast<float*>(smem + off + g.Dp * 8);  // [Dp] fp32 centre
    double* red = reinterpret_cast<double*>(smem);     // aliases the chunk buffers after the loop

    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);

    const int q_local = tid / sl.G;
    const int grp = tid - q_local * sl.G;
    const int q = cta * sl.npc + q_local;
    const bool active = (q_local < sl.npc) && (q < sl.n_pairs);
    int I = 0, J = 0;
    if (active) {  // column-major enumeration of the lower triangle of blocks
        int rem = q;
        while (rem >= g.nb - J) {
            rem -= g.nb - J;
            ++J;
        }
        I = J + rem;
    }

    if (g.Dp > g.D)  // padded dims stay zero in both buffers
        for (int i = tid; i < 2 * sl.CH * (g.Dp - g.D); i += nt) {
            const int r = i / (g.Dp - g.D), c = g.D + i % (g.Dp - g.D);
            vbuf0[size_t(r) * g.Dp + spos(c, g.nb)] = 0.f;
        }
    const int n0 = min(32, g.P);
    const bool use_async = !g.srp && (g.B % 4 == 0);
    // centre: fp64 mean of the first n0 (projected) pixels; from chunk 0 when it holds them all
    const bool cen_in_chunk = use_async && sl.CH >= n0;
    for (int j = tid; j < g.D; j += nt) {
        colsum[j] = 0.0;
        if (!cen_in_chunk) {
            double s = 0.0;
            for (int pp = 0; pp < n0; ++pp) s += proj(g, xl + size_t(pp) * g.B, j);
            cen[j] = float(s / double(n0));
        }
    }

    const int nchunks = (g.P + sl.CH - 1) / sl.CH;
    auto issue = [&](int c) {
        const int c0 = c * sl.CH, n = min(sl.CH, g.P - c0);
        float* dst = vbuf0 + (c & 1) * buf_floats;
        const int q4 = g.B / 4;
        const float* src = xl + size_t(c0) * g.B;
        for (int i = tid; i < n * q4; i += nt) {
            const int pp = i / q4, k = i - pp * q4;
            cp_async16(dst + size_t(pp) * g.Dp + ((k & 1) * g.nb + (k >> 1)) * 4, src + size_t(pp) * g.B + 4 * k);
        }
        cp_async_commit();
    };
    if (use_async) issue(0);
    __syncthreads();  // cen visible

    float acc2[kBlk][kBlk];
#pragma unroll
    for (int r = 0; r < kBlk; ++r)
#pragma unroll
        for (int c = 0; c < kBlk; ++c) acc2[r][c] = 0.f;

    for (int c = 0; c < nchunks; ++c) {
        const int c0 = c * sl.CH, n = min(sl.CH, g.P - c0);
        float* v = vbuf0 + (c & 1) * buf_floats;
        if (use_async) {
            if (c + 1 < nchunks) {
                issue(c + 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            // centre in place and take the column sums (one thread per dim; fp32 per chunk)
            for (int j = tid; j < g.D; j += nt) {
                {
                    float* col = v + spos(j, g.nb);
                    if (c == 0 && cen_in_chunk) {  // same sum, same order as the global path
                        double s = 0.0;
                        for (int pp = 0; pp < n0; ++pp) s += double(col[size_t(pp) * g.Dp]);
                        cen[j] = float(s / double(n0));
                    }
                    const float cj = cen[j];
                    float s = 0.f;
#pragma unroll 4
                    for (int pp = 0; pp < n; ++pp) {
                        const float val = col[size_t(pp) * g.Dp] - cj;
                        col[size_t(pp) * g.Dp] = val;
                        s += val;
                    }
                    colsum[j] += double(s);
                }
            }
        } else {
            for (int i = tid; i < n * g.D; i += nt) {
                const int pp = i / g.D, j = i - pp * g.D;
                v[size_t(pp) * g.Dp + spos(j, g.nb)] = float(proj(g, xl + size_t(c0 + pp) * g.B, j) - double(cen[j]));
            }
            __syncthreads();
            for (int j = tid; j < g.D; j += nt) {
                {
                    const float* col = v + spos(j, g.nb);
                    float s = 0.f;
                    for (int pp = 0; pp < n; ++pp) s += col[size_t(pp) * g.Dp];
                    colsum[j] += double(s);
                }
            }
        }
        __syncthreads();
        if (active) {
            // 8x8 outer products as paired FFMA2 (one operand broadcast from a
            // scalar register), next pixel's operands prefetched into registers
            float2 acc[kBlk][kBlk / 2];
#pragma unroll
            for (int r = 0; r < kBlk; ++r)
#pragma unroll
                for (int cc = 0; cc < kBlk / 2; ++cc) acc[r][cc] = make_float2(0.f, 0.f);
            const float* va0 = v + I * 4;
            const float* va1 = v + (g.nb + I) * 4;
            const float* vb0 = v + J * 4;
            const float* vb1 = v + (g.nb + J) * 4;
            const int G = sl.G;
            int pp = grp;
            float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
            if (pp < n) {
                const size_t o = size_t(pp) * g.Dp;
                a0 = *reinterpret_cast<const float4*>(va0 + o);
                a1 = *reinterpret_cast<const float4*>(va1 + o);
                b0 = *reinterpret_cast<const float4*>(vb0 + o);
                b1 = *reinterpret_cast<const float4*>(vb1 + o);
            }
            while (pp < n) {
                const int pn = pp + G;
                float4 na0 = a0, na1 = a1, nb0 = b0, nb1 = b1;
                if (pn < n) {
                    const size_t o = size_t(pn) * g.Dp;
                    na0 = *reinterpret_cast<const float4*>(va0 + o);
                    na1 = *reinterpret_cast<const float4*>(va1 + o);
                    nb0 = *reinterpret_cast<const float4*>(vb0 + o);
                    nb1 = *reinterpret_cast<const float4*>(vb1 + o);
                }
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                      make_float2(b1.z, b1.w)};
#pragma unroll
                for (int r = 0; r < kBlk; ++r)
#pragma unroll
                    for (int cc = 0; cc < kBlk / 2; ++cc)
                        acc[r][cc] = __ffma2_rn(make_float2(av[r], av[r]), bv[cc], acc[r][cc]);
                a0 = na0;
                a1 = na1;
                b0 = nb0;
                b1 = nb1;
                pp = pn;
            }
#pragma unroll
            for (int r = 0; r < kBlk; ++r)
#pragma unroll
                for (int cc = 0; cc < kBlk / 2; ++cc) {
                    acc2[r][2 * cc] += acc[r][cc].x;
                    acc2[r][2 * cc + 1] += acc[r][cc].y;
                }
        }
        __syncthreads();  // buffer (c & 1) is reissued at iteration c + 1
    }

    double* out = a.stats + size_t(line) * (g.SE + g.D);
    if (cta == 0) {
        for (int j = tid; j < g.D; j += nt) {
            out[j] = double(cen[j]);
            out[g.D + j] = colsum[j];
        }
    }
    if (sl.G > 1) {
#pragma unroll
        for (int r = 0; r < kBlk; ++r)
#pragma unroll
            for (int cc = 0; cc < kBlk; ++cc) red[tid * 64 + r * 8 + cc] = double(acc2[r][cc]);
        __syncthreads();
    }
    if (active && grp == 0) {
        double* S = out + 2 * g.D;
#pragma unroll
        for (int r = 0; r < kBlk; ++r) {
            const int ai = I * kBlk + r;
#pragma unroll
            for (int cc = 0; cc < kBlk; ++cc) {
                const int bj = J * kBlk + cc;
                if (ai < g.D && bj <= ai) {
                    double s;
                    if (sl.G > 1) {
                        s = 0.0;
                        for (int gg = 0; gg < sl.G; ++gg) s += red[(q_local * sl.G + gg) * 64 + r * 8 + cc];
                    } else {
                        s = double(acc2[r][cc]);
                    }
                    S[tri(ai, bj)] = s;
                }
            }
        }
    }
}

}  // namespace

StatsLaunch plan_stats(const Geometry& g) {
    StatsLaunch sl{};
    sl.minb = 1;
    sl.n_pairs = g.nb * (g.nb + 1) / 2;
    if (sl.n_pairs <= 64) {
        sl.G = 128 / sl.n_pairs;
        sl.npc = sl.n_pairs;
        sl.cpl = 1;
        sl.NT = 128;
    } else {
        // one thread per block pair, the pairs split evenly over the line's CTAs
        // up to D = 255 (configs[1]): <= 256 threads and two CTAs per SM (the second-level
        // accumulators spill to L1, touched once per chunk); beyond: up to 384 threads, one CTA
        sl.G = 1;
        const int maxnt = sl.n_pairs <= 512 ? 256 : 384;
        sl.cpl = (sl.n_pairs + maxnt - 1) / maxnt;
        sl.npc = (sl.n_pairs + sl.cpl - 1) / sl.cpl;
        sl.NT = (sl.npc + 31) / 32 * 32;
        sl.minb = maxnt <= 256 ? 2 : 1;
    }
    const size_t per_px = size_t(g.Dp) * 4 * 2;  // double buffered
    int ch = 64;
    if (sl.G > 1) ch = 256;
    size_t cap = 120 * 1024;
    if (sl.minb == 2) cap = 96 * 1024;
    while (ch > 16 && size_t(ch) * per_px > cap) ch /= 2;
    sl.CH = ch;
    size_t off = align_up(size_t(ch) * per_px, 16);
    const size_t red_bytes = (sl.G > 1) ? size_t(128) * 64 * 8 : 0;
    off = off > red_bytes ? off : red_bytes;
    sl.smem = off + size_t(g.Dp) * 12;  // colsum (fp64) + centre (fp32)
    return sl;
}

void launch_stats(const Geometry& g, const StatsLaunch& sl, const float* x, int n_per_stream, int in_stride,
                  int n_lines_total, double* stats, cudaStream_t st) {
    StatsArgs a{g, sl, x, n_per_stream, in_stride, stats};
    if (sl.minb == 2) {
        ensure_smem(stats_kernel<256, 2>, 110 * 1024);
        stats_kernel<256, 2><<<n_lines_total * sl.cpl, sl.NT, sl.smem, st>>>(a);
    } else {
        ensure_smem(stats_kernel<384, 1>, 200 * 1024);
        stats_kernel<384, 1><<<n_lines_total * sl.cpl, sl.NT, sl.smem, st>>>(a);
    }
}

}  // namespace erxk
