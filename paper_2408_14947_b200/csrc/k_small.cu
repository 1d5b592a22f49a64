// k_small.cu — the small-D path (D <= 16: the paper's default d = 5 sparse
// random projection, and narrow multispectral lines such as configs[2]).
// At these sizes the path is HBM-bound, so the design goal is
// one read of each line:
//
//   stats_small  one CTA per line: cp.async-stages pixel rows, projects each
//                pixel once (project_line, projection.hpp:31-34; fp64 sums),
//                accumulates sum(v) and sum(v v^T) with v = z - c
//                (line_stats, erx.hpp:38-40), and writes v (fp32, dim-major)
//                to a small per-line cache — D floats per pixel instead of B.
//                Identity projection (narrow lines, configs[2]): warps stream
//                their own chunks, a lane per pixel, no per-chunk barrier;
//                SRP (d = 5 default): (dim, pixel) items over shared stages;
//   score_small  one CTA per line: reads the cache, whitens with W = L^{-1}
//                (forward_substitute, linalg.hpp:21), and z-normalises the
//                line in the same kernel (normalize_scores, detector.hpp:29-32).
//
// Stats slot contract as k_stats.cu: [c | s | S packed lower], fp64.
#include <algorithm>
#include <cstdlib>

#include "erx_common.cuh"
#include "tc_common.cuh"

namespace erxk {
namespace {

constexpr int kSmallThreads = 256;       // score_small
constexpr int kStatsSmallThreads = 128;  // stats_small: 4 warps per line, two lines per SM

struct SmallArgs {
    Geometry g;
    SmallLaunch sm;
    const float* x;
    int n;
    int in_stride;
    double* stats;
    float* vcache;  // [line][D][P]
};

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem_src));
}

// One CTA (kStatsSmallThreads / 32 warps) per line.  The warps stream the line's pixel chunks
// round-robin, each through its own double-buffered cp.async stage (no CTA barrier inside the line):
// a lane projects whole pixels (every output dim, fp64), writes v = z - c to the cache and keeps fp32
// partial sums of v and v v^T; one barrier at the end reduces the warps' partials in fixed order.
// Warp 0 derives the centre c (fp64 mean of the first min(32, P) projected pixels) while the first
// chunks load.
template <int DM>
__global__ void __launch_bounds__(kStatsSmallThreads, DM <= 8 ? 4 : (DM <= 10 ? 2 : 1)) stats_small_kernel(SmallArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int kW = kStatsSmallThreads / 32;
    constexpr int DT = DM * (DM + 1) / 2;
    const Geometry& g = a.g;
    const int line = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = g.D, B = g.B, P = g.P;
    const int CH = a.sm.CH;  // pixels per warp chunk
    float* buf = reinterpret_cast<float*>(smem) + size_t(warp) * 2 * CH * B;  // [2][CH][B] per warp
    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
    float* vc = a.vcache + size_t(line) * D * P;

    __shared__ double cen_s[DM];
    // SRP table padded to srp_wmax entries per dim (weight 0 past a dim's nonzeros, band = its first
    // band), [DM][wmax] in shared memory after the stages: the dims' chains interleave, and a zero
    // term leaves the fp64 sum unchanged (same value as the sequential CSC sum)
    const int WM = g.srp ? g.srp_wmax : 0;
    double* ew = reinterpret_cast<double*>(smem + a.sm.smem_stats - size_t(DM) * WM * 12);
    int* eb = reinterpret_cast<int*>(ew + DM * WM);
    auto zrow = [&](const float* row, double (&z)[DM]) {  // all projected dims of a pixel row, fp64
        if (g.srp) {
            double acc[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j) acc[j] = 0.0;
            for (int k = 0; k < WM; ++k) {
#pragma unroll
                for (int j = 0; j < DM; ++j)
                    if (j < D) acc[j] += double(row[eb[j * WM + k]]) * ew[j * WM + k];
            }
#pragma unroll
            for (int j = 0; j < DM; ++j) z[j] = acc[j] * g.srp_scale;
        } else {
#pragma unroll
            for (int j = 0; j < DM; ++j) z[j] = (j < D) ? double(row[j]) : 0.0;
        }
    };
    const int nck = (P + CH - 1) / CH;
    auto issue = [&](int ci, int b) {
        const int p0 = ci * CH, n = min(CH, P - p0);
        const float* src = xl + size_t(p0) * B;
        float* dst = buf + b * CH * B;
        const int nfl = n * B;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (nfl & 3) == 0) {
            for (int i = lane; i < nfl / 4; i += 32) cp_async16(dst + 4 * i, src + 4 * i);
        } else {
            for (int i = lane; i < nfl; i += 32) cp_async4(dst + i, src + i);
        }
        cp_async_commit();
    };
    // each warp keeps two chunks in flight: chunk ci in stage it & 1, refilled with ci + 2 kW
    if (warp < nck) issue(warp, 0);
    if (warp + kW < nck) issue(warp + kW, 1);
    for (int q = tid; q < D * WM; q += kStatsSmallThreads) {
        const int j = q / WM, k = q - j * WM;
        const int b0 = __ldg(g.srp_ptr + j), nz = __ldg(g.srp_ptr + j + 1) - b0;
        eb[j * WM + k] = nz > 0 ? __ldg(g.srp_band + b0 + (k < nz ? k : 0)) : 0;
        ew[j * WM + k] = k < nz ? double(__ldg(g.srp_w + b0 + k)) : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
        // centre: lane p < n0 projects pixel p (from warp 0's first staged chunk when it holds them,
        // else from global memory), fp64 butterfly sum
        const int n0 = min(32, P);
        const bool staged = CH >= n0;
        if (staged) {
            if (kW < nck) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncwarp();
        }
        double z[DM];
        const int pl = min(lane, n0 - 1);
        zrow(staged ? buf + pl * B : xl + size_t(pl) * B, z);
#pragma unroll
        for (int j = 0; j < DM; ++j) {
            double v = lane < n0 ? z[j] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && j < D) cen_s[j] = v / double(n0);
        }
    }
    __syncthreads();
    // fp64 partial sums: the fp32 products v_a v_b are exact in fp64 (48-bit significands), so the
    // only rounding left is v = fl32(z - c) itself (an ill-conditioned background, e.g. radiance-scale
    // lines with little sensor noise, amplifies fp32 product rounding ~1e5-fold into the scores)
    double s1[DM], s2[DT];
#pragma unroll
    for (int j = 0; j < DM; ++j) s1[j] = 0.0;
#pragma unroll
    for (int j = 0; j < DT; ++j) s2[j] = 0.0;
    for (int ci = warp, it = 0; ci < nck; ci += kW, ++it) {
        if (ci + kW < nck) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncwarp();
        const float* st = buf + (it & 1) * CH * B;
        const int p0 = ci * CH, n = min(CH, P - p0);
        for (int pp = lane; pp < n; pp += 32) {
            double z[DM];
            zrow(st + pp * B, z);
            float v[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j) {
                v[j] = 0.f;
                if (j < D) {
                    v[j] = float(z[j] - cen_s[j]);
                    vc[size_t(j) * P + p0 + pp] = v[j];
                }
            }
#pragma unroll
            for (int i = 0; i < DM; ++i) {
                const double vi = double(v[i]);
                s1[i] += vi;
#pragma unroll
                for (int j = 0; j <= i; ++j) s2[i * (i + 1) / 2 + j] = fma(vi, double(v[j]), s2[i * (i + 1) / 2 + j]);
            }
        }
        __syncwarp();  // the stage is refilled next
        if (ci + 2 * kW < nck) issue(ci + 2 * kW, it & 1);
    }
    // warp partials in fp64 (over the stage buffers, once every warp is done with them), then the
    // warps in fixed order
    const int NT = D * (D + 1) / 2, NV = D + NT;
    double (*red)[DM + DT] = reinterpret_cast<double (*)[DM + DT]>(smem);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < DM; ++i) {
        double v = s1[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && i < D) red[warp][i] = v;
    }
#pragma unroll
    for (int i = 0; i < DM; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double v = s2[i * (i + 1) / 2 + j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && i < D) red[warp][D + i * (i + 1) / 2 + j] = v;
        }
    __syncthreads();
    double* out = a.stats + size_t(line) * (g.SE + D);
    for (int q = tid; q < NV; q += kStatsSmallThreads) {
        double v = 0.0;
        for (int w = 0; w < kW; ++w) v += red[w][q];
        if (q < D) {
            out[q] = cen_s[q];
            out[D + q] = v;
        } else {
            out[2 * D + (q - D)] = v;
        }
    }
}

// Identity projection, a WARP per line (D = B <= 12: configs[2]).  The CTA-per-line kernel above spends
// its time outside the rank-1 updates on narrow lines (ncu, configs[2]: 247 registers -> 8 warps per SM,
// 24 % of the stalls at its CTA barriers, and 40 % of its instructions in the 65-value block reduction
// every 8 pixels per lane).  Here each warp streams a whole line through its own double-buffered
// cp.async stage -- no CTA barrier anywhere, one butterfly reduction per line (32 pixels per lane at
// P = 1024) -- and the warps of an SM hide one another's start-up latency.  Same per-pixel arithmetic:
// centre = fp64 mean of the first min(32, P) pixels, v = fl32(z - c), exact fp64 products.
// EX: D == DM (configs[2]'s 10 bands, d = 5): every `j < D` folds at compile time.
template <int DM, bool EX>
__global__ void __launch_bounds__(kStatsSmallThreads, 2) stats_small_wl_kernel(SmallArgs a, int n_lines) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int kW = kStatsSmallThreads / 32;
    constexpr int DT = DM * (DM + 1) / 2;
    const Geometry& g = a.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int line = blockIdx.x * kW + warp;
    if (line >= n_lines) return;  // (no CTA barrier below)
    const int D = EX ? DM : g.D, B = EX ? DM : g.B, P = g.P;  // (identity projection: B == D)
    const int CH = a.sm.CH;
    float* buf = reinterpret_cast<float*>(smem) + size_t(warp) * 2 * CH * B;  // [2][CH][B]
    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
    float* vc = a.vcache + size_t(line) * D * P;
    const int nck = (P + CH - 1) / CH;
    auto issue = [&](int ci, int b) {
        const int p0 = ci * CH, n = min(CH, P - p0);
        const float* src = xl + size_t(p0) * B;
        float* dst = buf + b * CH * B;
        const int nfl = n * B;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (nfl & 3) == 0) {
            for (int i = lane; i < nfl / 4; i += 32) cp_async16(dst + 4 * i, src + 4 * i);
        } else {
            for (int i = lane; i < nfl; i += 32) cp_async4(dst + i, src + i);
        }
        cp_async_commit();
    };
    issue(0, 0);
    if (1 < nck) issue(1, 1);
    if (1 < nck) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncwarp();
    // centre: lane p < n0 holds pixel p of chunk 0 (CH >= 32 or CH >= P), fp64 butterfly sum
    double cen[DM];
    {
        const int n0 = min(32, P);
        const float* row = buf + min(lane, n0 - 1) * B;
#pragma unroll
        for (int j = 0; j < DM; ++j) {
            double v = (lane < n0 && j < D) ? double(row[j]) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            cen[j] = v / double(n0);
        }
    }
    double s1[DM], s2[DT];
#pragma unroll
    for (int j = 0; j < DM; ++j) s1[j] = 0.0;
#pragma unroll
    for (int j = 0; j < DT; ++j) s2[j] = 0.0;
    for (int ci = 0; ci < nck; ++ci) {
        if (ci + 1 < nck) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncwarp();
        const float* st = buf + (ci & 1) * CH * B;
        const int p0 = ci * CH, n = min(CH, P - p0);
        // software pipeline over the lane's pixels: the load -> fp64 subtract -> fp32 round -> cache
        // store chain of pixel pp + 32 is issued before the rank-1 updates of pixel pp (ncu: half of
        // the stall samples sat on that chain when each iteration ran it first)
        // (straight-line: a warp-uniform `if (j < D)` around each dim's chain compiles to a branch per dim,
        // which serialises the ten load -> convert -> subtract -> convert chains; loads are clamped to a
        // real band instead and padded dims zeroed by a select)
        auto prep = [&](int pp, float (&v)[DM]) {
            const float* row = st + pp * B;
            float xr[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j) xr[j] = row[min(j, D - 1)];
#pragma unroll
            for (int j = 0; j < DM; ++j) v[j] = float(double(xr[j]) - cen[j]);
            float* vp = vc + p0 + pp;
#pragma unroll
            for (int j = 0; j < DM; ++j) {
                if (j < D) *vp = v[j];
                else v[j] = 0.f;
                vp += P;  // (one pointer add per dim instead of a 64-bit multiply)
            }
        };
        float vn[DM];
#pragma unroll
        for (int j = 0; j < DM; ++j) vn[j] = 0.f;
        if (lane < n) prep(lane, vn);
        for (int pp = lane; pp < n; pp += 32) {
            double vd[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j) vd[j] = double(vn[j]);
            if (pp + 32 < n) prep(pp + 32, vn);
#pragma unroll
            for (int i = 0; i < DM; ++i) {
                s1[i] += vd[i];
#pragma unroll
                for (int j = 0; j <= i; ++j) s2[i * (i + 1) / 2 + j] = fma(vd[i], vd[j], s2[i * (i + 1) / 2 + j]);
            }
        }
        __syncwarp();  // the stage is refilled next
        if (ci + 2 < nck) issue(ci + 2, ci & 1);
    }
    // one butterfly per value (every lane ends with the line's total), staged through the warp's
    // (now idle) buffer so the slot is written with coalesced stores
    double* red = reinterpret_cast<double*>(buf);
#pragma unroll
    for (int i = 0; i < DM; ++i) {
        double v = s1[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && i < D) {
            red[i] = cen[i];
            red[D + i] = v;
        }
    }
#pragma unroll
    for (int i = 0; i < DM; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double v = s2[i * (i + 1) / 2 + j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && i < D) red[2 * D + i * (i + 1) / 2 + j] = v;
        }
    __syncwarp();
    double* out = a.stats + size_t(line) * (g.SE + D);
    const int NV = 2 * D + D * (D + 1) / 2;
    for (int q = lane; q < NV; q += 32) out[q] = red[q];
}

// SRP variant (the reference default, d = 5): one CTA per line, all threads share each staged chunk;
// work items are (dim, pixel) pairs, consecutive threads on consecutive pixels of one dim, so a thread
// sums only its dim's nonzeros (measured faster than whole-pixel lanes when B >> D: configs[3] d = 5
// 0.180 vs 0.252 ms per 2048 lines).
template <int DM>
__global__ void __launch_bounds__(kStatsSmallThreads) stats_small_srp_kernel(SmallArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geometry& g = a.g;
    const SmallLaunch& sm = a.sm;  // sm.CH2: pixels per stage
    const int line = blockIdx.x;
    const int tid = threadIdx.x;
    const int D = g.D, B = g.B;
    const int NT = D * (D + 1) / 2;
    float* stage = reinterpret_cast<float*>(smem);                                  // [2][CH][B]
    double* red = reinterpret_cast<double*>(smem + align_up(size_t(2) * sm.CH2 * B * 4, 16));  // [warps][D + NT]
    float* vs = reinterpret_cast<float*>(red + (kStatsSmallThreads / 32) * (D + NT));          // [CH][DM]
    __shared__ double cen_s[16];
    __shared__ double zc[32 * 16];
    // W's CSC in shared memory: weights (fp64) then bands, then the D + 1 column starts
    double* sw = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(vs) + align_up(size_t(sm.CH2) * DM * 4, 16));
    int* sb = reinterpret_cast<int*>(sw + g.srp_nnz);
    int* sp = sb + g.srp_nnz;
    for (int q = threadIdx.x; q < g.srp_nnz; q += kStatsSmallThreads) {
        sw[q] = double(__ldg(g.srp_w + q));
        sb[q] = __ldg(g.srp_band + q);
    }
    for (int q = threadIdx.x; q <= g.D; q += kStatsSmallThreads) sp[q] = g.srp ? __ldg(g.srp_ptr + q) : 0;
    // z_j of a staged pixel row: two interleaved fp64 partial sums (halves the dependent chain)
    auto srp_dot = [&](const float* row, int j) {
        double z0 = 0.0, z1 = 0.0;
        const int k1 = sp[j + 1];
        int k = sp[j];
        for (; k + 1 < k1; k += 2) {
            z0 += double(row[sb[k]]) * sw[k];
            z1 += double(row[sb[k + 1]]) * sw[k + 1];
        }
        if (k < k1) z0 += double(row[sb[k]]) * sw[k];
        return (z0 + z1) * g.srp_scale;
    };
    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
    float* vc = a.vcache + size_t(line) * D * g.P;
    const int n0 = min(32, g.P);
    // 16-byte rows: a chunk is ONE bulk copy (cp.async.bulk, mbarrier transaction count) issued by thread 0
    // instead of ~40 cp.async per thread (ncu, configs[3] d = 5: 17 % of the kernel's instructions)
    const bool use_bulk = (B % 4) == 0 && (reinterpret_cast<uintptr_t>(xl) & 15) == 0;
    __shared__ __align__(8) uint64_t fullb[2];
    if (tid == 0) {
        tc::mbar_init(&fullb[0], 1);
        tc::mbar_init(&fullb[1], 1);
        tc::fence_barrier_init();
    }
    __syncthreads();
    const int nchunks = (g.P + sm.CH2 - 1) / sm.CH2;
    auto issue = [&](int c) {
        const int c0 = c * sm.CH2, n = min(sm.CH2, g.P - c0);
        float* dst = stage + (c & 1) * sm.CH2 * B;
        const float* src = xl + size_t(c0) * B;
        if (use_bulk) {
            if (tid == 0) {
                tc::fence_proxy_async();  // the stage's earlier generic-proxy reads (ordered by the CTA barrier)
                tc::mbar_expect_tx(&fullb[c & 1], uint32_t(n) * B * 4);
                tc::bulk_g2s(dst, src, uint32_t(n) * B * 4, &fullb[c & 1]);
            }
        } else {
            for (int i = tid; i < n * B; i += kStatsSmallThreads) dst[i] = __ldg(src + i);
        }
    };
    issue(0);
    __syncthreads();
    constexpr int DT = DM * (DM + 1) / 2;

    // per-thread partial sums over its pixels (few per thread), fp64 (exact products, as above)
    double s1[DM], s2[DT];
#pragma unroll
    for (int j = 0; j < DM; ++j) s1[j] = 0.0;
#pragma unroll
    for (int j = 0; j < DT; ++j) s2[j] = 0.0;

    for (int c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) issue(c + 1);
        if (use_bulk) tc::mbar_wait(&fullb[c & 1], uint32_t(c >> 1) & 1u);
        else __syncthreads();
        const int c0 = c * sm.CH2, n = min(sm.CH2, g.P - c0);
        const float* st = stage + (c & 1) * sm.CH2 * B;
        if (c == 0) {  // centre: fp64 mean of the first min(32, P) projected pixels, from the staged chunk
            for (int i = tid; i < n0 * D; i += kStatsSmallThreads) {
                const int j = i / n0, pp = i - j * n0;
                const float* row = st + pp * B;
                const double z = g.srp ? srp_dot(row, j) : double(row[j]);
                zc[pp * 16 + j] = z;
            }
            __syncthreads();
            if (tid < D) {
                double s = 0.0;
                for (int pp = 0; pp < n0; ++pp) s += zc[pp * 16 + tid];
                cen_s[tid] = s / double(n0);
            }
            __syncthreads();
        }
        // projection: one (dim, pixel) item per thread, consecutive threads on consecutive
        // pixels of one dim (coalesced cache writes, warp-uniform nnz loop bounds)
        // (j = i / n by a float reciprocal: (i + 0.5) / n is at least 0.5 / n away from an integer)
        const float rn = 1.f / float(n);
        for (int i = tid; i < n * D; i += kStatsSmallThreads) {
            const int j = int((float(i) + 0.5f) * rn), pp = i - j * n;
            const float* row = st + pp * B;
            const double z = g.srp ? srp_dot(row, j) : double(row[j]);
            const float v = float(z - cen_s[j]);
            vs[pp * DM + j] = v;
            vc[size_t(j) * g.P + c0 + pp] = v;
        }
        __syncthreads();
        // rank-1 updates: one pixel per thread
        for (int pp = tid; pp < n; pp += kStatsSmallThreads) {
            float v[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j) v[j] = (j < D) ? vs[pp * DM + j] : 0.f;
#pragma unroll
            for (int i = 0; i < DM; ++i) {
                const double vi = double(v[i]);
                s1[i] += vi;
#pragma unroll
                for (int j = 0; j <= i; ++j) s2[i * (i + 1) / 2 + j] = fma(vi, double(v[j]), s2[i * (i + 1) / 2 + j]);
            }
        }
        __syncthreads();  // stage (c & 1) and vs are refilled at iteration c + 1
    }
    // block reduction in fp64: warp shuffles, then one partial per warp in smem (fixed order)
    const int lane = tid & 31, warp = tid >> 5;
    const int NV = D + NT;
#pragma unroll
    for (int i = 0; i < DM; ++i) {
        if (i < D) {
            double v = double(s1[i]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[warp * NV + i] = v;
        }
    }
#pragma unroll
    for (int i = 0; i < DM; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j)
            if (i < D) {
                double v = double(s2[i * (i + 1) / 2 + j]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) red[warp * NV + D + i * (i + 1) / 2 + j] = v;
            }
    __syncthreads();
    double* out = a.stats + size_t(line) * (g.SE + D);
    for (int q = tid; q < NV; q += kStatsSmallThreads) {
        double v = 0.0;
        for (int w = 0; w < kStatsSmallThreads / 32; ++w) v += red[w * NV + q];
        if (q < D) {
            out[q] = cen_s[q];
            out[D + q] = v;
        } else {
            out[2 * D + (q - D)] = v;
        }
    }
}

// SRP with a WARP per line (the reference default d = 5 on batched windows: configs[3]).  The CTA-per-line
// kernel above is issue-bound (ncu: 39 % of its instructions in the per-item sparse dot products, three CTA
// barriers per 44-pixel chunk, 58 % issue-active at 76 % of the HBM peak).  Here each warp streams its own
// line in 32-pixel chunks -- one bulk copy per chunk into the warp's two stages, its own mbarriers, no CTA
// barrier -- and a lane owns a pixel: the dims' sums run as DM independent fp64 chains over a k-major
// padded table {band offset, sign} read by broadcast loads (padding: sign 0 on the dim's first band), then
// v = fl32(z - c), the cache store and the exact fp64 rank-1 updates; one butterfly per line.
// z sums at most srp_wmax fp32 values in fp64 (exact for any realistic exponent spread), the centre is the
// CTA kernel's sequential fp64 mean of the first min(32, P) pixels.
constexpr int kSrpWlWarps = 4;
struct SrpEnt {
    uint32_t off;  // band * 4 (byte offset inside a pixel row)
    float w;       // +1, -1, or 0 (padding)
};

template <int DM, bool EX>
__global__ void __launch_bounds__(kSrpWlWarps * 32, 2) stats_small_srp_wl_kernel(SmallArgs a, int n_lines) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[kSrpWlWarps][2];
    constexpr int DT = DM * (DM + 1) / 2;
    const Geometry& g = a.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = EX ? DM : g.D, B = g.B, P = g.P, WM = g.srp_wmax;
    const size_t stage_fl = size_t(32) * B;
    float* stage = reinterpret_cast<float*>(smem) + size_t(warp) * 2 * stage_fl;  // [2][32][B]
    SrpEnt* ent = reinterpret_cast<SrpEnt*>(smem + size_t(kSrpWlWarps) * 2 * stage_fl * 4);  // [WM][DM]
    for (int q = tid; q < WM * DM; q += kSrpWlWarps * 32) {
        const int k = q / DM, j = q - k * DM;
        SrpEnt e{0u, 0.f};
        if (j < D) {
            const int b0 = __ldg(g.srp_ptr + j), nz = __ldg(g.srp_ptr + j + 1) - b0;
            if (nz > 0) {
                e.off = uint32_t(__ldg(g.srp_band + b0 + (k < nz ? k : 0))) * 4u;
                e.w = k < nz ? __ldg(g.srp_w + b0 + k) : 0.f;
            }
        }
        ent[q] = e;
    }
    if (tid < kSrpWlWarps * 2) tc::mbar_init(&full[tid >> 1][tid & 1], 1);
    tc::fence_barrier_init();
    __syncthreads();
    const int line = blockIdx.x * kSrpWlWarps + warp;
    if (line >= n_lines) return;  // (no CTA barrier below)
    const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
    float* vc = a.vcache + size_t(line) * D * P;
    const int nck = (P + 31) / 32;
    auto issue = [&](int c) {
        if (lane == 0) {
            const uint32_t bytes = uint32_t(min(32, P - c * 32)) * B * 4;
            tc::fence_proxy_async();  // the stage's earlier generic-proxy reads (ordered by __syncwarp)
            tc::mbar_expect_tx(&full[warp][c & 1], bytes);
            tc::bulk_g2s(stage + (c & 1) * stage_fl, xl + size_t(c) * 32 * B, bytes, &full[warp][c & 1]);
        }
    };
    issue(0);
    if (nck > 1) issue(1);
    const double scale = g.srp_scale;
    // z of one staged pixel row: DM independent chains, every table entry one broadcast load
    auto zrow = [&](const unsigned char* row, double (&z)[DM]) {
#pragma unroll
        for (int j = 0; j < DM; ++j) z[j] = 0.0;
        for (int k = 0; k < WM; ++k) {
            const SrpEnt* ek = ent + k * DM;
#pragma unroll
            for (int j = 0; j < DM; ++j) {
                const SrpEnt e = ek[j];
                z[j] += double(*reinterpret_cast<const float*>(row + e.off) * e.w);
            }
        }
#pragma unroll
        for (int j = 0; j < DM; ++j) z[j] *= scale;
    };
    double cen[DM];
    double s1[DM], s2[DT];
#pragma unroll
    for (int j = 0; j < DM; ++j) s1[j] = 0.0;
#pragma unroll
    for (int j = 0; j < DT; ++j) s2[j] = 0.0;
    for (int c = 0; c < nck; ++c) {
        tc::mbar_wait(&full[warp][c & 1], uint32_t(c >> 1) & 1u);
        const int n = min(32, P - c * 32);
        const unsigned char* row =
            reinterpret_cast<const unsigned char*>(stage + (c & 1) * stage_fl + size_t(min(lane, n - 1)) * B);
        double z[DM];
        zrow(row, z);
        if (c == 0) {
            // centre: the fp64 mean of the first n0 = min(32, P) projected pixels, summed in pixel order
            // (the CTA kernel's order) by broadcast shuffles
            const int n0 = n;
#pragma unroll
            for (int j = 0; j < DM; ++j) {
                double sc = 0.0;
                for (int pp = 0; pp < n0; ++pp) sc += __shfl_sync(0xffffffffu, z[j], pp);
                cen[j] = sc / double(n0);
            }
        }
        if (lane < n) {
            double vd[DM];
            float* vp = vc + c * 32 + lane;
#pragma unroll
            for (int j = 0; j < DM; ++j) {
                const float v = float(z[j] - cen[j]);
                if (j < D) *vp = v;
                vp += P;
                vd[j] = (j < D) ? double(v) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < DM; ++i) {
                s1[i] += vd[i];
#pragma unroll
                for (int j = 0; j <= i; ++j) s2[i * (i + 1) / 2 + j] = fma(vd[i], vd[j], s2[i * (i + 1) / 2 + j]);
            }
        }
        __syncwarp();  // the stage is refilled next
        if (c + 2 < nck) issue(c + 2);
    }
    // one butterfly per value, staged through the warp's (idle) buffer for coalesced stores of the slot
    __syncwarp();
    double* red = reinterpret_cast<double*>(stage);
#pragma unroll
    for (int i = 0; i < DM; ++i) {
        double v = s1[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && i < D) {
            red[i] = cen[i];
            red[D + i] = v;
        }
    }
#pragma unroll
    for (int i = 0; i < DM; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double v = s2[i * (i + 1) / 2 + j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && i < D) red[2 * D + i * (i + 1) / 2 + j] = v;
        }
    __syncwarp();
    double* out = a.stats + size_t(line) * (g.SE + D);
    const int NV = 2 * D + D * (D + 1) / 2;
    for (int q = lane; q < NV; q += 32) out[q] = red[q];
}

// score_small + normalize.  W: packed lower 8x8 blocks (column-major inside).
template <int DM>
__global__ void __launch_bounds__(kSmallThreads, 4) score_small_kernel(Geometry g, const double* __restrict__ stats,
                                                                    const double* __restrict__ prior,
                                                                    const float* __restrict__ Wp,
                                                                    const float* __restrict__ vcache,
                                                                    float* __restrict__ raw, float* __restrict__ norm,
                                                                    int* __restrict__ status, int* __restrict__ fixlist) {
    extern __shared__ __align__(16) unsigned char smem[];
    float* dl = reinterpret_cast<float*>(smem);  // raw scores of the line [P]
    __shared__ float Wd[16][16];
    __shared__ float off[16];
    __shared__ double red[8];
    __shared__ double mean_s, sd_s;
    const int line = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = g.D;
    const int nblk = g.nb * (g.nb + 1) / 2;
    const float* W = Wp + size_t(line) * nblk * 64;
    for (int i = tid; i < 256; i += kSmallThreads) {
        const int r = i / 16, c = i % 16;
        float w = 0.f;
        if (r < D && c <= r) {
            const int I = r / 8, J = c / 8;
            w = W[(I * (I + 1) / 2 + J) * 64 + (c % 8) * 8 + (r % 8)];
        }
        Wd[r][c] = w;
    }
    if (tid < 16) {
        // u = v - (mu_{t-1} - c_t): v is centred on this line's c_t
        const double* st = stats + size_t(line) * (g.SE + D);
        const double* pr = prior + size_t(line) * g.SE;
        off[tid] = (tid < D) ? float(pr[tid] - st[tid]) : 0.f;
    }
    __syncthreads();
    const float* vc = vcache + size_t(line) * D * g.P;
    double ls = 0.0;
    // kPX pixels per thread per pass, every cache load of the pass issued before the first is used
    constexpr int kPX = DM <= 8 ? 4 : 2;
    for (int p0 = tid; p0 < g.P; p0 += kPX * kSmallThreads) {
        float u[kPX][DM];
#pragma unroll
        for (int x = 0; x < kPX; ++x) {
            const int p = min(p0 + x * kSmallThreads, g.P - 1);
            // (unconditional loads clamped to the last real dim: a warp-uniform `j < D` around each load
            // compiles to a branch per dim; W = 0 in the padded columns)
            const float* vp = vc + p;
#pragma unroll
            for (int j = 0; j < DM; ++j) {
                u[x][j] = __ldg(vp) - off[j];
                if (j + 1 < D) vp += g.P;
            }
        }
#pragma unroll
        for (int x = 0; x < kPX; ++x) {
            const int p = p0 + x * kSmallThreads;
            float ssq = 0.f;
#pragma unroll
            for (int r = 0; r < DM; ++r) {
                if (r < D) {
                    float m = 0.f;
#pragma unroll
                    for (int c = 0; c <= r; ++c) m = fmaf(Wd[r][c], u[x][c], m);
                    ssq = fmaf(m, m, ssq);
                }
            }
            if (p < g.P) {
                const float d = sqrtf(ssq);
                dl[p] = d;
                raw[size_t(line) * g.P + p] = d;
                ls += double(d);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    if (lane == 0) red[warp] = ls;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kSmallThreads / 32; ++w) s += red[w];
        mean_s = s / double(g.P);
    }
    __syncthreads();
    const double mean = mean_s;
    double lv = 0.0;
    for (int p = tid; p < g.P; p += kSmallThreads) {
        const double dd = double(dl[p]) - mean;
        lv += dd * dd;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lv += __shfl_xor_sync(0xffffffffu, lv, o);
    __syncthreads();
    if (lane == 0) red[warp] = lv;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kSmallThreads / 32; ++w) s += red[w];
        sd_s = sqrt(s / double(g.P));
    }
    __syncthreads();
    const double sd = sd_s;
    if (tid == 0 && fixlist && flat_line(mean, sd) && status[line] != -2) list_for_fixup(fixlist, status, line);
    for (int p = tid; p < g.P; p += kSmallThreads)
        norm[size_t(line) * g.P + p] = (sd < 1e-12) ? 0.f : float((double(dl[p]) - mean) / sd);
}

// score_small + normalize with a WARP per line (narrow lines): W (packed lower, <= 78 values) lives in
// registers, the line's raw scores in the warp's own shared-memory strip; no CTA barrier.  The mean / std
// sums are fp64 per lane then one butterfly (the CTA kernel sums per thread, per warp, then over warps:
// a different, equally fixed order).
constexpr int kScoreWlWarps = 4;
template <int DM, bool EX>
__global__ void __launch_bounds__(kScoreWlWarps * 32, 4) score_small_wl_kernel(Geometry g, const double* __restrict__ stats,
                                                                           const double* __restrict__ prior,
                                                                           const float* __restrict__ Wp,
                                                                           const float* __restrict__ vcache,
                                                                           float* __restrict__ raw, float* __restrict__ norm,
                                                                           int* __restrict__ status, int* __restrict__ fixlist,
                                                                           int n_lines) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int DT = DM * (DM + 1) / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int line = blockIdx.x * kScoreWlWarps + warp;
    if (line >= n_lines) return;
    const int D = EX ? DM : g.D, P = g.P;
    float* dl = reinterpret_cast<float*>(smem) + size_t(warp) * P;  // raw scores of the line [P]
    const int nblk = g.nb * (g.nb + 1) / 2;
    const float* W = Wp + size_t(line) * nblk * 64;
    float Wr[DT], off[DM];
#pragma unroll
    for (int r = 0; r < DM; ++r) {
#pragma unroll
        for (int c = 0; c <= r; ++c) {
            const int I = r / 8, J = c / 8;
            const float w = __ldg(W + (I * (I + 1) / 2 + J) * 64 + (c % 8) * 8 + (r % 8));  // (the blocks cover Dp >= DM rows)
            Wr[r * (r + 1) / 2 + c] = (r < D) ? w : 0.f;
        }
    }
    {
        // u = v - (mu_{t-1} - c_t): v is centred on this line's c_t
        const double* st = stats + size_t(line) * (g.SE + D);
        const double* pr = prior + size_t(line) * g.SE;
#pragma unroll
        for (int j = 0; j < DM; ++j) off[j] = (j < D) ? float(__ldg(pr + j) - __ldg(st + j)) : 0.f;
    }
    const float* vc = vcache + size_t(line) * D * P;
    double ls = 0.0;
    constexpr int kPX = DM <= 8 ? 4 : 2;  // pixels per lane per pass, all their loads in flight first
    for (int p0 = lane; p0 < P; p0 += kPX * 32) {
        float u[kPX][DM];
#pragma unroll
        for (int x = 0; x < kPX; ++x) {
            const int p = min(p0 + x * 32, P - 1);
            // (unconditional clamped loads: no branch per dim; W = 0 in the padded columns)
            const float* vp = vc + p;
#pragma unroll
            for (int j = 0; j < DM; ++j) {
                u[x][j] = __ldg(vp) - off[j];
                if (j + 1 < D) vp += P;  // (clamped to the last real dim)
            }
        }
#pragma unroll
        for (int x = 0; x < kPX; ++x) {
            const int p = p0 + x * 32;
            float ssq = 0.f;
#pragma unroll
            for (int r = 0; r < DM; ++r) {
                float m = 0.f;
#pragma unroll
                for (int c = 0; c <= r; ++c) m = fmaf(Wr[r * (r + 1) / 2 + c], u[x][c], m);
                ssq = fmaf(m, m, ssq);  // (rows r >= D: W = 0, m = 0)
            }
            if (p < P) {
                const float d = sqrtf(ssq);
                dl[p] = d;
                raw[size_t(line) * P + p] = d;
                ls += double(d);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    const double mean = ls / double(P);
    __syncwarp();
    double lv = 0.0;
    for (int p = lane; p < P; p += 32) {
        const double dd = double(dl[p]) - mean;
        lv += dd * dd;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lv += __shfl_xor_sync(0xffffffffu, lv, o);
    const double sd = sqrt(lv / double(P));
    if (lane == 0 && fixlist && flat_line(mean, sd) && status[line] != -2) list_for_fixup(fixlist, status, line);
    for (int p = lane; p < P; p += 32)
        norm[size_t(line) * P + p] = (sd < 1e-12) ? 0.f : float((double(dl[p]) - mean) / sd);
}

}  // namespace

bool small_path(const Geometry& g) { return g.D <= 16; }

constexpr int kSmallWlMinLines = 2048;
static bool small_wl() {  // A/B switch of the warp-per-line kernels (default on)
    static const bool on = [] {
        const char* e = std::getenv("ERX_SMALL_WL");
        return !(e && e[0] == '0');
    }();
    return on;
}

SmallLaunch plan_small(const Geometry& g, size_t capacity_lines) {
    SmallLaunch sm{};
    // warp-per-line kernels for engines whose windows hold >= 2048 lines (decided once per engine, so every
    // window of a run -- the ragged last one included -- takes the same kernels and arithmetic)
    sm.wl = small_wl() && capacity_lines >= size_t(kSmallWlMinLines);
    // identity projection (B = D <= 16): per-warp stages of ~6 KB (4 warps x 2 stages = 48 KB, four
    // lines per SM); a lane owns one pixel of a chunk (a multiple of 32 pixels)
    int ch = int(std::min<size_t>(256, std::max<size_t>(4, size_t(6144) / (size_t(g.B) * 4))));
    if (ch >= 32) ch = ch / 32 * 32;
    sm.CH = ch;
    // SRP variant: two shared stages of ~20 KB, five CTAs per SM at B = 108 (a sweep of 14-34 KB
    // stages on configs[3] d = 5: 20 KB fastest, 0.132 ms per 2048 lines vs 0.170 at 26 KB)
    int ch2 = int(std::min<size_t>(256, std::max<size_t>(32, (size_t(20) * 1024) / (size_t(g.B) * 4))));
    ch2 = ch2 / 4 * 4;
    sm.CH2 = ch2;
    if (g.srp) {
        const int NT = g.D * (g.D + 1) / 2;
        const int dm = (g.D == 5 && g.B <= 128) ? 5 : (g.D <= 8 ? 8 : (g.D <= 12 ? 12 : 16));
        sm.smem_stats = align_up(size_t(2) * ch2 * g.B * 4, 16) + size_t(kStatsSmallThreads / 32) * (g.D + NT) * 8 +
                        align_up(size_t(ch2) * dm * 4, 16) + size_t(g.srp_nnz) * 12 + size_t(g.D + 1) * 4;
        sm.smem_score = size_t(g.P) * 4;
        return sm;
    }
    const int dm = (g.D == 5 || g.D == 10) ? g.D : (g.D <= 8 ? 8 : (g.D <= 12 ? 12 : 16));  // the kernel's DM
    sm.smem_stats = std::max(size_t(kStatsSmallThreads / 32) * 2 * ch * g.B * 4,
                             size_t(kStatsSmallThreads / 32) * (dm + dm * (dm + 1) / 2) * 8) +
                    size_t(dm) * (g.srp ? g.srp_wmax : 0) * 12;
    sm.smem_score = size_t(g.P) * 4;
    return sm;
}

void launch_stats_small(const Geometry& g, const SmallLaunch& sm, const float* x, int n_per_stream, int in_stride,
                        int n_lines_total, double* stats, float* vcache, cudaStream_t st) {
    {
        ensure_smem(stats_small_srp_kernel<5>, 200 * 1024);
        ensure_smem(stats_small_srp_kernel<8>, 200 * 1024);
        ensure_smem(stats_small_srp_kernel<12>, 200 * 1024);
        ensure_smem(stats_small_srp_kernel<16>, 200 * 1024);
        ensure_smem(stats_small_kernel<5>, 200 * 1024);
        ensure_smem(stats_small_kernel<8>, 200 * 1024);
        ensure_smem(stats_small_kernel<10>, 200 * 1024);
        ensure_smem(stats_small_kernel<12>, 200 * 1024);
        ensure_smem(stats_small_kernel<16>, 200 * 1024);
    }
    SmallArgs a{g, sm, x, n_per_stream, in_stride, stats, vcache};
    // SRP on batched windows: a warp per line while two CTAs of four warps (two 32-pixel stages each) fit
    // an SM (B <= 109) and the padded table stays small
    const size_t srp_wl_smem = size_t(kSrpWlWarps) * 2 * 32 * g.B * 4 + size_t(g.srp_wmax) * 16 * sizeof(SrpEnt);
    if (g.srp && sm.wl && g.D <= 12 && (g.B % 4) == 0 &&
        (reinterpret_cast<uintptr_t>(x) & 15) == 0 && srp_wl_smem <= 112 * 1024) {
        const int grid = (n_lines_total + kSrpWlWarps - 1) / kSrpWlWarps;
#define ERX_SRP_WL(DMV, EXV)                                                      \
    do {                                                                          \
        ensure_smem(stats_small_srp_wl_kernel<DMV, EXV>, 200 * 1024);             \
        stats_small_srp_wl_kernel<DMV, EXV><<<grid, kSrpWlWarps * 32, srp_wl_smem, st>>>(a, n_lines_total); \
    } while (0)
        if (g.D == 5) ERX_SRP_WL(5, true);
        else if (g.D == 8) ERX_SRP_WL(8, true);
        else if (g.D < 8) ERX_SRP_WL(8, false);
        else ERX_SRP_WL(12, false);
#undef ERX_SRP_WL
        return;
    }
    if (g.srp) {
        if (g.D == 5 && g.B <= 128)  // the reference default (measured: DM = 8 is faster at B = 224)
            stats_small_srp_kernel<5><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
        else if (g.D <= 8)
            stats_small_srp_kernel<8><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
        else if (g.D <= 12)
            stats_small_srp_kernel<12><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
        else
            stats_small_srp_kernel<16><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
        return;
    }
    // narrow identity lines: a warp per line (stats_small_wl_kernel) while a chunk holds the centre's
    // pixels; ERX_SMALL_WL=0 keeps the CTA-per-line kernels (A/B)
    // (from ~2048 lines per launch: below, warps-per-line leave SMs idle -- configs[1] d = 5 at 256 lines:
    // score 0.0106 -> 0.0166 ms)
    if (sm.wl && g.D <= 12 && (sm.CH >= 32 || sm.CH >= g.P)) {
        constexpr int kW = kStatsSmallThreads / 32;
        const int grid = (n_lines_total + kW - 1) / kW;
        // ~10 KB stages (8 pixels per lane per chunk at 10 bands: the pipeline restarts once per chunk)
        int chw = int(std::min<size_t>(256, size_t(10240) / (size_t(g.B) * 4))) / 32 * 32;
        if (chw > sm.CH) a.sm.CH = chw;
        const size_t smw = size_t(kW) * 2 * a.sm.CH * g.B * 4;
#define ERX_STATS_WL(DMV, EXV)                                              \
    do {                                                                    \
        ensure_smem(stats_small_wl_kernel<DMV, EXV>, 200 * 1024);           \
        stats_small_wl_kernel<DMV, EXV><<<grid, kStatsSmallThreads, smw, st>>>(a, n_lines_total); \
    } while (0)
        if (g.D == 5) ERX_STATS_WL(5, true);
        else if (g.D == 8) ERX_STATS_WL(8, true);
        else if (g.D < 8) ERX_STATS_WL(8, false);
        else if (g.D == 10) ERX_STATS_WL(10, true);
        else ERX_STATS_WL(12, false);
#undef ERX_STATS_WL
        return;
    }
    if (g.D == 5)  // the reference default, d = 5
        stats_small_kernel<5><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
    else if (g.D <= 8)
        stats_small_kernel<8><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
    else if (g.D == 10)  // configs[2]
        stats_small_kernel<10><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
    else if (g.D <= 12)
        stats_small_kernel<12><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
    else
        stats_small_kernel<16><<<n_lines_total, kStatsSmallThreads, sm.smem_stats, st>>>(a);
}

void launch_score_small(const Geometry& g, const SmallLaunch& sm, const double* stats, const double* prior,
                        const float* whiten, const float* vcache, int n_lines_total, float* raw, float* norm,
                        int* status, int* fixlist, cudaStream_t st) {
    {
        ensure_smem(score_small_kernel<8>, 200 * 1024);
        ensure_smem(score_small_kernel<5>, 200 * 1024);
        ensure_smem(score_small_kernel<10>, 200 * 1024);
        ensure_smem(score_small_kernel<12>, 200 * 1024);
        ensure_smem(score_small_kernel<16>, 200 * 1024);
    }
    if (sm.wl && g.D <= 12 && size_t(kScoreWlWarps) * g.P * 4 <= 48 * 1024) {
        const int grid = (n_lines_total + kScoreWlWarps - 1) / kScoreWlWarps;
        const size_t smw = size_t(kScoreWlWarps) * g.P * 4;
#define ERX_SCORE_WL(DMV, EXV)                                                                                   \
    score_small_wl_kernel<DMV, EXV><<<grid, kScoreWlWarps * 32, smw, st>>>(g, stats, prior, whiten, vcache, raw, \
                                                                           norm, status, fixlist, n_lines_total)
        if (g.D == 5) ERX_SCORE_WL(5, true);
        else if (g.D == 8) ERX_SCORE_WL(8, true);
        else if (g.D < 8) ERX_SCORE_WL(8, false);
        else if (g.D == 10) ERX_SCORE_WL(10, true);
        else ERX_SCORE_WL(12, false);
#undef ERX_SCORE_WL
        return;
    }
    if (g.D == 5)  // the reference default, d = 5
        score_small_kernel<5><<<n_lines_total, kSmallThreads, sm.smem_score, st>>>(g, stats, prior, whiten, vcache,
                                                                                   raw, norm, status, fixlist);
    else if (g.D <= 8)
        score_small_kernel<8><<<n_lines_total, kSmallThreads, sm.smem_score, st>>>(g, stats, prior, whiten, vcache,
                                                                                   raw, norm, status, fixlist);
    else if (g.D == 10)  // configs[2]
        score_small_kernel<10><<<n_lines_total, kSmallThreads, sm.smem_score, st>>>(g, stats, prior, whiten, vcache,
                                                                                    raw, norm, status, fixlist);
    else if (g.D <= 12)
        score_small_kernel<12><<<n_lines_total, kSmallThreads, sm.smem_score, st>>>(g, stats, prior, whiten, vcache,
                                                                                    raw, norm, status, fixlist);
    else
        score_small_kernel<16><<<n_lines_total, kSmallThreads, sm.smem_score, st>>>(g, stats, prior, whiten, vcache,
                                                                                    raw, norm, status, fixlist);
}

}  // namespace erxk
