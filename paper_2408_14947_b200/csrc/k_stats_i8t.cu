// k_stats_i8t.cu — line_stats (erx.hpp:38-40) on the tcgen05
// tensor cores with EXACT integer accumulation for WIDE lines (127 < D <= 512:
// configs[1]'s 224 and configs[4]'s 448 bands), the k_stats_i8.cu scheme
// tiled over 128-dim blocks.
//
// The second moment S = sum_p v_p v_p^T is D x D; one CTA's TMEM holds the four
// s32 class accumulators of ONE 128 x 128 block (4 x 128 columns).  So a line
// is cut into work items, one per lower-triangle pair of 128-dim tiles
// (mt, nt), nt <= mt — 3 items at 224 bands, 10 at 448 — each computing
// S[mt dims][nt dims] over all pixels:
//
//   range   (range_kernel, once per line for all dims) the centre c = fp32(mean
//           of the first min(32, P) pixels) (k_stats.cu's rule) and the
//           per-dim range max_p |fl32(x - c)|
//   main    the item's dims of every 32-pixel chunk (2D TMA boxes of 128 dims x
//           32 pixels from the line: cp.async.bulk.tensor, zero fill past B,
//           L2 hits for all but the first item of a line): v = fl32(x - c) rounded ONCE to
//           q = rint(v s_d), s_d = R / max|v|, R < 2^22, split into three
//           balanced int8 digits (i8_common.cuh), written as the MMA's K-major
//           A (mt dims) and B (nt dims) digit planes; 8 digit-pair MMAs
//           (M = 128, N = roundup16(nt dims), K = 32) per chunk into the four
//           s32 class accumulators
//   epilogue  S = (sum_c 2^(8(c+1)) acc_c [+ class 0 on the diagonal]) / (s_a s_b)
//           straight into the packed-lower stats slot; diagonal items also
//           write c and s = sum v (the quantiser's exact int64 sum of q / s_d).
// Consecutive items are the pairs of one line, so the CTAs working on them run
// together and all but the first read the line from L2.  Every s32 class sum
// is exact (|class sum| <= 3 2^14 P < 2^31 for P < 43690); the class-0 digit
// products d0 d0 are summed exactly on the diagonal by the quantiser (dp4a) and
// dropped off it (zero-mean, 2^-30 relative) — the same arithmetic as
// k_stats_i8.cu, so the same parity.
//
// Warp roles: 8 compute warps (range, quantisation, epilogue), 1 producer warp
// (TMA ring), 1 MMA warp.  Hand-offs through mbarriers only.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "erx_common.cuh"
#include "i8_common.cuh"
#include "tc_common.cuh"

namespace erxk {
namespace {

constexpr int kCh = 32;             // pixels per chunk (one K-step)
constexpr int kTile = 128;          // dims per tile
constexpr int kThreads = 256;       // compute threads
constexpr int kStages = 5;          // TMA ring depth
constexpr uint32_t kBox = kCh * kTile * 4;     // one 128-dim x 32-pixel fp32 box (16 KB)
constexpr uint32_t kPlane = tc::kSliceBytes;   // 128 rows x 32 K int8 (4 KB)
constexpr uint32_t kOps = 6 * kPlane;          // A digit planes 0-2, B digit planes 0-2
constexpr size_t kSmem = size_t(kStages) * 2 * kBox + 2 * size_t(kOps) + 1024;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            tc::smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar))
        : "memory");
}
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(m)) : "memory");
}
__device__ __forceinline__ float fmin_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

struct StatsI8TArgs {
    Geometry g;
    int n;           // lines per stream in the window
    int in_stride;   // lines per stream in the input buffer
    int n_lines;
    int ntile;       // ceil(D / 128)
    int npair;       // ntile (ntile + 1) / 2
    int nptile;      // 128-pixel tiles per line (v planes)
    double* stats;   // [line][c | s | S packed lower]
    const float* cen;  // [line][D] centre c (range_kernel)
    const float* vmax; // [line][D] max_p |fl32(x - c)|, NaN for a dim with a non-finite value (range_kernel)
    unsigned char* vplanes;  // [line][pixel tile][dim tile][3][16 KB] v digit planes (k_score_i8w), may be null
};

__device__ __forceinline__ void pair_of(int p, int& mt, int& nt) {  // p -> (mt, nt), nt <= mt, row-major
    mt = 0;
    while ((mt + 1) * (mt + 2) / 2 <= p) ++mt;
    nt = p - mt * (mt + 1) / 2;
}

__global__ void __launch_bounds__(kThreads + 64, 1) stats_i8t_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                     StatsI8TArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], pfull[2], pempty[2], accfull, accempty;
    __shared__ float cen_s[2][kTile], scl_s[2][kTile];
    __shared__ double inv_s[2][kTile];
    __shared__ long long sq_s[2][kTile];   // sum_p q per dim (diagonal items), per pixel half
    __shared__ int c0_s[2][kTile];         // sum_p d0^2 per dim (diagonal items), per pixel half
    __shared__ int bad_s;

    const Geometry& g = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int D = g.D, P = g.P;
    const int nch = (P + kCh - 1) / kCh;
    const int n_items = a.n_lines * a.npair;
    const int my_items = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    unsigned char* ring = smem;                              // [kStages][2 boxes]
    unsigned char* ops = smem + size_t(kStages) * 2 * kBox;  // [2][A d0 d1 d2 | B d0 d1 d2]

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
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

    auto item_geo = [&](int k, int& line, int& m0, int& n0, int& mr, int& nr) {
        // last line first: the range pass just streamed the window in line order, so its last lines are
        // the ones still in L2
        const int it = n_items - 1 - (blockIdx.x + k * gridDim.x);
        line = it / a.npair;
        int mt, nt;
        pair_of(it - line * a.npair, mt, nt);
        m0 = mt * kTile;
        n0 = nt * kTile;
        mr = min(kTile, D - m0);
        nr = min(kTile, D - n0);
    };
    auto line_row = [&](int line) {  // first pixel row of the line in the window buffer
        const int s = line / a.n, t = line - s * a.n;
        return (s * a.in_stride + t) * P;
    };

    if (warp == 8) {
        // ---------------- producer: for each item its chunks (A box [+ B box])
        if (lane == 0) {
            int j = 0;
            for (int k = 0; k < my_items; ++k) {
                int line, m0, n0, mr, nr;
                item_geo(k, line, m0, n0, mr, nr);
                const bool diag = m0 == n0;
                const int r0 = line_row(line);
                for (int c = 0; c < nch; ++c) {
                        const int st = j % kStages;
                        if (j >= kStages) tc::mbar_wait(&empty[st], uint32_t(j / kStages - 1) & 1u);
                        tc::mbar_expect_tx(&full[st], diag ? kBox : 2 * kBox);
                        unsigned char* dst = ring + size_t(st) * 2 * kBox;
                        tma_load_2d(dst, &tmap, m0, r0 + c * kCh, &full[st]);
                        if (!diag) tma_load_2d(dst + kBox, &tmap, n0, r0 + c * kCh, &full[st]);
                        ++j;
                }
            }
        }
        return;
    }
    if (warp == 9) {
        // ---------------- MMA issuer: 8 digit-pair MMAs (K = 32) per chunk of pass 2
        if (lane == 0) {
            const int pr[8][3] = {{0, 1, 0}, {1, 0, 0}, {0, 2, 1}, {1, 1, 1}, {2, 0, 1}, {1, 2, 2}, {2, 1, 2}, {2, 2, 3}};
            int k2 = 0;
            for (int k = 0; k < my_items; ++k) {
                int line, m0, n0, mr, nr;
                item_geo(k, line, m0, n0, mr, nr);
                const uint32_t idesc = tc::idesc_s8_s32(128, (nr + 15) / 16 * 16);
                const bool diag = m0 == n0;
                if (k >= 1) tc::mbar_wait(&accempty, uint32_t(k - 1) & 1u);
                for (int c = 0; c < nch; ++c, ++k2) {
                    const int buf = k2 & 1;
                    tc::mbar_wait(&pfull[buf], uint32_t(k2 >> 1) & 1u);
                    tc::tc_fence_after();
                    const uint32_t base = tc::smem_u32(ops + buf * kOps);
                    const uint32_t bbase = diag ? base : base + 3 * kPlane;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const uint64_t ad = tc::smem_desc(base + pr[q][0] * kPlane);
                        const uint64_t bd = tc::smem_desc(bbase + pr[q][1] * kPlane);
                        const bool first = c == 0 && (q == 0 || q == 2 || q == 5 || q == 7);
                        tc::mma_s8(tmem + uint32_t(pr[q][2]) * 128u, ad, bd, idesc, first ? 0u : 1u);
                    }
                    tc::mma_commit(&pempty[buf]);
                }
                tc::mma_commit(&accfull);
            }
        }
        return;
    }

    // ---------------- compute warps 0-7: thread = (dim d of the tile, pixel half h: 16 pixels)
    const int d = tid & (kTile - 1), h = tid >> 7;
    int j = 0, k2 = 0;
    for (int k = 0; k < my_items; ++k) {
        int line, m0, n0, mr, nr;
        item_geo(k, line, m0, n0, mr, nr);
        const bool diag = m0 == n0;
        const int nsets = diag ? 1 : 2;
        // ---- the centre and range of both dim sets (range_kernel, one pass over the line before)
        if (tid == 0) bad_s = 0;
        bar_compute();
        if (tid < nsets * kTile) {
            const int set = tid >> 7, dd = tid & (kTile - 1);
            const int rdim = (set == 0 ? m0 : n0) + dd, rcount = set == 0 ? mr : nr;
            float cd = 0.f, sc = 0.f;
            if (dd < rcount) {
                cd = a.cen[size_t(line) * D + rdim];
                const float m = a.vmax[size_t(line) * D + rdim];
                if (!(m >= 0.f && m <= 3.402823466e38f)) bad_s = 1;  // a non-finite value in this dim
                sc = i8::v_scale(m);
            }
            cen_s[set][dd] = cd;
            scl_s[set][dd] = sc;
            inv_s[set][dd] = sc > 0.f ? 1.0 / double(sc) : 0.0;
        }
        bar_compute();
        // ---- pass 2: quantise into the A (and B) digit planes; exact sum q and class-0 diagonal
        long long sq = 0;
        int c0 = 0;
        const float cA = cen_s[0][d], sA = scl_s[0][d];
        const float cB = nsets > 1 ? cen_s[1][d] : 0.f, sB = nsets > 1 ? scl_s[1][d] : 0.f;
        for (int c = 0; c < nch; ++c, ++k2) {
            const int st = j % kStages;
            const int buf = k2 & 1;
            tc::mbar_wait(&full[st], uint32_t(j / kStages) & 1u);
            ++j;
            if (k2 >= 2) tc::mbar_wait(&pempty[buf], uint32_t((k2 - 2) >> 1) & 1u);
            const float* box = reinterpret_cast<const float*>(ring + size_t(st) * 2 * kBox);
            unsigned char* op = ops + buf * kOps;
            const int n = min(kCh, P - c * kCh);
            for (int set = 0; set < nsets; ++set) {
                const float* bx = box + set * (kBox / 4);
                const float cc = set ? cB : cA, ss = set ? sB : sA;
                uint32_t w[3][4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    uint32_t u[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int p = h * 16 + jj * 4 + e;
                        const float x = bx[p * kTile + d];
                        u[e] = i8::quant_u(x - cc, ss);
                        if (p >= n) u[e] = 0x808080u;
                    }
                    i8::pack_digits(u, w[0][jj], w[1][jj], w[2][jj]);
                    if (diag) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) sq += (long long)(int(u[e]) - 0x808080);
                        c0 = __dp4a(int(w[0][jj]), int(w[0][jj]), c0);
                    }
                }
                const uint32_t off = tc::kmajor_off_s8(d, h * 16);
#pragma unroll
                for (int pl = 0; pl < 3; ++pl)
                    *reinterpret_cast<uint4*>(op + (set * 3 + pl) * kPlane + off) =
                        make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]);
                if (diag && a.vplanes) {
                    // the same digits as the wide score's MN-major A operand (i8_common.cuh: vplane_off)
                    const int p = c * kCh + h * 16;
                    unsigned char* vt = a.vplanes +
                                        ((size_t(line) * a.nptile + (p >> 7)) * a.ntile + m0 / kTile) * (3 * 16384);
                    const uint64_t stream_out = tc::policy_evict_first();
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl)
                        tc::st16_hint(vt + i8::vplane_off(pl, d, p & 127), make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]),
                                      stream_out);
                }
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[st]);
                mbar_arrive(&pfull[buf]);
            }
        }
        if (diag) {
            sq_s[h][d] = sq;
            c0_s[h][d] = c0;
        }
        // ---- epilogue: S block -> the stats slot (TMEM lane = row dim of mt, column = dim of nt)
        tc::mbar_wait(&accfull, uint32_t(k) & 1u);
        tc::tc_fence_after();
        bar_compute();  // sq_s / c0_s of this item
        const int lane_grp = warp & 3, colh = warp >> 2;
        const int row = lane_grp * 32 + lane;
        const uint32_t lane_base = uint32_t(lane_grp * 32) << 16;
        const int ngrp = (nr + 15) / 16;
        const int g0 = colh ? (ngrp + 1) / 2 : 0, g1 = colh ? ngrp : (ngrp + 1) / 2;
        double* out = a.stats + size_t(line) * (g.SE + D);
        const double poison = bad_s ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
        const int gi_row = m0 + row;
        for (int gi = g0; gi < g1; ++gi) {
            uint32_t v[4][16];
            tc::tmem_ld16x4(tmem + lane_base + uint32_t(gi * 16), 128u, v);
            if (row < mr) {
                const double ia = inv_s[0][row];
#pragma unroll
                for (int ii = 0; ii < 16; ++ii) {
                    const int col = gi * 16 + ii;
                    const int gj = n0 + col;
                    if (col < nr && gj <= gi_row) {
                        long long si = (static_cast<long long>(int(v[3][ii])) << 32) +
                                       (static_cast<long long>(int(v[2][ii])) << 24) +
                                       (static_cast<long long>(int(v[1][ii])) << 16) +
                                       (static_cast<long long>(int(v[0][ii])) << 8);
                        if (diag && col == row) si += (long long)(c0_s[0][row]) + c0_s[1][row];
                        out[2 * D + tri(gi_row, gj)] = double(si) * ia * inv_s[diag ? 0 : 1][col] + poison;
                    }
                }
            }
        }
        tc::tc_fence_before();
        bar_compute();
        if (tid == 0) mbar_arrive(&accempty);  // TMEM free for the next item's MMAs
        if (diag && tid < mr) {
            const long long q = sq_s[0][tid] + sq_s[1][tid];
            out[m0 + tid] = double(cen_s[0][tid]) + poison;
            out[D + m0 + tid] = double(q) * inv_s[0][tid] + poison;
        }
        bar_compute();  // cen_s / inv_s / sq_s / c0_s / bad_s are rewritten by the next item
    }
    if (warp == 0) tc::tmem_free<512>(tmem);
}

// Per (line, dim): the centre c = fp32(fp64 mean of the first min(32, P) pixels) (k_stats.cu's rule) and
// the range max_p |fl32(x - c)| (NaN when the dim holds a non-finite value), one pass over the line.
__global__ void __launch_bounds__(256) range_kernel(Geometry g, const float* __restrict__ x, int n, int in_stride,
                                                    float* __restrict__ cen, float* __restrict__ vmax) {
    // thread = (4-dim quad, pixel group of 4): 16-byte loads, 8 rows in flight per thread
    __shared__ float lo_s[4][256], hi_s[4][256];
    __shared__ double cs_s[4][256];
    const int line = blockIdx.x, D = g.D, P = g.P, B = g.B;
    const float* xl = line_ptr(x, line, n, in_stride, g);
    const int nq = B / 4, tid = threadIdx.x;
    const int n0 = min(32, P);
    // (one CTA per 64-quad block of the line: blockIdx.y; at 448 bands two CTAs per line double the loads in flight)
    for (int q0 = 64 * blockIdx.y; q0 < nq; q0 += 64 * gridDim.y) {
        const int q = q0 + (tid & 63), pg = tid >> 6;
        float4 lo = make_float4(3.402823466e38f, 3.402823466e38f, 3.402823466e38f, 3.402823466e38f);
        float4 hi = make_float4(-3.402823466e38f, -3.402823466e38f, -3.402823466e38f, -3.402823466e38f);
        double cs[4] = {0.0, 0.0, 0.0, 0.0};
        if (q < nq) {
            for (int p0 = pg; p0 < P; p0 += 32) {
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int p = p0 + 4 * u;
                    v[u] = p < P ? __ldg(reinterpret_cast<const float4*>(xl + size_t(p) * B) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int p = p0 + 4 * u;
                    if (p < P) {
                        lo.x = fmin_nan(lo.x, v[u].x); lo.y = fmin_nan(lo.y, v[u].y);
                        lo.z = fmin_nan(lo.z, v[u].z); lo.w = fmin_nan(lo.w, v[u].w);
                        hi.x = fmaxf(hi.x, v[u].x); hi.y = fmaxf(hi.y, v[u].y);
                        hi.z = fmaxf(hi.z, v[u].z); hi.w = fmaxf(hi.w, v[u].w);
                        if (p < n0) {
                            cs[0] += double(v[u].x); cs[1] += double(v[u].y);
                            cs[2] += double(v[u].z); cs[3] += double(v[u].w);
                        }
                    }
                }
            }
        }
        const int ql = tid & 63;
        lo_s[pg][4 * ql] = lo.x; lo_s[pg][4 * ql + 1] = lo.y; lo_s[pg][4 * ql + 2] = lo.z; lo_s[pg][4 * ql + 3] = lo.w;
        hi_s[pg][4 * ql] = hi.x; hi_s[pg][4 * ql + 1] = hi.y; hi_s[pg][4 * ql + 2] = hi.z; hi_s[pg][4 * ql + 3] = hi.w;
#pragma unroll
        for (int e = 0; e < 4; ++e) cs_s[pg][4 * ql + e] = cs[e];
        __syncthreads();
        {
            {
                const int dd = tid, d = 4 * q0 + dd;
                if (d < D) {
                    const float l = fmin_nan(fmin_nan(lo_s[0][dd], lo_s[1][dd]), fmin_nan(lo_s[2][dd], lo_s[3][dd]));
                    const float h = fmaxf(fmaxf(hi_s[0][dd], hi_s[1][dd]), fmaxf(hi_s[2][dd], hi_s[3][dd]));
                    const float c = float(((cs_s[0][dd] + cs_s[1][dd]) + (cs_s[2][dd] + cs_s[3][dd])) / double(n0));
                    const bool fin = isfinite(l) && isfinite(h);
                    cen[size_t(line) * D + d] = c;
                    vmax[size_t(line) * D + d] = fin ? fmaxf(h - c, c - l) : __int_as_float(0x7fc00000);
                }
            }
        }
        __syncthreads();
    }
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace

bool stats_i8t_eligible(const Geometry& g) {
    return !g.srp && g.D > 127 && g.D <= 512 && (g.B % 4) == 0 && g.P < 43690 && tensor_map_encoder() != nullptr;
}

int launch_stats_i8t(const Geometry& g, const float* x, int n_per_stream, int in_stride, int n_streams,
                     double* stats, float* cen, float* vmax, unsigned char* vplanes, cudaStream_t st) {
    auto encode = tensor_map_encoder();
    if (!encode) return 1;
    // the window's lines as one 2D tensor: rows = pixels of every (stream, line slot), B floats each
    CUtensorMap map;
    const cuuint64_t gdim[2] = {cuuint64_t(g.B), cuuint64_t(n_streams) * cuuint64_t(in_stride) * cuuint64_t(g.P)};
    const cuuint64_t gstride[1] = {cuuint64_t(g.B) * 4};
    const cuuint32_t box[2] = {cuuint32_t(kTile), cuuint32_t(kCh)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), gdim, gstride, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 2;
    const int ntile = (g.D + kTile - 1) / kTile;
    StatsI8TArgs a{g, n_per_stream, in_stride, n_streams * n_per_stream, ntile, ntile * (ntile + 1) / 2,
                   (g.P + kTile - 1) / kTile, stats, cen, vmax, vplanes};
    range_kernel<<<dim3(a.n_lines, (g.B / 4 + 63) / 64), 256, 0, st>>>(g, x, n_per_stream, in_stride, cen, vmax);
    const int items = a.n_lines * a.npair;
    const int grid = items < sm_count() ? items : sm_count();
    ensure_smem(stats_i8t_kernel, kSmem);
    stats_i8t_kernel<<<grid, kThreads + 64, kSmem, st>>>(map, a);
    return 0;
}

}  // namespace erxk
