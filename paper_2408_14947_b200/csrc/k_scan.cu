// k_scan.cu — the background recurrence over a window: ema_update
// (erx.hpp:42-44) or welford_batch_update (linalg.hpp:33-36), element-wise
// over (mu, packed K) and sequential over the window's lines in the
// reference's own order, fp64.  Writes, per line, the PRE-update background
// (score-then-update).  The first line ever initialises the
// background with its own statistics (erx.hpp:54-55).
//
// Input per line (k_stats.cu): [c | s | S]; line statistics are finished
// here:  mu_hat = c + s/P,  K_hat = (S - s_a s_b / P) / (P - 1).
#include "scan_rec.cuh"

#ifndef SCAN_MINB
#define SCAN_MINB 1
#endif
#ifndef SCAN_KB
#define SCAN_KB 8
#endif

namespace erxk {
namespace {

__global__ void __launch_bounds__(128, SCAN_MINB) scan_kernel(Geometry g, const double* __restrict__ stats,
                                                   double* __restrict__ prior, StateRef sref, int n, double alpha,
                                                   int incremental, float* __restrict__ kblk) {
    const double* __restrict__ st_in = sref.in();
    double* __restrict__ st_out = sref.out();
    const int initialized = sref.meta->initialized;
    const long long n_seen0 = sref.meta->welford_n;
    const int s = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.SE) return;
    const int D = g.D, SS = g.SE + g.D;  // stats slot stride
    const double P = double(g.P), invP = 1.0 / P, invP1 = 1.0 / (P - 1.0);
    int a = e, b = e;
    if (e >= D) unpack_tri(e - D, a, b);
    // with kblk, the pre-update covariance goes out as fp32 packed lower 8x8 blocks (the blocked
    // factor's shared-memory image) and only the mean as fp64
    const int nblk = g.nb * (g.nb + 1) / 2;
    const bool to_blk = kblk != nullptr && e >= D;
    // the factor's swizzled block rows (k_factor.cu: swz): element (r, c) at r * 8 + (c ^ (r & 4))
    const int boff = ((a >> 3) * ((a >> 3) + 1) / 2 + (b >> 3)) * 64 + (a & 7) * 8 + ((b & 7) ^ (a & 4));
    auto put = [&](size_t l, double pr) {
        if (to_blk)
            kblk[l * nblk * 64 + boff] = float(pr);
        else
            prior[l * g.SE + e] = pr;
    };
    const double* in = st_in + size_t(s) * g.SE;
    const size_t l0 = size_t(s) * n;
    // line statistics of line l, this element (and the two means it couples)
    auto mu_hat = [&](const double* st, int j) { return finish_stat(true, st[j], st[D + j], 0.0, invP, invP1); };
    auto k_hat = [&](const double* st) { return finish_stat(false, st[2 * D + (e - D)], st[D + a], st[D + b], invP, invP1); };
    if (!incremental) {
        const double om = 1.0 - alpha;
        double state = in[e];
        // the line statistics do not depend on the recurrence: they are loaded a batch
        // ahead (double-buffered registers) so the sequential EMA never waits on memory
        constexpr int kB = SCAN_KB;
        double cur[kB], nxt[kB];
        // branch-free loads (clamped line index, select after) so all 3 x kB loads issue back to back
        const bool is_mu = e < D;
        const int o0 = is_mu ? e : 2 * D + (e - D), o1 = D + a, o2 = D + b;
        auto load = [&](int t0, double* buf) {
            double x0[kB], x1[kB], x2[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const double* st = stats + (l0 + min(t0 + u, n - 1)) * SS;
                x0[u] = __ldg(st + o0);
                x1[u] = __ldg(st + o1);
                x2[u] = __ldg(st + o2);
            }
#pragma unroll
            for (int u = 0; u < kB; ++u)
                buf[u] = finish_stat(is_mu, x0[u], x1[u], x2[u], invP, invP1);
        };
        load(0, cur);
        for (int t0 = 0; t0 < n; t0 += kB) {
            if (t0 + kB < n) load(t0 + kB, nxt);
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int t = t0 + u;
                if (t < n) {
                    double pr;
                    if (!initialized && t == 0) {
                        pr = cur[u];
                        state = cur[u];
                    } else {
                        pr = state;
                        state = ema_step(state, cur[u], om, alpha);
                    }
                    put(l0 + t, pr);
                }
            }
#pragma unroll
            for (int u = 0; u < kB; ++u) cur[u] = nxt[u];
        }
        st_out[size_t(s) * g.SE + e] = state;
    } else {
        const bool is_cov = e >= D;
        WelfordElem w{in[a], in[b], is_cov ? in[e] : 0.0, double(n_seen0)};
        const double nb = P;
        for (int t = 0; t < n; ++t) {
            const size_t l = l0 + t;
            const double* st = stats + l * SS;
            const double mha = mu_hat(st, a), mhb = mu_hat(st, b);
            const double kh = is_cov ? k_hat(st) : 0.0;
            double pr;
            if (!initialized && t == 0) {
                w.ma = mha;
                w.mb = mhb;
                if (is_cov) w.cov = kh;
                w.nseen = nb;
                pr = is_cov ? w.cov : w.ma;
            } else {
                pr = is_cov ? w.cov : w.ma;
                welford_step(w, is_cov, mha, mhb, kh, nb);
            }
            put(l, pr);
        }
        const double ma = w.ma, cov = w.cov;
        st_out[size_t(s) * g.SE + e] = (e < D) ? ma : cov;
    }
}


// ---------------------------------------------------------------------------
// Short windows (EMA, n <= kTileLines: the batched configs[3] geometry, 32 lines per stream): one CTA
// takes 128 elements of one stream and first copies everything its recurrence reads into shared
// memory with cp.async -- its elements' line values for all n lines and the prefix of each line's
// sum vector s its elements touch -- so the sequential EMA never waits on global memory.  Same
// per-element arithmetic and order as scan_kernel (bit-identical results).
// ---------------------------------------------------------------------------
constexpr int kTileLines = 64;

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem_src));
}

__global__ void __launch_bounds__(128) scan_tile_kernel(Geometry g, const double* __restrict__ stats,
                                                        double* __restrict__ prior, StateRef sref, int n,
                                                        double alpha, float* __restrict__ kblk) {
    extern __shared__ __align__(16) double tsm[];
    const double* __restrict__ st_in = sref.in();
    double* __restrict__ st_out = sref.out();
    const int initialized = sref.meta->initialized;
    const int s = blockIdx.y, tid = threadIdx.x;
    const int e0 = blockIdx.x * 128, e = e0 + tid;
    const int D = g.D, SS = g.SE + g.D;
    const double P = double(g.P), invP = 1.0 / P, invP1 = 1.0 / (P - 1.0);
    // the sum-vector prefix this CTA touches: dims 0 .. amax (rows of its last covariance element)
    const int e_last = min(e0 + 127, g.SE - 1);
    int amax = e_last, bdummy = 0;
    if (e_last >= D) unpack_tri(e_last - D, amax, bdummy);
    if (e0 < D) amax = max(amax, min(e0 + 127, D - 1));
    const int ns = amax + 1;
    double* xv = tsm;             // [n][128] the elements' own line values (c_a or S_ab)
    double* sv = tsm + n * 128;   // [n][ns] the line sums s_0 .. s_amax
    const size_t l0 = size_t(s) * n;
    int a = e, b = e;
    if (e >= D) unpack_tri(e - D, a, b);
    const bool live = e < g.SE;
    const bool is_mu = e < D;
    const int o0 = is_mu ? e : 2 * D + (e - D);
    if (live)
        for (int t = 0; t < n; ++t) cp_async8(xv + t * 128 + tid, stats + (l0 + t) * SS + o0);
    for (int q = tid; q < n * ns; q += 128) {
        const int t = q / ns, j = q - t * ns;
        cp_async8(sv + q, stats + (l0 + t) * SS + D + j);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (!live) return;
    const int nblk = g.nb * (g.nb + 1) / 2;
    const bool to_blk = kblk != nullptr && e >= D;
    const int boff = ((a >> 3) * ((a >> 3) + 1) / 2 + (b >> 3)) * 64 + (a & 7) * 8 + ((b & 7) ^ (a & 4));
    const double om = 1.0 - alpha;
    double state = st_in[size_t(s) * g.SE + e];
#pragma unroll 4
    for (int t = 0; t < n; ++t) {
        const double* svt = sv + t * ns;
        const double cur = finish_stat(is_mu, xv[t * 128 + tid], svt[a], svt[b], invP, invP1);
        double pr;
        if (!initialized && t == 0) {
            pr = cur;
            state = cur;
        } else {
            pr = state;
            state = ema_step(state, cur, om, alpha);
        }
        if (to_blk)
            kblk[(l0 + t) * nblk * 64 + boff] = float(pr);
        else
            prior[(l0 + t) * g.SE + e] = pr;
    }
    st_out[size_t(s) * g.SE + e] = state;
}

// ---------------------------------------------------------------------------
// Few elements, long windows (a single stream at small D: configs[2] has 20
// state elements and up to thousands of lines per window): the element-
// parallel kernel above runs one warp through every line, each step waiting on
// its own global loads.  Here one CTA takes 32 elements of one stream; per
// chunk of TC (192 or 32) lines the other warps finish the line statistics into shared memory
// (all loads in flight at once) and write back the chunk before last, while
// warp 0 runs the recurrence over the previous chunk from shared memory.  The
// per-element arithmetic and its order are exactly the kernel above's (EMA
// mode), so the results are bit-identical.
// ---------------------------------------------------------------------------
// E: state elements per CTA (32, or 8 where even 32-element CTAs leave most SMs idle: configs[2]'s 65
// elements run as 9 CTAs whose loader warps finish a chunk under the recurrence of the previous one)
template <int TC, int NTH, int kU, int E = 32>
__global__ void __launch_bounds__(NTH) scan_chunk_kernel(Geometry g, const double* __restrict__ stats,
                                                         double* __restrict__ prior, StateRef sref, int n,
                                                         double alpha, float* __restrict__ kblk) {
    const double* __restrict__ st_in = sref.in();
    double* __restrict__ st_out = sref.out();
    const int initialized = sref.meta->initialized;
    extern __shared__ __align__(16) unsigned char smem[];
    double* kh = reinterpret_cast<double*>(smem);  // [2][TC][E] finished line statistics
    double* ps = kh + 2 * TC * E;                  // [2][TC][E] pre-update background
    __shared__ int o0_s[E], o1_s[E], o2_s[E], boff_s[E];
    const int s = blockIdx.y, e0 = blockIdx.x * E;
    const int ne = min(E, g.SE - e0);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int D = g.D, SS = g.SE + g.D;
    const double P = double(g.P), invP = 1.0 / P, invP1 = 1.0 / (P - 1.0);
    const int nblk = g.nb * (g.nb + 1) / 2;
    if (tid < E) {
        const int e = e0 + min(tid, ne - 1);
        int a = e, b = e;
        if (e >= D) unpack_tri(e - D, a, b);
        const bool is_mu = e < D;
        o0_s[tid] = is_mu ? e : 2 * D + (e - D);
        o1_s[tid] = D + a;
        o2_s[tid] = D + b;
        boff_s[tid] = (kblk != nullptr && e >= D)
                          ? ((a >> 3) * ((a >> 3) + 1) / 2 + (b >> 3)) * 64 + (a & 7) * 8 + ((b & 7) ^ (a & 4))
                          : -1;
    }
    __syncthreads();
    const size_t l0 = size_t(s) * n;
    const int nch = (n + TC - 1) / TC;
    double state = (lane < ne) ? st_in[size_t(s) * g.SE + e0 + lane] : 0.0;
    const double om = 1.0 - alpha;
    for (int it = 0; it <= nch + 1; ++it) {
        if (warp == 0) {
            // recurrence over chunk it - 1
            const int c = it - 1;
            if (c >= 0 && c < nch) {
                const double* kc = kh + (c & 1) * TC * E;
                double* pc = ps + (c & 1) * TC * E;
                const int nt = min(TC, n - c * TC);
#pragma unroll 8
                for (int t = 0; t < nt; ++t) {
                    const double cur = kc[t * E + (lane & (E - 1))];
                    double pr;
                    if (!initialized && c == 0 && t == 0) {
                        pr = cur;
                        state = cur;
                    } else {
                        pr = state;
                        state = ema_step(state, cur, om, alpha);
                    }
                    if (lane < E) pc[t * E + lane] = pr;
                }
            }
        } else {
            const int q0 = tid - 32, nq = NTH - 32;
            // finish the line statistics of chunk it
            if (it < nch) {
                double* kc = kh + (it & 1) * TC * E;
                const int nt = min(TC, n - it * TC);
                // batches of kU items per thread: all 3 kU loads in flight before any is used
                for (int qb = q0; qb < nt * E; qb += kU * nq) {
                    double x0[kU], x1[kU], x2[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int q = min(qb + u * nq, nt * E - 1);
                        const int t = q / E, j = q & (E - 1);
                        const double* st = stats + (l0 + size_t(it) * TC + t) * SS;
                        x0[u] = __ldg(st + o0_s[j]);
                        x1[u] = __ldg(st + o1_s[j]);
                        x2[u] = __ldg(st + o2_s[j]);
                    }
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int q = qb + u * nq;
                        if (q < nt * E) kc[q] = finish_stat(e0 + (q & (E - 1)) < D, x0[u], x1[u], x2[u], invP, invP1);
                    }
                }
            }
            // write back chunk it - 2
            const int c = it - 2;
            if (c >= 0) {
                const double* pc = ps + (c & 1) * TC * E;
                const int nt = min(TC, n - c * TC);
                for (int q = q0; q < nt * E; q += nq) {
                    const int t = q / E, j = q & (E - 1);
                    if (j >= ne) continue;
                    const size_t l = l0 + size_t(c) * TC + t;
                    if (boff_s[j] >= 0)
                        kblk[l * nblk * 64 + boff_s[j]] = float(pc[q]);
                    else
                        prior[l * g.SE + e0 + j] = pc[q];
                }
            }
        }
        __syncthreads();
    }
    if (warp == 0 && lane < ne) st_out[size_t(s) * g.SE + e0 + lane] = state;
}

__global__ void window_advance_kernel(WinMeta* meta, int n_lines, long long pixels_per_line, int incremental) {
    meta->lines_seen += n_lines;
    if (incremental) meta->welford_n += (long long)(n_lines) * pixels_per_line;
    meta->initialized = 1;
    meta->cur ^= 1;
}

}  // namespace

void launch_window_advance(WinMeta* meta, int n_lines, long long pixels_per_line, int incremental, cudaStream_t st) {
    window_advance_kernel<<<1, 1, 0, st>>>(meta, n_lines, pixels_per_line, incremental);
}

void launch_scan(const Geometry& g, const double* stats, double* prior, StateRef state, int n_streams,
                 int n_per_stream, double alpha, int incremental, cudaStream_t st, float* kblk) {
    const int blocks_plain = (g.SE + 127) / 128 * n_streams;
    // (configs[3] on one GPU's share of 8: 376 plain blocks, T = 256 -> chunked 0.074 vs 0.092 ms;
    // shares of 4 and 2 (752 / 1504 blocks) stay faster element-parallel)
    if (!incremental && blocks_plain < 4 * sm_count() && n_per_stream >= 64) {
        // too few elements to hide the per-line load latency: chunked variant
        dim3 grid((g.SE + 31) / 32, n_streams);
        const int ctas = int(grid.x * grid.y);
        const int ctas8 = (g.SE + 7) / 8 * n_streams;
        if (4 * ctas <= sm_count() && ctas8 <= sm_count() && n_per_stream >= 512) {
            // a handful of elements (configs[2]: 65): 8 per CTA, so a CTA's loader warps finish a chunk
            // under the recurrence of the previous one
            dim3 grid8((g.SE + 7) / 8, n_streams);
            const size_t sm = 2 * size_t(2) * 192 * 8 * sizeof(double);
            ensure_smem(scan_chunk_kernel<192, 256, 7, 8>, sm);
            scan_chunk_kernel<192, 256, 7, 8><<<grid8, 256, sm, st>>>(g, stats, prior, state, n_per_stream, alpha, kblk);
        } else if (ctas <= sm_count()) {
            const size_t sm = 2 * size_t(2) * 192 * 32 * sizeof(double);
            ensure_smem(scan_chunk_kernel<192, 512, 13>, sm);  // 6144 items per chunk: one batch per thread
            scan_chunk_kernel<192, 512, 13><<<grid, 512, sm, st>>>(g, stats, prior, state, n_per_stream, alpha, kblk);
        } else {
            const size_t sm = 2 * size_t(2) * 32 * 32 * sizeof(double);
            ensure_smem(scan_chunk_kernel<32, 256, 5>, sm);  // 1024 items per chunk
            scan_chunk_kernel<32, 256, 5><<<grid, 256, sm, st>>>(g, stats, prior, state, n_per_stream, alpha, kblk);
        }
        return;
    }
    dim3 grid((g.SE + 127) / 128, n_streams);
    const size_t tile_smem = size_t(n_per_stream) * (128 + g.D) * sizeof(double);
    if (!incremental && n_per_stream <= kTileLines && tile_smem <= 100 * 1024) {
        ensure_smem(scan_tile_kernel, 100 * 1024);
        scan_tile_kernel<<<grid, 128, tile_smem, st>>>(g, stats, prior, state, n_per_stream, alpha, kblk);
        return;
    }
    scan_kernel<<<grid, 128, 0, st>>>(g, stats, prior, state, n_per_stream, alpha, incremental, kblk);
}

}  // namespace erxk
