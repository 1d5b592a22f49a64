// k_fixup.cu — fp64 rescue of the lines the fp32 factor cannot take.
//
// The fast factor kernels (k_factor.cu: factor_blk / factor_big) run
// cholesky_lower (linalg.hpp:12-15) in fp32 and stop on a line whose
// factorisation is not trustworthy in that precision:
//   * a pivot that fails (<= 0, or NaN) at the configured eps, or
//   * a pivot L_ii^2 below A_ii / kCondTau (A = K_{t-1} + eps I): the
//     squared multiple correlation of dim i with the dims before it is above
//     1 - 1/kCondTau, and fp32 loses the digits the score needs (emulated:
//     median raw-score error grows like 2e-9 x A_ii / L_ii^2).
// Such a line goes on a device-side list instead of being escalated in fp32
// (where the escalation decision itself could differ from the fp64
// reference).  This kernel then redoes the whole per-line chain for every
// listed line in fp64, as the reference does (erx.hpp:51-71):
//   1. the pre-update background (mu_{t-1}, K_{t-1}) by the window scan's own
//      element recurrence from the window-start state (scan_rec.cuh: the same
//      bits the scan produced);
//   2. L = chol(K_{t-1} + eps I) with the eps x10 escalation up to 1e-1
//      (SPEC.md:306), failing pivot -> status + latch (FactorizationError);
//   3. X = L^{-1}; delta_i = ||X (z_i - mu)|| for every pixel from the line
//      itself (z = x, or the fp64 SRP projection);
//   4. normalize_scores (detector.hpp:29-32) from the fp64 deltas.
// It runs after the score / normalize kernels of the window and overwrites the
// raw / norm rows of its lines.  The normalisation kernels list lines too: a
// line whose fp32 scores are flat to within kFlatRel (erx_common.cuh) gets its
// zero-variance decision made on fp64 deltas.  With nothing listed (every BASELINE config:
// A_ii / L_ii^2 stays below ~500 there) it is one short launch that reads the
// list count and resets the list.
#include "f64_factor.cuh"
#include "scan_rec.cuh"

#include <algorithm>

namespace erxk {
namespace {

constexpr int kFixThreads = 256;
constexpr int kFixPx = 32;  // pixels per scoring pass

__global__ void __launch_bounds__(kFixThreads) fixup_kernel(FixupArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_fail;
    __shared__ double red[kFixThreads];
    const Geometry& g = a.g;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int D = g.D, Dp = g.Dp, SE = g.SE, SS = SE + D;
    double* A = a.work + size_t(blockIdx.x) * (2 * size_t(Dp) * Dp + g.P);
    double* X = A + size_t(Dp) * Dp;                // pristine K_{t-1} during the factor, then L^{-1}
    double* dl = X + size_t(Dp) * Dp;               // [P] fp64 deltas of the line
    double* mu = reinterpret_cast<double*>(smem);   // [Dp]
    double* dyn = mu + Dp;                          // factor / inverse / scoring scratch
    const int count = a.list[0];
    // nothing listed (the usual window): no CTA touches the list, so there is nothing to reset either --
    // skip the fence / atomic hand-shake below (the empty launch: 6.2 -> ~3 us)
    if (count == 0) return;
    const int initialized = a.state.meta->initialized;
    const long long n_seen0 = a.state.meta->welford_n;
    const double Pd = double(g.P), invP = 1.0 / Pd, invP1 = 1.0 / (Pd - 1.0), om = 1.0 - a.alpha;
    for (int q = blockIdx.x; q < count; q += gridDim.x) {
        const int line = a.list[2 + q];
        const int s = line / a.n, t = line - s * a.n;
        // ---- 1. pre-update background of line (s, t)
        const double* in = a.state.in() + size_t(s) * SE;
        for (int e = tid; e < SE; e += nt) {
            const ScanElem el = scan_elem(D, e);
            double pr = 0.0;
            if (!a.incremental) {
                double state = in[e];
                for (int u = 0; u <= t; ++u) {
                    const double* st = a.stats + (size_t(s) * a.n + u) * SS;
                    const double cur = finish_stat(el.is_mu, st[el.o0], st[el.o1], st[el.o2], invP, invP1);
                    if (!initialized && u == 0) {
                        pr = cur;
                        state = cur;
                    } else {
                        pr = state;
                        state = ema_step(state, cur, om, a.alpha);
                    }
                }
            } else {
                const bool is_cov = !el.is_mu;
                WelfordElem w{in[el.a], in[el.b], is_cov ? in[e] : 0.0, double(n_seen0)};
                for (int u = 0; u <= t; ++u) {
                    const double* st = a.stats + (size_t(s) * a.n + u) * SS;
                    const double mha = finish_stat(true, st[el.a], st[D + el.a], 0.0, invP, invP1);
                    const double mhb = finish_stat(true, st[el.b], st[D + el.b], 0.0, invP, invP1);
                    const double kh = is_cov ? finish_stat(false, st[el.o0], st[el.o1], st[el.o2], invP, invP1) : 0.0;
                    if (!initialized && u == 0) {
                        w.ma = mha;
                        w.mb = mhb;
                        if (is_cov) w.cov = kh;
                        w.nseen = Pd;
                        pr = is_cov ? w.cov : w.ma;
                    } else {
                        pr = is_cov ? w.cov : w.ma;
                        welford_step(w, is_cov, mha, mhb, kh, Pd);
                    }
                }
            }
            if (el.is_mu)
                mu[e] = pr;
            else
                X[size_t(el.a) * Dp + el.b] = pr;
        }
        __syncthreads();
        const float* xl = line_ptr(a.x, line, a.n, a.in_stride, g);
        if (!initialized && t == 0) {
            // the initialising line is its own background (erx.hpp:54-55): its statistics straight
            // from the line in fp64 (line_stats, erx.hpp:38-40), not from the stats kernel's
            // centred / quantised sums — a two-pixel line scored against itself then has exactly
            // symmetric deltas, as in the reference
            for (int j = tid; j < D; j += nt) {
                double sm = 0.0;
                for (int p = 0; p < g.P; ++p) sm += proj(g, xl + size_t(p) * g.B, j);
                mu[j] = sm / Pd;
            }
            __syncthreads();
            for (int e = tid; e < D * (D + 1) / 2; e += nt) {
                int i, j;
                unpack_tri(e, i, j);
                double sm = 0.0;
                for (int p = 0; p < g.P; ++p) {
                    const float* row = xl + size_t(p) * g.B;
                    sm += (proj(g, row, i) - mu[i]) * (proj(g, row, j) - mu[j]);
                }
                X[size_t(i) * Dp + j] = sm / (Pd - 1.0);
            }
            __syncthreads();
        }
        // ---- 2. L = chol(K + eps I), eps x10 up to 1e-1
        double eps = a.eps0;
        int fail;
        while (true) {
            for (int idx = tid; idx < D * D; idx += nt) {
                const int i = idx / D, j = idx - i * D;
                if (j <= i) A[size_t(i) * Dp + j] = X[size_t(i) * Dp + j] + (i == j ? eps : 0.0);
            }
            __syncthreads();
            fail = chol_blocked(A, D, Dp, dyn, dyn + kNB * (kNB + 1), &s_fail);
            __syncthreads();
            if (fail < 0) break;
            const double next = eps * 10.0;
            if (!(next <= 1e-1 * (1.0 + 1e-9))) break;
            eps = next;
        }
        if (fail >= 0) {
            if (tid == 0) {
                a.status[line] = fail;
                if (atomicCAS(a.latch, 0ull, 1ull) == 0ull) {
                    a.latch[1] = static_cast<unsigned long long>(a.state.meta->lines_seen * a.line_mult + a.line_off + line);
                    a.latch[2] = static_cast<unsigned long long>(fail);
                }
            }
            __syncthreads();
            continue;
        }
        // ---- 3. X = L^{-1}
        tri_inverse_blocked(A, X, D, Dp, dyn);
        __syncthreads();
        // ---- 4. delta_i = || X (z_i - mu) || for every pixel, fp64
        float* rawl = a.raw + size_t(line) * g.P;
        const int LDV = D + 1;  // odd stride: the 32 pixels of a warp hit distinct bank pairs
        double* V = dyn;        // [kFixPx][LDV]
        const int pp = tid & (kFixPx - 1), rg = tid / kFixPx, nrg = nt / kFixPx;
        for (int p0 = 0; p0 < g.P; p0 += kFixPx) {
            const int np = min(kFixPx, g.P - p0);
            for (int idx = tid; idx < np * D; idx += nt) {
                const int p = idx / D, j = idx - p * D;
                V[p * LDV + j] = proj(g, xl + size_t(p0 + p) * g.B, j) - mu[j];
            }
            __syncthreads();
            double acc = 0.0;
            if (pp < np) {
                for (int i = rg; i < D; i += nrg) {
                    const double* xr = X + size_t(i) * Dp;
                    double m0 = 0.0, m1 = 0.0;
                    int j = 0;
                    for (; j + 1 <= i; j += 2) {
                        m0 = fma(xr[j], V[pp * LDV + j], m0);
                        m1 = fma(xr[j + 1], V[pp * LDV + j + 1], m1);
                    }
                    if (j == i) m0 = fma(xr[j], V[pp * LDV + j], m0);
                    const double m = m0 + m1;
                    acc = fma(m, m, acc);
                }
            }
            red[tid] = acc;
            __syncthreads();
            if (tid < np) {
                double sum = 0.0;
                for (int r = 0; r < nrg; ++r) sum += red[r * kFixPx + tid];
                const double d = sqrt(sum);
                dl[p0 + tid] = d;
                rawl[p0 + tid] = float(d);
            }
            __syncthreads();
        }
        // ---- 5. normalize_scores (detector.hpp:29-32) from the fp64 deltas: population std, and the
        // zero-variance rule std < 1e-12 -> 0 decided on fp64 values as the reference does
        if (warp == 0) {
            const int P = g.P;
            double sm = 0.0;
            for (int i = lane; i < P; i += 32) sm += dl[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
            const double mean = sm / double(P);
            double v = 0.0;
            for (int i = lane; i < P; i += 32) {
                const double d = dl[i] - mean;
                v += d * d;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            const double sd = sqrt(v / double(P));
            float* out = a.norm + size_t(line) * P;
            for (int i = lane; i < P; i += 32) out[i] = (sd < 1e-12) ? 0.f : float((dl[i] - mean) / sd);
            if (lane == 0) a.status[line] = -1;
        }
        __syncthreads();
    }
    // the last CTA out resets the list for the next window (every CTA has read the count)
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&a.list[1], 1) == int(gridDim.x) - 1) {
            a.list[a.list_cap + 2] += a.list[0];  // running total of rescued lines (erx_rescued_lines)
            a.list[0] = 0;
            a.list[1] = 0;
            __threadfence();
        }
    }
}

}  // namespace

int fixup_ctas(const Geometry& g, int n_lines_total) {
    // enough CTAs for a burst of listed lines, few enough that the empty launch stays short and the
    // fp64 workspace (2 Dp^2 doubles per CTA) small
    const int cap = g.Dp > 256 ? 16 : 32;
    return n_lines_total < cap ? n_lines_total : cap;
}

size_t fixup_work_doubles(const Geometry& g, int n_lines_total) {
    return size_t(fixup_ctas(g, n_lines_total)) * (2 * size_t(g.Dp) * g.Dp + g.P);
}

void launch_fixup(const FixupArgs& a, int n_lines_total, cudaStream_t st) {
    const Geometry& g = a.g;
    const size_t chol = size_t(kNB) * (kNB + 1) + size_t(g.D) * (kNB + 1);
    const size_t inv = size_t(kNB) * (g.D + 1);
    const size_t scr = size_t(kFixPx) * (g.D + 1);
    const size_t sm = (size_t(g.Dp) + std::max(chol, std::max(inv, scr))) * sizeof(double);
    ensure_smem(fixup_kernel, sm);
    fixup_kernel<<<fixup_ctas(g, n_lines_total), kFixThreads, sm, st>>>(a);
}

}  // namespace erxk
