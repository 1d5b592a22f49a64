// k_scan.cu — the background recurrence over a window: ema_update
// (erx.hpp:42-44) or welford_batch_update (linalg.hpp:33-36), element-wise
// over (mu, packed K), sequential over the window's lines in the reference's
// own order and rounding.
#include "erx_common.cuh"

namespace erxk {
namespace {

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

}  // namespace

void launch_scan(const Geometry& g, const double* stats, double* prior, const double* state_in, double* state_out,
                 int n_streams, int n_per_stream, int initialized, double alpha, int incremental, int64_t n_seen0,
                 cudaStream_t st) {
    dim3 grid((g.SE + 127) / 128, n_streams);
    scan_kernel<<<grid, 128, 0, st>>>(g, stats, prior, state_in, state_out, n_per_stream, initialized, alpha,
                                      incremental, n_seen0);
}

}  // namespace erxk
