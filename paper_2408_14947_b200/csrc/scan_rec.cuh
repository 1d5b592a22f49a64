// scan_rec.cuh — the per-element background recurrence of ema_update
// (erx.hpp:42-44) and welford_batch_update (linalg.hpp:33-36), shared by the
// window scan (k_scan.cu) and the fp64 line rescue (k_fixup.cu) so both
// produce the same bits for the same (element, line).  Every operation is an
// explicit round-to-nearest intrinsic: no FMA contraction can make the two
// kernels disagree.
#pragma once

#include "erx_common.cuh"

namespace erxk {

// mu_hat = c + s / P or K_hat = (S - s_a s_b / P) / (P - 1) from the stats slot values x0 (c or S),
// x1, x2 (s_a, s_b)
__device__ __forceinline__ double finish_stat(bool is_mu, double x0, double x1, double x2, double invP, double invP1) {
    return is_mu ? __dadd_rn(x0, __dmul_rn(x1, invP))
                 : __dmul_rn(__dsub_rn(x0, __dmul_rn(__dmul_rn(x1, x2), invP)), invP1);
}

__device__ __forceinline__ void unpack_tri(int k, int& a, int& b) {
    a = int((sqrt(8.0 * k + 1.0) - 1.0) * 0.5);
    while (a * (a + 1) / 2 > k) --a;
    while ((a + 1) * (a + 2) / 2 <= k) ++a;
    b = k - a * (a + 1) / 2;
}

// One state element: e < D is mu_e, e >= D the packed covariance entry (a, b); o0..o2 are its stats-slot
// offsets ([c | s | S] per line, k_stats.cu contract).
struct ScanElem {
    int a, b;
    bool is_mu;
    int o0, o1, o2;
};
__device__ __forceinline__ ScanElem scan_elem(int D, int e) {
    ScanElem r;
    r.a = e;
    r.b = e;
    if (e >= D) unpack_tri(e - D, r.a, r.b);
    r.is_mu = e < D;
    r.o0 = r.is_mu ? e : 2 * D + (e - D);
    r.o1 = D + r.a;
    r.o2 = D + r.b;
    return r;
}

// EMA: state <- (1 - alpha) state + alpha * line value
__device__ __forceinline__ double ema_step(double state, double cur, double om, double alpha) {
    return __dadd_rn(__dmul_rn(om, state), __dmul_rn(alpha, cur));
}

// Batched Welford (Chan) merge of one line of P pixels into the running (means ma / mb, covariance
// entry cov, count nseen); cov is only meaningful for covariance elements.
struct WelfordElem {
    double ma, mb, cov, nseen;
};
__device__ __forceinline__ void welford_step(WelfordElem& w, bool is_cov, double mha, double mhb, double khat,
                                             double nb) {
    const double na = w.nseen, nn = __dadd_rn(na, nb);
    const double da = __dsub_rn(mha, w.ma), db = __dsub_rn(mhb, w.mb);
    if (is_cov) {
        const double m2a = (na >= 2.0) ? __dmul_rn(w.cov, __dsub_rn(na, 1.0)) : 0.0;
        const double m2b = __dmul_rn(khat, __dsub_rn(nb, 1.0));
        const double m2 = __dadd_rn(__dadd_rn(m2a, m2b), __dmul_rn(__dmul_rn(da, db), __ddiv_rn(__dmul_rn(na, nb), nn)));
        w.cov = (nn >= 2.0) ? __ddiv_rn(m2, __dsub_rn(nn, 1.0)) : 0.0;
    }
    const double f = __ddiv_rn(nb, nn);
    w.ma = __dadd_rn(w.ma, __dmul_rn(da, f));
    w.mb = __dadd_rn(w.mb, __dmul_rn(db, f));
    w.nseen = nn;
}

}  // namespace erxk
