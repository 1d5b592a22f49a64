// erx_oracle.cpp — CPU fp64 restatement of the reference ERX path.
//
// TEST INFRASTRUCTURE ONLY (see erx_oracle.h).  Each function cites the
// reference contract it restates.  The reference ships declarations only
// (no .cpp bodies), so the ERX bodies below follow SPEC.md
// line by line.  Pins:
//   * had::Rng / mix_seed against golden vectors produced by compiling the
//     reference's own rng.hpp (oracle/_ref, tests/golden/rng_golden.json);
//   * every SPEC.md known-answer example for linalg / erx / projection /
//     metrics (tests/test_oracle_kats.py);
//   * an independent dense-inverse numpy oracle at 1e-8.
// Beyond those the detector restatement is "parity unpinned" (no reference
// implementation exists to run).

#include "erx_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- Rng
// rng.hpp:18-72: std::mt19937_64 engine with hand-rolled transforms.
class Rng {
  public:
    explicit Rng(uint64_t seed) : eng_(seed) {}
    uint64_t next_u64() { return eng_(); }
    double uniform() { return double(eng_() >> 11) * 0x1.0p-53; }           // rng.hpp:25
    float uniform_f32() { return float(eng_() >> 40) * 0x1.0p-24f; }        // rng.hpp:28
    uint64_t below(uint64_t bound) {                                          // rng.hpp:31-37
        const uint64_t thr = (0 - bound) % bound;
        while (true) {
            uint64_t r = eng_();
            if (r >= thr) return r % bound;
        }
    }
    double normal() {                                                         // rng.hpp:40-53
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        double u2 = uniform();
        double rad = std::sqrt(-2.0 * std::log(u1));
        double ang = 6.283185307179586476925286766559 * u2;
        spare_ = rad * std::sin(ang);
        spare_ok_ = true;
        return rad * std::cos(ang);
    }
    std::vector<uint32_t> sample_indices(uint32_t n, uint32_t k) {           // rng.hpp:56-66
        std::vector<uint32_t> pool(n);
        for (uint32_t i = 0; i < n; ++i) pool[i] = i;
        k = std::min(k, n);
        for (uint32_t i = 0; i < k; ++i) {
            uint32_t j = i + uint32_t(below(n - i));
            std::swap(pool[i], pool[j]);
        }
        pool.resize(k);
        return pool;
    }

  private:
    std::mt19937_64 eng_;
    bool spare_ok_ = false;
    double spare_ = 0.0;
};

inline uint64_t mix_seed(uint64_t seed, uint64_t n) {                        // rng.hpp:75-83
    uint64_t x = seed ^ (0x9e3779b97f4a7c15ULL + n * 0xbf58476d1ce4e5b9ULL);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// ---------------------------------------------------------------- linalg
// cholesky_lower (linalg.hpp:12-15): row-oriented
// Cholesky–Banachiewicz, lower triangle read only; a pivot that is not > 0
// (including NaN) fails with its index.
int cholesky_lower(const double* a, int n, double* l) {
    std::fill(l, l + size_t(n) * n, 0.0);
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n; ++i) {
            double s = a[size_t(i) * n + j];
            for (int k = 0; k < j; ++k) s -= l[size_t(i) * n + k] * l[size_t(j) * n + k];
            if (i == j) {
                if (!(s > 0.0)) return j;
                l[size_t(j) * n + j] = std::sqrt(s);
            } else {
                l[size_t(i) * n + j] = s / l[size_t(j) * n + j];
            }
        }
    }
    return -1;
}

// forward_substitute_inplace (linalg.hpp:17-21).
int forward_substitute(const double* l, int n, double* x) {
    for (int i = 0; i < n; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s -= l[size_t(i) * n + k] * x[k];
        double d = l[size_t(i) * n + i];
        if (d == 0.0) return i;
        x[i] = s / d;
    }
    return -1;
}

// line_stats (erx.hpp:38-40): column mean and the unbiased
// 1/(p-1) covariance, two-pass.
int line_stats(const double* z, int p, int d, double* mu, double* cov) {
    if (p < 2) return 3;
    for (int j = 0; j < d; ++j) mu[j] = 0.0;
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < d; ++j) mu[j] += z[size_t(i) * d + j];
    for (int j = 0; j < d; ++j) mu[j] /= double(p);
    std::fill(cov, cov + size_t(d) * d, 0.0);
    std::vector<double> c(d);
    for (int i = 0; i < p; ++i) {
        for (int j = 0; j < d; ++j) c[j] = z[size_t(i) * d + j] - mu[j];
        for (int a = 0; a < d; ++a)
            for (int b = 0; b <= a; ++b) cov[size_t(a) * d + b] += c[a] * c[b];
    }
    for (int a = 0; a < d; ++a)
        for (int b = 0; b <= a; ++b) {
            double v = cov[size_t(a) * d + b] / double(p - 1);
            cov[size_t(a) * d + b] = v;
            cov[size_t(b) * d + a] = v;
        }
    return 0;
}

// welford_batch_update (linalg.hpp:33-36): Chan et al.
// pairwise combination of the running (mean, M2 = cov*(n-1), n) with the
// batch's own two-pass statistics.
int welford_batch_update(double* mean, double* cov, int64_t* n_seen, const double* batch, int k, int n) {
    if (k < 1) return 3;
    std::vector<double> mb(n, 0.0), m2b(size_t(n) * n, 0.0), c(n);
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < n; ++j) mb[j] += batch[size_t(i) * n + j];
    for (int j = 0; j < n; ++j) mb[j] /= double(k);
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j < n; ++j) c[j] = batch[size_t(i) * n + j] - mb[j];
        for (int a = 0; a < n; ++a)
            for (int b = 0; b <= a; ++b) m2b[size_t(a) * n + b] += c[a] * c[b];
    }
    const double na = double(*n_seen), nb = double(k), nn = na + nb;
    std::vector<double> delta(n);
    for (int j = 0; j < n; ++j) delta[j] = mb[j] - mean[j];
    for (int a = 0; a < n; ++a)
        for (int b = 0; b <= a; ++b) {
            double m2a = (*n_seen >= 2) ? cov[size_t(a) * n + b] * (na - 1.0) : 0.0;
            double m2 = m2a + m2b[size_t(a) * n + b] + delta[a] * delta[b] * (na * nb / nn);
            double v = (nn >= 2.0) ? m2 / (nn - 1.0) : 0.0;
            cov[size_t(a) * n + b] = v;
            cov[size_t(b) * n + a] = v;
        }
    for (int j = 0; j < n; ++j) mean[j] += delta[j] * (nb / nn);
    *n_seen += k;
    return 0;
}

// ---------------------------------------------------------------- projection
// generate_srp (projection.hpp:11-26): b x d, entries
// independent: +sqrt(s)/sqrt(d) w.p. 1/(2s), -sqrt(s)/sqrt(d) w.p. 1/(2s),
// else 0, s = sqrt(b).  Draw order pinned: row-major b x d,
// one uniform() per entry: u < 1/(2s) -> +, u < 1/s -> -, else 0.
void generate_srp(uint32_t b, uint32_t d, uint64_t seed, double* w) {
    Rng rng(seed);
    const double s = std::sqrt(double(b));
    const double v = std::sqrt(s) / std::sqrt(double(d));
    const double p_half = 1.0 / (2.0 * s), p_one = 1.0 / s;
    for (uint32_t i = 0; i < b; ++i)
        for (uint32_t j = 0; j < d; ++j) {
            double u = rng.uniform();
            w[size_t(i) * d + j] = (u < p_half) ? v : (u < p_one ? -v : 0.0);
        }
}

// project_line (projection.hpp:31-34): Z = X W in fp64,
// bands summed in ascending order; identity bypass copies X (no_srp).
int project_line(const float* x, uint32_t p, uint32_t b, const double* w, uint32_t w_rows, uint32_t d, int identity,
                 double* z) {
    if (w_rows != b) return 2;
    if (identity) {
        for (size_t i = 0; i < size_t(p) * b; ++i) z[i] = double(x[i]);
        return 0;
    }
    for (uint32_t i = 0; i < p; ++i)
        for (uint32_t j = 0; j < d; ++j) {
            double s = 0.0;
            for (uint32_t k = 0; k < b; ++k) s += double(x[size_t(i) * b + k]) * w[size_t(k) * d + j];
            z[size_t(i) * d + j] = s;
        }
    return 0;
}

// normalize_scores (detector.hpp:29-32): population std,
// std < 1e-12 -> zeros.
void normalize_scores(const double* raw, int p, double* norm) {
    double m = 0.0;
    for (int i = 0; i < p; ++i) m += raw[i];
    m /= double(p);
    double v = 0.0;
    for (int i = 0; i < p; ++i) v += (raw[i] - m) * (raw[i] - m);
    double sd = std::sqrt(v / double(p));
    for (int i = 0; i < p; ++i) norm[i] = (sd < 1e-12) ? 0.0 : (raw[i] - m) / sd;
}

// ---------------------------------------------------------------- detector
// ErxDetector (erx.hpp:51-71).
struct Erx {
    orc_erx_config cfg;
    uint32_t bands = 0;
    int d = 0;
    std::vector<double> w;  // bands x d (empty when no_srp)
    std::vector<double> mu, cov;
    int64_t lines_seen = 0, welford_n = 0;
    bool initialized = false;
    std::vector<double> z, l, mhat, khat, m;
};

static int validate(const orc_erx_config* c, uint32_t bands, std::string& msg) {
    // ErxConfig::validate (erx.hpp:23): 0<alpha<=1, eps>0, d>=1;
    // d <= b unless no_srp.
    if (!(c->alpha > 0.0 && c->alpha <= 1.0)) { msg = "alpha must be in (0, 1]"; return 2; }
    if (!(c->epsilon > 0.0)) { msg = "epsilon must be > 0"; return 2; }
    if (bands < 1) { msg = "bands must be >= 1"; return 2; }
    if (!c->no_srp) {
        if (c->dims < 1) { msg = "dims must be >= 1"; return 2; }
        if (uint32_t(c->dims) > bands) { msg = "dims must be <= bands"; return 2; }
    }
    return 0;
}

static void put(char* dst, size_t n, const std::string& s) {
    if (dst && n) {
        std::snprintf(dst, n, "%s", s.c_str());
    }
}

int erx_process(Erx& e, int64_t index, uint32_t p, uint32_t b, const float* data, double* raw, double* norm,
                uint8_t* warmup, int* pivot, std::string& msg) {
    if (b != e.bands) { msg = "band count mismatch"; return 2; }      // projection.hpp:31-32
    if (p < 2) { msg = "line needs p >= 2 pixels"; return 3; }          // erx.hpp:39
    const int d = e.d;
    e.z.resize(size_t(p) * d);
    project_line(data, p, b, e.w.data(), b, d, e.cfg.no_srp, e.z.data());
    e.mhat.resize(d);
    e.khat.resize(size_t(d) * d);
    line_stats(e.z.data(), int(p), d, e.mhat.data(), e.khat.data());
    const bool first = !e.initialized;
    if (first) {                                                         // erx.hpp:54-55
        e.mu = e.mhat;
        e.cov = e.khat;
        if (e.cfg.use_incremental) e.welford_n = p;  // "incremental mode only" (erx.hpp:32)
        e.initialized = true;
    }
    // Cholesky of K + eps I with eps escalation x10 up to 1e-1 (§9.2).
    std::vector<double> a(size_t(d) * d);
    e.l.resize(size_t(d) * d);
    double eps = e.cfg.epsilon;
    int piv = -1;
    while (true) {
        for (size_t i = 0; i < a.size(); ++i) a[i] = e.cov[i];
        for (int j = 0; j < d; ++j) a[size_t(j) * d + j] += eps;
        piv = cholesky_lower(a.data(), d, e.l.data());
        if (piv < 0) break;
        double next = eps * 10.0;
        if (!(next <= 1e-1 * (1.0 + 1e-9))) {
            if (pivot) *pivot = piv;
            msg = "Cholesky failed at pivot " + std::to_string(piv) + " after epsilon escalation";
            return 5;
        }
        eps = next;
    }
    // Score every pixel against the pre-update background.
    e.m.resize(d);
    for (uint32_t i = 0; i < p; ++i) {
        for (int j = 0; j < d; ++j) e.m[j] = e.z[size_t(i) * d + j] - e.mu[j];
        forward_substitute(e.l.data(), d, e.m.data());
        double s = 0.0;
        for (int j = 0; j < d; ++j) s += e.m[j] * e.m[j];
        raw[i] = std::sqrt(s);
    }
    // Fold this line into the background (score-then-update).
    // The initialising line is already the whole background.
    if (!first) {
        if (e.cfg.use_incremental) {
            welford_batch_update(e.mu.data(), e.cov.data(), &e.welford_n, e.z.data(), int(p), d);
        } else {                                                         // erx.hpp:42-44
            const double al = e.cfg.alpha;
            for (int j = 0; j < d; ++j) e.mu[j] = (1.0 - al) * e.mu[j] + al * e.mhat[j];
            for (size_t k = 0; k < e.cov.size(); ++k) e.cov[k] = (1.0 - al) * e.cov[k] + al * e.khat[k];
        }
    }
    e.lines_seen += 1;
    if (norm) normalize_scores(raw, int(p), norm);
    if (warmup) *warmup = (index < int64_t(e.cfg.buffer_len)) ? 1 : 0;
    return 0;
}

// Exact ROC AUC with ties grouped (metrics.hpp:25-28):
// trapezoid over the (fpr, tpr) steps at every unique score.
double roc_auc(const double* s, const uint8_t* y, size_t n, int* status) {
    size_t npos = 0;
    for (size_t i = 0; i < n; ++i) npos += y[i] ? 1 : 0;
    size_t nneg = n - npos;
    if (npos == 0 || nneg == 0) {
        if (status) *status = 4;
        return 0.0;
    }
    std::vector<size_t> idx(n);
    for (size_t i = 0; i < n; ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return s[a] > s[b]; });
    double auc = 0.0, tp = 0, fp = 0, ptp = 0, pfp = 0;
    size_t i = 0;
    while (i < n) {
        size_t j = i;
        while (j < n && s[idx[j]] == s[idx[i]]) {
            if (y[idx[j]]) tp += 1; else fp += 1;
            ++j;
        }
        auc += (fp - pfp) / double(nneg) * (tp + ptp) / (2.0 * double(npos));
        ptp = tp;
        pfp = fp;
        i = j;
    }
    if (status) *status = 0;
    return auc;
}

}  // namespace orc

using namespace orc;

extern "C" {

void* orc_rng_new(uint64_t seed) { return new Rng(seed); }
void orc_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t orc_rng_next_u64(void* r) { return static_cast<Rng*>(r)->next_u64(); }
double orc_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
float orc_rng_uniform_f32(void* r) { return static_cast<Rng*>(r)->uniform_f32(); }
uint64_t orc_rng_below(void* r, uint64_t bound) { return static_cast<Rng*>(r)->below(bound); }
double orc_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
void orc_rng_sample_indices(void* r, uint32_t n, uint32_t k, uint32_t* out, uint32_t* out_k) {
    auto v = static_cast<Rng*>(r)->sample_indices(n, k);
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    if (out_k) *out_k = uint32_t(v.size());
}
uint64_t orc_mix_seed(uint64_t seed, uint64_t n) { return mix_seed(seed, n); }

int orc_cholesky_lower(const double* a, int n, double* l) { return cholesky_lower(a, n, l); }
int orc_forward_substitute(const double* l, int n, double* x) { return forward_substitute(l, n, x); }
int orc_welford_batch_update(double* mean, double* cov, int64_t* n_seen, const double* batch, int k, int n) {
    return welford_batch_update(mean, cov, n_seen, batch, k, n);
}
void orc_generate_srp(uint32_t bands, uint32_t dims, uint64_t seed, double* w) { generate_srp(bands, dims, seed, w); }
int orc_project_line(const float* x, uint32_t p, uint32_t b, const double* w, uint32_t w_rows, uint32_t d,
                     int identity, double* z) {
    return project_line(x, p, b, w, w_rows, d, identity, z);
}
int orc_line_stats(const double* z, int p, int d, double* mu, double* cov) { return line_stats(z, p, d, mu, cov); }
void orc_normalize_scores(const double* raw, int p, double* norm) { normalize_scores(raw, p, norm); }
void orc_apply_threshold(const double* norm, int p, double tau, uint8_t* out) {   // erx.hpp:46-47
    for (int i = 0; i < p; ++i) out[i] = norm[i] >= tau ? 1 : 0;
}

void* orc_erx_new(const orc_erx_config* cfg, uint32_t bands, int* status, char* msg, size_t msglen) {
    std::string m;
    int st = validate(cfg, bands, m);
    if (status) *status = st;
    if (st) {
        put(msg, msglen, m);
        return nullptr;
    }
    Erx* e = new Erx();
    e->cfg = *cfg;
    e->bands = bands;
    if (cfg->no_srp) {
        e->d = int(bands);                                                   // projection.hpp:28-29
    } else {
        e->d = cfg->dims;
        e->w.resize(size_t(bands) * cfg->dims);
        generate_srp(bands, uint32_t(cfg->dims), cfg->seed, e->w.data());
    }
    return e;
}
void orc_erx_free(void* h) { delete static_cast<Erx*>(h); }
int orc_erx_dims(void* h) { return static_cast<Erx*>(h)->d; }

int orc_erx_process(void* h, int64_t index, uint32_t p, uint32_t b, const float* data, double* raw, double* norm,
                    uint8_t* warmup, int* pivot, char* msg, size_t msglen) {
    std::string m;
    int st = erx_process(*static_cast<Erx*>(h), index, p, b, data, raw, norm, warmup, pivot, m);
    if (st) put(msg, msglen, m);
    return st;
}

// Install a background (mu, K, lines_seen, welford_n): the detector continues as if it had
// reached this state itself.  ErxState is a plain value type (erx.hpp:27-34) that SPEC.md:337
// lets move between threads between lines; tests use this to pin states the stream would only
// reach by rounding accidents (an indefinite K that forces the eps escalation of SPEC.md:306).
int orc_erx_set_state(void* h, const double* mu, const double* cov, int64_t lines_seen, int64_t welford_n) {
    Erx* e = static_cast<Erx*>(h);
    e->mu.assign(mu, mu + e->d);
    e->cov.assign(cov, cov + size_t(e->d) * e->d);
    e->lines_seen = lines_seen;
    e->welford_n = welford_n;
    e->initialized = true;
    return 0;
}

int orc_erx_state(void* h, double* mu, double* cov, int64_t* lines_seen, int64_t* welford_n, int* initialized,
                  double* weights) {
    Erx* e = static_cast<Erx*>(h);
    if (mu && e->initialized) std::memcpy(mu, e->mu.data(), sizeof(double) * e->d);
    if (cov && e->initialized) std::memcpy(cov, e->cov.data(), sizeof(double) * e->d * e->d);
    if (lines_seen) *lines_seen = e->lines_seen;
    if (welford_n) *welford_n = e->welford_n;
    if (initialized) *initialized = e->initialized ? 1 : 0;
    if (weights && !e->w.empty()) std::memcpy(weights, e->w.data(), sizeof(double) * e->w.size());
    return 0;
}

int orc_erx_run_streams(const orc_erx_config* cfg, uint32_t bands, uint32_t n_streams, uint32_t n_lines,
                        uint32_t p, const float* lines, double* raw, double* norm, int threads) {
    std::atomic<uint32_t> next{0};
    std::atomic<int> err{0};
    auto worker = [&]() {
        std::vector<double> r(p), nm(p);
        while (true) {
            uint32_t s = next.fetch_add(1);
            if (s >= n_streams || err.load()) return;
            int st = 0;
            Erx* e = static_cast<Erx*>(orc_erx_new(cfg, bands, &st, nullptr, 0));
            if (!e) { err = st; return; }
            std::string m;
            for (uint32_t t = 0; t < n_lines; ++t) {
                const float* x = lines + (size_t(s) * n_lines + t) * p * bands;
                double* ro = raw ? raw + (size_t(s) * n_lines + t) * p : r.data();
                double* no = norm ? norm + (size_t(s) * n_lines + t) * p : nm.data();
                st = erx_process(*e, int64_t(t), p, bands, x, ro, no, nullptr, nullptr, m);
                if (st) { err = st; break; }
            }
            delete e;
        }
    };
    int nt = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int i = 0; i < nt; ++i) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    return err.load();
}

double orc_roc_auc(const double* scores, const uint8_t* labels, size_t n, int* status) {
    return roc_auc(scores, labels, n, status);
}

}  // extern "C"
