// datagen.cpp — the BASELINE.json synthetic line-scan workloads
// (include/erx_datagen.h).  Input generation only (not the scored path).
//
// Pinned laws:
//  * stream-level draws from Rng(mix_seed(seed, 0x5EED)) in this order:
//    base spectra (one per scene), drift direction, loading matrix A
//    (row-major b x r), random scene-change lines, then anomalies
//    (line, pixel, shape, target / offset / mixture fraction);
//  * line t draws from Rng(mix_seed(seed, t + 1)): per pixel, r factor
//    normals z then b noise normals e;  x = base(t) + A z + e;
//  * smooth spectrum = 4 Gaussians (amplitude U(0.2,1), centre U(0,b),
//    width U(b/20, b/4)) min-max scaled into [0.05, 0.6];
//  * drift(t) = drift * (t / L) * d, d a smooth spectrum mapped to [-1, 1].
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/erx_datagen.h"
#include "datagen_plan.hpp"
#include "host_rng.hpp"

using erx_host::mix_seed;
using erx_host::Rng;

namespace {

std::vector<double> smooth_spectrum(Rng& g, uint32_t B) {
    std::vector<double> s(B, 0.0);
    const double wlo = std::max(0.5, B / 20.0), whi = std::max(wlo, B / 4.0);
    for (int k = 0; k < 4; ++k) {
        const double amp = 0.2 + 0.8 * g.uniform();
        const double c = g.uniform() * B;
        const double w = wlo + g.uniform() * (whi - wlo);
        for (uint32_t b = 0; b < B; ++b) {
            const double u = (double(b) - c) / w;
            s[b] += amp * std::exp(-0.5 * u * u);
        }
    }
    const double lo = *std::min_element(s.begin(), s.end());
    const double hi = *std::max_element(s.begin(), s.end());
    for (auto& v : s) v = (hi > lo) ? 0.05 + 0.55 * (v - lo) / (hi - lo) : 0.3;
    return s;
}

struct Cell {
    int dl, dp;
};

struct Anomaly {
    int64_t line0;
    int64_t pix0;
    std::vector<Cell> cells;
    std::vector<double> spec;  // target spectrum or offset vector
    double f = 0.0;            // mixture fraction
};

struct Stream {
    std::vector<std::vector<double>> base;  // per scene
    std::vector<double> drift;              // direction in [-1, 1]
    std::vector<double> A;                  // B x r
    std::vector<int64_t> changes;           // sorted scene-change lines
    std::vector<Anomaly> anoms;
};

Stream build(const erx_gen_spec& s) {
    Stream st;
    Rng g(mix_seed(s.seed, 0x5EED));
    const uint32_t B = s.bands;
    for (uint32_t k = 0; k <= s.n_scene_changes; ++k) {
        if (s.base_kind == ERX_BASE_UNIFORM) {
            std::vector<double> b(B);
            for (auto& v : b) v = 0.05 + 0.45 * g.uniform();
            st.base.push_back(b);
        } else {
            st.base.push_back(smooth_spectrum(g, B));
        }
    }
    st.drift = smooth_spectrum(g, B);
    for (auto& v : st.drift) v = (v - 0.325) / 0.275;
    st.A.resize(size_t(B) * s.n_factors);
    for (auto& v : st.A) v = g.normal() * s.loading_sd;
    for (uint32_t k = 0; k < s.n_scene_changes && k < 4; ++k) {
        int64_t c = s.scene_change_line[k];
        if (c < 0) c = int64_t(s.lines / 10) + int64_t(g.below(std::max<uint64_t>(1, 8ull * s.lines / 10)));
        st.changes.push_back(c);
    }
    std::sort(st.changes.begin(), st.changes.end());
    double avg = 1.0;
    if (s.anomaly_kind == ERX_ANOM_BLOB3X3) avg = 9.0;
    if (s.anomaly_kind == ERX_ANOM_BLOB2TO5) avg = 3.5;
    const uint64_t n_anom = uint64_t(std::llround(s.anomaly_frac * double(s.lines) * double(s.pixels) / avg));
    for (uint64_t i = 0; i < n_anom; ++i) {
        Anomaly a;
        a.line0 = int64_t(g.below(s.lines));
        a.pix0 = int64_t(g.below(s.pixels));
        switch (s.anomaly_kind) {
            case ERX_ANOM_BLOB3X3:
                for (int dl = 0; dl < 3; ++dl)
                    for (int dp = 0; dp < 3; ++dp) a.cells.push_back({dl, dp});
                a.spec = smooth_spectrum(g, B);
                break;
            case ERX_ANOM_BLOB2TO5: {
                const int k = 2 + int(g.below(4));
                if (k == 2) a.cells = {{0, 0}, {0, 1}};
                if (k == 3) a.cells = {{0, 0}, {0, 1}, {0, 2}};
                if (k == 4) a.cells = {{0, 0}, {0, 1}, {1, 0}, {1, 1}};
                if (k == 5) a.cells = {{0, 1}, {1, 0}, {1, 1}, {1, 2}, {2, 1}};
                a.spec = smooth_spectrum(g, B);
                break;
            }
            case ERX_ANOM_OFFSET:
                a.cells = {{0, 0}};
                a.spec.resize(B);
                for (auto& v : a.spec) v = g.normal() * s.offset_sd;
                break;
            default:
                a.cells = {{0, 0}};
                a.f = s.mix_lo + (s.mix_hi - s.mix_lo) * g.uniform();
                a.spec = smooth_spectrum(g, B);
                break;
        }
        st.anoms.push_back(std::move(a));
    }
    return st;
}

// build() costs ~4 ms for c3 (a smooth spectrum per anomaly): keep the last few streams
std::shared_ptr<const Stream> build_cached(const erx_gen_spec& in) {
    erx_gen_spec s;
    std::memset(&s, 0, sizeof(s));  // padding bytes zero: the cache compares whole structs
    s.lines = in.lines; s.pixels = in.pixels; s.bands = in.bands; s.n_factors = in.n_factors;
    s.loading_sd = in.loading_sd; s.noise_sd = in.noise_sd; s.base_kind = in.base_kind;
    s.drift = in.drift; s.n_scene_changes = in.n_scene_changes;
    for (int k = 0; k < 4; ++k) s.scene_change_line[k] = in.scene_change_line[k];
    s.anomaly_frac = in.anomaly_frac; s.anomaly_kind = in.anomaly_kind; s.offset_sd = in.offset_sd;
    s.mix_lo = in.mix_lo; s.mix_hi = in.mix_hi; s.seed = in.seed;
    static std::mutex mu;
    static std::vector<std::pair<erx_gen_spec, std::shared_ptr<const Stream>>> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : cache)
        if (std::memcmp(&e.first, &s, sizeof(s)) == 0) return e.second;
    auto st = std::make_shared<const Stream>(build(s));
    if (cache.size() >= 8) cache.erase(cache.begin());
    cache.push_back({s, st});
    return st;
}

void gen_line(const erx_gen_spec& s, const Stream& st, const std::vector<std::vector<std::pair<int, int>>>& hits,
              uint32_t t, uint32_t rel, float* out, uint8_t* mask) {
    const uint32_t B = s.bands, P = s.pixels, R = s.n_factors;
    size_t scene = 0;
    while (scene < st.changes.size() && int64_t(t) >= st.changes[scene]) ++scene;
    std::vector<double> base(B);
    const double dt = s.drift * double(t) / double(std::max<uint32_t>(1, s.lines));
    for (uint32_t b = 0; b < B; ++b) base[b] = st.base[scene][b] + dt * st.drift[b];
    Rng r(mix_seed(s.seed, uint64_t(t) + 1));
    std::vector<double> z(R), e(B);
    std::vector<double> bg(size_t(P) * B), noise(size_t(P) * B);
    for (uint32_t p = 0; p < P; ++p) {
        for (auto& v : z) v = r.normal();
        for (uint32_t b = 0; b < B; ++b) e[b] = r.normal() * s.noise_sd;
        for (uint32_t b = 0; b < B; ++b) {
            double v = base[b] + e[b];
            const double* a = st.A.data() + size_t(b) * R;
            for (uint32_t k = 0; k < R; ++k) v += a[k] * z[k];
            bg[size_t(p) * B + b] = v;
            noise[size_t(p) * B + b] = e[b];
        }
    }
    if (mask) std::memset(mask, 0, P);
    for (const auto& h : hits[rel]) {
        const Anomaly& a = st.anoms[h.first];
        const uint32_t p = uint32_t(h.second);
        double* px = bg.data() + size_t(p) * B;
        const double* ns = noise.data() + size_t(p) * B;
        for (uint32_t b = 0; b < B; ++b) {
            switch (s.anomaly_kind) {
                case ERX_ANOM_OFFSET: px[b] += a.spec[b]; break;
                case ERX_ANOM_MIXTURE: px[b] = (1.0 - a.f) * px[b] + a.f * a.spec[b]; break;
                default: px[b] = a.spec[b] + ns[b]; break;
            }
        }
        if (mask) mask[p] = 1;
    }
    for (size_t i = 0; i < bg.size(); ++i) out[i] = float(bg[i]);
}

}  // namespace

namespace erx_host {

// The stream-level draws flattened for the device generator (k_datagen.cu): the same build()
// and the same per-line hit lists as erx_gen_lines.
int gen_plan(const erx_gen_spec& s, uint32_t first, uint32_t n, GenPlan& pl) {
    if (s.pixels < 1 || s.bands < 1 || s.lines < 1) return 2;
    const auto stp = build_cached(s);
    const Stream& st = *stp;
    pl.B = s.bands;
    pl.P = s.pixels;
    pl.R = s.n_factors;
    pl.base.clear();
    for (const auto& b : st.base) pl.base.insert(pl.base.end(), b.begin(), b.end());
    pl.drift = st.drift;
    pl.A = st.A;
    pl.changes = st.changes;
    std::vector<std::vector<std::pair<int, int>>> hits(n);
    for (size_t i = 0; i < st.anoms.size(); ++i) {
        const Anomaly& a = st.anoms[i];
        for (const Cell& c : a.cells) {
            const int64_t l = a.line0 + c.dl, p = a.pix0 + c.dp;
            if (l < int64_t(first) || l >= int64_t(first) + n || p >= int64_t(s.pixels) || l >= int64_t(s.lines))
                continue;
            hits[size_t(l - first)].push_back({int(i), int(p)});
        }
    }
    pl.hit_off.assign(1, 0u);
    pl.hit_pix.clear();
    pl.hit_anom.clear();
    pl.anom_spec.clear();
    pl.anom_f.clear();
    std::vector<int> slot(st.anoms.size(), -1);
    for (uint32_t l = 0; l < n; ++l) {
        for (const auto& h : hits[l]) {
            if (slot[h.first] < 0) {
                slot[h.first] = int(pl.anom_f.size());
                pl.anom_f.push_back(st.anoms[h.first].f);
                const auto& sp = st.anoms[h.first].spec;
                pl.anom_spec.insert(pl.anom_spec.end(), sp.begin(), sp.end());
            }
            pl.hit_pix.push_back(uint32_t(h.second));
            pl.hit_anom.push_back(uint32_t(slot[h.first]));
        }
        pl.hit_off.push_back(uint32_t(pl.hit_pix.size()));
    }
    return 0;
}

}  // namespace erx_host

extern "C" {

int erx_gen_preset(int id, uint32_t stream, erx_gen_spec* o) {
    std::memset(o, 0, sizeof(*o));
    for (auto& c : o->scene_change_line) c = -1;
    o->drift = 0.05;
    o->base_kind = ERX_BASE_SMOOTH;
    switch (id) {
        case 0:
            o->lines = 2000; o->pixels = 384; o->bands = 108; o->n_factors = 8;
            o->loading_sd = 0.02; o->noise_sd = 0.005;
            o->anomaly_frac = 0.003; o->anomaly_kind = ERX_ANOM_BLOB3X3; o->seed = 0;
            break;
        case 1:
            o->lines = 10000; o->pixels = 640; o->bands = 224; o->n_factors = 12;
            o->loading_sd = 0.02; o->noise_sd = 0.005;
            o->n_scene_changes = 1; o->scene_change_line[0] = 5000;
            o->anomaly_frac = 0.002; o->anomaly_kind = ERX_ANOM_BLOB2TO5; o->seed = 0;
            break;
        case 2:
            o->lines = 20000; o->pixels = 1024; o->bands = 10; o->n_factors = 3;
            o->loading_sd = 0.03; o->noise_sd = 0.01; o->base_kind = ERX_BASE_UNIFORM;
            o->anomaly_frac = 0.005; o->anomaly_kind = ERX_ANOM_OFFSET; o->offset_sd = 0.1; o->seed = 0;
            break;
        case 3:
            o->lines = 5000; o->pixels = 640; o->bands = 108; o->n_factors = 8;
            o->loading_sd = 0.02; o->noise_sd = 0.005;
            o->anomaly_frac = 0.003; o->anomaly_kind = ERX_ANOM_BLOB3X3; o->seed = stream;
            break;
        case 4:
            o->lines = 3000; o->pixels = 1280; o->bands = 448; o->n_factors = 16;
            o->loading_sd = 0.015; o->noise_sd = 0.003; o->n_scene_changes = 2;
            o->anomaly_frac = 0.002; o->anomaly_kind = ERX_ANOM_MIXTURE; o->mix_lo = 0.3; o->mix_hi = 0.7;
            o->seed = stream;
            break;
        default:
            return 2;
    }
    return 0;
}

int erx_gen_lines(const erx_gen_spec* spec, uint32_t first, uint32_t n, float* out, uint8_t* mask, int threads) {
    if (!spec || spec->pixels < 1 || spec->bands < 1 || spec->lines < 1) return 2;
    const erx_gen_spec s = *spec;
    const auto stp = build_cached(s);
    const Stream& st = *stp;
    std::vector<std::vector<std::pair<int, int>>> hits(n);
    for (size_t i = 0; i < st.anoms.size(); ++i) {
        const Anomaly& a = st.anoms[i];
        for (const Cell& c : a.cells) {
            const int64_t l = a.line0 + c.dl, p = a.pix0 + c.dp;
            if (l < int64_t(first) || l >= int64_t(first) + n || p >= int64_t(s.pixels) || l >= int64_t(s.lines))
                continue;
            hits[size_t(l - first)].push_back({int(i), int(p)});
        }
    }
    int nt = threads > 0 ? threads : int(std::max(1u, std::thread::hardware_concurrency()));
    nt = std::min<int>(nt, int(std::max<uint32_t>(1, n)));
    std::atomic<uint32_t> next{0};
    auto work = [&]() {
        for (;;) {
            const uint32_t i = next.fetch_add(1);
            if (i >= n) return;
            gen_line(s, st, hits, first + i, i, out + size_t(i) * s.pixels * s.bands,
                     mask ? mask + size_t(i) * s.pixels : nullptr);
        }
    };
    std::vector<std::thread> pool;
    for (int k = 0; k < nt; ++k) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    return 0;
}

int erx_gen_scene_changes(const erx_gen_spec* spec, int64_t* out) {
    if (!spec || spec->pixels < 1 || spec->bands < 1 || spec->lines < 1) return -1;
    const auto stp = build_cached(*spec);
    for (size_t k = 0; k < stp->changes.size(); ++k) out[k] = stp->changes[k];
    return int(stp->changes.size());
}

uint64_t erx_mix_seed(uint64_t seed, uint64_t n) { return mix_seed(seed, n); }

void erx_rng_probe(uint64_t seed, int kind, uint32_t n, uint64_t* u64_out, double* f64_out) {
    Rng r(seed);
    for (uint32_t i = 0; i < n; ++i) {
        switch (kind) {
            case 0: u64_out[i] = r.next_u64(); break;
            case 1: f64_out[i] = r.uniform(); break;
            case 2: f64_out[i] = double(r.uniform_f32()); break;
            case 3: f64_out[i] = r.normal(); break;
            default: u64_out[i] = r.below(u64_out[i]); break;  // bound given in u64_out[i]
        }
    }
}

}  // extern "C"
