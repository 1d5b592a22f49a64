// Drop-in check: code written against the reference interface
// (had::ErxDetector / had::LineDetector / had::SpectralLine / had::ScoredLine and
// the free functions of proj/include/hadkit/{erx,detector,cube,projection}.hpp),
// including the reference's own include paths ("hadkit/erx.hpp"), compiled
// against include/ and linked to liberx_b200.so.  Runs the
// reference line-scan loop (SPEC.md:642-650 shape) on a generated cube and
// prints one JSON summary line for tests/test_cpp_mirror.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "erx_datagen.h"
#include "hadkit/detector.hpp"
#include "hadkit/erx.hpp"
#include "hadkit/projection.hpp"

static int run_loop(had::LineDetector& det, const std::vector<float>& cube, std::uint32_t lines, std::uint32_t p,
                    std::uint32_t b, std::vector<had::ScoredLine>& out) {
    for (std::uint32_t t = 0; t < lines; ++t) {
        had::SpectralLine line{std::int64_t(t), p, b, cube.data() + size_t(t) * p * b};
        det.process(line, out);
    }
    det.finish(out);
    return int(out.size());
}

int main() {
    erx_gen_spec spec;
    erx_gen_preset(0, 0, &spec);
    const std::uint32_t L = 40, P = spec.pixels, B = spec.bands;
    std::vector<float> cube(size_t(L) * P * B);
    erx_gen_lines(&spec, 0, L, cube.data(), nullptr, 0);

    had::ErxDetector det(had::ErxConfig{.alpha = 0.1, .no_srp = true}, B, /*window_lines=*/16);
    std::vector<had::ScoredLine> out;
    const int n = run_loop(det, cube, L, P, B, out);
    bool order_ok = n == int(L);
    for (int i = 0; i < n; ++i) order_ok = order_ok && out[size_t(i)].index == i && out[size_t(i)].raw.size() == P;
    double mean_norm = 0.0;
    for (double v : out.back().norm) mean_norm += v;
    mean_norm /= P;
    const auto st = det.state();

    int cfg_err = 0, data_err = 0, fact_err = 0, pivot = -1;
    try {
        had::ErxDetector bad(had::ErxConfig{.alpha = 0.0}, B);
    } catch (const had::ConfigError& e) {
        cfg_err = e.exit_code();
    }
    try {
        std::vector<float> one(B, 0.5f);
        had::SpectralLine l{0, 1, B, one.data()};
        std::vector<had::ScoredLine> o;
        det.process(l, o);
    } catch (const had::DataError& e) {
        data_err = e.exit_code();
    }
    try {
        had::ErxDetector d2(had::ErxConfig{.no_srp = true}, 3, 1);
        std::vector<float> x(8 * 3, 0.25f);
        x[1] = NAN;
        had::SpectralLine l{0, 8, 3, x.data()};
        std::vector<had::ScoredLine> o;
        d2.process(l, o);
    } catch (const had::FactorizationError& e) {
        fact_err = int(e.kind());
        pivot = e.pivot;
    }
    // the reference's free functions (detector.hpp:32, projection.hpp:15-34, erx.hpp:38-47)
    const std::vector<double> nz = had::normalize_scores(out.back().raw);
    double nz_err = 0.0;
    for (size_t i = 0; i < nz.size(); ++i) nz_err = std::fmax(nz_err, std::fabs(nz[i] - out.back().norm[i]));
    had::ErxDetector srp_det(had::ErxConfig{.dims = 5, .seed = 7}, B, 4);
    std::vector<had::ScoredLine> o2;
    for (std::uint32_t t = 0; t < 5; ++t) srp_det.process(had::SpectralLine{std::int64_t(t), P, B, cube.data() + size_t(t) * P * B}, o2);
    srp_det.finish(o2);
    const auto w = had::generate_srp(B, 5, 7);
    const bool w_same = srp_det.state().weights.weights.v == w.weights.v && srp_det.state().weights.nonzero_count() == w.nonzero_count();
    const auto z = had::project_line(had::SpectralLine{0, P, B, cube.data()}, w);
    auto [mh, kh] = had::erx::line_stats(z);
    had::ErxState es;
    es.mu = mh;
    es.cov = kh;
    had::erx::ema_update(es, mh, kh, 0.3);
    double ema_dev = 0.0;  // EMA of a state with its own statistics is a fixed point (to rounding)
    for (long jj = 0; jj < mh.size(); ++jj) ema_dev = std::fmax(ema_dev, std::fabs(es.mu(jj) - mh(jj)) / std::fabs(mh(jj)));
    const bool ema_fixed = ema_dev < 1e-14;
    const auto thr = had::erx::apply_threshold({-1.0, 0.0, 2.0}, 1.0);
    const bool ident = had::identity_projection(B).nonzero_count() == B && had::identity_projection(B).identity;
    std::printf("{\"normalize_err\": %.3e, \"srp_weights_match\": %s, \"z_rows\": %ld, \"z_cols\": %ld, "
                "\"stats_d\": %ld, \"ema_fixed\": %s, \"threshold\": [%d, %d, %d], \"identity_ok\": %s, "
                "\"srp_lines\": %d}\n",
                nz_err, w_same ? "true" : "false", z.rows(), z.cols(), kh.rows(), ema_fixed ? "true" : "false",
                thr[0], thr[1], thr[2], ident ? "true" : "false", int(o2.size()));
    std::printf("{\"lines\": %d, \"order_ok\": %s, \"name\": \"%s\", \"norm_mean\": %.3e, \"lines_seen\": %lld, "
                "\"dims\": %ld, \"warmup0\": %s, \"config_exit\": %d, \"data_exit\": %d, \"numeric_kind\": %d, "
                "\"pivot\": %d}\n",
                n, order_ok ? "true" : "false", std::string(det.name()).c_str(), mean_norm,
                (long long)st.lines_seen, st.mu.size(), out[0].warmup ? "true" : "false", cfg_err, data_err,
                fact_err, pivot);
    return 0;
}
