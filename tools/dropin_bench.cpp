// dropin_bench.cpp — the drop-in single-stream number: BASELINE configs[0]
// (384 px x 108 bands) fed through had::ErxDetector::process ONE host line per
// call (detector.hpp:19, cube.hpp:45-55; the reference line-scan loop), scores
// returned as ScoredLine fp64 vectors, timed by the wall clock from the first
// line fed to the last ScoredLine.  Lag T = window_lines (the
// contract allows pipelined detectors to lag, detector.hpp:11-14); T = 1 is the
// lag-0 per-line latency.  Prints one JSON line.
//   g++ -std=c++20 -O2 -I include tools/dropin_bench.cpp -L paper_2408_14947_b200 -l:liberx_b200.so
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "erx_datagen.h"
#include "hadkit/erx.hpp"

static double run(const had::ErxConfig& cfg, const std::vector<float>& cube, std::uint32_t L, std::uint32_t P,
                  std::uint32_t B, std::uint32_t window, std::uint32_t warm) {
    had::ErxDetector det(cfg, B, window);
    std::vector<had::ScoredLine> out;
    out.reserve(L);
    for (std::uint32_t t = 0; t < warm; ++t) det.process(had::SpectralLine{std::int64_t(t), P, B, cube.data() + size_t(t) * P * B}, out);
    const auto t0 = std::chrono::steady_clock::now();
    for (std::uint32_t t = warm; t < L; ++t) det.process(had::SpectralLine{std::int64_t(t), P, B, cube.data() + size_t(t) * P * B}, out);
    det.finish(out);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (out.size() != L) std::abort();
    return double(L - warm) / el;
}

int main(int argc, char** argv) {
    const std::uint32_t L = argc > 1 ? std::uint32_t(std::atoi(argv[1])) : 2000;
    erx_gen_spec spec;
    erx_gen_preset(0, 0, &spec);
    const std::uint32_t P = spec.pixels, B = spec.bands;
    std::vector<float> cube(size_t(L) * P * B);
    erx_gen_lines(&spec, 0, L, cube.data(), nullptr, 0);
    std::string js = "{\"workload\": \"configs[0] (384 px x 108 bands), had::ErxDetector::process one host line per call\"";
    for (int srp = 0; srp < 2; ++srp) {
        had::ErxConfig cfg;
        cfg.no_srp = srp == 0;
        for (std::uint32_t w : {32u, 1u}) {
            const double lps = run(cfg, cube, L, P, B, w, 64);
            char buf[160];
            std::snprintf(buf, sizeof buf, ", \"%s_window%u\": {\"lines_per_s\": %.1f, \"ms_per_line\": %.4f}",
                          srp ? "srp" : "full", w, lps, 1e3 / lps);
            js += buf;
        }
    }
    std::printf("%s}\n", js.c_str());
    return 0;
}
