// hadkit_b200.hpp — header-only C++20 mirror of the reference detector
// interface (proj/include/hadkit/{errors,cube,detector,erx}.hpp) over the
// erx_b200 C ABI.  Code written against had::ErxDetector / had::LineDetector
// compiles against this header and runs on the B200 engine:
//
//   had::ErxDetector det(had::ErxConfig{.alpha = 0.1}, bands);   // erx.hpp:58
//   det.process(line, out);                                       // detector.hpp:19
//   det.finish(out);                                              // detector.hpp:21
//
// The reference's include paths work too: include/hadkit/{erx,detector,cube,
// projection,errors}.hpp forward here, so `#include "hadkit/erx.hpp"` with
// -I include compiles unchanged.
//
// Differences from the reference headers, all additive:
//   * ErxDetector takes an optional window (pipelining lag, detector.hpp:11-14)
//     and device ordinal;
//   * vectors / matrices use the small dense types below (b200::Vec / Mat,
//     with the Eigen members the reference code calls: rows(), cols(),
//     operator(), size(), data()) instead of Eigen (not vendored with the
//     reference, proj/.gitignore:2);
//   * state() returns a snapshot of the device-resident background by value
//     (erx.hpp:65 returns a reference to host state);
//   * a CUDA failure throws had::DeviceError (no reference analogue).
// Exceptions are rethrown from C ABI status codes; none crosses the ABI.
//
// The free functions of the reference API (normalize_scores, generate_srp,
// identity_projection, project_line, erx::line_stats / ema_update /
// apply_threshold) are host utilities here, as in the reference: the
// detector's own per-line path never calls them (it runs on the device).
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../erx_b200.h"

namespace had {

// ------------------------------------------------------------------ errors.hpp:12-79
enum class ErrorKind { config = 2, data = 3, metric_undefined = 4, numeric = 5, io = 6 };

class Error : public std::runtime_error {
  public:
    Error(ErrorKind k, const std::string& m) : std::runtime_error(m), kind_(k) {}
    ErrorKind kind() const { return kind_; }
    int exit_code() const {
        if (kind_ == ErrorKind::config) return 2;
        if (kind_ == ErrorKind::metric_undefined) return 4;
        return 3;
    }

  private:
    ErrorKind kind_;
};
struct ConfigError : Error {
    explicit ConfigError(const std::string& m) : Error(ErrorKind::config, m) {}
};
struct DataError : Error {
    explicit DataError(const std::string& m) : Error(ErrorKind::data, m) {}
};
struct MetricUndefinedError : Error {
    explicit MetricUndefinedError(const std::string& m) : Error(ErrorKind::metric_undefined, m) {}
};
struct FactorizationError : Error {
    FactorizationError(int p, const std::string& m) : Error(ErrorKind::numeric, m), pivot(p) {}
    int pivot;
};
struct SingularSolveError : Error {
    explicit SingularSolveError(const std::string& m) : Error(ErrorKind::numeric, m) {}
};
struct UpdateInstabilityError : Error {
    explicit UpdateInstabilityError(const std::string& m) : Error(ErrorKind::numeric, m) {}
};
// Malformed or truncated file; `offset` is the byte position of the problem (errors.hpp:67-75).
struct FormatError : Error {
    FormatError(std::string file_path, std::size_t byte_offset, const std::string& m)
        : Error(ErrorKind::data, m + " (file '" + file_path + "', offset " + std::to_string(byte_offset) + ")"),
          path(std::move(file_path)),
          offset(byte_offset) {}
    std::string path;
    std::size_t offset;
};
struct IoError : Error {
    explicit IoError(const std::string& m) : Error(ErrorKind::io, m) {}
};
struct DeviceError : Error {
    explicit DeviceError(const std::string& m) : Error(ErrorKind::io, m) {}
};

namespace b200 {
inline void throw_status(int st, const std::string& msg, int pivot = -1) {
    switch (st) {
        case ERX_OK: return;
        case ERX_ERR_CONFIG: throw ConfigError(msg);
        case ERX_ERR_DATA: throw DataError(msg);
        case ERX_ERR_METRIC: throw MetricUndefinedError(msg);
        case ERX_ERR_NUMERIC: throw FactorizationError(pivot, msg);
        case ERX_ERR_IO: throw IoError(msg);
        default: throw DeviceError("[" + std::to_string(st) + "] " + msg);
    }
}

// Minimal dense containers standing in for Eigen::VectorXd / MatrixXd.
struct Vec {
    std::vector<double> v;
    Vec() = default;
    explicit Vec(long n) : v(size_t(n), 0.0) {}
    long size() const { return long(v.size()); }
    long rows() const { return size(); }
    double operator()(long i) const { return v[size_t(i)]; }
    double& operator()(long i) { return v[size_t(i)]; }
    const double* data() const { return v.data(); }
    double* data() { return v.data(); }
};
struct Mat {
    long r = 0, c = 0;
    std::vector<double> v;  // row-major
    Mat() = default;
    Mat(long rows, long cols) : r(rows), c(cols), v(size_t(rows * cols), 0.0) {}
    long rows() const { return r; }
    long cols() const { return c; }
    double operator()(long i, long j) const { return v[size_t(i * c + j)]; }
    double& operator()(long i, long j) { return v[size_t(i * c + j)]; }
    const double* data() const { return v.data(); }
    double* data() { return v.data(); }
};
}  // namespace b200

// ------------------------------------------------------------------ cube.hpp:48-82
struct SpectralLine {
    std::int64_t index = 0;
    std::uint32_t pixels = 0;
    std::uint32_t bands = 0;
    const float* data = nullptr;  // pixels x bands, band fastest
};

struct ScoredLine {
    std::int64_t index = 0;
    std::vector<double> raw;
    std::vector<double> norm;
    std::optional<std::vector<std::uint8_t>> decisions;
    bool warmup = false;
};

// ------------------------------------------------------------------ detector.hpp:15-32
// Per-line z-score of the raw distances, population std; std < 1e-12 -> zeros (detector.hpp:29-32).
inline std::vector<double> normalize_scores(const std::vector<double>& raw) {
    const size_t p = raw.size();
    std::vector<double> out(p, 0.0);
    if (!p) return out;
    double mean = 0.0;
    for (double d : raw) mean += d;
    mean /= double(p);
    double var = 0.0;
    for (double d : raw) var += (d - mean) * (d - mean);
    const double sd = std::sqrt(var / double(p));
    if (sd < 1e-12) return out;
    for (size_t i = 0; i < p; ++i) out[i] = (raw[i] - mean) / sd;
    return out;
}

class LineDetector {
  public:
    virtual ~LineDetector() = default;
    virtual void process(const SpectralLine& line, std::vector<ScoredLine>& out) = 0;
    virtual void finish(std::vector<ScoredLine>& out) { (void)out; }
    virtual std::string_view name() const = 0;
    virtual bool emits_normalized_scores() const { return false; }
};

// ------------------------------------------------------------------ projection.hpp:15-34
struct SrpMatrix {
    b200::Mat weights;  // b x d, explicit zeros
    std::uint64_t seed = 0;
    double sparsity = 0.0;  // s = sqrt(b)
    bool identity = false;  // no-SRP bypass: weights are the b x b identity
    std::int64_t nonzero_count() const {
        std::int64_t n = 0;
        for (double w : weights.v) n += (w != 0.0) ? 1 : 0;
        return n;
    }
    int input_dims() const { return static_cast<int>(weights.rows()); }
    int output_dims() const { return static_cast<int>(weights.cols()); }
};

// The engine's own generator (erx_generate_srp): the same W the detector uploads for this seed.
inline SrpMatrix generate_srp(std::uint32_t bands, std::uint32_t dims, std::uint64_t seed) {
    SrpMatrix m;
    m.weights = b200::Mat(bands, dims);
    m.seed = seed;
    m.sparsity = std::sqrt(double(bands));
    b200::throw_status(erx_generate_srp(bands, dims, seed, m.weights.data()), "generate_srp: bands and dims >= 1");
    return m;
}

inline SrpMatrix identity_projection(std::uint32_t bands) {
    SrpMatrix m;
    m.weights = b200::Mat(bands, bands);
    for (std::uint32_t i = 0; i < bands; ++i) m.weights(i, i) = 1.0;
    m.sparsity = 1.0;
    m.identity = true;
    return m;
}

// Z = X W, p x d in double precision; ConfigError on a band-count mismatch (projection.hpp:31-34).
inline b200::Mat project_line(const b200::Mat& pixels, const SrpMatrix& w) {
    if (pixels.cols() != w.weights.rows()) throw ConfigError("project_line: band count mismatch");
    const long p = pixels.rows(), b = pixels.cols(), d = w.weights.cols();
    b200::Mat z(p, d);
    for (long i = 0; i < p; ++i)
        for (long k = 0; k < b; ++k) {
            const double x = pixels(i, k);
            for (long j = 0; j < d; ++j) z(i, j) += x * w.weights(k, j);
        }
    return z;
}
inline b200::Mat project_line(const SpectralLine& line, const SrpMatrix& w) {
    b200::Mat x(line.pixels, line.bands);
    for (size_t i = 0; i < x.v.size(); ++i) x.v[i] = double(line.data[i]);
    return project_line(x, w);
}

// ------------------------------------------------------------------ erx.hpp:14-71
struct ErxConfig {
    int dims = 5;
    double alpha = 0.1;
    std::uint32_t buffer_len = 99;
    double epsilon = 1e-5;
    std::uint64_t seed = 0;
    bool no_srp = false;
    bool use_incremental = false;

    erx_config c() const {
        return erx_config{dims, alpha, buffer_len, epsilon, seed, no_srp ? 1 : 0, use_incremental ? 1 : 0};
    }
    void validate() const {
        erx_config k = c();
        char msg[256] = {0};
        b200::throw_status(erx_config_validate(&k, 1u << 30, msg, sizeof msg), msg);
    }
};

struct ErxState {
    SrpMatrix weights;  // b x d (identity b x b when no_srp)
    b200::Vec mu;
    b200::Mat cov;
    std::int64_t lines_seen = 0;
    std::int64_t welford_n = 0;
    bool initialized = false;
};

namespace erx {
// Column mean and unbiased (1/(p-1)) covariance of a projected line; DataError for p < 2 (erx.hpp:38-40).
inline std::pair<b200::Vec, b200::Mat> line_stats(const b200::Mat& z) {
    const long p = z.rows(), d = z.cols();
    if (p < 2) throw DataError("line_stats: a line needs p >= 2 pixels (1/(p-1) covariance)");
    b200::Vec mu(d);
    b200::Mat cov(d, d);
    for (long i = 0; i < p; ++i)
        for (long j = 0; j < d; ++j) mu(j) += z(i, j);
    for (long j = 0; j < d; ++j) mu(j) /= double(p);
    for (long i = 0; i < p; ++i)
        for (long a = 0; a < d; ++a)
            for (long b = 0; b <= a; ++b) cov(a, b) += (z(i, a) - mu(a)) * (z(i, b) - mu(b));
    for (long a = 0; a < d; ++a)
        for (long b = 0; b <= a; ++b) cov(b, a) = cov(a, b) = cov(a, b) / double(p - 1);
    return {mu, cov};
}
// mu <- (1-alpha) mu + alpha mu_hat, same for cov (erx.hpp:42-44).
inline void ema_update(ErxState& state, const b200::Vec& mu_hat, const b200::Mat& cov_hat, double alpha) {
    for (long j = 0; j < mu_hat.size(); ++j) state.mu(j) = (1.0 - alpha) * state.mu(j) + alpha * mu_hat(j);
    for (size_t k = 0; k < cov_hat.v.size(); ++k) state.cov.v[k] = (1.0 - alpha) * state.cov.v[k] + alpha * cov_hat.v[k];
}
// y_i = 1 iff norm_scores[i] >= tau (erx.hpp:46-47).
inline std::vector<std::uint8_t> apply_threshold(const std::vector<double>& norm, double tau) {
    std::vector<std::uint8_t> y(norm.size());
    for (size_t i = 0; i < norm.size(); ++i) y[i] = norm[i] >= tau ? 1 : 0;
    return y;
}
}  // namespace erx

class ErxDetector : public LineDetector {
  public:
    ErxDetector(const ErxConfig& cfg, std::uint32_t bands, std::uint32_t window_lines = 32, int device = 0)
        : cfg_(cfg), bands_(bands) {
        erx_config k = cfg.c();
        erx_engine* e = nullptr;
        char msg[512] = {0};
        b200::throw_status(erx_create(&k, bands, 1, window_lines, device, &e, msg, sizeof msg), msg);
        eng_.reset(e);
    }

    void process(const SpectralLine& line, std::vector<ScoredLine>& out) override {
        if (line.bands != bands_) throw ConfigError("band count mismatch");  // projection.hpp:31-32
        check(erx_push_host(eng_.get(), line.index, 1, line.pixels, line.bands, line.data), out);
    }
    void finish(std::vector<ScoredLine>& out) override { check(erx_finish(eng_.get()), out); }
    std::string_view name() const override { return "erx"; }
    bool emits_normalized_scores() const override { return true; }
    const ErxConfig& config() const { return cfg_; }

    // Snapshot of the device-resident background (erx.hpp:65 returns a reference;
    // the B200 state lives in HBM, so this returns a copy).
    ErxState state() const {
        ErxState s;
        const int d = erx_dims(eng_.get());
        s.mu.v.resize(size_t(d));
        s.cov.r = s.cov.c = d;
        s.cov.v.resize(size_t(d) * d);
        int ini = 0;
        b200::throw_status(erx_get_state(eng_.get(), 0, s.mu.v.data(), s.cov.v.data(), &s.lines_seen,
                                         &s.welford_n, &ini),
                           erx_last_error(eng_.get()));
        s.initialized = ini != 0;
        if (!cfg_.no_srp) {
            s.weights.weights = b200::Mat(bands_, d);
            s.weights.seed = cfg_.seed;
            s.weights.sparsity = std::sqrt(double(bands_));
            erx_get_weights(eng_.get(), s.weights.weights.data());
        } else {
            s.weights = identity_projection(bands_);
        }
        return s;
    }

  private:
    struct Del {
        void operator()(erx_engine* e) const { erx_destroy(e); }
    };

    void drain(std::vector<ScoredLine>& out) {
        while (const std::uint32_t n = erx_ready(eng_.get())) drain_run(out, n, erx_next_pixels(eng_.get()));
    }
    void drain_run(std::vector<ScoredLine>& out, std::uint32_t n, std::uint32_t pixels) {
        std::vector<std::int64_t> idx(n);
        std::vector<std::uint8_t> wu(n);
        std::vector<double> raw(size_t(n) * pixels), norm(size_t(n) * pixels);
        const int got = erx_pop(eng_.get(), n, idx.data(), wu.data(), raw.data(), norm.data());
        for (int k = 0; k < got; ++k) {
            ScoredLine s;
            s.index = idx[size_t(k)];
            s.warmup = wu[size_t(k)] != 0;
            s.raw.assign(raw.begin() + long(k) * pixels, raw.begin() + long(k + 1) * pixels);
            s.norm.assign(norm.begin() + long(k) * pixels, norm.begin() + long(k + 1) * pixels);
            out.push_back(std::move(s));
        }
    }
    void check(int st, std::vector<ScoredLine>& out) {
        drain(out);  // lines scored before a failure are still emitted
        b200::throw_status(st, erx_last_error(eng_.get()), erx_last_pivot(eng_.get()));
    }

    ErxConfig cfg_;
    std::uint32_t bands_;
    std::unique_ptr<erx_engine, Del> eng_;
};

}  // namespace had
