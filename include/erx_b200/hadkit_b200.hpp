// hadkit_b200.hpp — header-only C++20 mirror of the reference detector
// interface (proj/include/hadkit/{errors,cube,detector,erx}.hpp) over the
// erx_b200 C ABI.  Code written against had::ErxDetector / had::LineDetector
// compiles against this header and runs on the B200 engine:
//
//   had::ErxDetector det(had::ErxConfig{.alpha = 0.1}, bands);   // erx.hpp:58
//   det.process(line, out);                                       // detector.hpp:19
//   det.finish(out);                                              // detector.hpp:21
//
// Differences from the reference headers, all additive:
//   * ErxDetector takes an optional window (pipelining lag, detector.hpp:11-14)
//     and device ordinal;
//   * ErxState's vectors use the small dense types below instead of Eigen
//     (Eigen is not vendored with the reference, proj/.gitignore:2);
//   * a CUDA failure throws had::DeviceError (no reference analogue).
// Exceptions are rethrown from C ABI status codes; none crosses the ABI.
#pragma once

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
struct FactorizationError : Error {
    FactorizationError(int p, const std::string& m) : Error(ErrorKind::numeric, m), pivot(p) {}
    int pivot;
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
        case ERX_ERR_NUMERIC: throw FactorizationError(pivot, msg);
        default: throw DeviceError("[" + std::to_string(st) + "] " + msg);
    }
}

// Minimal dense containers standing in for Eigen::VectorXd / MatrixXd.
struct Vec {
    std::vector<double> v;
    long size() const { return long(v.size()); }
    long rows() const { return size(); }
    double operator()(long i) const { return v[size_t(i)]; }
    const double* data() const { return v.data(); }
};
struct Mat {
    long r = 0, c = 0;
    std::vector<double> v;  // row-major
    long rows() const { return r; }
    long cols() const { return c; }
    double operator()(long i, long j) const { return v[size_t(i * c + j)]; }
    const double* data() const { return v.data(); }
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

// ------------------------------------------------------------------ detector.hpp:15-27
class LineDetector {
  public:
    virtual ~LineDetector() = default;
    virtual void process(const SpectralLine& line, std::vector<ScoredLine>& out) = 0;
    virtual void finish(std::vector<ScoredLine>& out) { (void)out; }
    virtual std::string_view name() const = 0;
    virtual bool emits_normalized_scores() const { return false; }
};

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
    b200::Mat weights;  // b x d (empty when no_srp)
    b200::Vec mu;
    b200::Mat cov;
    std::int64_t lines_seen = 0;
    std::int64_t welford_n = 0;
    bool initialized = false;
};

namespace erx {
inline std::vector<std::uint8_t> apply_threshold(const std::vector<double>& norm, double tau) {  // erx.hpp:46-47
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
            s.weights.r = bands_;
            s.weights.c = d;
            s.weights.v.resize(size_t(bands_) * d);
            erx_get_weights(eng_.get(), s.weights.v.data());
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
