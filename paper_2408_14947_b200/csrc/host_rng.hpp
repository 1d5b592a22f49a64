// host_rng.hpp — product-side restatement of had::Rng / had::mix_seed
// (proj/include/hadkit/rng.hpp:18-83) and generate_srp
// (projection.hpp:11-26).  Pinned bit-for-bit against golden vectors from
// the reference's own rng.hpp (tests/golden/ref_golden.json,
// tests/test_capi_host.py).  Host-only: used at engine construction (SRP
// weights) and by the synthetic input generator.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace erx_host {

class Rng {
  public:
    explicit Rng(uint64_t seed) : eng_(seed) {}
    uint64_t next_u64() { return eng_(); }
    double uniform() { return double(eng_() >> 11) * 0x1.0p-53; }
    float uniform_f32() { return float(eng_() >> 40) * 0x1.0p-24f; }
    uint64_t below(uint64_t bound) {
        const uint64_t thr = (0 - bound) % bound;
        for (;;) {
            const uint64_t r = eng_();
            if (r >= thr) return r % bound;
        }
    }
    double normal() {
        if (have_) {
            have_ = false;
            return spare_;
        }
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double ang = 6.283185307179586476925286766559 * u2;
        spare_ = rad * std::sin(ang);
        have_ = true;
        return rad * std::cos(ang);
    }

  private:
    std::mt19937_64 eng_;
    bool have_ = false;
    double spare_ = 0.0;
};

inline uint64_t mix_seed(uint64_t seed, uint64_t n) {
    uint64_t x = seed ^ (0x9e3779b97f4a7c15ULL + n * 0xbf58476d1ce4e5b9ULL);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// SRP law: +-sqrt(s)/sqrt(d) w.p. 1/(2s) each, s = sqrt(b).
// Draw order: row-major b x d, one uniform() per entry.
inline void generate_srp(uint32_t b, uint32_t d, uint64_t seed, double* w) {
    Rng rng(seed);
    const double s = std::sqrt(double(b));
    const double v = std::sqrt(s) / std::sqrt(double(d));
    const double p_half = 1.0 / (2.0 * s), p_one = 1.0 / s;
    for (uint32_t i = 0; i < b; ++i)
        for (uint32_t j = 0; j < d; ++j) {
            const double u = rng.uniform();
            w[size_t(i) * d + j] = (u < p_half) ? v : (u < p_one ? -v : 0.0);
        }
}

}  // namespace erx_host
