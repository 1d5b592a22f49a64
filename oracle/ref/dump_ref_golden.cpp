// dump_ref_golden.cpp — compiled AGAINST THE REFERENCE'S OWN HEADERS
// (/root/reference/proj/include/hadkit/rng.hpp and errors.hpp, the only two
// reference headers with complete inline bodies) into
// oracle/_ref/dump_ref_golden.  It prints golden vectors as JSON; the
// committed fixture tests/golden/ref_golden.json is produced by
// tests/golden/make_golden.py and pins the oracle's and the product's
// restatements of had::Rng / had::mix_seed / had::ErrorKind.
// Nothing here is shipped; it only runs in the build container.
#include <cstdio>
#include <cstdint>
#include <vector>

#include "hadkit/errors.hpp"
#include "hadkit/rng.hpp"

static void u64s(const char* key, std::vector<std::uint64_t> v, bool last = false) {
    std::printf("  \"%s\": [", key);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)v[i]);
    std::printf("]%s\n", last ? "" : ",");
}
static void f64s(const char* key, std::vector<double> v) {
    std::printf("  \"%s\": [", key);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
    std::printf("],\n");
}

int main() {
    const std::uint64_t seeds[] = {0, 1, 42, 0xdeadbeefULL};
    std::printf("{\n");
    for (std::uint64_t seed : seeds) {
        char key[64];
        {
            had::Rng r(seed);
            std::vector<std::uint64_t> v;
            for (int i = 0; i < 16; ++i) v.push_back(r.next_u64());
            std::snprintf(key, sizeof key, "next_u64_seed%llu", (unsigned long long)seed);
            u64s(key, v);
        }
        {
            had::Rng r(seed);
            std::vector<double> v;
            for (int i = 0; i < 16; ++i) v.push_back(r.uniform());
            std::snprintf(key, sizeof key, "uniform_seed%llu", (unsigned long long)seed);
            f64s(key, v);
        }
        {
            had::Rng r(seed);
            std::vector<double> v;
            for (int i = 0; i < 16; ++i) v.push_back(double(r.uniform_f32()));
            std::snprintf(key, sizeof key, "uniform_f32_seed%llu", (unsigned long long)seed);
            f64s(key, v);
        }
        {
            had::Rng r(seed);
            std::vector<double> v;
            for (int i = 0; i < 17; ++i) v.push_back(r.normal());
            std::snprintf(key, sizeof key, "normal_seed%llu", (unsigned long long)seed);
            f64s(key, v);
        }
        {
            had::Rng r(seed);
            std::vector<std::uint64_t> v;
            const std::uint64_t bounds[] = {1, 2, 3, 7, 10, 100, 1000003, 0x8000000000000001ULL};
            for (int rep = 0; rep < 2; ++rep)
                for (std::uint64_t b : bounds) v.push_back(r.below(b));
            std::snprintf(key, sizeof key, "below_seed%llu", (unsigned long long)seed);
            u64s(key, v);
        }
        {
            had::Rng r(seed);
            auto idx = r.sample_indices(50, 12);
            std::vector<std::uint64_t> v(idx.begin(), idx.end());
            std::snprintf(key, sizeof key, "sample_indices_50_12_seed%llu", (unsigned long long)seed);
            u64s(key, v);
        }
        {
            // normal() interleaved with uniform(): pins the cached-spare behaviour.
            had::Rng r(seed);
            std::vector<double> v;
            for (int i = 0; i < 6; ++i) {
                v.push_back(r.normal());
                v.push_back(r.uniform());
            }
            std::snprintf(key, sizeof key, "normal_uniform_mix_seed%llu", (unsigned long long)seed);
            f64s(key, v);
        }
    }
    {
        std::vector<std::uint64_t> v;
        for (std::uint64_t s : seeds)
            for (std::uint64_t n : {0ULL, 1ULL, 2ULL, 99ULL, 5000ULL, 0xffffffffffffffffULL}) v.push_back(had::mix_seed(s, n));
        u64s("mix_seed", v);
    }
    {
        // ErrorKind values and exit codes (errors.hpp:12-37,51-56).
        had::ConfigError ce("c");
        had::DataError de("d");
        had::MetricUndefinedError me("m");
        had::FactorizationError fe(7, "f");
        had::SingularSolveError se("s");
        had::IoError ie("i");
        std::printf("  \"error_kinds\": {\"config\": %d, \"data\": %d, \"metric_undefined\": %d, \"numeric\": %d, \"io\": %d},\n",
                    int(ce.kind()), int(de.kind()), int(me.kind()), int(fe.kind()), int(ie.kind()));
        std::printf("  \"exit_codes\": {\"config\": %d, \"data\": %d, \"metric_undefined\": %d, \"numeric\": %d, \"singular\": %d, \"io\": %d},\n",
                    ce.exit_code(), de.exit_code(), me.exit_code(), fe.exit_code(), se.exit_code(), ie.exit_code());
        std::printf("  \"factorization_pivot\": %d\n", fe.pivot);
    }
    std::printf("}\n");
    return 0;
}
