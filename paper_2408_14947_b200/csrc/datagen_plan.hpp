// datagen_plan.hpp — the stream-level draws of the synthetic generator
// (datagen.cpp: build) flattened for the device generator (k_datagen.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/erx_datagen.h"

namespace erx_host {

struct GenPlan {
    uint32_t B = 0, P = 0, R = 0;
    std::vector<double> base;       // [scene][B]
    std::vector<double> drift;      // [B], direction in [-1, 1]
    std::vector<double> A;          // [B][R] loading matrix
    std::vector<int64_t> changes;   // sorted scene-change lines
    std::vector<uint32_t> hit_off;  // [n + 1] CSR over the requested lines (hits in anomaly order)
    std::vector<uint32_t> hit_pix;  // pixel of each hit
    std::vector<uint32_t> hit_anom; // row of anom_spec / anom_f
    std::vector<double> anom_spec;  // [used][B] target spectrum or offset vector
    std::vector<double> anom_f;     // [used] mixture fraction
};

int gen_plan(const erx_gen_spec& s, uint32_t first, uint32_t n, GenPlan& out);

}  // namespace erx_host
