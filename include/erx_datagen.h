/*
 * erx_datagen.h — seeded synthetic line-scan generator for the BASELINE.json
 * workloads (configs[0..4]).  Input generation only: it feeds the parity
 * tests, the benchmark and the CPU baseline identical lines; it is not part
 * of the scored path.  Deterministic per (seed, line) through
 * had::mix_seed (rng.hpp:75-83), so lines can be generated in parallel and
 * in any order.  Pinned generator laws are listed in DESIGN.md §Inputs.
 */
#ifndef ERX_DATAGEN_H
#define ERX_DATAGEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ERX_BASE_SMOOTH 0   /* sum of 4 random Gaussians over the band index, scaled into [0.05, 0.6] */
#define ERX_BASE_UNIFORM 1  /* iid uniform [0.05, 0.5] per band */

#define ERX_ANOM_BLOB3X3 0   /* 3x3 (line x pixel) blobs replaced by a random smooth spectrum */
#define ERX_ANOM_BLOB2TO5 1  /* blobs of 2-5 pixels replaced by a random smooth spectrum */
#define ERX_ANOM_OFFSET 2    /* single pixels: background + per-band offset N(0, offset_sd) */
#define ERX_ANOM_MIXTURE 3   /* single pixels: (1-f) bg + f target, f ~ U(mix_lo, mix_hi) */

typedef struct {
    uint32_t lines, pixels, bands;
    uint32_t n_factors;     /* columns of the loading matrix A */
    double loading_sd;      /* A ~ N(0, loading_sd) */
    double noise_sd;        /* iid N(0, noise_sd) per band */
    int32_t base_kind;
    double drift;           /* amplitude of the slow linear drift over the whole stream */
    uint32_t n_scene_changes;
    int64_t scene_change_line[4]; /* -1: drawn uniformly in [L/10, 9L/10) */
    double anomaly_frac;
    int32_t anomaly_kind;
    double offset_sd;
    double mix_lo, mix_hi;
    uint64_t seed;
} erx_gen_spec;

/* BASELINE.json configs[config_id] (0..4) for stream `stream` (seeds: the
 * stream index for configs 3/4, 0 otherwise).  Returns 0, or 2 for a bad id. */
int erx_gen_preset(int config_id, uint32_t stream, erx_gen_spec* out);

/* Lines [first_line, first_line + n_lines) of one stream: out [n][P][B] fp32,
 * mask [n][P] u8 (1 = anomaly) or NULL.  threads <= 0: all host cores. */
int erx_gen_lines(const erx_gen_spec* spec, uint32_t first_line, uint32_t n_lines, float* out, uint8_t* mask,
                  int threads);

/* The stream's scene-change lines as drawn (sorted; out holds up to 4): returns their count, or -1
 * for a bad spec. */
int erx_gen_scene_changes(const erx_gen_spec* spec, int64_t* out);

/* The same lines generated on the device (k_datagen.cu): d_out [n][P][B] fp32 and
 * d_mask [n][P] u8 (or NULL) in device memory, on `stream` (a cudaStream_t; NULL = the legacy
 * default stream), returning when done.  Identical random streams and fp64 operation order as
 * erx_gen_lines; only the last-place results of log / sin / cos may differ (fp32 values then
 * differ by at most one ulp, rarely).  Returns 0 (ERX_OK), 2 bad spec, 3 if a Box-Muller u1 = 0
 * draw occurred (host redraws; p = 2^-53 per pair), 16 on a CUDA error. */
int erx_gen_lines_device(const erx_gen_spec* spec, uint32_t first_line, uint32_t n_lines, float* d_out,
                         uint8_t* d_mask, void* stream);

/* Host RNG restatement probes (had::mix_seed, had::Rng; rng.hpp:18-83), for
 * pinning against the reference's golden vectors.  kind: 0 next_u64 ->
 * u64_out, 1 uniform, 2 uniform_f32, 3 normal -> f64_out, 4 below(u64_out[i]). */
uint64_t erx_mix_seed(uint64_t seed, uint64_t n);
void erx_rng_probe(uint64_t seed, int kind, uint32_t n, uint64_t* u64_out, double* f64_out);

#ifdef __cplusplus
}
#endif

#endif
