/*
 * erx_oracle.h — C ABI of the CPU fp64 oracle for the ERX hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is a CPU restatement of the
 * reference algorithm (SPEC.md §erx, §linalg, §projection, §metrics and the
 * header contracts under proj/include/hadkit/).  Only tests/, the
 * __graft_entry__.smoke() checker and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The shipped product (liberx_b200.so) never
 * links, loads or calls it.
 *
 * Return codes follow had::ErrorKind (errors.hpp:12-18):
 *   0 ok, 2 config, 3 data, 4 metric_undefined, 5 numeric.
 */
#ifndef ERX_ORACLE_H
#define ERX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors had::ErxConfig (erx.hpp:14-24). */
typedef struct {
    int32_t dims;
    double alpha;
    uint32_t buffer_len;
    double epsilon;
    uint64_t seed;
    int32_t no_srp;
    int32_t use_incremental;
} orc_erx_config;

/* ---- had::Rng restatement (rng.hpp:18-83) ---- */
void* orc_rng_new(uint64_t seed);
void orc_rng_free(void* r);
uint64_t orc_rng_next_u64(void* r);
double orc_rng_uniform(void* r);
float orc_rng_uniform_f32(void* r);
uint64_t orc_rng_below(void* r, uint64_t bound);
double orc_rng_normal(void* r);
void orc_rng_sample_indices(void* r, uint32_t n, uint32_t k, uint32_t* out, uint32_t* out_k);
uint64_t orc_mix_seed(uint64_t seed, uint64_t n);

/* ---- linalg (linalg.hpp:12-36) ---- */
/* Returns -1 on success, else the failing pivot index. Reads the lower triangle only. */
int orc_cholesky_lower(const double* a, int n, double* l);
/* In place; returns -1 on success, else the index of the zero diagonal entry. */
int orc_forward_substitute(const double* l, int n, double* x);
int orc_welford_batch_update(double* mean, double* cov, int64_t* n_seen, const double* batch, int k, int n);

/* ---- projection (projection.hpp:15-34) ---- */
void orc_generate_srp(uint32_t bands, uint32_t dims, uint64_t seed, double* w /* bands x dims */);
int orc_project_line(const float* x, uint32_t p, uint32_t b, const double* w, uint32_t w_rows, uint32_t d,
                     int identity, double* z /* p x d */);

/* ---- erx free functions (erx.hpp:36-49, detector.hpp:29-32) ---- */
int orc_line_stats(const double* z, int p, int d, double* mu, double* cov);
void orc_normalize_scores(const double* raw, int p, double* norm);
void orc_apply_threshold(const double* norm, int p, double tau, uint8_t* out);

/* ---- the streaming detector (erx.hpp:51-71) ---- */
void* orc_erx_new(const orc_erx_config* cfg, uint32_t bands, int* status, char* msg, size_t msglen);
void orc_erx_free(void* h);
int orc_erx_dims(void* h);
int orc_erx_process(void* h, int64_t index, uint32_t p, uint32_t b, const float* data, double* raw, double* norm,
                    uint8_t* warmup, int* pivot, char* msg, size_t msglen);
int orc_erx_state(void* h, double* mu, double* cov, int64_t* lines_seen, int64_t* welford_n, int* initialized,
                  double* weights);

int orc_erx_set_state(void* h, const double* mu, const double* cov, int64_t lines_seen, int64_t welford_n);

/* ---- input generator: the shared seeded BASELINE.json generator
 * (paper_2408_14947_b200/csrc/datagen.cpp, compiled into this library too so
 * the CPU baseline / reference arm needs no product library).  Same
 * arguments as erx_gen_preset / erx_gen_lines (include/erx_datagen.h). ---- */
int orc_gen_preset(int config_id, uint32_t stream, void* spec_out);
int orc_gen_lines(const void* spec, uint32_t first_line, uint32_t n_lines, float* out, uint8_t* mask, int threads);
int orc_gen_scene_changes(const void* spec, int64_t* out);

/* Runs n_streams independent detectors over lines [S][L][P][B] with `threads`
 * host threads, one stream per thread at a time.  raw/norm
 * are [S][L][P]; either may be NULL.  Returns the first error code seen. */
int orc_erx_run_streams(const orc_erx_config* cfg, uint32_t bands, uint32_t n_streams, uint32_t n_lines,
                        uint32_t p, const float* lines, double* raw, double* norm, int threads);

/* ---- metrics (metrics.hpp:25-28) ---- */
double orc_roc_auc(const double* scores, const uint8_t* labels, size_t n, int* status);

#ifdef __cplusplus
}
#endif

#endif
