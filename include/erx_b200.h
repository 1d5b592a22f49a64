/*
 * erx_b200.h — C ABI of the B200-native ERX engine (liberx_b200.so).
 *
 * This is the drop-in boundary for the reference's per-line detector
 * (had::ErxDetector, proj/include/hadkit/erx.hpp:56-71, behind the
 * had::LineDetector interface, detector.hpp:15-27).  Plain pointers and
 * sizes only; no C++ or torch types cross it; no exception crosses it.
 * Every entry point below names the reference declaration it replaces.
 *
 * Status codes are the reference's had::ErrorKind values (errors.hpp:12-18)
 * so a wrapper can rethrow the same exception types:
 *   ERX_OK 0, ERX_ERR_CONFIG 2 (ConfigError), ERX_ERR_DATA 3 (DataError),
 *   ERX_ERR_METRIC 4 (MetricUndefinedError, metrics only),
 *   ERX_ERR_NUMERIC 5 (FactorizationError, pivot via erx_last_pivot),
 *   ERX_ERR_IO 6; plus ERX_ERR_DEVICE 16 for CUDA failures (no reference
 *   analogue) and ERX_ERR_STATE 17 for calls on a failed engine.
 *
 * Threading (detector.hpp:11): one engine per consumer
 * thread at a time; engines are independent and may run concurrently.
 */
#ifndef ERX_B200_H
#define ERX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ERX_OK 0
#define ERX_ERR_CONFIG 2
#define ERX_ERR_DATA 3
#define ERX_ERR_METRIC 4
#define ERX_ERR_NUMERIC 5
#define ERX_ERR_IO 6
#define ERX_ERR_DEVICE 16
#define ERX_ERR_STATE 17

/* Mirrors had::ErxConfig (erx.hpp:14-24) field for field. */
typedef struct {
    int32_t dims;            /* projected dimensions d (default 5) */
    double alpha;            /* EMA momentum in (0, 1] (default 0.1) */
    uint32_t buffer_len;     /* lines flagged warmup (default 99) */
    double epsilon;          /* Cholesky regularisation (default 1e-5) */
    uint64_t seed;           /* SRP seed (default 0) */
    int32_t no_srp;          /* identity projection, d = b */
    int32_t use_incremental; /* equal-weight Welford statistics instead of EMAs */
} erx_config;

typedef struct erx_engine erx_engine;

/* ErxConfig{} defaults (erx.hpp:15-21). */
void erx_config_default(erx_config* cfg);

/* ErxConfig::validate (erx.hpp:23) plus the d <= b rule. */
int erx_config_validate(const erx_config* cfg, uint32_t bands, char* msg, size_t msg_len);

/* generate_srp (projection.hpp:26): bands x dims, row-major, explicit zeros. */
int erx_generate_srp(uint32_t bands, uint32_t dims, uint64_t seed, double* weights);

/*
 * Replaces ErxDetector::ErxDetector(cfg, bands) (erx.hpp:58).  n_streams > 1
 * holds that many independent detector instances advanced in lock-step (the
 * batched multi-stream path).  window_lines is the pipelining
 * lag T permitted by detector.hpp:11-14: up to T lines per stream are scored
 * in one device pass (T = 1: no lag).  device: CUDA ordinal.
 */
int erx_create(const erx_config* cfg, uint32_t bands, uint32_t n_streams, uint32_t window_lines, int device,
               erx_engine** out, char* msg, size_t msg_len);
void erx_destroy(erx_engine* e);

/* Message / failing pivot of the last error (FactorizationError::pivot, errors.hpp:51-56). */
const char* erx_last_error(const erx_engine* e);
int erx_last_pivot(const erx_engine* e);

int erx_dims(const erx_engine* e);
uint32_t erx_streams(const erx_engine* e);
uint32_t erx_window(const erx_engine* e);

/*
 * Replaces LineDetector::process (detector.hpp:19) for all streams at once:
 * `lines` is HOST memory [n_streams][n_lines][pixels][bands] fp32 (the
 * SpectralLine payload, cube.hpp:48-55), line i of every stream carrying the
 * emission index first_index + i.  The data is copied before return.  Full
 * windows are scored immediately; results queue for erx_pop.
 */
int erx_push_host(erx_engine* e, int64_t first_index, uint32_t n_lines, uint32_t pixels, uint32_t bands,
                  const float* lines);

/* Replaces LineDetector::finish (detector.hpp:21): scores any partial window. */
int erx_finish(erx_engine* e);

/* Scored lines waiting per stream (the leading run that shares one pixel
 * count) and that pixel count (0 when nothing is queued). */
uint32_t erx_ready(const erx_engine* e);
uint32_t erx_next_pixels(const erx_engine* e);

/*
 * Pops up to max_lines scored lines of every stream, oldest first: the
 * ScoredLine fields (cube.hpp:76-82).  index/warmup: [n]; raw/norm:
 * [n_streams][n][pixels] fp64.  Any pointer may be NULL.  Returns the count
 * popped (>= 0) or a negative status.
 */
int erx_pop(erx_engine* e, uint32_t max_lines, int64_t* index, uint8_t* warmup, double* raw, double* norm);

/*
 * Device-resident path (no host copies): scores n_lines (<= window) lines
 * per stream already in HBM, d_lines [n_streams][n_lines][pixels][bands]
 * fp32, writing d_raw / d_norm [n_streams][n_lines][pixels] fp32.
 * Asynchronous on the engine's stream; numeric failures are latched on the
 * device and reported by erx_sync.
 */
int erx_run_device(erx_engine* e, int64_t first_index, uint32_t n_lines, uint32_t pixels, const float* d_lines,
                   float* d_raw, float* d_norm);
/* Background update only: line statistics and the EMA / Welford scan over
 * n_lines device-resident lines, no factor and no scores.  With
 * erx_set_state it is the building block of the line-range split of one
 * stream across devices (paper_2408_14947_b200/sharding.py:
 * range summary from a zero background, carry chain, then scoring). */
int erx_advance_device(erx_engine* e, int64_t first_index, uint32_t n_lines, uint32_t pixels, const float* d_lines);
int erx_sync(erx_engine* e);
void* erx_cuda_stream(erx_engine* e);

/* ErxDetector::state() (erx.hpp:65, ErxState erx.hpp:27-34) for one stream. */
int erx_get_state(erx_engine* e, uint32_t stream, double* mu, double* cov, int64_t* lines_seen,
                  int64_t* welford_n, int* initialized);
/* ErxState::weights (SrpMatrix, projection.hpp:15-24); bands x dims. */
int erx_get_weights(const erx_engine* e, double* weights);
/* Overwrites one stream's background (mu, cov row-major d x d, welford_n)
 * and marks the engine initialised: the carry hand-off for a line-range split
 * of one stream across devices. */
int erx_set_state(erx_engine* e, uint32_t stream, const double* mu, const double* cov, int64_t lines_seen,
                  int64_t welford_n);

/* Engine options.  ERX_OPT_FACTOR_PRECISION: 0 auto (blocked fp32 in shared
 * memory while the matrix fits, D <= 233, else blocked fp32 in the shared
 * memory of a 2/4/8-CTA thread-block cluster), 32, 30 (force the cluster
 * kernel), 31 (the fp32 kernel over an L2 workspace), 64 (fp64 in shared
 * memory, D <= 165, else the fp64 L2 kernel) or 1 (force the blocked fp64 L2
 * kernel).  erx_get_option reports the kernel in use once the first line has
 * fixed the geometry: 32, 30, 31, 64 or 0 (blocked fp64 L2).  The fp32 kernels
 * hand lines they cannot factor reliably to an fp64 rescue (k_fixup.cu). */
#define ERX_OPT_FACTOR_PRECISION 1
/* ERX_OPT_STATS_TENSOR: which kernels compute line_stats and the score.
 *   2 (default) exact-integer tcgen05 path (kind::i8 digit planes, s32 TMEM
 *     accumulation) where eligible (full covariance, B % 4 == 0): statistics and
 *     score for 16 < D <= 127; statistics for 127 < D <= 512 (128-dim tile
 *     pairs, 2D TMA boxes) with the FFMA score; the FFMA kernels elsewhere;
 *   0 the FFMA kernels.
 * (1, the round-1 bf16x3 tcgen05 statistics, is gone: fp32 TMEM accumulation
 * truncates and missed the median gate; ERX_ERR_CONFIG.)
 * erx_get_option reports the kind in use once the geometry is fixed. */
#define ERX_OPT_STATS_TENSOR 2
/* ERX_OPT_HOST_GROUPS: stream groups per host window of erx_push_host (the
 * host->device copy of group g+1 overlaps the kernels of group g).  0 (default)
 * sizes the groups at >= 8 MB of input each, 1..8 forces that count
 * (results are identical for every count: streams are independent). */
#define ERX_OPT_HOST_GROUPS 3
/* ERX_OPT_ASYNC_HOST: 0 (default) erx_push_host returns with every full window
 * scored and queued; 1 it returns once the window's input is on the device
 * (the source buffer is free) and the window stays in flight, so the next
 * push's host->device copy overlaps its kernels and result copies.  In-flight
 * windows are harvested by erx_ready / erx_pop (which wait for the oldest one
 * only when nothing is queued), erx_finish and every state / device call; a
 * FactorizationError is reported by the call that harvests it (erx_ready
 * defers it to the next erx_pop / push / finish). */
#define ERX_OPT_ASYNC_HOST 4
/* ERX_OPT_FACTOR_THREADS: threads per line of the blocked fp32 shared-memory
 * factor (precision 32).  0 (default) picks 128 when every SM holds >= 6 lines
 * of a launch, else 256; 64, 128, 256 or 512 force that CTA size (same results to
 * rounding; a tuning and test hook). */
#define ERX_OPT_FACTOR_THREADS 5
/* ERX_OPT_GRAPHS: 1 (default) erx_run_device captures a window's launches once
 * per (input, output, size) into a CUDA graph and replays it as one launch (the
 * single-stream lag-0 path: one launch per line); 0 launches kernel by kernel.
 * Per-kernel profiling (erx_set_profiling) bypasses the graphs. */
#define ERX_OPT_GRAPHS 6
/* ERX_OPT_DEVICE_GROUPS: 0 (default) auto, 1 or 2.  erx_run_device runs a window of >= 2 streams
 * as two stream groups on two CUDA streams (forked from and joined back into the engine stream, so
 * the call's stream-ordered contract is unchanged), each with its own rescue list, so the small
 * kernels and tails of one group overlap the other group's kernels; auto splits windows of >= 1024
 * lines.  Per-kernel profiling runs one group. */
#define ERX_OPT_DEVICE_GROUPS 7
/* ERX_OPT_STATS_SPLIT: 3 (default), 0..3.  The exact-integer statistics (16 < D <= 127) run the range
 * pass on its own warps with this many of the ring's stages (stats_i8_ws_kernel, where the ring holds
 * two more); 0 runs the single-role kernel (stats_i8_kernel).  Bit-identical results. */
#define ERX_OPT_STATS_SPLIT 8
/* ERX_OPT_STATS_ONEPASS: 0 (default), 2, 4, 8, 16 or 32.  Opt-in (measured: no faster than the two-pass
 * kernels on configs[3], 0.258 vs 0.254 ms per 2048 lines, and the wider predicted range fails the
 * radiance-scale ill-conditioned gates, so it is off by default).  With a non-zero headroom the
 * exact-integer statistics (16 < D <= 127) read every line ONCE: the per-dim quantisation range is
 * predicted as this factor times the range of the line's first 64 pixels, every quantised value is checked against the digit range, and a line with
 * any value outside (or a non-finite one) is redone by the two-pass kernel with its exact range
 * (stats_i8_op_kernel, then stats_i8_kernel over the listed lines).  0 runs the two-pass kernels for
 * every line (ERX_OPT_STATS_SPLIT picks which).  Lines of one chunk (<= 64 pixels) get their exact range
 * either way.  Results per line depend on that line only (window cuts do not change a bit); the wider
 * predicted range costs ~2.6 of the quantiser's 22 bits on a clean line.
 * ERX_OPT_STATS_REDONE (read-only): lines the two-pass kernel has redone so far. */
#define ERX_OPT_STATS_ONEPASS 9
#define ERX_OPT_STATS_REDONE 10
int erx_set_option(erx_engine* e, int option, int64_t value);
int64_t erx_get_option(const erx_engine* e, int option);

/* ---- instrumentation (bench / profiling; not part of the reference API) ---- */
#define ERX_KERNEL_STATS 0
#define ERX_KERNEL_SCAN 1
#define ERX_KERNEL_FACTOR 2
#define ERX_KERNEL_SCORE 3
#define ERX_KERNEL_NORMALIZE 4
#define ERX_KERNEL_FIXUP 5  /* fp64 rescue of lines the fp32 factor lists (k_fixup.cu) */
#define ERX_NUM_KERNELS 6
uint64_t erx_launch_count(const erx_engine* e);
/* When on, every kernel launch is bracketed by CUDA events on the engine stream. */
int erx_set_profiling(erx_engine* e, int on);
/* Lines whose per-line chain was redone in fp64 by the rescue kernel (k_fixup.cu: the fp32 factor
 * failed or found the background ill-conditioned, or the line's fp32 scores were flat), summed
 * over the engine's life; waits for queued work. */
int64_t erx_rescued_lines(erx_engine* e);

/* Per-kernel summed device ms and launch counts since profiling was enabled. */
int erx_kernel_times(erx_engine* e, double* ms, uint64_t* launches);

/* ---- parity-gate metrics on the device (k_metrics.cu) ----
 * Exact ROC AUC of fp32 device scores against u8 labels (non-zero = anomaly),
 * ties grouped into one ROC step: the AUC of had::roc_curve
 * (metrics.hpp:25-28) / evaluate_run (metrics.hpp:54-58) over the elements
 * with d_select[i] != 0 (NULL = all; e.g. the non-warmup pixels).  Computed
 * from one device radix sort as an exact integer ratio.  ERX_ERR_METRIC when
 * either class is empty (MetricUndefinedError).  npos / nneg may be NULL.
 * stream: a cudaStream_t (NULL = legacy default stream); returns synchronised. */
int erx_metrics_roc_auc(const float* d_scores, const uint8_t* d_labels, const uint8_t* d_select, size_t n,
                        void* stream, double* auc, uint64_t* npos, uint64_t* nneg);
/* Top-k set of fp32 device scores over the selected elements (the parity
 * gates' top-1% anomaly set): d_mask[i] = 1 for the k largest
 * (ties at the cutoff go to the lower index), else 0; *cutoff = the k-th
 * largest score (may be NULL).  ERX_ERR_DATA when k exceeds the selection. */
int erx_metrics_top_k(const float* d_scores, const uint8_t* d_select, size_t n, size_t k, void* stream,
                      uint8_t* d_mask, float* cutoff);

/* ---- HADC cube / mask files (hadc.cpp; SPEC.md:576-598 [MODULE] io) ----
 * Little-endian container: "HADC", version u16 (1), lines / pixels / bands u32, dtype u8
 * (1 = float32, 2 = u8 mask 0/1), layout u8 (1 = [line][pixel][band]), name_len u16 + UTF-8
 * name, then exactly lines*pixels*bands elements.  Format violations (bad magic / version /
 * dtype / layout, zero sizes, a size product overflowing 64 bits, payload length != declared,
 * mask value > 1) return ERX_ERR_DATA — had::FormatError, kind data (errors.hpp:67-75) — with
 * "at offset <n>" in erx_hadc_last_error (read_cube / read_mask errors);
 * failing to open or read the file returns ERX_ERR_IO (had::IoError, errors.hpp:77-79). */
typedef struct erx_hadc erx_hadc;
typedef struct {
    uint16_t version;
    uint32_t lines, pixels, bands;
    uint8_t dtype, layout;
    uint16_t name_len;
    char name[256]; /* NUL-terminated, truncated to 255 bytes */
} erx_hadc_info;
int erx_hadc_open(const char* path, erx_hadc** out, erx_hadc_info* info);
/* Message of the last failure on h (h = NULL: of this thread's last failed erx_hadc_open). */
const char* erx_hadc_last_error(const erx_hadc* h);
/* Lines [first, first + n) into host memory (mask values checked). */
int erx_hadc_read(erx_hadc* h, uint32_t first_line, uint32_t n_lines, void* dst);
/* The same lines into device memory through two pinned ~16 MB stages: the file read of one
 * chunk overlaps the H2D copy of the previous one on `stream` (a cudaStream_t, NULL = legacy
 * default); returns when the copies are done. */
int erx_hadc_read_device(erx_hadc* h, uint32_t first_line, uint32_t n_lines, void* d_dst, void* stream);
void erx_hadc_close(erx_hadc* h);
/* write_cube / write_mask (dtype 1 / 2); ERX_ERR_CONFIG for zero sizes, ERX_ERR_DATA for a mask
 * value > 1, ERX_ERR_IO for file errors. */
int erx_hadc_write(const char* path, const char* name, uint32_t lines, uint32_t pixels, uint32_t bands, int dtype,
                   const void* data);

/* CUDA events on the engine stream, for callers timing device work. */
int erx_event_record(erx_engine* e, int slot);
int erx_event_elapsed_ms(erx_engine* e, int slot_a, int slot_b, float* ms);

/* Memory helpers so callers need no CUDA runtime of their own. */
void* erx_host_alloc(size_t bytes);
void erx_host_free(void* p);
void* erx_device_alloc(int device, size_t bytes);
void erx_device_free(void* p);
int erx_copy(void* dst, const void* src, size_t bytes, int kind /* 1 h2d, 2 d2h, 3 d2d */, erx_engine* on_stream);

#ifdef __cplusplus
}
#endif

#endif
