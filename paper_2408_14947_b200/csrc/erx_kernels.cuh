// erx_kernels.cuh — device-side pieces of the windowed ERX pipeline.
//
// One window = n lines of each of S independent streams, line id
// l = s * n + t.  The five kernels map onto the reference per-line chain
// (erx.hpp:51-71) re-associated across lines:
//
//   stats      project_line + line_stats       (projection.hpp:33, erx.hpp:40)
//   scan       ema_update / welford_batch_update (erx.hpp:43, linalg.hpp:36)
//   factor     cholesky_lower(K + eps I) with eps escalation, then L^{-1}
//                                               (linalg.hpp:15)
//   score      forward_substitute as a whitening multiply m = L^{-1}(z - mu),
//              delta = ||m||                    (linalg.hpp:21)
//   normalize  normalize_scores                 (detector.hpp:29-32)
//
// Only line_stats is state-free, so every line of the window gets its
// statistics at once; the EMA is an exact element-wise scan (same rounding
// order as the sequential recurrence); factor and score then run for every
// line against its own pre-update background (score-then-update).
#pragma once

#include <cstddef>
#include <cstdint>

namespace erxk {

constexpr int kBlk = 8;          // register-block edge (stats / score)
constexpr int kNB = 32;          // panel width of the blocked factorisation

// Packed lower-triangular index (row-major, j <= i).
__host__ __device__ inline int tri(int i, int j) { return i * (i + 1) / 2 + j; }

struct Geometry {
    int P;         // pixels per line
    int B;         // bands
    int D;         // projected dims (B when no_srp)
    int Dp;        // D rounded up to a multiple of kBlk
    int nb;        // Dp / kBlk
    int SE;        // slot elements: D + D(D+1)/2 (mean followed by packed lower covariance)
    int srp;       // 1: sparse random projection, 0: identity
    const int* srp_ptr;    // [D+1] CSC starts per output dim
    const int* srp_band;   // [nnz] band index
    const float* srp_w;    // [nnz] sign of the weight (+1 / -1)
    double srp_scale;      // |w| = sqrt(s)/sqrt(d); z_j = scale * sum_k sign_k x_k (fp64)
    int srp_wmax;          // max nonzeros of one output dim (the small path's padded table width)
    int srp_nnz;           // nonzeros of W
};

// Per-engine window state, resident on the device so a captured window (CUDA graph) replays without
// host-side parameters: the scan, factor and rescue read it, window_advance_kernel moves it on.
struct WinMeta {
    long long lines_seen;  // lines per stream before this window
    long long welford_n;   // pixels folded into the background (incremental mode)
    int initialized;       // the background exists (else the window's first line initialises it)
    int cur;               // which half of the ping-pong state holds the background
};
// The window's background: state_base + cur * state_stride (+ stream group offset); the scan writes the
// other half.
struct StateRef {
    const WinMeta* meta;
    double* base;
    size_t stride;   // doubles per half (S * SE)
    size_t offset;   // the stream group's first element (s0 * SE)
    __host__ __device__ const double* in() const { return base + size_t(meta->cur) * stride + offset; }
    __host__ __device__ double* out() const { return base + size_t(meta->cur ^ 1) * stride + offset; }
};
void launch_window_advance(WinMeta* meta, int n_lines, long long pixels_per_line, int incremental, cudaStream_t st);

struct StatsLaunch {
    int CH;          // pixels staged per chunk
    int n_pairs;     // lower-triangular 8x8 block pairs
    int npc;         // pairs per CTA
    int G;           // pixel groups per pair (threads per pair)
    int cpl;         // CTAs per line
    int NT;          // threads per CTA
    int minb;        // kernel variant: 1 (<= 384 threads) or 2 (<= 256 threads, two CTAs per SM)
    size_t smem;     // dynamic shared memory bytes
};

struct SmallLaunch {
    int CH;             // pixels per warp chunk (identity projection)
    int CH2;            // pixels per shared stage (SRP variant)
    size_t smem_stats;
    size_t smem_score;
    bool wl;            // warp-per-line kernels (engines with >= 2048 lines per window)
};

// small-D path (k_small.cu): D <= 16, one CTA per line, fused normalisation
bool small_path(const Geometry& g);
SmallLaunch plan_small(const Geometry& g, size_t capacity_lines);
void launch_stats_small(const Geometry& g, const SmallLaunch& sm, const float* x, int n_per_stream, int in_stride,
                        int n_lines_total, double* stats, float* vcache, cudaStream_t st);
void launch_score_small(const Geometry& g, const SmallLaunch& sm, const double* stats, const double* prior,
                        const float* whiten, const float* vcache, int n_lines_total, float* raw, float* norm,
                        int* status, int* fixlist, cudaStream_t st);

struct ScoreLaunch {
    int npairs;      // row-block pairs {s, nb-1-s}
    int G;           // pixel lanes per pair
    int PT;          // pixels per CTA (4 per lane)
    int threads;     // CTA size
    int Dpad;        // smem row stride (floats), = 4 mod 32
    int tiles;       // CTAs per line
    int wsmem;       // 1: the line's W blocks are staged in shared memory
    size_t slab_off; // wsmem == 0: byte offset of the per-step W block ring (k_score.cu: score_slabs)
    size_t smem;
};

StatsLaunch plan_stats(const Geometry& g);
ScoreLaunch plan_score(const Geometry& g);
// floats of packed lower 8x8 W blocks per line (k_factor.cu: write_wblocks)
size_t whiten_floats_per_line(const Geometry& g);
// Factor precision actually used for a request (0 auto, 32, 64): 64 / 32 select the
// shared-memory kernel in that precision, 0 the blocked fp64 global-memory kernel.
int factor_precision(const Geometry& g, int requested, int lines_per_launch);
size_t factor_smem(const Geometry& g, int precision);

// Exact-integer tcgen05 stats kernel (k_stats_i8.cu): no_srp, 16 < D <= 127, B % 4 == 0.
bool stats_i8_eligible(const Geometry& g);
// vmax / vplanes (may be null): [line][D] max_p |fl32(x - c)| and the score's v digit planes
// (vplanes_bytes_per_line per line).  ring1 > 0: the range pass on its own warps with ring1 of the
// ring's stages (stats_i8_ws_kernel, where the ring holds ring1 + 2); 0: the single-role kernel.
// c0: [line][4][D] int32 scratch for the class-0 diagonal partials (folded into S_aa by a second,
// tiny kernel of this launcher).
// redo + headroom > 0: the one-pass kernel (stats_i8_op_kernel: range predicted as headroom x the range
// of the line's first chunk) followed by the exact two-pass kernel over the lines it lists in redo
// ([0] count, [1] running total, [2 ..] line ids; n_lines_total + 2 ints, zeroed once by the caller).
void launch_stats_i8(const Geometry& g, const float* x, int n_per_stream, int in_stride, int n_lines_total,
                     double* stats, float* vmax, unsigned char* vplanes, int* c0, cudaStream_t st,
                     int ring1 = 3, int* redo = nullptr, int headroom = 0);
// Exact-integer tcgen05 stats for wide lines (k_stats_i8t.cu): no_srp, 127 < D <= 512, B % 4 == 0;
// work items are the lower-triangle pairs of 128-dim tiles, 2D TMA boxes from the line.  Returns 0, or
// non-zero when the tensor map could not be encoded (nothing launched).
bool stats_i8t_eligible(const Geometry& g);
// cen / vmax: [line][D] scratch the range pass fills (vmax is also the score's per-dim range).
int launch_stats_i8t(const Geometry& g, const float* x, int n_per_stream, int in_stride, int n_streams,
                     double* stats, float* cen, float* vmax, unsigned char* vplanes, cudaStream_t st);
// Exact-integer tcgen05 score for wide lines (k_score_i8w.cu): the factor's fp32 W blocks are turned into
// the int8 operand by launch_wplanes_w (any factor kernel), then the score reads the stats' v planes.
bool score_i8w_eligible(const Geometry& g);
size_t wplanes_w_bytes_per_line(const Geometry& g);
size_t vplanes_w_bytes_per_line(const Geometry& g);
void launch_wplanes_w(const Geometry& g, const float* whiten, const double* stats, const double* prior,
                      const float* vmax, int n_lines_total, unsigned char* wpl, cudaStream_t st);
void launch_score_i8w(const Geometry& g, const unsigned char* vplanes, const unsigned char* wplanes, int n_lines_total,
                      float* raw, cudaStream_t st);
// Exact-integer tcgen05 score kernel (k_score_i8.cu): v planes from stats_i8, W planes from the factor.
bool score_i8_eligible(const Geometry& g);
size_t wplanes_bytes_per_line();
size_t vplanes_bytes_per_line(const Geometry& g);
void launch_score_i8(const Geometry& g, const unsigned char* vplanes, const unsigned char* wplanes, int n_lines_total,
                     float* raw, cudaStream_t st);

// Host launchers.  All asynchronous on `st`.
void launch_stats(const Geometry& g, const StatsLaunch& sl, const float* x, int n_per_stream, int in_stride,
                  int n_lines_total, double* stats, cudaStream_t st);
// kblk (may be null): write the pre-update covariance as fp32 packed lower 8x8 blocks (row-major
// inside a block, nb(nb+1)/2 * 64 floats per line) instead of fp64 into prior (the mean stays fp64).
void launch_scan(const Geometry& g, const double* stats, double* prior, StateRef state, int n_streams,
                 int n_per_stream, double alpha, int incremental, cudaStream_t st, float* kblk = nullptr);
// latch: {flag, line, pivot} of the first factorisation failure (sticky until the host clears it).
// vmax != null (precision 32 only): write the tensor path's int8 W planes (k_factor.cu: write_wplanes,
// i8::kWBytes per line) instead of the fp32 blocks.  The fp32 factors (precision 32 / 31) put lines
// they cannot take (failed or ill-conditioned pivot) on fixlist for launch_fixup instead of
// escalating eps in fp32; the fp64 ones escalate and latch themselves.
// line ids in the latch: meta->lines_seen * line_mult + line_off + line (streams x window rows)
void launch_factor(const Geometry& g, const double* prior, int n_lines_total, double eps0, double* work,
                   float* whiten, int* status, unsigned long long* latch, const WinMeta* meta, long long line_mult,
                   long long line_off, int precision, cudaStream_t st, int* fixlist, const double* stats = nullptr,
                   const float* vmax = nullptr, const float* kblk = nullptr, int blk_threads = 0);

// fp64 rescue of the lines on the fp32 factor's list (k_fixup.cu): background, factor with eps
// escalation, whitening and normalisation of every listed line redone in fp64 from the line and the
// window statistics; overwrites their raw / norm rows and writes their final status.
struct FixupArgs {
    Geometry g;
    const float* x;          // window lines: line l = s * n + t at line_ptr(x, l, n, in_stride)
    int n;
    int in_stride;
    const double* stats;     // [L][SE + D] the window's line statistics (k_stats.cu contract)
    StateRef state;          // background at the window start (+ initialized / welford count in its meta)
    double alpha;
    int incremental;
    double eps0;
    int* list;               // [0] count, [1] CTAs done, [2 .. list_cap + 1] listed lines, [list_cap + 2] total
    int list_cap;
    double* work;            // fixup_work_doubles(g, L)
    float* raw;
    float* norm;
    int* status;
    unsigned long long* latch;
    long long line_mult, line_off;  // latch line id = meta->lines_seen * line_mult + line_off + line
};
int fixup_ctas(const Geometry& g, int n_lines_total);
size_t fixup_work_doubles(const Geometry& g, int n_lines_total);
void launch_fixup(const FixupArgs& a, int n_lines_total, cudaStream_t st);
void launch_score(const Geometry& g, const ScoreLaunch& sc, const float* x, int n_per_stream, int in_stride,
                  const double* prior, const float* whiten, int n_lines_total, float* raw, cudaStream_t st);
// status / fixlist (may be null): lines whose scores are flat at fp32 resolution go to the fp64 rescue
void launch_normalize(const Geometry& g, const float* raw, int n_lines_total, float* norm, int* status, int* fixlist,
                      cudaStream_t st);

}  // namespace erxk
