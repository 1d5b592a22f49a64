// erx_engine.cu — host runtime behind the C ABI (include/erx_b200.h).
//
// An engine owns S independent ERX streams (S = 1 is the drop-in
// had::ErxDetector, erx.hpp:56-71) advanced in lock-step through windows of
// up to T lines.  It owns one CUDA stream, the SRP weights, the device-side
// background state (ping-pong buffers), the window workspaces and a pinned
// host staging area for the drop-in (host pointer) path.  No CPU fallback:
// every score is computed by the kernels in erx_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/erx_b200.h"
#include "erx_kernels.cuh"
#include "host_rng.hpp"

using erxk::Geometry;

namespace {

// One scored window of the drop-in path: pinned host arrays [S][n][P] written
// by the device-to-host copies directly (no re-packing per line).  Blocks are
// recycled through the engine's pool once every row has been popped.
struct ResultBlock {
    float* raw = nullptr;
    float* norm = nullptr;
    int* status = nullptr;  // [S][n] factor status per line (-1 ok, else the failing pivot)
    size_t cap = 0;         // floats per array
    uint32_t n = 0, P = 0;
};

// A window of the host path whose kernels / result copies may still be running
// (ERX_OPT_ASYNC_HOST): harvested into the queue once `done` has fired.
struct PendingWindow {
    std::shared_ptr<ResultBlock> blk;
    uint32_t n = 0, P = 0;
    std::vector<int64_t> index;
    cudaEvent_t done = nullptr;
};

struct ScoredRow {
    int64_t index;
    uint8_t warmup;
    uint32_t P;                        // pixels of this line
    uint32_t t;                        // row of the block
    std::shared_ptr<ResultBlock> blk;  // raw / norm of all streams
};

struct Timing {
    int kernel;
    cudaEvent_t a, b;
};

}  // namespace

struct erx_engine {
    erx_config cfg{};
    uint32_t B = 0, S = 1, T = 1;
    int device = 0;
    int D = 0, Dp = 0;
    cudaStream_t stream = nullptr;

    std::vector<double> W;  // B x D (SRP only)
    int* d_srp_ptr = nullptr;
    int* d_srp_band = nullptr;
    float* d_srp_sign = nullptr;
    double srp_scale = 1.0;
    int srp_wmax = 0;  // max nonzeros per output dim
    int srp_nnz = 0;

    uint32_t P = 0;  // pixels (set by the first line)
    Geometry geo{};
    erxk::StatsLaunch sl{};
    erxk::ScoreLaunch sc{};
    erxk::SmallLaunch smp{};
    bool small = false;       // D <= 16: stats_small / score_small path
    float* d_vcache = nullptr;  // [S*T][D][P] centred projections (small path)
    float* d_vmax = nullptr;    // [S*T][D] per-dim |x - c| range (tensor path)
    float* d_cen = nullptr;     // [S*T][D] per-dim centre (wide tensor path)
    unsigned char* d_vplanes = nullptr;  // [S*T][tiles][48 KB] quantised v digit planes (tensor path; wide:
                                         // [S*T][pixel tiles][dim tiles][48 KB])
    unsigned char* d_wplw = nullptr;     // [S*T][wplanes_w_bytes] the wide score's int8 W operand
    int* d_c0 = nullptr;        // [S*T][4][D] class-0 diagonal partials of the integer statistics (tensor path)
    int* d_redo = nullptr;      // [kDevGroups][S*T + 2] one-pass statistics: lines listed for the exact two-pass redo
    float* d_kblk = nullptr;    // [S*T][nb(nb+1)/2][64] pre-update K as fp32 blocks (blocked fp32 factor)
    int factor_req = 0;   // requested factor precision (0 auto, 32, 64)
    // ERX_OPT_STATS_TENSOR: 2 exact-integer tcgen05 stats + score where eligible (default), 0 FFMA kernels.
    int stats_tensor = 2;
    int factor_prec = 0;  // precision in use (0 = blocked fp64 global path)
    int factor_threads = 0;  // ERX_OPT_FACTOR_THREADS (0 auto)
    bool tensor = false;      // exact-integer tcgen05 stats + score in use (fixed at configure)
    bool wide_i8 = false;     // exact-integer tcgen05 stats + score for D > 127 (k_stats_i8t.cu, k_score_i8w.cu)
    size_t white_stride = 0;  // floats per line of d_white (fp32 W blocks or int8 W planes)

    // device buffers, capacity S*T lines
    float* d_lines = nullptr;
    double* d_stats = nullptr;
    double* d_prior = nullptr;
    double* d_state[2] = {nullptr, nullptr};  // halves of one allocation (d_state[1] = d_state[0] + S * SE)
    int cur = 0;                              // host mirror of d_meta->cur
    erxk::WinMeta* d_meta = nullptr;          // device-resident window state (erx_kernels.cuh)
    // CUDA graphs of the device path (erx_run_device): one captured window per (input, output, size) key
    struct GraphEntry {
        const float* x;
        float* raw;
        float* norm;
        uint32_t n, P, in_stride;
        cudaGraphExec_t exec;
        uint64_t kernels;
    };
    std::vector<GraphEntry> graphs;
    bool use_graphs = true;                   // ERX_OPT_GRAPHS
    double* d_work = nullptr;
    float* d_white = nullptr;
    float* d_raw = nullptr;
    float* d_norm = nullptr;
    int* d_status = nullptr;
    unsigned long long* d_latch = nullptr;  // {flag, line id, pivot} of the first device-path failure
    int* d_fix = nullptr;        // fp64 rescue list of the fp32 factor ([0] count, [1] done, [2..] lines)
    double* d_fixwork = nullptr; // the rescue's fp64 workspace
    int fix_cap = 0;             // list capacity (lines per window)
    size_t fixwork_doubles = 0;  // rescue workspace per device stream group
    // the device path runs a window as two stream groups on two CUDA streams (ERX_OPT_DEVICE_GROUPS), each
    // with its own rescue list / workspace, so one group's small kernels and tails overlap the other's
    static constexpr int kDevGroups = 2;
    int dev_groups = 0;          // 0 auto, 1 or 2
    int stats_split = 3;         // ERX_OPT_STATS_SPLIT: pass-1 stages of the split statistics kernel (0: single role)
    int stats_onepass = 0;       // ERX_OPT_STATS_ONEPASS: headroom of the one-pass statistics (0: the two-pass kernels)
    int64_t redone_before = 0;   // redone lines counted by earlier (re-planned) lists
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int64_t rescued_before = 0;  // rescued lines counted by earlier (re-planned) lists

    // pinned host staging (drop-in path)
    float* h_lines = nullptr;
    // drop-in path streams: host->device copies and device->host result copies run
    // beside the compute stream, one stream group at a time (run_host_window)
    cudaStream_t h2d = nullptr, d2h = nullptr;
    static constexpr int kMaxGroups = 8;
    cudaEvent_t ev_in[kMaxGroups] = {}, ev_out[kMaxGroups] = {}, ev_d2h[kMaxGroups] = {};
    int prev_groups = 0;  // stream groups of the previous host window (its events guard buffer reuse)
    std::vector<ResultBlock*> block_pool;
    int host_groups = 0;  // ERX_OPT_HOST_GROUPS (0 auto)
    bool async_host = false;  // ERX_OPT_ASYNC_HOST
    std::deque<PendingWindow> pending;
    std::vector<cudaEvent_t> done_pool;
    int pending_err = 0;  // a failure found by erx_ready, reported by the next call that can return it

    bool initialized = false;
    int64_t lines_seen = 0;
    int64_t welford_n = 0;
    uint32_t fill = 0;
    std::vector<int64_t> win_index;
    std::deque<ScoredRow> queue;

    std::string err;
    int pivot = -1;
    bool failed = false;

    uint64_t launches = 0;
    bool profiling = false;
    std::vector<Timing> timings;
    std::vector<cudaEvent_t> event_pool;
    double kms[ERX_NUM_KERNELS] = {};
    uint64_t kcount[ERX_NUM_KERNELS] = {};
    cudaEvent_t user_ev[8] = {};
};

namespace {

int fail(erx_engine* e, int code, const std::string& m) {
    if (e) e->err = m;
    return code;
}

#define CU(call)                                                                                 \
    do {                                                                                         \
        cudaError_t _r = (call);                                                                 \
        if (_r != cudaSuccess)                                                                   \
            return fail(e, ERX_ERR_DEVICE, std::string(#call) + ": " + cudaGetErrorString(_r)); \
    } while (0)

void put_msg(char* dst, size_t n, const std::string& s) {
    if (dst && n) std::snprintf(dst, n, "%s", s.c_str());
}

int validate(const erx_config* c, uint32_t bands, std::string& m) {
    // ErxConfig::validate (erx.hpp:23)
    if (!(c->alpha > 0.0 && c->alpha <= 1.0)) { m = "alpha must be in (0, 1]"; return ERX_ERR_CONFIG; }
    if (!(c->epsilon > 0.0)) { m = "epsilon must be > 0"; return ERX_ERR_CONFIG; }
    if (bands < 1) { m = "bands must be >= 1"; return ERX_ERR_CONFIG; }
    if (!c->no_srp) {
        if (c->dims < 1) { m = "dims must be >= 1"; return ERX_ERR_CONFIG; }
        if (uint32_t(c->dims) > bands) { m = "dims must be <= bands"; return ERX_ERR_CONFIG; }
    }
    const uint32_t d = c->no_srp ? bands : uint32_t(c->dims);
    if (d > 512) { m = "projected dims > 512 are not supported"; return ERX_ERR_CONFIG; }
    return ERX_OK;
}

cudaEvent_t take_event(erx_engine* e) {
    if (!e->event_pool.empty()) {
        cudaEvent_t ev = e->event_pool.back();
        e->event_pool.pop_back();
        return ev;
    }
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    return ev;
}

template <typename F>
void timed(erx_engine* e, int kernel, F&& launch) {
    if (e->profiling) {
        Timing t{kernel, take_event(e), take_event(e)};
        cudaEventRecord(t.a, e->stream);
        launch();
        cudaEventRecord(t.b, e->stream);
        e->timings.push_back(t);
    } else {
        launch();
    }
    e->launches += 1;
}

void collect_timings(erx_engine* e) {
    for (auto& t : e->timings) {
        cudaEventSynchronize(t.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t.a, t.b);
        e->kms[t.kernel] += ms;
        e->kcount[t.kernel] += 1;
        e->event_pool.push_back(t.a);
        e->event_pool.push_back(t.b);
    }
    e->timings.clear();
}

int64_t read_rescued(erx_engine* e) {
    if (!e->d_fix) return 0;
    int64_t tot = 0;
    cudaStreamSynchronize(e->stream);
    for (int gi = 0; gi < erx_engine::kDevGroups; ++gi) {
        int v = 0;
        cudaMemcpy(&v, e->d_fix + size_t(gi) * (e->fix_cap + 3) + e->fix_cap + 2, sizeof(int), cudaMemcpyDeviceToHost);
        tot += v;
    }
    return tot;
}

int64_t read_redone(erx_engine* e) {
    if (!e->d_redo) return 0;
    int64_t tot = 0;
    cudaStreamSynchronize(e->stream);
    for (int gi = 0; gi < erx_engine::kDevGroups; ++gi) {
        int v = 0;
        cudaMemcpy(&v, e->d_redo + size_t(gi) * (size_t(e->S) * e->T + 2) + 1, sizeof(int), cudaMemcpyDeviceToHost);
        tot += v;
    }
    return tot;
}

void free_window(erx_engine* e) {
    e->rescued_before += read_rescued(e);
    e->redone_before += read_redone(e);
    cudaFree(e->d_lines);
    cudaFree(e->d_stats);
    cudaFree(e->d_prior);
    cudaFree(e->d_work);
    cudaFree(e->d_white);
    cudaFree(e->d_raw);
    cudaFree(e->d_norm);
    cudaFree(e->d_status);
    cudaFree(e->d_vcache);
    e->d_vcache = nullptr;
    cudaFree(e->d_vmax);
    e->d_vmax = nullptr;
    cudaFree(e->d_cen);
    e->d_cen = nullptr;
    cudaFree(e->d_vplanes);
    e->d_vplanes = nullptr;
    cudaFree(e->d_wplw);
    e->d_wplw = nullptr;
    cudaFree(e->d_c0);
    e->d_c0 = nullptr;
    cudaFree(e->d_redo);
    e->d_redo = nullptr;
    cudaFree(e->d_kblk);
    e->d_kblk = nullptr;
    cudaFree(e->d_fix);
    e->d_fix = nullptr;
    cudaFree(e->d_fixwork);
    e->d_fixwork = nullptr;
    cudaFreeHost(e->h_lines);
    e->d_lines = nullptr;
    e->d_stats = e->d_prior = e->d_work = nullptr;
    e->d_white = e->d_raw = e->d_norm = nullptr;
    e->d_status = nullptr;
    e->h_lines = nullptr;
}

void free_block(ResultBlock* b) {
    cudaFreeHost(b->raw);
    cudaFreeHost(b->norm);
    cudaFreeHost(b->status);
    delete b;
}

int drain_pending(erx_engine* e);

// (Re)plan the geometry for P pixels and size the window buffers.
int configure(erx_engine* e, uint32_t P) {
    CU(cudaSetDevice(e->device));
    if (int st = drain_pending(e)) return st;  // in-flight host windows use the buffers
    if (P == e->P && e->d_stats) return ERX_OK;
    CU(cudaStreamSynchronize(e->stream));
    free_window(e);
    for (auto& ge : e->graphs) cudaGraphExecDestroy(ge.exec);  // they reference the old buffers
    e->graphs.clear();
    e->P = P;
    Geometry& g = e->geo;
    g.P = int(P);
    g.B = int(e->B);
    g.D = e->D;
    g.Dp = e->Dp;
    g.nb = e->Dp / erxk::kBlk;
    g.SE = e->D + e->D * (e->D + 1) / 2;
    g.srp = e->cfg.no_srp ? 0 : 1;
    g.srp_ptr = e->d_srp_ptr;
    g.srp_band = e->d_srp_band;
    g.srp_w = e->d_srp_sign;
    g.srp_scale = e->srp_scale;
    g.srp_wmax = e->srp_wmax;
    g.srp_nnz = e->srp_nnz;
    e->sl = erxk::plan_stats(g);
    e->sc = erxk::plan_score(g);
    e->small = erxk::small_path(g);
    if (e->small) e->smp = erxk::plan_small(g, size_t(e->S) * e->T);
    e->factor_prec = erxk::factor_precision(g, e->factor_req, int(e->S * e->T));
    // exact-integer tensor path: stats_i8 + factor writing int8 W planes + score_i8
    e->tensor = e->stats_tensor == 2 && erxk::stats_i8_eligible(g) && erxk::score_i8_eligible(g) &&
                e->factor_prec == 32;
    e->wide_i8 = !e->tensor && !e->small && e->stats_tensor == 2 && erxk::stats_i8t_eligible(g) &&
                 erxk::score_i8w_eligible(g);
    e->white_stride = e->tensor ? erxk::wplanes_bytes_per_line() / sizeof(float) : erxk::whiten_floats_per_line(g);
    const size_t L = size_t(e->S) * e->T;
    CU(cudaMalloc(&e->d_stats, L * (g.SE + g.D) * sizeof(double)));  // [c | s | S] per line
    CU(cudaMalloc(&e->d_prior, L * g.SE * sizeof(double)));
    if (e->factor_prec == 0 || e->factor_prec == 31) CU(cudaMalloc(&e->d_work, L * 2 * size_t(g.Dp) * g.Dp * sizeof(double)));
    CU(cudaMalloc(&e->d_white, L * std::max(erxk::whiten_floats_per_line(g),
                                            erxk::stats_i8_eligible(g) ? erxk::wplanes_bytes_per_line() / 4 : size_t(0)) *
                                    sizeof(float)));
    CU(cudaMalloc(&e->d_raw, L * P * sizeof(float)));
    CU(cudaMalloc(&e->d_norm, L * P * sizeof(float)));
    CU(cudaMalloc(&e->d_status, L * sizeof(int)));
    if (e->small) CU(cudaMalloc(&e->d_vcache, L * size_t(g.D) * P * sizeof(float)));
    if (erxk::stats_i8_eligible(g) || e->wide_i8) CU(cudaMalloc(&e->d_vmax, L * size_t(g.D) * sizeof(float)));
    if (e->tensor) CU(cudaMalloc(&e->d_vplanes, L * erxk::vplanes_bytes_per_line(g)));
    if (e->wide_i8) {
        CU(cudaMalloc(&e->d_vplanes, L * erxk::vplanes_w_bytes_per_line(g)));
        CU(cudaMalloc(&e->d_cen, L * size_t(g.D) * sizeof(float)));
        CU(cudaMalloc(&e->d_wplw, L * erxk::wplanes_w_bytes_per_line(g)));
    }
    if (e->tensor) CU(cudaMalloc(&e->d_c0, L * 4 * size_t(g.D) * sizeof(int)));
    if (e->tensor) {
        CU(cudaMalloc(&e->d_redo, erx_engine::kDevGroups * (L + 2) * sizeof(int)));
        CU(cudaMemset(e->d_redo, 0, erx_engine::kDevGroups * (L + 2) * sizeof(int)));
    }
    if (e->factor_prec == 32) CU(cudaMalloc(&e->d_kblk, L * erxk::whiten_floats_per_line(g) * sizeof(float)));
    // fp64 rescue list (fed by the fp32 factors and by the normalisation's flat-line check)
    CU(cudaMalloc(&e->d_fix, erx_engine::kDevGroups * (L + 3) * sizeof(int)));
    CU(cudaMemset(e->d_fix, 0, erx_engine::kDevGroups * (L + 3) * sizeof(int)));
    e->fix_cap = int(L);
    e->fixwork_doubles = erxk::fixup_work_doubles(g, int(L));
    CU(cudaMalloc(&e->d_fixwork, erx_engine::kDevGroups * e->fixwork_doubles * sizeof(double)));
    return ERX_OK;
}

int ensure_host_staging(erx_engine* e) {
    if (e->h_lines) return ERX_OK;
    const size_t L = size_t(e->S) * e->T;
    CU(cudaMalloc(&e->d_lines, L * e->P * e->B * sizeof(float)));
    CU(cudaMallocHost(&e->h_lines, L * e->P * e->B * sizeof(float)));
    if (!e->h2d) {
        CU(cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking));
        for (int k = 0; k < erx_engine::kMaxGroups; ++k) {
            CU(cudaEventCreateWithFlags(&e->ev_in[k], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&e->ev_out[k], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&e->ev_d2h[k], cudaEventDisableTiming));
        }
    }
    return ERX_OK;
}

// A pinned result block for S x n lines of P pixels (pool-recycled).
std::shared_ptr<ResultBlock> take_block(erx_engine* e, uint32_t n) {
    const size_t need = size_t(e->S) * e->T * e->P;
    ResultBlock* b = nullptr;
    while (!e->block_pool.empty() && !b) {
        b = e->block_pool.back();
        e->block_pool.pop_back();
        if (b->cap < need) {
            free_block(b);
            b = nullptr;
        }
    }
    if (!b) {
        b = new ResultBlock();
        if (cudaMallocHost(&b->raw, need * sizeof(float)) != cudaSuccess ||
            cudaMallocHost(&b->norm, need * sizeof(float)) != cudaSuccess ||
            cudaMallocHost(&b->status, size_t(e->S) * e->T * sizeof(int)) != cudaSuccess) {
            free_block(b);
            return nullptr;
        }
        b->cap = need;
    }
    b->n = n;
    b->P = e->P;
    auto* pool = &e->block_pool;
    return std::shared_ptr<ResultBlock>(b, [pool](ResultBlock* x) { pool->push_back(x); });
}

// Enqueue the five-kernel window pipeline for n lines of streams [s0, s0 + ns).
// x points at stream 0 of the window (stream stride in_stride lines); every
// per-line buffer holds line (s, t) at s * n + t, so a stream range is a
// contiguous line range and the groups are independent (no cross-stream data).
int enqueue_window(erx_engine* e, const float* x, uint32_t n, uint32_t in_stride, float* raw, float* norm,
                   uint32_t s0, uint32_t ns, bool score = true, int grp = 0) {
    // grp: device stream group (run_device_window) -- its own CUDA stream, rescue list and workspace
    cudaStream_t st = grp ? e->stream2 : e->stream;
    int* fix = e->d_fix + size_t(grp) * (e->fix_cap + 3);
    double* fixwork = e->d_fixwork + size_t(grp) * e->fixwork_doubles;
    const Geometry& g = e->geo;
    const int L = int(ns * n);
    const size_t l0 = size_t(s0) * n;
    const erxk::StateRef sref{e->d_meta, e->d_state[0], size_t(e->S) * g.SE, size_t(s0) * g.SE};
    const float* xg = x + size_t(s0) * in_stride * g.P * g.B;
    double* stats = e->d_stats + l0 * (g.SE + g.D);
    double* prior = e->d_prior + l0 * g.SE;
    double* work = e->d_work ? e->d_work + l0 * 2 * size_t(g.Dp) * g.Dp : nullptr;
    float* white = e->d_white + l0 * e->white_stride;
    float* vcache = e->d_vcache ? e->d_vcache + l0 * size_t(g.D) * g.P : nullptr;
    float* vmax = e->d_vmax ? e->d_vmax + l0 * size_t(g.D) : nullptr;
    float* cen = e->d_cen ? e->d_cen + l0 * size_t(g.D) : nullptr;
    const size_t vpl_line = e->wide_i8 ? erxk::vplanes_w_bytes_per_line(g) : erxk::vplanes_bytes_per_line(g);
    unsigned char* vplanes = e->d_vplanes ? e->d_vplanes + l0 * vpl_line : nullptr;
    unsigned char* wplw = e->d_wplw ? e->d_wplw + l0 * erxk::wplanes_w_bytes_per_line(g) : nullptr;
    float* kblk = e->d_kblk ? e->d_kblk + l0 * erxk::whiten_floats_per_line(g) : nullptr;
    int* c0 = (e->tensor && e->d_c0) ? e->d_c0 + l0 * 4 * size_t(g.D) : nullptr;
    int* redo = (e->d_redo && e->stats_onepass > 0) ? e->d_redo + size_t(grp) * (size_t(e->S) * e->T + 2) : nullptr;
    const bool tensor = e->tensor;
    int* status = e->d_status + l0;
    float* rawg = raw ? raw + l0 * g.P : nullptr;
    float* normg = norm ? norm + l0 * g.P : nullptr;
    int stats_rc = 0;
    timed(e, ERX_KERNEL_STATS, [&] {
        if (e->small)
            erxk::launch_stats_small(g, e->smp, xg, int(n), int(in_stride), L, stats, vcache, st);
        else if (tensor)
            erxk::launch_stats_i8(g, xg, int(n), int(in_stride), L, stats, vmax, vplanes, c0, st, e->stats_split,
                                  redo, e->stats_onepass);
        else if (e->wide_i8)
            stats_rc = erxk::launch_stats_i8t(g, xg, int(n), int(in_stride), int(ns), stats, cen, vmax, vplanes,
                                              st);
        else
            erxk::launch_stats(g, e->sl, xg, int(n), int(in_stride), L, stats, st);
    });
    if (stats_rc) return fail(e, ERX_ERR_DEVICE, "stats_i8t: cannot encode the TMA tensor map");
#ifdef ERX_X_STATSONLY
    return ERX_OK;  // A/B timing builds (tools/ab_build.sh): the statistics kernel alone
#endif
    timed(e, ERX_KERNEL_SCAN, [&] {
        erxk::launch_scan(g, stats, prior, sref, int(ns), int(n), e->cfg.alpha, e->cfg.use_incremental, st,
                          kblk);
    });
    if (!score) {  // background update only (erx_advance_device): statistics and the scan
        cudaError_t r = cudaGetLastError();
        if (r != cudaSuccess) return fail(e, ERX_ERR_DEVICE, std::string("kernel launch: ") + cudaGetErrorString(r));
        return ERX_OK;
    }
    timed(e, ERX_KERNEL_FACTOR, [&] {
        erxk::launch_factor(g, prior, L, e->cfg.epsilon, work, white, status, e->d_latch, e->d_meta, (long long)(e->S),
                            (long long)(l0), e->factor_prec, st, fix, stats, tensor ? vmax : nullptr, kblk,
                            e->factor_threads);
    });
    if (e->small) {  // score + normalisation fused
        timed(e, ERX_KERNEL_SCORE, [&] {
            erxk::launch_score_small(g, e->smp, stats, prior, white, vcache, L, rawg, normg, status, fix,
                                     st);
        });
    } else {
        timed(e, ERX_KERNEL_SCORE, [&] {
            if (tensor) {
                erxk::launch_score_i8(g, vplanes, reinterpret_cast<const unsigned char*>(white), L, rawg, st);
            } else if (e->wide_i8) {
                erxk::launch_wplanes_w(g, white, stats, prior, vmax, L, wplw, st);
                erxk::launch_score_i8w(g, vplanes, wplw, L, rawg, st);
            } else
                erxk::launch_score(g, e->sc, xg, int(n), int(in_stride), prior, white, L, rawg, st);
        });
        timed(e, ERX_KERNEL_NORMALIZE, [&] { erxk::launch_normalize(g, rawg, L, normg, status, fix, st); });
    }
    {
        timed(e, ERX_KERNEL_FIXUP, [&] {
            erxk::FixupArgs fa{g, xg, int(n), int(in_stride), stats, sref, e->cfg.alpha, e->cfg.use_incremental,
                               e->cfg.epsilon, fix, e->fix_cap, fixwork, rawg, normg, status, e->d_latch,
                               (long long)(e->S), (long long)(l0)};
            erxk::launch_fixup(fa, L, st);
        });
    }
    cudaError_t r = cudaGetLastError();
    if (r != cudaSuccess) return fail(e, ERX_ERR_DEVICE, std::string("kernel launch: ") + cudaGetErrorString(r));
    return ERX_OK;
}

// The window's state transition, once all of its stream groups are enqueued: on the device (the next
// window's kernels read it) and in the host mirror.
void enqueue_advance(erx_engine* e, uint32_t n) {
    erxk::launch_window_advance(e->d_meta, int(n), (long long)(e->P), e->cfg.use_incremental, e->stream);
    e->launches += 1;
}
void commit_window(erx_engine* e, uint32_t n) {
    e->cur ^= 1;
    if (e->cfg.use_incremental) e->welford_n += int64_t(n) * e->P;
    e->initialized = true;
    e->lines_seen += n;
}

// Stream groups of one host window: enough that the copy of group g+1 hides
// the kernels of group g, few enough that each copy stays >= ~8 MB (full
// PCIe efficiency) and each launch still fills the GPU.
uint32_t host_groups(const erx_engine* e, uint32_t n) {
    if (e->host_groups > 0) return std::min<uint32_t>(uint32_t(e->host_groups), e->S);
    const double bytes = double(e->S) * n * e->P * e->B * sizeof(float);
    uint32_t G = uint32_t(std::min(double(erx_engine::kMaxGroups), std::floor(bytes / (8.0 * 1024 * 1024))));
    return std::max<uint32_t>(1, std::min<uint32_t>(G, e->S));
}

// Move finished host windows into the queue, oldest first.  block_oldest: wait
// for the oldest pending window (the others are taken only if already done).
// A window with a failing line queues the lines before it, fails the engine
// and drops every later window.
int harvest(erx_engine* e, bool block_oldest) {
    while (!e->pending.empty()) {
        PendingWindow& pw = e->pending.front();
        if (block_oldest) {
            CU(cudaEventSynchronize(pw.done));
            block_oldest = false;
        } else {
            const cudaError_t q = cudaEventQuery(pw.done);
            if (q == cudaErrorNotReady) break;
            if (q != cudaSuccess) return fail(e, ERX_ERR_DEVICE, std::string("host window: ") + cudaGetErrorString(q));
        }
        const uint32_t n = pw.n;
        int bad_t = -1, bad_piv = -1;  // first failing line in emission order (then stream order)
        for (uint32_t t = 0; t < n && bad_t < 0; ++t)
            for (uint32_t s = 0; s < e->S; ++s) {
                if (pw.blk->status[s * n + t] == -2) {  // listed for the fp64 rescue, never rescued
                    e->failed = true;
                    return fail(e, ERX_ERR_DEVICE, "internal: a line listed for the fp64 rescue was not rescued");
                }
                if (pw.blk->status[s * n + t] >= 0) {
                    bad_t = int(t);
                    bad_piv = pw.blk->status[s * n + t];
                    break;
                }
            }
        const uint32_t good = bad_t < 0 ? n : uint32_t(bad_t);
        for (uint32_t t = 0; t < good; ++t) {
            ScoredRow row;
            row.index = pw.index[t];
            row.warmup = (row.index < int64_t(e->cfg.buffer_len)) ? 1 : 0;
            row.P = pw.P;
            row.t = t;
            row.blk = pw.blk;
            e->queue.push_back(std::move(row));
        }
        const int64_t bad_index = bad_t >= 0 ? pw.index[bad_t] : -1;
        e->done_pool.push_back(pw.done);
        e->pending.pop_front();
        if (bad_t >= 0) {
            cudaStreamSynchronize(e->d2h);  // later windows are dropped: let their copies land first
            cudaStreamSynchronize(e->stream);
            for (auto& later : e->pending) e->done_pool.push_back(later.done);
            e->pending.clear();
            e->failed = true;
            e->pivot = bad_piv;
            return fail(e, ERX_ERR_NUMERIC,
                        "Cholesky of K + eps*I failed at pivot " + std::to_string(bad_piv) + " for line index " +
                            std::to_string(bad_index) + " after epsilon escalation to 1e-1");
        }
    }
    return ERX_OK;
}

int drain_pending(erx_engine* e) {
    while (!e->pending.empty()) {
        const int st = harvest(e, true);
        if (st) return st;
    }
    return ERX_OK;
}

// Score one window of the drop-in path.  src holds stream s at src + s *
// src_pitch floats (n lines of P x B each): the caller's buffer (direct path)
// or the pinned staging buffer.  The window is cut into stream groups: group
// g's host->device copy (h2d stream) overlaps the kernels of group g-1
// (compute stream), whose results drain on the d2h stream.  The call returns
// once the input is on the device (the source buffer is free again, the
// per-call contract of the reference's process()); by default it also waits
// for the scores and queues them, with ERX_OPT_ASYNC_HOST the window stays in
// flight (its copy-in then overlaps the previous window's kernels and result
// copies) until erx_ready / erx_pop / erx_finish harvest it.
// One window of the device path.  Every per-window value the kernels need is either a buffer pointer
// (fixed for a given input / output) or in the device-resident window state, so the window's launches
// (6-8 kernels and the state advance) are captured once per (input, output, size) into a CUDA graph
// and replayed as ONE launch: the single-stream lag-0 path costs one graph launch per line — the host
// path's windows always qualify (fixed staging buffers), device-path callers when they reuse a few
// buffers (an 8-entry cache) (ERX_OPT_GRAPHS; off while per-kernel profiling is on).
// Both device stream groups of one window: group 0 on the engine stream, group 1 forked onto stream2
// and joined back before the state advance (no shared buffers: per-line buffers are indexed by
// stream, rescue lists and workspaces are per group).
int enqueue_device_window(erx_engine* e, const float* d_lines, uint32_t n, uint32_t in_stride, float* d_raw,
                          float* d_norm) {
    const bool split = !e->profiling && e->S >= 2 &&
                       (e->dev_groups == 2 || (e->dev_groups == 0 && uint64_t(e->S) * n >= 1024));
    if (!split) {
        if (int st = enqueue_window(e, d_lines, n, in_stride, d_raw, d_norm, 0, e->S)) return st;
        enqueue_advance(e, n);
        return ERX_OK;
    }
    const uint32_t sh = e->S / 2;
    CU(cudaEventRecord(e->ev_fork, e->stream));
    CU(cudaStreamWaitEvent(e->stream2, e->ev_fork, 0));
    if (int st = enqueue_window(e, d_lines, n, in_stride, d_raw, d_norm, 0, sh, true, 0)) return st;
    if (int st = enqueue_window(e, d_lines, n, in_stride, d_raw, d_norm, sh, e->S - sh, true, 1)) return st;
    CU(cudaEventRecord(e->ev_join, e->stream2));
    CU(cudaStreamWaitEvent(e->stream, e->ev_join, 0));
    enqueue_advance(e, n);
    return ERX_OK;
}

int run_device_window(erx_engine* e, const float* d_lines, uint32_t n, uint32_t in_stride, float* d_raw,
                      float* d_norm) {
    if (!e->use_graphs || e->profiling) return enqueue_device_window(e, d_lines, n, in_stride, d_raw, d_norm);
    for (auto& ge : e->graphs)
        if (ge.x == d_lines && ge.raw == d_raw && ge.norm == d_norm && ge.n == n && ge.P == e->P &&
            ge.in_stride == in_stride) {
            CU(cudaGraphLaunch(ge.exec, e->stream));
            e->launches += ge.kernels;
            return ERX_OK;
        }
    const uint64_t k0 = e->launches;
    CU(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    int st = enqueue_device_window(e, d_lines, n, in_stride, d_raw, d_norm);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(e->stream, &graph);
    if (st) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (ce != cudaSuccess) return fail(e, ERX_ERR_DEVICE, std::string("graph capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return fail(e, ERX_ERR_DEVICE, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    if (e->graphs.size() >= 8) {  // a small cache: callers cycle through a few buffers
        cudaGraphExecDestroy(e->graphs.front().exec);
        e->graphs.erase(e->graphs.begin());
    }
    e->graphs.push_back({d_lines, d_raw, d_norm, n, e->P, in_stride, exec, e->launches - k0});
    CU(cudaGraphLaunch(exec, e->stream));
    return ERX_OK;
}

int run_host_window_body(erx_engine* e, const float* src, size_t src_pitch);

// Any failure inside a host window leaves the engine failed with the window dropped (its lines
// cannot be scored any more; the reference leaves continuation after a throw unspecified).
int run_host_window(erx_engine* e, const float* src, size_t src_pitch) {
    const int st = run_host_window_body(e, src, src_pitch);
    if (st && e->fill) {
        e->fill = 0;
        e->failed = true;
    }
    return st;
}

int run_host_window_body(erx_engine* e, const float* src, size_t src_pitch) {
    if (e->fill == 0) return ERX_OK;
    const uint32_t n = e->fill;
    const size_t line_f = size_t(e->P) * e->B;
    auto blk = take_block(e, n);
    if (!blk) return fail(e, ERX_ERR_DEVICE, "cudaMallocHost (result block)");
    const uint32_t G = host_groups(e, n);
    const int pg = e->prev_groups;
    for (uint32_t gi = 0; gi < G; ++gi) {
        const uint32_t s0 = uint32_t(uint64_t(e->S) * gi / G), s1 = uint32_t(uint64_t(e->S) * (gi + 1) / G);
        const uint32_t ns = s1 - s0;
        if (!ns) continue;
        // the previous window's group (or, with another grouping, all of it) must be done with
        // d_lines before this copy overwrites it, and its results must have left d_raw / d_norm
        const int prev = pg == int(G) ? int(gi) : pg - 1;
        if (pg) CU(cudaStreamWaitEvent(e->h2d, e->ev_out[prev], 0));
        CU(cudaMemcpy2DAsync(e->d_lines + size_t(s0) * e->T * line_f, size_t(e->T) * line_f * sizeof(float),
                             src + size_t(s0) * src_pitch, src_pitch * sizeof(float), n * line_f * sizeof(float), ns,
                             cudaMemcpyHostToDevice, e->h2d));
        CU(cudaEventRecord(e->ev_in[gi], e->h2d));
        CU(cudaStreamWaitEvent(e->stream, e->ev_in[gi], 0));
        if (pg) CU(cudaStreamWaitEvent(e->stream, e->ev_d2h[prev], 0));
        // one group: the whole window (and the state advance) as one replayable graph
        int st = G == 1 ? run_device_window(e, e->d_lines, n, e->T, e->d_raw, e->d_norm)
                        : enqueue_window(e, e->d_lines, n, e->T, e->d_raw, e->d_norm, s0, ns);
        if (st) return st;
        CU(cudaEventRecord(e->ev_out[gi], e->stream));
        CU(cudaStreamWaitEvent(e->d2h, e->ev_out[gi], 0));
        const size_t l0 = size_t(s0) * n, nl = size_t(ns) * n;
        CU(cudaMemcpyAsync(blk->raw + l0 * e->P, e->d_raw + l0 * e->P, nl * e->P * sizeof(float),
                           cudaMemcpyDeviceToHost, e->d2h));
        CU(cudaMemcpyAsync(blk->norm + l0 * e->P, e->d_norm + l0 * e->P, nl * e->P * sizeof(float),
                           cudaMemcpyDeviceToHost, e->d2h));
        CU(cudaMemcpyAsync(blk->status + l0, e->d_status + l0, nl * sizeof(int), cudaMemcpyDeviceToHost, e->d2h));
        CU(cudaEventRecord(e->ev_d2h[gi], e->d2h));
    }
    if (G > 1) enqueue_advance(e, n);
    commit_window(e, n);
    e->prev_groups = int(G);
    PendingWindow pw;
    pw.blk = blk;
    pw.n = n;
    pw.P = e->P;
    pw.index.assign(e->win_index.begin(), e->win_index.begin() + n);
    if (!e->done_pool.empty()) {
        pw.done = e->done_pool.back();
        e->done_pool.pop_back();
    } else {
        CU(cudaEventCreateWithFlags(&pw.done, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(pw.done, e->d2h));
    e->pending.push_back(std::move(pw));
    e->fill = 0;
    CU(cudaStreamSynchronize(e->h2d));  // the source buffer is free again
    return e->async_host ? ERX_OK : drain_pending(e);
}

int run_staged_window(erx_engine* e) {
    return run_host_window(e, e->h_lines, size_t(e->T) * e->P * e->B);
}

}  // namespace

extern "C" {

void erx_config_default(erx_config* c) {
    c->dims = 5;
    c->alpha = 0.1;
    c->buffer_len = 99;
    c->epsilon = 1e-5;
    c->seed = 0;
    c->no_srp = 0;
    c->use_incremental = 0;
}

int erx_config_validate(const erx_config* cfg, uint32_t bands, char* msg, size_t msg_len) {
    std::string m;
    int st = validate(cfg, bands, m);
    if (st) put_msg(msg, msg_len, m);
    return st;
}

int erx_generate_srp(uint32_t bands, uint32_t dims, uint64_t seed, double* w) {
    if (bands < 1 || dims < 1) return ERX_ERR_CONFIG;
    erx_host::generate_srp(bands, dims, seed, w);
    return ERX_OK;
}

int erx_create(const erx_config* cfg, uint32_t bands, uint32_t n_streams, uint32_t window_lines, int device,
               erx_engine** out, char* msg, size_t msg_len) {
    *out = nullptr;
    std::string m;
    int st = validate(cfg, bands, m);
    if (!st && (n_streams < 1 || window_lines < 1)) {
        m = "n_streams and window_lines must be >= 1";
        st = ERX_ERR_CONFIG;
    }
    if (st) {
        put_msg(msg, msg_len, m);
        return st;
    }
    erx_engine* e = new erx_engine();
    e->cfg = *cfg;
    e->B = bands;
    e->S = n_streams;
    e->T = window_lines;
    e->device = device;
    e->D = cfg->no_srp ? int(bands) : cfg->dims;
    e->Dp = (e->D + erxk::kBlk - 1) / erxk::kBlk * erxk::kBlk;
    e->win_index.resize(window_lines);
    auto bail = [&](const std::string& why) {
        put_msg(msg, msg_len, why);
        erx_destroy(e);
        return ERX_ERR_DEVICE;
    };
    cudaError_t r = cudaSetDevice(device);
    if (r != cudaSuccess) return bail(std::string("cudaSetDevice: ") + cudaGetErrorString(r));
    r = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
    if (r != cudaSuccess) return bail(std::string("cudaStreamCreate: ") + cudaGetErrorString(r));
    if (cudaStreamCreateWithFlags(&e->stream2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return bail("cudaStreamCreate (device group stream)");
    // SRP weights (generate_srp, projection.hpp:26) -> CSC of signs per output dim
    std::vector<int> ptr(e->D + 1, 0), band;
    std::vector<float> sign;
    if (!cfg->no_srp) {
        e->W.resize(size_t(bands) * e->D);
        erx_host::generate_srp(bands, uint32_t(e->D), cfg->seed, e->W.data());
        const double s = std::sqrt(double(bands));
        e->srp_scale = std::sqrt(s) / std::sqrt(double(e->D));
        for (int j = 0; j < e->D; ++j) {
            ptr[j] = int(band.size());
            for (uint32_t k = 0; k < bands; ++k) {
                double w = e->W[size_t(k) * e->D + j];
                if (w != 0.0) {
                    band.push_back(int(k));
                    sign.push_back(w > 0 ? 1.f : -1.f);
                }
            }
        }
        ptr[e->D] = int(band.size());
        for (int j = 0; j < e->D; ++j) e->srp_wmax = std::max(e->srp_wmax, ptr[j + 1] - ptr[j]);
        e->srp_nnz = ptr[e->D];
    }
    const size_t nnz = std::max<size_t>(band.size(), 1);
    if (cudaMalloc(&e->d_srp_ptr, ptr.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&e->d_srp_band, nnz * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&e->d_srp_sign, nnz * sizeof(float)) != cudaSuccess)
        return bail("cudaMalloc (srp)");
    cudaMemcpy(e->d_srp_ptr, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (!band.empty()) {
        cudaMemcpy(e->d_srp_band, band.data(), band.size() * sizeof(int), cudaMemcpyHostToDevice);
        cudaMemcpy(e->d_srp_sign, sign.data(), sign.size() * sizeof(float), cudaMemcpyHostToDevice);
    }
    const int SE = e->D + e->D * (e->D + 1) / 2;
    if (cudaMalloc(&e->d_state[0], 2 * size_t(n_streams) * SE * sizeof(double)) != cudaSuccess)
        return bail("cudaMalloc (state)");
    cudaMemset(e->d_state[0], 0, 2 * size_t(n_streams) * SE * sizeof(double));
    e->d_state[1] = e->d_state[0] + size_t(n_streams) * SE;
    if (cudaMalloc(&e->d_meta, sizeof(erxk::WinMeta)) != cudaSuccess) return bail("cudaMalloc (meta)");
    cudaMemset(e->d_meta, 0, sizeof(erxk::WinMeta));
    if (cudaMalloc(&e->d_latch, 4 * sizeof(unsigned long long)) != cudaSuccess) return bail("cudaMalloc (latch)");
    cudaMemset(e->d_latch, 0, 4 * sizeof(unsigned long long));
    for (auto& ev : e->user_ev) cudaEventCreate(&ev);
    *out = e;
    return ERX_OK;
}

void erx_destroy(erx_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    if (e->d2h) cudaStreamSynchronize(e->d2h);
    for (auto& pw : e->pending) cudaEventDestroy(pw.done);
    e->pending.clear();
    for (auto ev : e->done_pool) cudaEventDestroy(ev);
    e->done_pool.clear();
    e->queue.clear();  // returns result blocks to the pool
    for (auto* b : e->block_pool) free_block(b);
    e->block_pool.clear();
    free_window(e);
    cudaFree(e->d_srp_ptr);
    cudaFree(e->d_srp_band);
    cudaFree(e->d_srp_sign);
    cudaFree(e->d_state[0]);
    cudaFree(e->d_meta);
    for (auto& ge : e->graphs) cudaGraphExecDestroy(ge.exec);
    e->graphs.clear();
    cudaFree(e->d_latch);
    for (auto& t : e->timings) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    for (auto ev : e->event_pool) cudaEventDestroy(ev);
    for (auto ev : e->user_ev)
        if (ev) cudaEventDestroy(ev);
    for (int k = 0; k < erx_engine::kMaxGroups; ++k) {
        if (e->ev_in[k]) cudaEventDestroy(e->ev_in[k]);
        if (e->ev_out[k]) cudaEventDestroy(e->ev_out[k]);
        if (e->ev_d2h[k]) cudaEventDestroy(e->ev_d2h[k]);
    }
    if (e->h2d) cudaStreamDestroy(e->h2d);
    if (e->stream2) cudaStreamDestroy(e->stream2);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    if (e->d2h) cudaStreamDestroy(e->d2h);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

const char* erx_last_error(const erx_engine* e) { return e ? e->err.c_str() : "null engine"; }
int erx_last_pivot(const erx_engine* e) { return e ? e->pivot : -1; }
int erx_dims(const erx_engine* e) { return e->D; }
uint32_t erx_streams(const erx_engine* e) { return e->S; }
uint32_t erx_window(const erx_engine* e) { return e->T; }

int report_pending(erx_engine* e) {
    const int st = e->pending_err;
    e->pending_err = 0;
    return st;
}

int erx_push_host(erx_engine* e, int64_t first_index, uint32_t n_lines, uint32_t pixels, uint32_t bands,
                  const float* lines) {
    if (int st = report_pending(e)) return st;
    if (e->failed) return fail(e, ERX_ERR_STATE, "engine is in a failed state: " + e->err);
    if (int st = harvest(e, false)) return st;
    if (bands != e->B) return fail(e, ERX_ERR_CONFIG, "band count mismatch");  // projection.hpp:31-32
    if (pixels < 2) return fail(e, ERX_ERR_DATA, "a line needs p >= 2 pixels (1/(p-1) covariance)");  // erx.hpp:39
    if (n_lines == 0) return ERX_OK;
    if (pixels != e->P || !e->d_stats) {
        int st = run_staged_window(e);
        if (st) return st;
        st = configure(e, pixels);
        if (st) return st;
    }
    int st = ensure_host_staging(e);
    if (st) return st;
    const size_t line_f = size_t(pixels) * bands;
    uint32_t i = 0;
    while (i < n_lines) {
        if (e->fill == 0 && n_lines - i >= e->T) {
            // a whole window straight from the caller's buffer (pinned memory: DMA; pageable: staged by CUDA)
            for (uint32_t k = 0; k < e->T; ++k) e->win_index[k] = first_index + int64_t(i + k);
            e->fill = e->T;
            st = run_host_window(e, lines + size_t(i) * line_f, size_t(n_lines) * line_f);
            if (st) return st;
            i += e->T;
            continue;
        }
        if (e->fill >= e->T) return fail(e, ERX_ERR_STATE, "internal: staging window overfull");
        for (uint32_t s = 0; s < e->S; ++s)
            std::memcpy(e->h_lines + (size_t(s) * e->T + e->fill) * line_f,
                        lines + (size_t(s) * n_lines + i) * line_f, line_f * sizeof(float));
        e->win_index[e->fill] = first_index + int64_t(i);
        e->fill += 1;
        i += 1;
        if (e->fill == e->T) {
            st = run_staged_window(e);
            if (st) return st;
        }
    }
    return ERX_OK;
}

int erx_finish(erx_engine* e) {
    if (int st = report_pending(e)) return st;
    if (e->failed) return fail(e, ERX_ERR_STATE, "engine is in a failed state: " + e->err);
    if (int st = run_staged_window(e)) return st;
    return drain_pending(e);
}

// Harvest finished host windows; when nothing is queued, wait for the oldest in-flight one.
void ready_harvest(erx_engine* e) {
    if (e->pending_err || e->failed) return;
    int st = harvest(e, false);
    if (!st && e->queue.empty() && !e->pending.empty()) st = harvest(e, true);
    if (st) e->pending_err = st;
}

uint32_t erx_ready(const erx_engine* ce) {
    erx_engine* e = const_cast<erx_engine*>(ce);  // opaque handle: harvesting is not observable state
    ready_harvest(e);
    // the leading run of queued lines that share one pixel count
    uint32_t n = 0;
    for (const auto& r : e->queue) {
        if (r.P != e->queue.front().P) break;
        ++n;
    }
    return n;
}

uint32_t erx_next_pixels(const erx_engine* e) { return e->queue.empty() ? 0u : e->queue.front().P; }

int erx_pop(erx_engine* e, uint32_t max_lines, int64_t* index, uint8_t* warmup, double* raw, double* norm) {
    const uint32_t n = std::min<uint32_t>(max_lines, erx_ready(e));
    if (!n) return -report_pending(e);
    const size_t P = e->queue.front().P;
    for (uint32_t k = 0; k < n; ++k) {
        const ScoredRow& r = e->queue[k];
        if (index) index[k] = r.index;
        if (warmup) warmup[k] = r.warmup;
    }
    // widen fp32 -> fp64 (ScoredLine payload), streams split across host threads for big pops
    auto widen = [&](uint32_t s_lo, uint32_t s_hi) {
        for (uint32_t k = 0; k < n; ++k) {
            const ScoredRow& r = e->queue[k];
            const ResultBlock& b = *r.blk;
            for (uint32_t s = s_lo; s < s_hi; ++s) {
                const float* fr = b.raw + (size_t(s) * b.n + r.t) * P;
                const float* fn = b.norm + (size_t(s) * b.n + r.t) * P;
                double* dr = raw ? raw + (size_t(s) * n + k) * P : nullptr;
                double* dn = norm ? norm + (size_t(s) * n + k) * P : nullptr;
                if (dr)
                    for (size_t p = 0; p < P; ++p) dr[p] = double(fr[p]);
                if (dn)
                    for (size_t p = 0; p < P; ++p) dn[p] = double(fn[p]);
            }
        }
    };
    const size_t elems = size_t(e->S) * n * P;
    const uint32_t hw = std::max(1u, std::thread::hardware_concurrency());
    const uint32_t nt = std::min<uint32_t>({e->S, 16u, hw, uint32_t(elems >> 17) + 1});
    if (nt <= 1) {
        widen(0, e->S);
    } else {
        std::vector<std::thread> pool;
        for (uint32_t i = 1; i < nt; ++i)
            pool.emplace_back(widen, uint32_t(uint64_t(e->S) * i / nt), uint32_t(uint64_t(e->S) * (i + 1) / nt));
        widen(0, uint32_t(e->S / nt));
        for (auto& th : pool) th.join();
    }
    for (uint32_t k = 0; k < n; ++k) e->queue.pop_front();
    return int(n);
}

int erx_run_device(erx_engine* e, int64_t first_index, uint32_t n_lines, uint32_t pixels, const float* d_lines,
                   float* d_raw, float* d_norm) {
    (void)first_index;
    if (int st = report_pending(e)) return st;
    if (!e->failed)
        if (int st = drain_pending(e)) return st;
    if (e->failed) return fail(e, ERX_ERR_STATE, "engine is in a failed state: " + e->err);
    if (pixels < 2) return fail(e, ERX_ERR_DATA, "a line needs p >= 2 pixels (1/(p-1) covariance)");
    if (n_lines == 0) return ERX_OK;
    if (n_lines > e->T) return fail(e, ERX_ERR_CONFIG, "n_lines exceeds the engine window");
    if (e->fill) return fail(e, ERX_ERR_STATE, "host lines pending; call erx_finish first");
    int st = configure(e, pixels);
    if (st) return st;
    st = run_device_window(e, d_lines, n_lines, n_lines, d_raw, d_norm);
    if (st) return st;
    commit_window(e, n_lines);
    return ERX_OK;
}

int erx_advance_device(erx_engine* e, int64_t first_index, uint32_t n_lines, uint32_t pixels, const float* d_lines) {
    (void)first_index;
    if (int st = report_pending(e)) return st;
    if (!e->failed)
        if (int st = drain_pending(e)) return st;
    if (e->failed) return fail(e, ERX_ERR_STATE, "engine is in a failed state: " + e->err);
    if (pixels < 2) return fail(e, ERX_ERR_DATA, "a line needs p >= 2 pixels (1/(p-1) covariance)");
    if (n_lines == 0) return ERX_OK;
    if (n_lines > e->T) return fail(e, ERX_ERR_CONFIG, "n_lines exceeds the engine window");
    if (e->fill) return fail(e, ERX_ERR_STATE, "host lines pending; call erx_finish first");
    int st = configure(e, pixels);
    if (st) return st;
    st = enqueue_window(e, d_lines, n_lines, n_lines, nullptr, nullptr, 0, e->S, /*score=*/false);
    if (st) return st;
    enqueue_advance(e, n_lines);
    commit_window(e, n_lines);
    return ERX_OK;
}

int erx_sync(erx_engine* e) {
    if (int st = report_pending(e)) return st;
    if (int st = drain_pending(e)) return st;
    CU(cudaStreamSynchronize(e->stream));
    unsigned long long latch[4];
    CU(cudaMemcpy(latch, e->d_latch, sizeof(latch), cudaMemcpyDeviceToHost));
    if (latch[0]) {
        e->failed = true;
        e->pivot = int(latch[2]);
        return fail(e, ERX_ERR_NUMERIC, "Cholesky of K + eps*I failed at pivot " + std::to_string(latch[2]) +
                                            " (window line id " + std::to_string(latch[1]) + ")");
    }
    return ERX_OK;
}

void* erx_cuda_stream(erx_engine* e) { return reinterpret_cast<void*>(e->stream); }

int erx_get_state(erx_engine* e, uint32_t stream, double* mu, double* cov, int64_t* lines_seen,
                  int64_t* welford_n, int* initialized) {
    if (stream >= e->S) return fail(e, ERX_ERR_CONFIG, "stream index out of range");
    if (lines_seen) *lines_seen = e->lines_seen;
    if (welford_n) *welford_n = e->welford_n;
    if (initialized) *initialized = e->initialized ? 1 : 0;
    if (!e->initialized || (!mu && !cov)) return ERX_OK;
    const int D = e->D, SE = D + D * (D + 1) / 2;
    std::vector<double> h(SE);
    if (!e->failed)
        if (int st = drain_pending(e)) return st;
    CU(cudaStreamSynchronize(e->stream));
    CU(cudaMemcpy(h.data(), e->d_state[e->cur] + size_t(stream) * SE, SE * sizeof(double), cudaMemcpyDeviceToHost));
    if (mu) std::memcpy(mu, h.data(), D * sizeof(double));
    if (cov)
        for (int i = 0; i < D; ++i)
            for (int j = 0; j <= i; ++j) {
                const double v = h[D + erxk::tri(i, j)];
                cov[size_t(i) * D + j] = v;
                cov[size_t(j) * D + i] = v;
            }
    return ERX_OK;
}

int erx_get_weights(const erx_engine* e, double* w) {
    if (e->cfg.no_srp) return ERX_ERR_CONFIG;
    std::memcpy(w, e->W.data(), e->W.size() * sizeof(double));
    return ERX_OK;
}

int erx_set_state(erx_engine* e, uint32_t stream, const double* mu, const double* cov, int64_t lines_seen,
                  int64_t welford_n) {
    if (stream >= e->S) return fail(e, ERX_ERR_CONFIG, "stream index out of range");
    const int D = e->D, SE = D + D * (D + 1) / 2;
    std::vector<double> h(SE);
    std::memcpy(h.data(), mu, D * sizeof(double));
    for (int i = 0; i < D; ++i)
        for (int j = 0; j <= i; ++j) h[D + erxk::tri(i, j)] = cov[size_t(i) * D + j];
    if (int st = drain_pending(e)) return st;
    CU(cudaStreamSynchronize(e->stream));
    CU(cudaMemcpy(e->d_state[e->cur] + size_t(stream) * SE, h.data(), SE * sizeof(double), cudaMemcpyHostToDevice));
    e->initialized = true;
    e->lines_seen = lines_seen;
    e->welford_n = welford_n;
    const erxk::WinMeta m{lines_seen, welford_n, 1, e->cur};
    CU(cudaMemcpy(e->d_meta, &m, sizeof(m), cudaMemcpyHostToDevice));
    return ERX_OK;
}

uint64_t erx_launch_count(const erx_engine* e) { return e->launches; }

int64_t erx_rescued_lines(erx_engine* e) {
    if (!e->failed) drain_pending(e);
    return e->rescued_before + read_rescued(e);
}

int erx_set_option(erx_engine* e, int option, int64_t value) {
    if (!e->graphs.empty()) {  // captured windows bake in the current options
        cudaStreamSynchronize(e->stream);
        for (auto& ge : e->graphs) cudaGraphExecDestroy(ge.exec);
        e->graphs.clear();
    }
    if (option == ERX_OPT_ASYNC_HOST) {
        if (value != 0 && value != 1) return fail(e, ERX_ERR_CONFIG, "async host: 0 or 1");
        if (!value)
            if (int st = drain_pending(e)) return st;
        e->async_host = value != 0;
        return ERX_OK;
    }
    if (option == ERX_OPT_FACTOR_THREADS) {
        if (value != 0 && value != 64 && value != 128 && value != 256 && value != 512)
            return fail(e, ERX_ERR_CONFIG, "factor threads: 0, 64, 128, 256 or 512");
        e->factor_threads = int(value);
        return ERX_OK;
    }
    if (option == ERX_OPT_STATS_SPLIT) {
        if (value < 0 || value > 3) return fail(e, ERX_ERR_CONFIG, "stats split: 0..3");
        e->stats_split = int(value);
        return ERX_OK;
    }
    if (option == ERX_OPT_STATS_ONEPASS) {
        if (value != 0 && value != 2 && value != 4 && value != 8 && value != 16 && value != 32)
            return fail(e, ERX_ERR_CONFIG, "stats one-pass headroom: 0, 2, 4, 8, 16 or 32");
        e->stats_onepass = int(value);
        return ERX_OK;
    }
    if (option == ERX_OPT_DEVICE_GROUPS) {
        if (value < 0 || value > erx_engine::kDevGroups) return fail(e, ERX_ERR_CONFIG, "device groups: 0, 1 or 2");
        e->dev_groups = int(value);
        return ERX_OK;
    }
    if (option == ERX_OPT_GRAPHS) {
        if (value != 0 && value != 1) return fail(e, ERX_ERR_CONFIG, "graphs: 0 or 1");
        e->use_graphs = value != 0;
        return ERX_OK;
    }
    if (option == ERX_OPT_HOST_GROUPS) {
        if (value < 0 || value > erx_engine::kMaxGroups) return fail(e, ERX_ERR_CONFIG, "host groups: 0..8");
        e->host_groups = int(value);
        return ERX_OK;
    }
    if (option == ERX_OPT_STATS_TENSOR) {
        if (value != 0 && value != 2) return fail(e, ERX_ERR_CONFIG, "stats tensor: 0 or 2");
        if (int st = run_staged_window(e)) return st;  // staged lines are scored with the old plan
        if (int st = drain_pending(e)) return st;
        e->stats_tensor = int(value);
        if (e->d_stats) {
            const uint32_t P = e->P;
            e->P = 0;  // re-plan (the tensor path changes the whitening operand's format)
            return configure(e, P);
        }
        return ERX_OK;
    }
    if (option == ERX_OPT_FACTOR_PRECISION) {
        if (value != 0 && value != 1 && value != 30 && value != 31 && value != 32 && value != 64)
            return fail(e, ERX_ERR_CONFIG, "factor precision: 0, 1, 30, 31, 32 or 64");
        if (int st = run_staged_window(e)) return st;
        if (int st = drain_pending(e)) return st;
        e->factor_req = int(value);
        if (e->d_stats) {
            const uint32_t P = e->P;
            e->P = 0;  // force a re-plan with the new precision
            return configure(e, P);
        }
        return ERX_OK;
    }
    return fail(e, ERX_ERR_CONFIG, "unknown option");
}

int64_t erx_get_option(const erx_engine* e, int option) {
    if (option == ERX_OPT_FACTOR_PRECISION) return e->d_stats ? e->factor_prec : e->factor_req;
    if (option == ERX_OPT_HOST_GROUPS) return e->host_groups;
    if (option == ERX_OPT_GRAPHS) return e->use_graphs ? 1 : 0;
    if (option == ERX_OPT_DEVICE_GROUPS) return e->dev_groups;
    if (option == ERX_OPT_STATS_SPLIT) return e->stats_split;
    if (option == ERX_OPT_STATS_ONEPASS) return e->stats_onepass;
    if (option == ERX_OPT_STATS_REDONE) return const_cast<erx_engine*>(e)->redone_before + read_redone(const_cast<erx_engine*>(e));
    if (option == ERX_OPT_FACTOR_THREADS) return e->factor_threads;
    if (option == ERX_OPT_ASYNC_HOST) return e->async_host ? 1 : 0;
    if (option == ERX_OPT_STATS_TENSOR) {
        if (!e->d_stats) return e->stats_tensor;
        if (e->tensor || e->wide_i8) return 2;
        return 0;
    }
    return -1;
}

int erx_set_profiling(erx_engine* e, int on) {
    collect_timings(e);
    e->profiling = on != 0;
    for (int k = 0; k < ERX_NUM_KERNELS; ++k) {
        e->kms[k] = 0;
        e->kcount[k] = 0;
    }
    return ERX_OK;
}

int erx_kernel_times(erx_engine* e, double* ms, uint64_t* launches) {
    collect_timings(e);
    for (int k = 0; k < ERX_NUM_KERNELS; ++k) {
        if (ms) ms[k] = e->kms[k];
        if (launches) launches[k] = e->kcount[k];
    }
    return ERX_OK;
}

int erx_event_record(erx_engine* e, int slot) {
    if (slot < 0 || slot >= 8) return ERX_ERR_CONFIG;
    CU(cudaEventRecord(e->user_ev[slot], e->stream));
    return ERX_OK;
}

int erx_event_elapsed_ms(erx_engine* e, int a, int b, float* ms) {
    if (a < 0 || a >= 8 || b < 0 || b >= 8) return ERX_ERR_CONFIG;
    CU(cudaEventSynchronize(e->user_ev[b]));
    CU(cudaEventElapsedTime(ms, e->user_ev[a], e->user_ev[b]));
    return ERX_OK;
}

void* erx_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}
void erx_host_free(void* p) { cudaFreeHost(p); }
void* erx_device_alloc(int device, size_t bytes) {
    void* p = nullptr;
    cudaSetDevice(device);
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}
void erx_device_free(void* p) { cudaFree(p); }

int erx_copy(void* dst, const void* src, size_t bytes, int kind, erx_engine* e) {
    cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice : kind == 2 ? cudaMemcpyDeviceToHost
                                                                     : cudaMemcpyDeviceToDevice;
    if (e) {
        CU(cudaMemcpyAsync(dst, src, bytes, k, e->stream));
    } else {
        CU(cudaMemcpy(dst, src, bytes, k));
    }
    return ERX_OK;
}

}  // extern "C"
