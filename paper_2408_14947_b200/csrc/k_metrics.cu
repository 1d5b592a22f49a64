// k_metrics.cu — the parity-gate metrics on the device:
// exact ROC AUC with tied scores grouped (metrics.hpp:25-28 roc_curve /
// evaluate_run :54-58) and the top-k anomaly set
// over pooled scores, so a c3 evaluation (≈200 M non-warmup scores) does not
// need a host sort.
//
// Both reduce to one stable LSD radix sort of 32-bit keys with a 32-bit
// payload (4 passes of 8 bits): keys are the fp32 scores mapped to unsigned
// order (negative: ~bits, else bits | sign), so equal scores are equal keys.
// Per pass: (1) per-tile digit histograms, (2) one exclusive scan of the
// digit-major [256][tiles] counts, (3) a scatter in which each tile ranks its
// elements stably (warp match + per-warp digit counts, rounds in element
// order).
//
// AUC (Mann-Whitney form of the trapezoid over the tie-grouped ROC):
//   2 npos nneg AUC = sum over tie groups g of pos_g (2 negbelow_g + neg_g)
// computed in exact integers from the ascending sort (label payload): the
// negative prefix count C at each group head and at the next head gives
// negbelow_g = C[h_g] and neg_g = C[h_{g+1}] - C[h_g], pos_g likewise.
// The top-k set sorts descending (key complement) with the element index as
// payload; ties at the cutoff resolve to the lower index (stable sort).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <utility>

#include "erx_common.cuh"
#include "../../include/erx_b200.h"

namespace erxk {
namespace {

constexpr int kSortThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kSortThreads * kItems;  // 2048 elements per tile
constexpr int kScanBlock = 1024;

__device__ __forceinline__ uint32_t key_of(float f) {
    const uint32_t b = f == 0.f ? 0u : __float_as_uint(f);  // -0 ties with +0, as in the oracle's ==

    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// ---------------------------------------------------------------- exclusive scan (u32, in place ok)
__global__ void __launch_bounds__(kScanBlock) scan_block_kernel(const uint32_t* __restrict__ in,
                                                                uint32_t* __restrict__ out, size_t n,
                                                                uint32_t* __restrict__ block_sums) {
    __shared__ uint32_t ws[32];
    const size_t i = size_t(blockIdx.x) * kScanBlock + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t v = i < n ? in[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = ws[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        ws[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const uint32_t excl = x - v + (warp ? ws[warp - 1] : 0u);
    if (i < n) out[i] = excl;
    if (threadIdx.x == kScanBlock - 1 && block_sums) block_sums[blockIdx.x] = ws[31];
}

__global__ void scan_add_kernel(uint32_t* __restrict__ out, size_t n, const uint32_t* __restrict__ block_off) {
    const size_t i = size_t(blockIdx.x) * kScanBlock + threadIdx.x;
    if (i < n && blockIdx.x) out[i] += block_off[blockIdx.x];
}

// exclusive scan of n u32 (wrap-around arithmetic); tmp: scan_tmp_words(n) words
size_t scan_tmp_words(size_t n) {
    size_t w = 0;
    while (n > kScanBlock) {
        n = (n + kScanBlock - 1) / kScanBlock;
        w += n;
    }
    return w + 1;
}

void scan_exclusive(const uint32_t* in, uint32_t* out, size_t n, uint32_t* tmp, cudaStream_t st) {
    if (n == 0) return;
    const size_t nb = (n + kScanBlock - 1) / kScanBlock;
    if (nb == 1) {
        scan_block_kernel<<<1, kScanBlock, 0, st>>>(in, out, n, nullptr);
        return;
    }
    uint32_t* sums = tmp;
    scan_block_kernel<<<unsigned(nb), kScanBlock, 0, st>>>(in, out, n, sums);
    scan_exclusive(sums, sums, nb, tmp + nb, st);
    scan_add_kernel<<<unsigned(nb), kScanBlock, 0, st>>>(out, n, sums);
}

// ---------------------------------------------------------------- radix sort passes
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const uint32_t* __restrict__ keys, size_t n,
                                                                  int shift, uint32_t* __restrict__ counts,
                                                                  int ntiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0u;
    __syncthreads();
    const size_t base = size_t(blockIdx.x) * kTile;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const size_t e = base + size_t(it) * kSortThreads + threadIdx.x;
        if (e < n) atomicAdd(&h[(keys[e] >> shift) & 255u], 1u);
    }
    __syncthreads();
    counts[size_t(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(const uint32_t* __restrict__ keys,
                                                                     const uint32_t* __restrict__ vals, size_t n,
                                                                     int shift, const uint32_t* __restrict__ offs,
                                                                     int ntiles, uint32_t* __restrict__ keys_out,
                                                                     uint32_t* __restrict__ vals_out) {
    constexpr int kWarps = kSortThreads / 32;
    __shared__ uint32_t cnt[kWarps][256];
    __shared__ uint32_t run[256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    run[tid] = offs[size_t(tid) * ntiles + blockIdx.x];
    const size_t base = size_t(blockIdx.x) * kTile;
    for (int it = 0; it < kItems; ++it) {  // rounds in element order: stable
        const size_t e = base + size_t(it) * kSortThreads + tid;
        const bool ok = e < n;
        const uint32_t k = ok ? keys[e] : 0u;
        const uint32_t v = ok ? vals[e] : 0u;
        const uint32_t d = ok ? ((k >> shift) & 255u) : 256u + lane;  // out-of-range lanes match nobody
        for (int q = tid; q < kWarps * 256; q += kSortThreads) (&cnt[0][0])[q] = 0u;
        __syncthreads();
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & lt);
        if (ok && rank == 0) cnt[warp][d] = __popc(peers);
        __syncthreads();
        {   // thread = digit: exclusive prefix over warps, carried across rounds
            uint32_t r = run[tid];
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t t = cnt[w][tid];
                cnt[w][tid] = r;
                r += t;
            }
            run[tid] = r;
        }
        __syncthreads();
        if (ok) {
            const uint32_t pos = cnt[warp][d] + rank;
            keys_out[pos] = k;
            vals_out[pos] = v;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- element kernels
// keys = order-mapped scores (complemented when descending), vals = label or index; compaction by
// select (nullable) with positions from an exclusive scan of the flags
__global__ void select_flags_kernel(const uint8_t* __restrict__ sel, size_t n, uint32_t* __restrict__ flags) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = sel[i] ? 1u : 0u;
}

__global__ void gather_kernel(const float* __restrict__ scores, const uint8_t* __restrict__ labels,
                              const uint8_t* __restrict__ sel, const uint32_t* __restrict__ pos, size_t n,
                              bool descending, bool label_payload, uint32_t* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (sel && !sel[i]) return;
    const size_t o = sel ? pos[i] : i;
    const uint32_t k = key_of(scores[i]);
    keys[o] = descending ? ~k : k;
    vals[o] = label_payload ? (labels[i] ? 1u : 0u) : uint32_t(i);
}

__global__ void neg_flags_kernel(const uint32_t* __restrict__ lab, size_t n, uint32_t* __restrict__ f) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) f[i] = lab[i] ? 0u : 1u;
}

__global__ void head_flags_kernel(const uint32_t* __restrict__ keys, size_t n, uint32_t* __restrict__ f) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) f[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void head_list_kernel(const uint32_t* __restrict__ keys, size_t n, const uint32_t* __restrict__ hpos,
                                 uint32_t* __restrict__ heads) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && (i == 0 || keys[i] != keys[i - 1])) heads[hpos[i]] = uint32_t(i);
}

// one thread per tie group: pos_g (2 C[h_g] + neg_g), exact u64, block-reduced then atomically added
__global__ void __launch_bounds__(256) auc_groups_kernel(const uint32_t* __restrict__ heads, size_t ngroups,
                                                         const uint32_t* __restrict__ C, size_t n, uint32_t nneg,
                                                         unsigned long long* __restrict__ total) {
    __shared__ unsigned long long red[8];
    const size_t g = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long v = 0ull;
    if (g < ngroups) {
        const uint32_t h0 = heads[g];
        const uint32_t h1 = g + 1 < ngroups ? heads[g + 1] : uint32_t(n);
        const uint32_t c0 = C[h0];
        const uint32_t c1 = g + 1 < ngroups ? C[h1] : nneg;
        const uint32_t neg = c1 - c0, pos = (h1 - h0) - neg;
        v = (unsigned long long)pos * (2ull * c0 + neg);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0ull;
        for (int w = 0; w < 8; ++w) s += red[w];
        atomicAdd(total, s);
    }
}

__global__ void topk_mark_kernel(const uint32_t* __restrict__ idx, size_t k, uint8_t* __restrict__ mask) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < k) mask[idx[i]] = 1u;
}

inline unsigned blocks_for(size_t n, int t) { return unsigned((n + t - 1) / t); }

// Workspace: keys/vals double-buffered (4 n words), scan flags/positions (2 n words), radix counts
// (256 x tiles words) and scan temporaries.
// The device buffer is cached per process (grow-only, one per device; calls serialise on a mutex)
// so repeated evaluations do not pay cudaMalloc / cudaFree.
struct WsCache {
    std::mutex mu;
    void* base[64] = {};
    size_t bytes[64] = {};
};
WsCache& ws_cache() {
    static WsCache c;
    return c;
}

struct Ws {
    uint32_t *k0, *v0, *k1, *v1, *f, *p, *cnt, *tmp;
    unsigned long long* acc;
    void* base = nullptr;
    int ntiles = 0;
    std::unique_lock<std::mutex> lock{ws_cache().mu};
    cudaStream_t st = nullptr;
    explicit Ws(cudaStream_t s) : st(s) {}
    ~Ws() { cudaStreamSynchronize(st); }  // no work may still use the cached buffer on return
    bool alloc(size_t n) {
        ntiles = int((n + kTile - 1) / kTile);
        const size_t ncnt = size_t(256) * ntiles;
        const size_t words = 4 + 6 * n + ncnt + scan_tmp_words(std::max(n, ncnt));
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
        WsCache& c = ws_cache();
        if (c.bytes[dev] < words * 4) {
            if (c.base[dev]) cudaFree(c.base[dev]);
            c.base[dev] = nullptr;
            c.bytes[dev] = 0;
            if (cudaMalloc(&c.base[dev], words * 4) != cudaSuccess) return false;
            c.bytes[dev] = words * 4;
        }
        base = c.base[dev];
        acc = static_cast<unsigned long long*>(base);
        uint32_t* w = static_cast<uint32_t*>(base) + 4;
        k0 = w; v0 = k0 + n; k1 = v0 + n; v1 = k1 + n; f = v1 + n; p = f + n; cnt = p + n; tmp = cnt + ncnt;
        return true;
    }
};

// sort (k0, v0) of n elements ascending, result in (k0, v0)
void radix_sort(Ws& w, size_t n, cudaStream_t st) {
    for (int shift = 0; shift < 32; shift += 8) {
        radix_hist_kernel<<<unsigned(w.ntiles), kSortThreads, 0, st>>>(w.k0, n, shift, w.cnt, w.ntiles);
        scan_exclusive(w.cnt, w.cnt, size_t(256) * w.ntiles, w.tmp, st);
        radix_scatter_kernel<<<unsigned(w.ntiles), kSortThreads, 0, st>>>(w.k0, w.v0, n, shift, w.cnt, w.ntiles,
                                                                           w.k1, w.v1);
        std::swap(w.k0, w.k1);
        std::swap(w.v0, w.v1);
    }
}

// gather the selected elements into (k0, v0); returns the selected count
size_t gather(Ws& w, const float* scores, const uint8_t* labels, const uint8_t* sel, size_t n, bool descending,
              bool label_payload, cudaStream_t st) {
    size_t m = n;
    if (sel) {
        select_flags_kernel<<<blocks_for(n, 256), 256, 0, st>>>(sel, n, w.f);
        scan_exclusive(w.f, w.p, n, w.tmp, st);
        uint32_t last_pos = 0, last_flag = 0;
        cudaMemcpyAsync(&last_pos, w.p + n - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&last_flag, w.f + n - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        m = size_t(last_pos) + last_flag;
    }
    gather_kernel<<<blocks_for(n, 256), 256, 0, st>>>(scores, labels, sel, w.p, n, descending, label_payload, w.k0,
                                                      w.v0);
    return m;
}

}  // namespace
}  // namespace erxk

using namespace erxk;

extern "C" {

int erx_metrics_roc_auc(const float* d_scores, const uint8_t* d_labels, const uint8_t* d_select, size_t n,
                        void* stream, double* auc, uint64_t* npos_out, uint64_t* nneg_out) {
    if (!auc || (n && (!d_scores || !d_labels)) || n >= (size_t(1) << 32)) return ERX_ERR_CONFIG;
    *auc = 0.0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n == 0) return ERX_ERR_METRIC;
    Ws w(st);
    if (!w.alloc(n)) return ERX_ERR_DEVICE;
    const size_t m = gather(w, d_scores, d_labels, d_select, n, false, true, st);
    if (m == 0) return ERX_ERR_METRIC;
    w.ntiles = int((m + kTile - 1) / kTile);
    radix_sort(w, m, st);
    // negative prefix counts, tie-group heads
    neg_flags_kernel<<<blocks_for(m, 256), 256, 0, st>>>(w.v0, m, w.f);
    scan_exclusive(w.f, w.p, m, w.tmp, st);  // p = C
    uint32_t cl = 0, fl = 0;
    cudaMemcpyAsync(&cl, w.p + m - 1, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&fl, w.f + m - 1, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return ERX_ERR_DEVICE;
    const uint32_t nneg = cl + fl, npos = uint32_t(m) - nneg;
    if (npos_out) *npos_out = npos;
    if (nneg_out) *nneg_out = nneg;
    if (npos == 0 || nneg == 0) return ERX_ERR_METRIC;  // roc_curve needs both classes (MetricUndefinedError)
    head_flags_kernel<<<blocks_for(m, 256), 256, 0, st>>>(w.k0, m, w.f);
    scan_exclusive(w.f, w.v1, m, w.tmp, st);  // v1 = head positions
    uint32_t hl = 0, hf = 0;
    cudaMemcpyAsync(&hl, w.v1 + m - 1, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&hf, w.f + m - 1, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return ERX_ERR_DEVICE;
    const size_t ngroups = size_t(hl) + hf;
    head_list_kernel<<<blocks_for(m, 256), 256, 0, st>>>(w.k0, m, w.v1, w.k1);  // k1 = heads
    unsigned long long* total = w.acc;
    cudaMemsetAsync(total, 0, 8, st);
    auc_groups_kernel<<<blocks_for(ngroups, 256), 256, 0, st>>>(w.k1, ngroups, w.p, m, nneg, total);
    unsigned long long tot = 0;
    cudaMemcpyAsync(&tot, total, 8, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) return ERX_ERR_DEVICE;
    *auc = double(tot) / (2.0 * double(npos) * double(nneg));
    return ERX_OK;
}

int erx_metrics_top_k(const float* d_scores, const uint8_t* d_select, size_t n, size_t k, void* stream,
                      uint8_t* d_mask, float* cutoff) {
    if ((n && (!d_scores || !d_mask)) || n >= (size_t(1) << 32)) return ERX_ERR_CONFIG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n == 0) return k == 0 ? ERX_OK : ERX_ERR_DATA;
    if (cudaMemsetAsync(d_mask, 0, n, st) != cudaSuccess) return ERX_ERR_DEVICE;
    Ws w(st);
    if (!w.alloc(n)) return ERX_ERR_DEVICE;
    const size_t m = gather(w, d_scores, nullptr, d_select, n, true, false, st);
    if (k > m) return ERX_ERR_DATA;
    if (k == 0) return cudaStreamSynchronize(st) == cudaSuccess ? ERX_OK : ERX_ERR_DEVICE;
    w.ntiles = int((m + kTile - 1) / kTile);
    radix_sort(w, m, st);
    topk_mark_kernel<<<blocks_for(k, 256), 256, 0, st>>>(w.v0, k, d_mask);
    uint32_t ck = 0;
    cudaMemcpyAsync(&ck, w.k0 + k - 1, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) return ERX_ERR_DEVICE;
    if (cutoff) {
        const uint32_t key = ~ck;
        const uint32_t b = (key & 0x80000000u) ? (key & 0x7fffffffu) : ~key;
        std::memcpy(cutoff, &b, 4);
    }
    return ERX_OK;
}

}  // extern "C"
