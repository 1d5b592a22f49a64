// k_datagen.cu — the synthetic line-scan generator (include/erx_datagen.h,
// datagen.cpp) on the device, so a full c3 run (88 GB of
// input) needs no host generation or H2D traffic.
//
// Same laws and the same random streams as the host generator: line t draws
// from had::Rng(mix_seed(seed, t + 1)) (rng.hpp:18-83; mt19937_64, uniform =
// (u64 >> 11) 2^-53, Box-Muller normals cos-then-sin), per pixel r factor
// normals then b noise normals, x = fl32(base(t) + e + sum_k A_bk z_k) in the
// host's fp64 operation order (explicit _rn ops: no FMA contraction), then the
// anomaly overrides in anomaly order.  The stream-level draws (spectra, A,
// scene changes, anomaly placement) are the host's (datagen.cpp gen_plan).
//
// One kernel, one warp per line: the mt19937_64 state and a ring of the
// line's normals sit in shared memory; each 312-word refill runs as two
// lane-parallel halves (words 0..155 read only old words, 156..311 read the
// new words 0..155), its 156 Box-Muller pairs go to the ring, and every pixel
// whose r + b normals are complete is emitted (lanes over bands) before the
// next refill.  No scratch in HBM: the kernel writes only x and the mask.
// Exactness: everything is bit-identical to the host except log / sin / cos,
// whose CUDA and glibc results can differ in the last fp64 place; after the
// fp32 rounding of x that shows up in a vanishing fraction of values, by at
// most one fp32 ulp (tests/test_gpu_datagen.py measures it).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/erx_b200.h"
#include "../../include/erx_datagen.h"
#include "datagen_plan.hpp"
#include "erx_common.cuh"
#include "host_rng.hpp"

namespace erxk {
namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull, kMatA = 0xB5026F5AA96619E9ull;

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

__device__ __forceinline__ uint64_t mix_seed_d(uint64_t seed, uint64_t n) {
    uint64_t x = seed ^ (0x9e3779b97f4a7c15ull + n * 0xbf58476d1ce4e5b9ull);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

struct GenDev {
    const double* base;
    const double* drift;
    const double* A;
    const int64_t* changes;
    int n_changes;
    const uint32_t* hit_off;
    const uint32_t* hit_pix;
    const uint32_t* hit_anom;
    const double* spec;
    const double* f;
    int kind;
    double drift_amp, noise_sd;
    uint32_t lines, P, B, R;
    uint32_t ring;  // normals ring per warp (power of two >= 312 + R + B)
};

constexpr int kLinesPerCta = 4;  // one warp per line

// One warp per line: refill the mt19937_64 state (two lane-parallel halves: words 0..155 read only
// old words, 156..311 read the new 0..155), turn the 312 tempered words into 156 Box-Muller pairs
// appended to a shared-memory ring of normals, and emit every pixel whose r + b normals are
// complete: lanes over bands, x = fl32(base + e + sum_k A_bk z_k) in the host's fp64 order, then
// the pixel's anomaly hits in anomaly order.
__global__ void __launch_bounds__(32 * kLinesPerCta) gen_lines_kernel(GenDev gd, uint64_t seed, uint32_t first,
                                                                      uint32_t n_lines, float* __restrict__ out,
                                                                      uint8_t* __restrict__ mask,
                                                                      int* __restrict__ flag) {
    extern __shared__ __align__(16) unsigned char gsm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t l = blockIdx.x * kLinesPerCta + w;
    if (l >= n_lines) return;
    uint64_t* x = reinterpret_cast<uint64_t*>(gsm) + size_t(w) * kN;
    double* ring = reinterpret_cast<double*>(gsm + size_t(kLinesPerCta) * kN * 8) + size_t(w) * gd.ring;
    const uint32_t rmask = gd.ring - 1;
    const uint32_t t = first + l;
    const uint32_t B = gd.B, R = gd.R, W = R + B;
    if (lane == 0) {  // mt19937_64::seed
        uint64_t v = mix_seed_d(seed, uint64_t(t) + 1);
        x[0] = v;
        for (int i = 1; i < kN; ++i) {
            v = 6364136223846793005ull * (v ^ (v >> 62)) + uint64_t(i);
            x[i] = v;
        }
    }
    __syncwarp();
    int scene = 0;
    while (scene < gd.n_changes && int64_t(t) >= gd.changes[scene]) ++scene;
    const double dt = __ddiv_rn(__dmul_rn(gd.drift_amp, double(t)), double(gd.lines > 1 ? gd.lines : 1));
    const double* base_s = gd.base + size_t(scene) * B;
    const uint32_t h0 = gd.hit_off[l], h1 = gd.hit_off[l + 1];
    float* xo = out + size_t(l) * gd.P * B;
    const uint32_t n_normals = gd.P * W;
    uint32_t produced = 0, pix = 0;
    constexpr int kPer = (kM + 31) / 32;  // 5 words per lane per half
    while (pix < gd.P) {
        uint64_t nv[kPer];
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
            const int i = lane + 32 * r;
            if (i < kM) {
                const uint64_t y = (x[i] & kUpper) | (x[i + 1] & kLower);
                nv[r] = x[i + kM] ^ (y >> 1) ^ ((y & 1ull) ? kMatA : 0ull);
            }
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < kPer; ++r)
            if (lane + 32 * r < kM) x[lane + 32 * r] = nv[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
            const int i = kM + lane + 32 * r;
            if (i < kN) {
                const uint64_t y = (x[i] & kUpper) | (x[(i + 1) % kN] & kLower);
                nv[r] = x[i - kM] ^ (y >> 1) ^ ((y & 1ull) ? kMatA : 0ull);
            }
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < kPer; ++r)
            if (kM + lane + 32 * r < kN) x[kM + lane + 32 * r] = nv[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
            const int q = lane + 32 * r;
            if (q < kM) {
                const double u1 = double(temper(x[2 * q]) >> 11) * 0x1.0p-53;
                const double u2 = double(temper(x[2 * q + 1]) >> 11) * 0x1.0p-53;
                if (!(u1 > 0.0) && produced + 2 * q < n_normals) atomicExch(flag, 1);  // host redraws u1
                const double rad = sqrt(__dmul_rn(-2.0, log(u1)));
                const double ang = __dmul_rn(6.283185307179586476925286766559, u2);
                double sn, cs;
                sincos(ang, &sn, &cs);
                ring[(produced + 2 * q) & rmask] = __dmul_rn(rad, cs);
                ring[(produced + 2 * q + 1) & rmask] = __dmul_rn(rad, sn);
            }
        }
        produced += kN;
        __syncwarp();
        // emit the pixels now complete
        for (; pix < gd.P && (pix + 1) * W <= produced; ++pix) {
            const uint32_t o = pix * W;
            bool hit = false;
            for (uint32_t b = lane; b < B; b += 32) {
                const double eb = __dmul_rn(ring[(o + R + b) & rmask], gd.noise_sd);
                double v = __dadd_rn(__dadd_rn(base_s[b], __dmul_rn(dt, gd.drift[b])), eb);
                const double* a = gd.A + size_t(b) * R;
                for (uint32_t k = 0; k < R; ++k) v = __dadd_rn(v, __dmul_rn(a[k], ring[(o + k) & rmask]));
                for (uint32_t h = h0; h < h1; ++h) {
                    if (gd.hit_pix[h] != pix) continue;
                    hit = true;
                    const uint32_t an = gd.hit_anom[h];
                    const double sp = gd.spec[size_t(an) * B + b];
                    if (gd.kind == ERX_ANOM_OFFSET) {
                        v = __dadd_rn(v, sp);
                    } else if (gd.kind == ERX_ANOM_MIXTURE) {
                        const double fa = gd.f[an];
                        v = __dadd_rn(__dmul_rn(__dsub_rn(1.0, fa), v), __dmul_rn(fa, sp));
                    } else {
                        v = __dadd_rn(sp, eb);
                    }
                }
                xo[size_t(pix) * B + b] = __double2float_rn(v);
            }
            if (mask && lane == 0) {
                if (!hit)  // B < 32 lanes: lane 0 checks the hit list itself
                    for (uint32_t h = h0; h < h1; ++h) hit |= gd.hit_pix[h] == pix;
                mask[size_t(l) * gd.P + pix] = hit ? 1 : 0;
            }
        }
        __syncwarp();  // ring slots of emitted pixels may be overwritten by the next refill
    }
}

// The plan's arrays packed into one pinned staging block and one device block (one copy)
struct Packer {
    std::vector<unsigned char> host;
    template <typename T>
    size_t add(const std::vector<T>& v) {
        const size_t off = (host.size() + 15) & ~size_t(15);
        host.resize(off + v.size() * sizeof(T));
        if (!v.empty()) std::memcpy(host.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
};

}  // namespace
}  // namespace erxk

using namespace erxk;

extern "C" int erx_gen_lines_device(const erx_gen_spec* spec, uint32_t first, uint32_t n, float* d_out,
                                    uint8_t* d_mask, void* stream) {
    if (!spec || (n && !d_out)) return ERX_ERR_CONFIG;
    if (n == 0) return ERX_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    erx_host::GenPlan pl;
    if (erx_host::gen_plan(*spec, first, n, pl)) return ERX_ERR_CONFIG;
    std::vector<void*> owned;
    auto cleanup = [&](int code) {
        cudaStreamSynchronize(st);
        for (void* p : owned) cudaFree(p);
        return code;
    };
    Packer pk;
    const size_t o_base = pk.add(pl.base), o_drift = pk.add(pl.drift), o_A = pk.add(pl.A),
                 o_ch = pk.add(pl.changes), o_hoff = pk.add(pl.hit_off), o_hpix = pk.add(pl.hit_pix),
                 o_hanom = pk.add(pl.hit_anom), o_spec = pk.add(pl.anom_spec), o_f = pk.add(pl.anom_f);
    const size_t o_flag = pk.add(std::vector<int>(4, 0));
    // device copy of the plan: cached per process and device (grow-only), calls serialise on it
    static std::mutex mu;
    static void* cache[64] = {};
    static size_t cache_bytes[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cleanup(ERX_ERR_DEVICE);
    if (cache_bytes[dev] < pk.host.size()) {
        if (cache[dev]) cudaFree(cache[dev]);
        cache[dev] = nullptr;
        cache_bytes[dev] = 0;
        if (cudaMalloc(&cache[dev], pk.host.size() * 2) != cudaSuccess) return cleanup(ERX_ERR_DEVICE);
        cache_bytes[dev] = pk.host.size() * 2;
    }
    void* dblk = cache[dev];
    if (cudaMemcpyAsync(dblk, pk.host.data(), pk.host.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
        return cleanup(ERX_ERR_DEVICE);
    auto at = [&](size_t off) { return static_cast<unsigned char*>(dblk) + off; };
    GenDev gd{};
    gd.base = reinterpret_cast<const double*>(at(o_base));
    gd.drift = reinterpret_cast<const double*>(at(o_drift));
    gd.A = reinterpret_cast<const double*>(at(o_A));
    gd.changes = reinterpret_cast<const int64_t*>(at(o_ch));
    gd.n_changes = int(pl.changes.size());
    gd.hit_off = reinterpret_cast<const uint32_t*>(at(o_hoff));
    gd.hit_pix = reinterpret_cast<const uint32_t*>(at(o_hpix));
    gd.hit_anom = reinterpret_cast<const uint32_t*>(at(o_hanom));
    gd.spec = reinterpret_cast<const double*>(at(o_spec));
    gd.f = reinterpret_cast<const double*>(at(o_f));
    int* flag = reinterpret_cast<int*>(at(o_flag));
    gd.kind = spec->anomaly_kind;
    gd.drift_amp = spec->drift;
    gd.noise_sd = spec->noise_sd;
    gd.lines = spec->lines;
    gd.P = pl.P;
    gd.B = pl.B;
    gd.R = pl.R;
    if (uint64_t(pl.P) * (pl.R + pl.B) >= (uint64_t(1) << 31)) return cleanup(ERX_ERR_CONFIG);
    uint32_t ring = 512;
    while (ring < uint32_t(kN) + pl.R + pl.B) ring *= 2;
    gd.ring = ring;
    const size_t smem = size_t(kLinesPerCta) * (size_t(kN) * 8 + size_t(ring) * 8);
    if (smem > 200 * 1024) return cleanup(ERX_ERR_CONFIG);  // bands beyond ~6000
    ensure_smem(gen_lines_kernel, smem);
    gen_lines_kernel<<<(n + kLinesPerCta - 1) / kLinesPerCta, 32 * kLinesPerCta, smem, st>>>(gd, spec->seed, first, n,
                                                                                             d_out, d_mask, flag);
    int h_flag = 0;
    cudaMemcpyAsync(&h_flag, flag, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) return cleanup(ERX_ERR_DEVICE);
    return cleanup(h_flag ? ERX_ERR_DATA : ERX_OK);
}
