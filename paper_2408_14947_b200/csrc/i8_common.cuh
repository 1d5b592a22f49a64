// i8_common.cuh — shared pieces of the exact-integer tensor-core path
// (k_stats_i8.cu, k_factor.cu plane writer, k_score_i8.cu).
//
// A value v with |v s| <= R < 2^22 is rounded ONCE to q = rint(v s) by
// fma(v, s, 1.5 * 2^23) (the integer lands in the low mantissa bits), and
// u = q + 0x808080 holds three balanced signed int8 digits
// (q = d0 + 2^8 d1 + 2^16 d2, digit i = byte i of u minus 128).
#pragma once

#include "tc_common.cuh"

namespace erxk {
namespace i8 {

constexpr float kR = 4194000.f;      // quantisation range, < 2^22
constexpr float kMagic = 12582912.f;  // 1.5 * 2^23

// W planes as the score kernel's MMA B operand (K-major): 3 digit planes x 4 K-slices x 128 rows
// x 32 B, then 128 fp32 row factors 256 / r_i and 128 fp32 offsets (W (mu - c))_i.  One line's
// block is copied to shared memory as is.
constexpr uint32_t kWPlane = 4 * tc::kSliceBytes;  // 16 KB
constexpr uint32_t kWAux = 2 * 128 * 4;
constexpr uint32_t kWBytes = 3 * kWPlane + kWAux;

// v planes as the score kernel's MMA A operand, MN-major (M = 128 pixels of a tile, K = 128 dims):
// per digit plane, K-step s (32 dims) at s * 4096, 8-dim group kg at kg * 1024 (descriptor LBO),
// 16-pixel group mg at mg * 128 (SBO), dim row d % 8 at 16 B, pixel % 16 the byte.  Dims are
// the slow index inside a K-step, so the dims a line never uses (>= 16 * ceil((D + 1) / 16)) form one
// contiguous tail of each plane that is neither written nor read (vplane_used_bytes).
constexpr uint32_t kVPlane = 16384;
constexpr uint32_t kTileBytes = 3 * kVPlane;  // one 128-pixel tile
constexpr uint32_t kVLbo = 1024, kVSbo = 128;
__host__ __device__ constexpr uint32_t vplane_off(int plane, int d, int p) {  // p: pixel within the tile (16-aligned)
    return uint32_t(plane) * kVPlane + uint32_t(d >> 5) * 4096u + uint32_t((d & 31) >> 3) * kVLbo +
           uint32_t(p >> 4) * kVSbo + uint32_t(d & 7) * 16u + uint32_t(p & 15);
}
// leading bytes of each plane that hold dims 0 .. D (the ones row included), in 16-dim units
__host__ __device__ constexpr uint32_t vplane_used_bytes(int D) {
    return ((D + 1 + 15) / 16) * 2048u < kVPlane ? ((D + 1 + 15) / 16) * 2048u : kVPlane;
}
__host__ __device__ constexpr int vplane_used_dims(int D) { return int(vplane_used_bytes(D) / 2048u) * 16; }

// The stats kernel's per-dim v scale, recomputed bit-identically by the factor's plane writer.
__device__ __forceinline__ float v_scale(float vmax) {
    return (vmax > 0.f && vmax <= 3.402823466e38f) ? kR / vmax : 0.f;
}

__device__ __forceinline__ uint32_t quant_u(float v, float k) {  // q + 0x808080, q = rint(v k)
    return __float_as_uint(fmaf(v, k, kMagic)) + (0x808080u - 0x4B400000u);
}

__device__ __forceinline__ void pack_digits(const uint32_t (&u)[4], uint32_t& w0, uint32_t& w1, uint32_t& w2) {
    const uint32_t t01 = __byte_perm(u[0], u[1], 0x5140), t23 = __byte_perm(u[2], u[3], 0x5140);
    w0 = __byte_perm(t01, t23, 0x5410) ^ 0x80808080u;
    w1 = __byte_perm(t01, t23, 0x7632) ^ 0x80808080u;
    const uint32_t r01 = __byte_perm(u[0], u[1], 0x0062), r23 = __byte_perm(u[2], u[3], 0x0062);
    w2 = __byte_perm(r01, r23, 0x5410) ^ 0x80808080u;
}

// Per-dim constants of the score's y = (x - c) - (mu - c): centre c, offset dc = fl32(mu - c) and
// scale s = R / bound, bound = (max_p |x - c| + |dc|)(1 + 2^-20) (0 when the dim has no range).
// Computed identically by the factor's plane writer (W' = W / s) and by the score kernel.
struct YScale {
    float c, dc, s;
};
__device__ __forceinline__ YScale y_scale(const double* stats_line, const double* prior_line, const float* vmax_line,
                                          int d) {
    YScale r;
    r.c = float(stats_line[d]);
    r.dc = float(prior_line[d] - stats_line[d]);
    const float bound = (vmax_line[d] + fabsf(r.dc)) * (1.f + 9.5367431640625e-07f);
    r.s = (bound > 0.f && bound <= 3.402823466e38f) ? kR / bound : 0.f;
    return r;
}

}  // namespace i8
}  // namespace erxk
