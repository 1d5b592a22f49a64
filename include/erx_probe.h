/*
 * erx_probe.h — design probes and tensor-core self-tests (liberx_probe.so).
 *
 * Not part of the ERX path: these measure the device the path runs on (the
 * FFMA peak that bench.py reports FFMA-bound kernels against, streaming
 * bandwidth of the global->shared copy paths) and check the tcgen05
 * descriptor layouts the exact-integer kernels rely on.  Kept out of
 * liberx_b200.so so the product library carries only the path.
 *
 * device: CUDA ordinal; stream: a cudaStream_t (NULL = legacy default).
 * Returns 0, 2 on bad arguments, 16 on a CUDA error.
 */
#ifndef ERX_PROBE_H
#define ERX_PROBE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FP32 FFMA throughput (TFLOP/s, best of 5): reg_form = register-tile outer
 * products (the FFMA kernels' instruction shape), const_form = FFMA with
 * constant-bank operands (highest issue rate).  Either may be NULL. */
int erx_probe_fp32_tflops(int device, void* stream, double* reg_form, double* const_form);
/* Same for the paired fma.rn.f32x2 (FFMA2) instruction. */
int erx_probe_ffma2_tflops(int device, void* stream, double* tflops);
/* Streaming global->shared throughput, GB/s: mode 0 cp.async.bulk ring (one
 * issuing thread), 1 LDG.128 by 256 threads, 2 cp.async by 256 threads;
 * chunk_bytes per stage (multiple of 1 KB), 1..8 stages, ctas_per_sm
 * persistent CTAs. */
int erx_probe_stream(int device, void* stream, int mode, uint32_t chunk_bytes, int stages, int ctas_per_sm,
                     uint64_t bytes, double* gbs);
/* tcgen05 kind::f16 self-test on device buffers: D[128][128] = A[128][K] . B[128][K]^T
 * from bf16 operands (split = 0) or the 3-way bf16 split with 6 products
 * (split = 1).  K a multiple of 16, <= 256. */
int erx_tc_selftest(int device, void* stream, const float* dA, const float* dB, int K, int split, float* dD);
/* kind::i8 check (exact s32): D[128][N] = A[128][K] B[N][K]^T with A staged K-major or MN-major
 * (a_mn; layout strides ms / ks between 16-row M groups / 8-row K groups, descriptor lbo / sbo). */
int erx_tc_selftest_i8(int device, void* stream, const int8_t* dA, const int8_t* dB, int K, int N, int a_mn,
                       int ms, int ks, int lbo, int sbo, int* dD);

#ifdef __cplusplus
}
#endif

#endif
