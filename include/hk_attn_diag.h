/* hk_attn_diag.h — diagnostic entry points of libhkattn_diag.so (not the hot path; kept
 * out of libhkattn.so, whose C ABI allocates nothing).
 *
 * hk_diag_last_error: thread-local text of this library's last non-OK status.
 *
 * hk_diag_umma: one 128 x N output tile through tcgen05, to pin the
 * UMMA instruction/shared-memory descriptor encodings the attention kernels
 * rely on, in isolation.
 *   A : device bf16 [128][K] row-major.
 *   B : device bf16; b_mn == 0: [N][K] row-major and D = A * B^T (B K-major);
 *                    b_mn != 0: [K][N] row-major and D = A * B   (B MN-major).
 *   D : device fp32 [128][N] row-major, overwritten.
 *   a_tmem != 0 stages A in tensor memory (the P*V / dS*K operand form),
 *   otherwise A is read from shared memory (K-major).
 * Supported: N in {64, 128}, K in {64, 128}. Same error conventions as hk_attn.h.
 *
 * hk_diag_bwd_phase: exactly the work of hk_attn_bwd (same arguments, same
 * validation) but enqueues only one of its three kernels, so a profiler or
 * bench can time each on the stream in isolation:
 *   phase 0 = D-preprocess (writes the workspace), 1 = dK/dV pass, 2 = dQ pass.
 * Phases 1 and 2 read the workspace written by phase 0.
 *
 * hk_diag_rates: micro-benchmarks. kind 0: pipe issue rate of op `param`
 * (0 ex2.f32, 1 cvt.bf16x2.f32, 2 fma.f32, 3 max.f32, 4 ex2.bf16x2, 5 add.f32),
 * 148 CTAs x 512 threads x iters x 8 ops; out[cta] = clock64 cycles.
 * kind 2: tcgen05.ld (32x32b.x32) bandwidth with `param` warps x 128 columns.
 * kind 3: forward softmax step, param = 10 * (emulated exps per 8) + warpgroups.
 * kind 4: TMA load throughput per SM with boxes of `param` rows x 128 B.
 * kind 5: fp32 red.global.add.v4 throughput into a `param` x 64 KB region.
 * kind 6: bulk-async (TMA) fp32 reduce-add of 128 x 128 tiles (64 KB) from shared memory
 * into a [row_tiles*128][32][128] fp32 region (dQ-like), param = mode * 100000 + row_tiles;
 * mode 0 = one cp.reduce.async.bulk.tensor.2d per tile, 1 = 128 row-wise cp.reduce.async.bulk.
 * kind 1: tcgen05.mma pacing, mode = param / 1000 (0 SS, 1 TS, 2 SS with B
 * MN-major), N = param % 1000 in {64,128,256}; out[cta] = cycles per MMA.
 * `out` is a device pointer to >= 148 floats.
 *
 * hk_diag_trace_read: copy the in-kernel event table of an HK_TRACE build
 * (64 events x 1024 slots of u64 clock64, slot = (event, iteration mod 1024),
 * 0 = not recorded; 512 KiB) into the host buffer `dst` (capacity `bytes`);
 * zero-fills `dst` on non-trace builds. reset != 0 clears the table.
 */
#ifndef HK_ATTN_DIAG_H_
#define HK_ATTN_DIAG_H_
#include "hk_attn.h"
#ifdef __cplusplus
extern "C" {
#endif
const char* hk_diag_last_error(void);
hk_status hk_diag_umma(const void* A, const void* B, float* D, int N, int K, int a_tmem, int b_mn,
                       cudaStream_t stream);
hk_status hk_diag_bwd_phase(int phase, const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                            const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                            int B, int Hq, int Hkv, int N, int d, int causal, cudaStream_t stream);
hk_status hk_diag_rates(int kind, int param, int iters, float* out, cudaStream_t stream);
hk_status hk_diag_trace_read(void* dst, size_t bytes, int reset);
#ifdef __cplusplus
}
#endif
#endif
