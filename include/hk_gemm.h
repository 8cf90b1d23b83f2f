/* hk_gemm.h — C ABI of the BF16 GEMM in libhkattn.so.
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, arXiv 2511.08083):
 *   C[m, n] = sum_k A[m, k] * B[n, k]        (C = A B^T)
 * the paper's GEMM listing accumulates mma_ABt(C, A_tile, B_tile, C) over
 * K_STEP slices of row-major A and B, 256x256 output tiles
 * (P:1044), benchmarked at M = N = K = 8192 on N(0,1) inputs.
 * bf16 operands, fp32 accumulation in tensor memory, bf16 output rounded to
 * nearest even (the listing's epilogue is not shown; reading #18).
 *
 * Layouts: A [M][K], B [N][K], C [M][N], all bf16, row-major, contiguous.
 * Supported: M % 256 == 0, N % 256 == 0, K % 64 == 0 (K >= 64); other shapes
 * return HK_ERR_UNSUPPORTED.
 *
 * Ownership: device pointers owned by the caller; no device memory is
 * allocated; the work is enqueued on `stream`. C is fully overwritten and
 * bitwise reproducible (fixed accumulation order, no atomics).
 *
 * Errors: as in hk_attn.h -- validated before anything is enqueued,
 * HK_ERR_INVALID_ARGUMENT for null / misaligned (16 B) pointers, non-positive
 * sizes or C overlapping A or B; the message is in hk_attn_last_error().
 */
#ifndef HK_GEMM_H_
#define HK_GEMM_H_

#include "hk_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

hk_status hk_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HK_GEMM_H_ */
