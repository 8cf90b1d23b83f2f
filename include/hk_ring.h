/* hk_ring.h — C ABI of the context-parallel (ring) attention building blocks in
 * libhkattn.so ("context-parallel ring attention over
 * NVLink 5 ... with an LSE merge").
 *
 * Ring attention splits the sequence over ranks; each rank combines, for its
 * query rows, partial attention results over disjoint key sets (one per ring
 * step, each from hk_attn_fwd / hk_attn_fwd_qk) with the same rescale-and-add
 * the forward applies between key tiles (O is rescaled by
 * exp(m_old - m_new) before the new block accumulates), written in LSE form:
 *   LSE   = ln(e^LSE_acc + e^LSE_part)
 *   O_acc = e^(LSE_acc - LSE) O_acc + e^(LSE_part - LSE) O_part
 * Rows where both LSEs are -inf (no key seen yet) stay O = 0, LSE = -inf.
 * The backward needs no merge: with the final O and LSE, each step's hk_attn_bwd
 * returns that key set's exact share of dQ, dK, dV, which hk_accum_bf16 sums.
 *
 * Layouts: O_acc fp32 [B][N][H][d]; O_part, O_out bf16 [B][N][H][d];
 * LSE_acc, LSE_part fp32 [B][H][N]; all contiguous, 16-B aligned; d % 8 == 0,
 * d <= 256. Ownership, streams and errors as in hk_attn.h.
 */
#ifndef HK_RING_H_
#define HK_RING_H_

#include "hk_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

/* init != 0: O_acc = O_part, LSE_acc = LSE_part (the first partial; inputs of the
 * accumulator are not read). O_out != NULL: also write bf16(O_acc) after the merge. */
hk_status hk_attn_merge(float* O_acc, float* LSE_acc, const void* O_part, const float* LSE_part, void* O_out, int B,
                        int N, int H, int d, int init, cudaStream_t stream);

/* Gradient accumulation over ring steps, n bf16 elements x (n % 8 == 0):
 *   out == NULL:  acc = (init ? 0 : acc) + x          (fp32)
 *   out != NULL:  out = bf16((init ? 0 : acc) + x)     (the last step; acc not written)
 * x may be NULL (treated as 0) when out != NULL and init == 0: out = bf16(acc). */
hk_status hk_accum_bf16(float* acc, const void* x, void* out, size_t n, int init, cudaStream_t stream);

/* acc += x over n fp32 elements (n % 4 == 0, 16-B aligned, no overlap; ABI 5): the ring backward
 * adds the dK/dV accumulator received from the previous rank to this rank's own contributions for
 * the same key chunk, which were formed while that accumulator was in flight. */
hk_status hk_accum_f32(float* acc, const float* x, size_t n, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HK_RING_H_ */
