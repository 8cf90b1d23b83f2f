/* hk_membound.h — C ABI of the memory-bound kernels in libhkattn.so
 * ("Memory bound").
 *
 * hk_ln_dropout_residual — fused dropout + residual + LayerNorm, the paper's
 * listing P:1214-1267, per row of D elements:
 *   x~ = x * keep / (1 - p)        keep(i) = lowbias32(i * 0x9E3779B9 + seed) >= floor(p 2^32),
 *                                  i = row * D + col (reading #20)
 *   out_resid = bf16(residual + x~)
 *   out = (r - mean) / sqrt(var + eps) * weight + bias, r = out_resid,
 *   mean and the centred variance in fp32 (the listing uses bf16; reading #20).
 * Layouts: x, residual, out, out_resid [rows][D]; weight, bias [D]; all bf16,
 * contiguous, 16-B aligned. Supported: D % 8 == 0, 8 <= D <= 8192,
 * rows * D < 2^32, 0 <= p < 1, eps > 0.
 *
 * hk_rope — rotary positional encoding (B=16, H=16, d=128), rotate-half
 * form (reading #21): for x [B][N][H][d] bf16 and cos, sin [N][d/2] fp32,
 *   out[.., i] = x_i cos - x_{i+d/2} sin,  out[.., i+d/2] = x_{i+d/2} cos + x_i sin.
 * Supported: d % 16 == 0, 16 <= d <= 512. `out` may equal `x` (in place).
 *
 * Ownership, streams and errors as in hk_attn.h (device pointers owned by the
 * caller, no allocation, enqueued on `stream`, validation before any launch,
 * message in hk_attn_last_error()).
 */
#ifndef HK_MEMBOUND_H_
#define HK_MEMBOUND_H_

#include "hk_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

hk_status hk_ln_dropout_residual(const void* x, const void* residual, const void* weight, const void* bias, void* out,
                                 void* out_resid, int rows, int D, float p, unsigned int seed, float eps,
                                 cudaStream_t stream);

hk_status hk_rope(const void* x, const float* cos, const float* sin, void* out, int B, int N, int H, int d,
                  cudaStream_t stream);
/* inverse != 0: the inverse rotation (sin negated): out_i = x_i cos + x_{i+d/2} sin,
 * out_{i+d/2} = x_{i+d/2} cos - x_i sin — the gradient of a rotated tensor maps back through it. */
hk_status hk_rope_ex(const void* x, const float* cos, const float* sin, void* out, int B, int N, int H, int d,
                     int inverse, cudaStream_t stream);

/* hk_attn_fwd_rope — rotary fused into the attention forward (SURVEY §8(f) NEXT #3, P:559,
 * P:583): O, LSE = attention(rope(Q), rope(K), V), dense self-attention (Nq = Nk = N), positions
 * 0..N-1, cos / sin [N][d/2] fp32 as hk_rope. Q tiles are rotated in shared memory by the
 * forward kernel (each is read once per CTA, so the rotation costs no HBM pass); K, re-read by
 * every query tile of its group, is rotated once into the caller's Kr [B][N][Hkv][d] bf16 (an
 * output: the backward and a KV cache need the rotated keys). Bitwise equal to hk_rope on Q and K
 * followed by hk_attn_fwd. Other arguments, layouts and errors as hk_attn_fwd. */
hk_status hk_attn_fwd_rope(const void* Q, const void* K, const void* V, const float* cos, const float* sin, void* O,
                           float* LSE, void* Kr, int B, int Hq, int Hkv, int N, int d, int causal,
                           cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HK_MEMBOUND_H_ */
