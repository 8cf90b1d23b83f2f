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

#ifdef __cplusplus
}
#endif
#endif /* HK_MEMBOUND_H_ */
