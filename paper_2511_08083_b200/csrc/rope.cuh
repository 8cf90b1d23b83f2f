// Rotate-half rotary embedding of one 8-wide chunk pair (reading #21):
// for element i of the first half (a) and i + d/2 of the second (b) at position n,
//   lo = a cos - b sin,  hi = b cos + a sin   (sin negated for the inverse rotation).
// Shared by the standalone hk_rope kernels and the forward's fused Q rotation, so the two give
// bitwise the same rotated values.
#pragma once
#include <cuda_bf16.h>

namespace hk {

// 8 bf16 <-> 8 fp32 (round to nearest even)
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __bfloat1622float2(h[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
  return v;
}


__device__ __forceinline__ void rope_pair8(const float (&a)[8], const float (&b)[8], const float (&c)[8],
                                           const float (&s)[8], float (&lo)[8], float (&hi)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    lo[e] = fmaf(a[e], c[e], -b[e] * s[e]);
    hi[e] = fmaf(b[e], c[e], a[e] * s[e]);
  }
}

// cos, sin [N][d/2] fp32: the 8 values of chunk ch at position n; sgn = -1 gives the inverse
__device__ __forceinline__ void rope_load_cs(const float* cosp, const float* sinp, size_t n, int half, int ch,
                                             float sgn, float (&c)[8], float (&s)[8]) {
  const float4* cp = reinterpret_cast<const float4*>(cosp + n * half + ch * 8);
  const float4* sp = reinterpret_cast<const float4*>(sinp + n * half + ch * 8);
  const float4 c0 = __ldg(cp), c1 = __ldg(cp + 1), s0 = __ldg(sp), s1 = __ldg(sp + 1);
  c[0] = c0.x, c[1] = c0.y, c[2] = c0.z, c[3] = c0.w, c[4] = c1.x, c[5] = c1.y, c[6] = c1.z, c[7] = c1.w;
  s[0] = sgn * s0.x, s[1] = sgn * s0.y, s[2] = sgn * s0.z, s[3] = sgn * s0.w;
  s[4] = sgn * s1.x, s[5] = sgn * s1.y, s[6] = sgn * s1.z, s[7] = sgn * s1.w;
}

}  // namespace hk
