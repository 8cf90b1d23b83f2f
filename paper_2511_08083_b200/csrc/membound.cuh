// The paper's memory-bound kernels (PAPER.md P:554-562,
// P:583): fused dropout + residual + LayerNorm (listing P:1214-1267) and rotary
// positional encoding. Both are HBM-roofline kernels on B200: 16-byte vector
// loads/stores, one pass over HBM, statistics in fp32 registers.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "rope.cuh"

namespace hk {

// ---------------------------------------------------------------- dropout hash
// keep(i) = lowbias32(i * 0x9E3779B9 + seed) >= thresh, thresh = floor(p * 2^32)
// (reading #20; the oracle implements the same counter-based hash).
__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// ---------------------------------------------------------------- LayerNorm
struct LnParams {
  const __nv_bfloat16* x;         // [rows][D]
  const __nv_bfloat16* residual;  // [rows][D]
  const __nv_bfloat16* weight;    // [D]
  const __nv_bfloat16* bias;      // [D]
  __nv_bfloat16* out;             // [rows][D]
  __nv_bfloat16* out_resid;       // [rows][D]
  int rows, D;
  uint32_t thresh;  // dropout keep threshold (0 = no dropout)
  uint32_t seed;
  float scale;      // 1 / (1 - p)
  float eps;
};

// One warp per row (rows grid-strided over warps). Lane l owns the 8-element
// vectors l, l+32, ... of its row (VPL = vectors per lane, compile-time max).
// r = bf16(residual + dropout(x)) is kept packed in registers (it is stored
// rounded anyway) for the two-pass mean / centred variance.
template <int VPL>
__global__ void __launch_bounds__(256) ln_dropout_residual_kernel(const LnParams p) {
  const int lane = threadIdx.x & 31;
  const int nv = p.D / 8;
  const size_t gwarp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const size_t nwarps = (size_t)gridDim.x * blockDim.x / 32;
  const float inv_d = 1.f / (float)p.D;
  for (size_t row = gwarp; row < (size_t)p.rows; row += nwarps) {
    const uint4* xr = reinterpret_cast<const uint4*>(p.x + row * p.D);
    const uint4* rr = reinterpret_cast<const uint4*>(p.residual + row * p.D);
    // every load of the row is issued before any store (the stores could alias the
    // inputs as far as the compiler knows, which would serialise one round trip per vector)
    uint4 xv[VPL], rv[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int v = lane + 32 * k;
      if (v < nv) {
        xv[k] = __ldcs(xr + v);  // streamed once: evict-first
        rv[k] = __ldcs(rr + v);
      }
    }
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int v = lane + 32 * k;
      if (v < nv) {
        float xf[8], rf[8];
        unpack8(xv[k], xf);
        unpack8(rv[k], rf);
        const uint32_t base = (uint32_t)(row * p.D + (size_t)v * 8);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float xt = xf[e];
          if (p.thresh) xt = lowbias32((base + e) * 0x9E3779B9u + p.seed) >= p.thresh ? xt * p.scale : 0.f;
          rf[e] += xt;
        }
        rv[k] = pack8(rf);
        float q[8];
        unpack8(rv[k], q);  // the stored (rounded) values feed the statistics
#pragma unroll
        for (int e = 0; e < 8; ++e) sum += q[e];
        __stcs(reinterpret_cast<uint4*>(p.out_resid + row * p.D) + v, rv[k]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum * inv_d;
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (lane + 32 * k < nv) {
        float q[8];
        unpack8(rv[k], q);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float c = q[e] - mean;
          ss = fmaf(c, c, ss);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float rstd = rsqrtf(ss * inv_d + p.eps);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int v = lane + 32 * k;
      if (v < nv) {
        float q[8], w[8], b[8];
        unpack8(rv[k], q);
        unpack8(__ldg(reinterpret_cast<const uint4*>(p.weight) + v), w);
        unpack8(__ldg(reinterpret_cast<const uint4*>(p.bias) + v), b);
#pragma unroll
        for (int e = 0; e < 8; ++e) q[e] = fmaf((q[e] - mean) * rstd, w[e], b[e]);
        __stcs(reinterpret_cast<uint4*>(p.out + row * p.D) + v, pack8(q));
      }
    }
  }
}

// ---------------------------------------------------------------- rotary
struct RopeParams {
  const __nv_bfloat16* x;  // [B][N][H][d]
  const float* cos;        // [N][d/2]
  const float* sin;        // [N][d/2]
  __nv_bfloat16* out;      // [B][N][H][d]
  size_t rows;             // B * N * H
  int N, H, d;
  float sgn;               // +1: rotate by theta; -1: the inverse rotation (gradients)
};

// One thread per (row, 8-wide chunk of the first half): it loads the matching
// chunks of both halves (16 B each) and the 8 cos/sin values of its position.
// I: index type of the chunk counter — uint32_t when the chunk count fits (32-bit divisions;
// 64-bit ones compile to a long subroutine and made the memory-bound kernels ALU-bound).
template <typename I>
__global__ void __launch_bounds__(256) rope_kernel(const RopeParams p) {
  const int half = p.d / 2, cpr = half / 8;  // chunks per row
  const I total = (I)(p.rows * cpr);
  for (I t = (I)(blockIdx.x * blockDim.x + threadIdx.x); t < total; t += (I)(gridDim.x * blockDim.x)) {
    const I row = t / (I)cpr;
    const int ch = (int)(t - row * (I)cpr);
    const int n = (int)((row / (I)p.H) % (I)p.N);
    const __nv_bfloat16* xr = p.x + (size_t)row * p.d;  // 64-bit offset whatever I is
    float a[8], b[8], c[8], s[8];
    unpack8(__ldcs(reinterpret_cast<const uint4*>(xr) + ch), a);
    unpack8(__ldcs(reinterpret_cast<const uint4*>(xr + half) + ch), b);
    rope_load_cs(p.cos, p.sin, (size_t)n, half, ch, p.sgn, c, s);
    float lo[8], hi[8];
    rope_pair8(a, b, c, s, lo, hi);
    __nv_bfloat16* orow = p.out + (size_t)row * p.d;
    __stcs(reinterpret_cast<uint4*>(orow) + ch, pack8(lo));
    __stcs(reinterpret_cast<uint4*>(orow + half) + ch, pack8(hi));
  }
}

// Rotary, head-loop form (HK_ROPE_HLOOP): one thread per (b, n, 8-wide chunk) walks all H heads,
// so the position's cos/sin chunk is loaded once instead of once per head (the per-head form
// moves twice as many cos/sin bytes through L1 as x bytes).
template <typename I>
__global__ void __launch_bounds__(256) rope_hloop_kernel(const RopeParams p) {
  const int half = p.d / 2, cpr = half / 8;
  const I units = (I)(p.rows / p.H * cpr);  // (b, n) positions x chunks
  for (I t = (I)(blockIdx.x * blockDim.x + threadIdx.x); t < units; t += (I)(gridDim.x * blockDim.x)) {
    const size_t bn = t / (I)cpr;
    const int ch = (int)(t - (I)bn * (I)cpr);
    const int n = (int)((I)bn % (I)p.N);
    float c[8], s[8];
    rope_load_cs(p.cos, p.sin, (size_t)n, half, ch, p.sgn, c, s);
    constexpr int HG = 4;  // heads per group: their loads go out together
    for (int h0 = 0; h0 < p.H; h0 += HG) {
      uint4 va[HG], vb[HG];
#pragma unroll
      for (int u = 0; u < HG; ++u) {
        if (h0 + u < p.H) {
          const __nv_bfloat16* xr = p.x + (bn * p.H + h0 + u) * p.d;
          va[u] = __ldcs(reinterpret_cast<const uint4*>(xr) + ch);
          vb[u] = __ldcs(reinterpret_cast<const uint4*>(xr + half) + ch);
        }
      }
#pragma unroll
      for (int u = 0; u < HG; ++u) {
        if (h0 + u < p.H) {
          float a[8], b[8], lo[8], hi[8];
          unpack8(va[u], a);
          unpack8(vb[u], b);
          rope_pair8(a, b, c, s, lo, hi);
          __nv_bfloat16* orow = p.out + (bn * p.H + h0 + u) * p.d;
          __stcs(reinterpret_cast<uint4*>(orow) + ch, pack8(lo));
          __stcs(reinterpret_cast<uint4*>(orow + half) + ch, pack8(hi));
        }
      }
    }
  }
}

}  // namespace hk
