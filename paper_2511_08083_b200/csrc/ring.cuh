// Context-parallel (ring) attention building blocks (include/hk_ring.h): the
// LSE merge of partial attention results and the fp32 gradient accumulator.
// Both are HBM-bound elementwise passes: 16-B vector loads, one pass each.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "membound.cuh"  // unpack8 / pack8

namespace hk {

struct MergeParams {
  float* o_acc;          // [B][N][H][d] fp32
  float* lse_acc;        // [B][H][N]
  const __nv_bfloat16* o_part;
  const float* lse_part;
  __nv_bfloat16* o_out;  // optional bf16 copy of the merged O
  int B, N, H, d, init;
};

// d/8 lanes per (b, n, h) row, rows grid-strided; all lanes of a row sit in one
// warp, so the row's LSE reads precede lane 0's LSE write (__syncwarp).
__global__ void __launch_bounds__(256) attn_merge_kernel(const MergeParams p) {
  const int lpr = p.d / 8;  // lanes per row (power of two not required: rows never straddle a warp)
  const int rpw = 32 / lpr;  // rows per warp
  const int lane = threadIdx.x & 31;
  const int sub = lane % lpr, lrow = lane / lpr;
  const size_t rows = (size_t)p.B * p.N * p.H;
  const size_t gwarp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const size_t nwarps = (size_t)gridDim.x * blockDim.x / 32;
  for (size_t base = gwarp * rpw; base < rows; base += nwarps * rpw) {
    const size_t row = base + lrow;
    const bool ok = lrow < rpw && row < rows;
    size_t li = 0;
    float wa = 0.f, wb = 1.f, L = 0.f;
    if (ok) {
      // 32-bit divisions when the row count fits (64-bit ones are a long subroutine)
      size_t h, n, b;
      if (rows < ((size_t)1 << 31)) {
        const uint32_t r32 = (uint32_t)row, q = r32 / (uint32_t)p.H;
        h = r32 - q * (uint32_t)p.H;
        n = q % (uint32_t)p.N;
        b = q / (uint32_t)p.N;
      } else {
        h = row % p.H;
        n = (row / p.H) % p.N;
        b = row / ((size_t)p.H * p.N);
      }
      li = (b * p.H + h) * p.N + n;
      const float lb = p.lse_part[li];
      if (p.init) {
        L = lb;
      } else {
        const float la = p.lse_acc[li];
        const float m = fmaxf(la, lb);
        if (m == -INFINITY) {  // neither partial has seen a key
          L = -INFINITY;
          wa = wb = 0.f;
        } else {
          const float ea = expf(la - m), eb = expf(lb - m);
          const float s = ea + eb;
          L = m + logf(s);
          wa = ea / s;
          wb = eb / s;
        }
      }
    }
    __syncwarp();
    if (ok) {
      float a[8], o[8];
      unpack8(*reinterpret_cast<const uint4*>(p.o_part + row * p.d + sub * 8), o);
      float4* acc = reinterpret_cast<float4*>(p.o_acc + row * p.d + sub * 8);
      if (p.init) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = o[k];
      } else {
        const float4 x0 = acc[0], x1 = acc[1];
        const float in[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = wa * in[k] + wb * o[k];
      }
      acc[0] = make_float4(a[0], a[1], a[2], a[3]);
      acc[1] = make_float4(a[4], a[5], a[6], a[7]);
      if (p.o_out) *reinterpret_cast<uint4*>(p.o_out + row * p.d + sub * 8) = pack8(a);
      if (sub == 0) p.lse_acc[li] = L;
    }
  }
}

// acc += x, fp32, 4 per thread-iteration (16-B loads).
__global__ void __launch_bounds__(256) accum_f32_kernel(float* __restrict__ acc, const float* __restrict__ x,
                                                        size_t n4) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<const float4*>(acc)[i];
    const float4 b = reinterpret_cast<const float4*>(x)[i];
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    reinterpret_cast<float4*>(acc)[i] = a;
  }
}

// acc / out over n elements, 8 per thread-iteration (16-B bf16 loads).
__global__ void __launch_bounds__(256) accum_bf16_kernel(float* __restrict__ acc, const __nv_bfloat16* __restrict__ x,
                                                         __nv_bfloat16* __restrict__ out, size_t n8, int init) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (x) unpack8(reinterpret_cast<const uint4*>(x)[i], v);  // x == nullptr: cast acc to bf16
    if (!init) {
      const float4 a0 = reinterpret_cast<const float4*>(acc)[2 * i], a1 = reinterpret_cast<const float4*>(acc)[2 * i + 1];
      v[0] += a0.x; v[1] += a0.y; v[2] += a0.z; v[3] += a0.w;
      v[4] += a1.x; v[5] += a1.y; v[6] += a1.z; v[7] += a1.w;
    }
    if (out) {
      reinterpret_cast<uint4*>(out)[i] = pack8(v);
    } else {
      reinterpret_cast<float4*>(acc)[2 * i] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(acc)[2 * i + 1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

}  // namespace hk
