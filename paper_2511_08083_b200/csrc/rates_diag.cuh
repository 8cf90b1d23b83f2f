// Diagnostic micro-benchmarks (not the hot path): issue rates of the pipes the
// softmax uses, and tcgen05.mma pacing for the operand forms the kernels use.
#pragma once
#include "ptx.cuh"
#include "softmax.cuh"

namespace hk {

// op: 0 ex2.approx.f32, 1 cvt.rn.bf16x2.f32, 2 fma.rn.f32 (3 regs), 3 max.f32,
//     4 ex2.approx.ftz.bf16x2, 5 add.f32
template <int OP>
__global__ void __launch_bounds__(512) pipe_rate_kernel(int iters, float* out_cycles, float* sink) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  uint32_t u[8] = {};
  const float b = 1.0001f, c = 0.9999f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) {  // dependent chain: the packed result feeds the next conversion
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        a[i] = __uint_as_float(u[i]);
      }
      if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
      if (OP == 3) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]));
      if (OP == 4) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
      if (OP == 5) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (OP == 6) {  // fma.rn.f32x2 on register pairs (a[i], a[i^1])
        if ((i & 1) == 0) {
          float2 v = fma2(make_float2(a[i], a[i + 1]), make_float2(b, c), make_float2(a[(i + 2) & 7], a[(i + 3) & 7]));
          a[i] = v.x;
          a[i + 1] = v.y;
        }
      }
      if (OP == 7) {
        if ((i & 1) == 0) {
          float2 v = add2(make_float2(a[i], a[i + 1]), make_float2(a[(i + 2) & 7], a[(i + 3) & 7]));
          a[i] = v.x;
          a[i + 1] = v.y;
        }
      }
      if (OP == 8) a[i] = max3f(a[i], a[(i + 3) & 7], a[(i + 5) & 7]);
      if (OP == 9) a[i] = __int_as_float(__float_as_int(a[i]) + (__float_as_int(a[(i + 3) & 7]) << 23));
      if (OP == 10) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]), "f"(a[(i + 5) & 7]));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
  if (s == 12345.f) sink[0] = s;
  if (threadIdx.x == 0) out_cycles[blockIdx.x] = (float)(t1 - t0);
}

// tcgen05.mma pacing: one CTA per SM, one thread issues iters x 8 MMAs
// (M=128, N, K=16) on resident smem / TMEM operands; out = cycles per MMA.
// mode 0: SS (A 128 rows K-major, B N rows K-major); mode 1: TS (A in TMEM,
// B MN-major [16][N] slices); mode 2: SS with B MN-major.
template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int iters, float* out_cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  // zero the operand tiles so the MMAs see finite data
  for (int i = threadIdx.x; i < (128 * 128 * 2 + 256 * 128 * 2) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp_id() == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  const uint32_t a_s = smem_u32(smem), b_s = a_s + 128 * 128 * 2;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, N, 0, MODE == 0 ? 0 : 1);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0)
          umma_ss(tb, sdesc_sw128(a_s + (kk / 4) * 128 * 128 + (kk % 4) * 32, 16, 1024),
                  sdesc_sw128(b_s + (kk / 4) * N * 128 + (kk % 4) * 32, 16, 1024), idesc, 1);
        else if (MODE == 1)
          umma_ts(tb, tb + 256 + kk * 8, sdesc_sw128(b_s + kk * 16 * 128, 128 * 128, 1024), idesc, 1);
        else
          umma_ss(tb, sdesc_sw128(a_s + (kk / 4) * 128 * 128 + (kk % 4) * 32, 16, 1024),
                  sdesc_sw128(b_s + kk * 16 * 128, 128 * 128, 1024), idesc, 1);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out_cycles[blockIdx.x] = (float)(t1 - t0) / (iters * 8);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tb);
}

// TMEM -> register bandwidth: W warps (W/4 warpgroups) each repeatedly load
// their 32 lanes x NC columns with tcgen05.ld.32x32b.x32; out = cycles.
template <int NC>
__global__ void tmem_ld_rate_kernel(int iters, float* out_cycles, float* sink) {
  __shared__ uint32_t tbase_s;
  if (warp_id() == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s + ((warp_id() & 3) * 32 << 16) + (warp_id() / 4) * NC;
  float acc = 0.f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c0 = 0; c0 < NC; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tb + c0, r);
      tmem_wait_ld();
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 1234.5f) sink[0] = acc;
  if (threadIdx.x == 0) out_cycles[blockIdx.x] = (float)(t1 - t0);
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tbase_s);
}

// Forward softmax step throughput in isolation (no MMAs): NWG warpgroups each
// run softmax_step on their own 128-column TMEM score tile `iters` times;
// out = cycles per step (clock64, thread 0). The running max is reset every
// step so the (rare) O-rescale branch is not exercised.
template <int EMU_OF_8>
__global__ void softmax_rate_kernel(int iters, float* out_cycles, float* sink) {
  __shared__ uint32_t tbase_s;
  if (warp_id() == 0) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int t = warp_id() / 4;
  const uint32_t lane_base = (warp_id() & 3) * 32;
  const int r = lane_base + lane_id();
  const uint32_t tS = tbase_s + 128 * t, tO = tbase_s + 256 + 128 * t;
  uint32_t init[32];
  for (int c0 = 0; c0 < 128; c0 += 32) {
    for (int k = 0; k < 32; ++k) {
      uint32_t hsh = (r * 131 + c0 + k) * 2654435761u;
      init[k] = __float_as_uint(((hsh >> 8) & 0xFFFF) / 6553.6f - 5.f);
    }
    tmem_st32(tmem_addr(tS, lane_base, c0), init);
  }
  tmem_wait_st();
  __syncthreads();
  const float c = 1.4426950408889634f / sqrtf(128.f);
  float l = 0.f, msum = 0.f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float m = -INFINITY;
    softmax_step<128, EMU_OF_8>(tS, tO, lane_base, r, c, m, l, 1 << 20, false);
    msum += m;
  }
  tmem_wait_st();
  const long long t1 = clock64();
  if (l + msum == 1234.5f) sink[0] = l;
  if (threadIdx.x == 0) out_cycles[blockIdx.x] = (float)(t1 - t0) / iters;
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tbase_s);
}

// TMA load throughput: one CTA per SM, one thread streams `iters` boxes of
// 64 x ROWS bf16 (ROWS x 128 B) through an 8-slot ring from an L2-resident
// [rows][64] tensor; a consumer warp frees each slot when it lands.
// out[cta] = cycles.
template <int ROWS>
__global__ void __launch_bounds__(64, 1) tma_rate_kernel(const __grid_constant__ CUtensorMap map, int iters,
                                                          int total_rows, float* out_cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int SLOTS = 8;
  constexpr uint32_t BYTES = ROWS * 128;
  __shared__ uint64_t full[SLOTS], empty[SLOTS];
  if (threadIdx.x == 0) {
    for (int i = 0; i < SLOTS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_last();
    for (int it = 0; it < iters; ++it) {
      const int s = it % SLOTS;
      mbar_wait(&empty[s], ((it / SLOTS) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], BYTES);
      const int row = ((blockIdx.x * 7 + it) * ROWS) % total_rows;
      tma_load_4d(&map, &full[s], smem + s * BYTES, 0, 0, row, 0, pol);
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % SLOTS;
      mbar_wait(&full[s], (it / SLOTS) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out_cycles[blockIdx.x] = (float)(t1 - t0);
}

// fp32 reduce-add throughput into L2: each CTA adds `iters` 128x128 fp32 tiles
// (64 KB, rows of 512 B like a dQ accumulator row) into a `tiles`-tile region
// with red.global.add.v4.f32; out[cta] = cycles.
__global__ void __launch_bounds__(256) red_rate_kernel(float* dst, int tiles, int iters, float* out_cycles) {
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float* tile = dst + (size_t)((blockIdx.x * 7 + it * 13) % tiles) * 128 * 128;
    // thread t: row t/2, half (t%2) of the row: 64 floats = 16 x v4
    float* rowp = tile + (threadIdx.x / 2) * 128 + (threadIdx.x % 2) * 64;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float v = 1e-3f * (k + 1);
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(rowp + 4 * k), "f"(v), "f"(v), "f"(v),
                   "f"(v)
                   : "memory");
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out_cycles[blockIdx.x] = (float)(t1 - t0);
}

// fp32 reduce-add of whole 128 x 128 tiles (64 KB) from shared memory into global memory by the
// bulk-async (TMA) engine: the instruction SURVEY §8(f) NEXT #1 names for accumulating dQ inside
// the dK/dV pass. The destination mimics dQ [rows][H][128] fp32 of one (b, kvh) window: a tile
// is 128 rows of one head, rows H * 512 B apart. MODE 0: one cp.reduce.async.bulk.tensor.2d
// per tile (box 128 x 128 fp32, no swizzle); MODE 1: 128 row-wise cp.reduce.async.bulk (512 B
// each). One thread per CTA issues, keeping up to INFLIGHT tiles outstanding. out[cta] = cycles.
template <int MODE>
__global__ void __launch_bounds__(128) bulk_red_rate_kernel(const __grid_constant__ CUtensorMap map, float* dst,
                                                            int row_tiles, int H, int iters, float* out_cycles) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  float* sm = reinterpret_cast<float*>(sm_raw);
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) sm[i] = 1e-3f * (i & 7);
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int t = (blockIdx.x * 7 + it * 13) % (row_tiles * H);
      const int rt = t / H, h = t % H;
      if (MODE == 0) {
        asm volatile(
            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                reinterpret_cast<uint64_t>(&map)),
            "r"(smem_u32(sm)), "r"(h * 128), "r"(rt * 128)
            : "memory");
      } else {
        float* base = dst + ((size_t)rt * 128 * H + h) * 128;
        for (int r = 0; r < 128; ++r)
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;" ::"l"(
                           base + (size_t)r * H * 128),
                       "r"(smem_u32(sm + r * 128))
                       : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    const long long t1 = clock64();
    out_cycles[blockIdx.x] = (float)(t1 - t0);
  }
}

}  // namespace hk
