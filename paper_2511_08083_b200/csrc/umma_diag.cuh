// Diagnostic single-tile tcgen05 GEMM: D[128 x N] = A[128 x K] * op(B).
// Exercises exactly the operand forms the attention kernels use:
//   A from SMEM (K-major, TMA SWIZZLE_128B) or from TMEM (bf16 pairs per column),
//   B K-major ([N][K] in HBM, D = A B^T)  or  MN-major ([K][N] in HBM, D = A B).
// Not on the hot path: `hk_diag_umma` exists so tests can pin the descriptor
// encodings in isolation.
#pragma once
#include "ptx.cuh"

namespace hk {

template <int N, int K, bool A_TMEM, bool B_MN>
__global__ void __launch_bounds__(128, 1)
    umma_diag_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const __nv_bfloat16* __restrict__ A, float* __restrict__ D) {
  constexpr int M = 128;
  constexpr uint32_t A_BYTES = M * K * 2;
  constexpr uint32_t B_BYTES = N * K * 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp_id() == 0) tmem_alloc<256>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  const uint32_t tD = tbase;          // columns [0, N)
  const uint32_t tA = tbase + 128;    // columns [128, 128 + K/2)

  if (tid == 0) {
    uint64_t pol = policy_evict_normal();
    mbar_arrive_expect_tx(&bar_load, (A_TMEM ? 0 : A_BYTES) + B_BYTES);
    if (!A_TMEM)
      for (int p = 0; p < K / 64; ++p) tma_load_4d(&mapA, &bar_load, sA + p * M * 128, p * 64, 0, 0, 0, pol);
    if (!B_MN) {
      for (int p = 0; p < K / 64; ++p) tma_load_4d(&mapB, &bar_load, sB + p * N * 128, p * 64, 0, 0, 0, pol);
    } else {
      for (int p = 0; p < N / 64; ++p) tma_load_4d(&mapB, &bar_load, sB + p * K * 128, p * 64, 0, 0, 0, pol);
    }
  }
  if (A_TMEM) {
    // row = tid: pack A[row][2c], A[row][2c+1] into column c.
    const uint32_t lane_base = (warp_id() & 3) * 32;
    const __nv_bfloat16* arow = A + (size_t)tid * K;
#pragma unroll
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(arow + 2 * (c0 + c));
        r[c] = *reinterpret_cast<uint32_t*>(&v);
      }
      tmem_st16(tmem_addr(tA, lane_base, c0), r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();

  if (tid == 0) {
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    constexpr uint32_t idesc = idesc_bf16(M, N, 0, B_MN ? 1 : 0);
#pragma unroll
    for (int kk = 0; kk < K / 16; ++kk) {
      uint64_t bdesc;
      if (!B_MN)
        bdesc = sdesc_sw128(smem_u32(sB + (kk / 4) * N * 128 + (kk % 4) * 32), 16, 1024);
      else
        bdesc = sdesc_sw128(smem_u32(sB + kk * 16 * 128), K * 128, 1024);
      if (A_TMEM) {
        umma_ts(tD, tA + kk * 8, bdesc, idesc, kk > 0);
      } else {
        uint64_t adesc = sdesc_sw128(smem_u32(sA + (kk / 4) * M * 128 + (kk % 4) * 32), 16, 1024);
        umma_ss(tD, adesc, bdesc, idesc, kk > 0);
      }
    }
    tc_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const uint32_t lane_base = (warp_id() & 3) * 32;
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem_addr(tD, lane_base, c0), r);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 32; ++c) D[(size_t)tid * N + c0 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<256>(tbase);
}

}  // namespace hk
