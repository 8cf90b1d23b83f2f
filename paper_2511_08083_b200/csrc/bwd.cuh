// Backward fused attention for sm_100a: three stream-ordered kernels.
//
// The paper gives no backward algorithm (PAPER.md: "notoriously
// register heavy", multiple MFMA shapes, row+col loads of one shared tile);
// BASELINE.json prescribes the structure implemented here:
//   B0  bwd_pre_kernel   D = rowsum(dO * O) and LSE2 = LSE * log2(e)   (HBM-bound)
//   B1  bwd_dkdv_kernel  per (key tile j, kvh, b): loop h in the GQA group and
//       query blocks i; S^T = K_j Q_i^T, dP^T = V_j dO_i^T (tcgen05, TMEM),
//       P^T = exp2(c S^T - LSE2_i), dS^T = P^T (dP^T - D_i) in registers,
//       dV += P^T dO_i, dK += dS^T Q_i with bf16 P^T / dS^T read from TMEM.
//       The GQA group reduction is this in-kernel h-loop (no atomics).
//   B2  bwd_dq_kernel    per (query tile i, h, b): loop key blocks j;
//       S = Q_i K_j^T, dP = dO_i V_j^T, dS = P (dP - D_i), dQ += dS K_j.
// The elementwise work is split into a P phase and a dS phase with separate
// TMEM hand-offs so the exponentials of one block overlap tensor-core work of
// the neighbouring blocks (see the MMA order comments on each kernel).
#pragma once
#include <cstddef>
#include <cstdio>

#include "../../include/hk_attn.h"
#include "ptx.cuh"
#include "tma_host.h"

namespace hk {

// ---------------------------------------------------------------- B0
// One group of d/8 lanes per (b, n, h) row (16-B loads), rows in memory order.
template <int D>
__global__ void __launch_bounds__(256) bwd_pre_kernel(const __nv_bfloat16* __restrict__ O,
                                                      const __nv_bfloat16* __restrict__ dO,
                                                      const float* __restrict__ lse, float* __restrict__ Dout,
                                                      float* __restrict__ lse2, int B, int N, int H) {
  constexpr int LPR = D / 8;  // lanes per row
  constexpr int RPW = 32 / LPR;
  const size_t rows = (size_t)B * N * H;
  const int sub = threadIdx.x % LPR;
  const size_t gwarp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const size_t nwarps = (size_t)gridDim.x * blockDim.x / 32;
  const int lrow = (threadIdx.x % 32) / LPR;
  for (size_t base = gwarp * RPW; base < rows; base += nwarps * RPW) {
    const size_t row = base + lrow;
    float acc = 0.f;
    if (row < rows) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(O + row * D) + sub);
      const uint4 g = __ldg(reinterpret_cast<const uint4*>(dO + row * D) + sub);
      const __nv_bfloat162* ap = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&g);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 x = __bfloat1622float2(ap[k]), y = __bfloat1622float2(gp[k]);
        acc = fmaf(x.x, y.x, acc);
        acc = fmaf(x.y, y.y, acc);
      }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (row < rows && sub == 0) {
      const size_t h = row % H, n = (row / H) % N, b = row / ((size_t)H * N);
      const size_t idx = (b * H + h) * N + n;
      Dout[idx] = acc;
      lse2[idx] = lse[idx] * 1.4426950408889634f;
    }
  }
}

struct BwdParams {
  const float* Dv;    // [B][Hq][N]
  const float* lse2;  // [B][Hq][N]
  __nv_bfloat16* dq;  // [B][N][Hq][D]
  __nv_bfloat16* dk;  // [B][N][Hkv][D]
  __nv_bfloat16* dv;  // [B][N][Hkv][D]
  int B, Hq, Hkv, N;
};

// 128 x 128 tiles throughout: tcgen05.mma with N=64 paces at 48 cycles per
// K=16 step instead of 32 (measured, scripts/rates.py), N=128 at full rate.
template <int D>
struct BwdCfg {
  static constexpr int PANELS = D / 64;
  static constexpr uint32_t T128 = 128 * D * 2;  // a 128-row [rows][D] bf16 tile
  static constexpr int NS = (D == 128) ? 2 : 3;  // ring depth
  // B1: K_j, V_j resident + NS x {Q_i, dO_i, lse2_i, D_i}
  static constexpr uint32_t STAGE1 = 2 * T128 + 1024;
  static constexpr uint32_t SMEM1 = 2 * T128 + NS * STAGE1 + 1024;
  // B2: Q_i, dO_i resident + NS x {K_j, V_j}
  static constexpr uint32_t STAGE2 = 2 * T128;
  static constexpr uint32_t SMEM2 = 2 * T128 + NS * STAGE2 + 1024;
  static constexpr int THREADS = 320;  // 8 elementwise warps + TMA warp + MMA warp
};

// SMEM descriptor helpers for [rows][D] bf16 tiles stored as D/64 panels of rows x 128 B.
// K-major use (rows are M or N, D is the contraction): k-step kk of 16 elements.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int rows, int kk) {
  return sdesc_sw128(base + (kk / 4) * rows * 128 + (kk % 4) * 32, 16, 1024);
}
// MN-major use (rows are the contraction, D is N): k-step kk of 16 rows.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int rows, int kk) {
  return sdesc_sw128(base + kk * 16 * 128, rows * 128, 1024);
}
// Packed bf16 operand in TMEM written by two warpgroups: columns 16kk.. of the
// 128-wide contraction live at packed column kk*8 (kk < 4) or 64 + (kk-4)*8.
__device__ __forceinline__ uint32_t packed_col(int kk) { return kk < 4 ? kk * 8 : 64 + (kk - 4) * 8; }

__device__ __forceinline__ void lds_v4(const void* p, float& a, float& b, float& c, float& d) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(smem_u32(p)));
}

// Row of 64 fp32 TMEM columns -> registers.
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&v)[64]) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
  tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
}
__device__ __forceinline__ void tmem_st_packed64(uint32_t taddr, const float (&v)[64]) {
  uint32_t pk[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) pk[c] = pack_bf16(v[2 * c], v[2 * c + 1]);
  tmem_st32(taddr, pk);
}

// ---------------------------------------------------------------- B1: dK, dV
// CTA = (key tile jt, kvh, b); loop h in the GQA group x 128-row query blocks qi.
// TMEM: dV [0,D)  dK [D,2D)  S^T [2D,2D+128)  dP^T [2D+128,2D+256); bf16 P^T / dS^T
// overwrite the first half of each warpgroup's columns of S^T / dP^T.
// MMA order per block: dV(i) [needs P^T(i)], S^T(i+1), dK(i) [needs dS^T(i)],
// dP^T(i+1): the exponentials of block i+1 overlap dK(i)/dP^T(i+1) and the dS
// work overlaps dV(i+1)/S^T(i+2).
template <int D, bool CAUSAL>
__global__ void __launch_bounds__(320, 1)
    bwd_dkdv_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapdO,
                    const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                    const BwdParams p) {
  using C = BwdCfg<D>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::T128;
  uint8_t* sStage = smem + 2 * C::T128;  // stage s: Q [T128] dO [T128] lse2 [512 B] D [512 B]

  __shared__ uint64_t bar_kv, bar_full[NS], bar_empty[NS], bar_s, bar_dp, bar_p, bar_ds, bar_acc;
  __shared__ uint32_t tmem_base_s;

  const int warp = warp_id(), lane = lane_id();
  const int T = p.N / 128;
  const int jt = CAUSAL ? (T - 1 - (int)blockIdx.x) : (int)blockIdx.x;  // key tile (heaviest first)
  const int kvh = blockIdx.y, b = blockIdx.z;
  const int G = p.Hq / p.Hkv;
  const int i0 = CAUSAL ? jt : 0;  // first query block that sees key tile jt
  const int per_h = T - i0;
  const int n_it = G * per_h;

  if (threadIdx.x == 0) {
    mbar_init(&bar_kv, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    mbar_init(&bar_s, 1);
    mbar_init(&bar_dp, 1);
    mbar_init(&bar_p, 8);
    mbar_init(&bar_ds, 8);
    mbar_init(&bar_acc, 1);
    fence_barrier_init();
  }
  if (warp == 8) {
    tma_prefetch(&mapQ);
    tma_prefetch(&mapdO);
    tma_prefetch(&mapK);
    tma_prefetch(&mapV);
  }
  if (warp == 9) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base_s;
  const uint32_t tdV = tb, tdK = tb + D, tS = tb + 2 * D, tP = tb + 2 * D + 128;

  if (warp == 8) {
    // ================= TMA producer =================
    if (lane == 0) {
      const uint64_t pol_keep = policy_evict_last();
      const uint64_t pol_stream = policy_evict_normal();
      mbar_arrive_expect_tx(&bar_kv, 2 * C::T128);
      for (int pn = 0; pn < C::PANELS; ++pn) {
        tma_load_4d(&mapK, &bar_kv, sK + pn * 128 * 128, pn * 64, kvh, jt * 128, b, pol_stream);
        tma_load_4d(&mapV, &bar_kv, sV + pn * 128 * 128, pn * 64, kvh, jt * 128, b, pol_stream);
      }
      int h = kvh * G, qi = i0, s = 0;
      uint32_t ph = 0;
      for (int it = 0; it < n_it; ++it) {
        uint8_t* st = sStage + s * C::STAGE1;
        mbar_wait(&bar_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&bar_full[s], 2 * C::T128 + 1024);
        for (int pn = 0; pn < C::PANELS; ++pn) {
          tma_load_4d(&mapQ, &bar_full[s], st + pn * 128 * 128, pn * 64, h, qi * 128, b, pol_keep);
          tma_load_4d(&mapdO, &bar_full[s], st + C::T128 + pn * 128 * 128, pn * 64, h, qi * 128, b, pol_keep);
        }
        const size_t off = ((size_t)b * p.Hq + h) * p.N + (size_t)qi * 128;
        bulk_load(st + 2 * C::T128, p.lse2 + off, 512, &bar_full[s]);
        bulk_load(st + 2 * C::T128 + 512, p.Dv + off, 512, &bar_full[s]);
        if (++qi == T) {
          qi = i0;
          ++h;
        }
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t idesc_sp = idesc_bf16(128, 128, 0, 0);  // S^T / dP^T: M=128 keys, N=128 queries
      constexpr uint32_t idesc_acc = idesc_bf16(128, D, 0, 1);   // dV / dK: B = dO_i / Q_i MN-major
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
      auto stage_q = [&](int it) { return smem_u32(sStage + (it % NS) * C::STAGE1); };
      auto issue_s = [&](int it) {
        const uint32_t q = stage_q(it);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(tS, desc_kmajor(aK, 128, kk), desc_kmajor(q, 128, kk), idesc_sp, kk > 0);
        tc_commit(&bar_s);
      };
      auto issue_dp = [&](int it) {
        const uint32_t dO = stage_q(it) + C::T128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(tP, desc_kmajor(aV, 128, kk), desc_kmajor(dO, 128, kk), idesc_sp, kk > 0);
        tc_commit(&bar_dp);
      };
      mbar_wait(&bar_kv, 0);
      mbar_wait(&bar_full[0], 0);
      tc_fence_after();
      issue_s(0);
      issue_dp(0);
      for (int it = 0; it < n_it; ++it) {
        const uint32_t q = stage_q(it), dO = q + C::T128;
        const uint32_t acc = it > 0 ? 1u : 0u;
        mbar_wait(&bar_p, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tdV, tS + packed_col(kk), desc_mnmajor(dO, 128, kk), idesc_acc, (acc | kk) ? 1u : 0u);
        const bool more = it + 1 < n_it;
        if (more) {
          mbar_wait(&bar_full[(it + 1) % NS], ((it + 1) / NS) & 1);
          tc_fence_after();
          issue_s(it + 1);
        }
        mbar_wait(&bar_ds, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tdK, tP + packed_col(kk), desc_mnmajor(q, 128, kk), idesc_acc, (acc | kk) ? 1u : 0u);
        if (it + NS < n_it) tc_commit(&bar_empty[it % NS]);
        if (more) issue_dp(it + 1);
      }
      tc_commit(&bar_acc);
    }
  } else {
    // ================= elementwise warpgroups (warps 0-7) =================
    const int wg = warp >> 2;              // query columns [64 wg, 64 wg + 64) of each block
    const uint32_t lb = (warp & 3) * 32;   // TMEM lane base
    const int r = (warp & 3) * 32 + lane;  // key row within the tile
    const int key = jt * 128 + r;
    const float c = 1.4426950408889634f / sqrtf((float)D);
    const uint32_t cS = tS + 64 * wg, cP = tP + 64 * wg;
    int qi = i0, s = 0;
    for (int it = 0; it < n_it; ++it) {
      const uint8_t* vec = sStage + s * C::STAGE1 + 2 * C::T128;  // lse2 [128], then D [128]
      const uint32_t par = it & 1;
      float v[64];
      // ---- phase 1: P^T = exp2(c S^T - LSE2) (masked), bf16 into TMEM for dV += P^T dO
      mbar_wait(&bar_s, par);
      tc_fence_after();
      tmem_ld64(tmem_addr(cS, lb, 0), v);
      tmem_wait_ld();
      const int q0 = qi * 128 + 64 * wg;
#pragma unroll
      for (int c4 = 0; c4 < 64; c4 += 4) {
        float l0, l1, l2, l3;
        lds_v4(vec + 4 * (64 * wg + c4), l0, l1, l2, l3);
        v[c4 + 0] = ex2(fmaf(v[c4 + 0], c, -l0));
        v[c4 + 1] = ex2(fmaf(v[c4 + 1], c, -l1));
        v[c4 + 2] = ex2(fmaf(v[c4 + 2], c, -l2));
        v[c4 + 3] = ex2(fmaf(v[c4 + 3], c, -l3));
      }
      if (CAUSAL && qi == jt) {
#pragma unroll
        for (int cc = 0; cc < 64; ++cc)
          if (q0 + cc < key) v[cc] = 0.f;  // query < key is masked
      }
      tmem_st_packed64(tmem_addr(cS, lb, 0), v);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p);
      // ---- phase 2: dS^T = P^T (dP^T - D), bf16 into TMEM for dK += dS^T Q
      mbar_wait(&bar_dp, par);
      tc_fence_after();
      float dp[64];
      tmem_ld64(tmem_addr(cP, lb, 0), dp);
      tmem_wait_ld();
#pragma unroll
      for (int c4 = 0; c4 < 64; c4 += 4) {
        float d0, d1, d2, d3;
        lds_v4(vec + 512 + 4 * (64 * wg + c4), d0, d1, d2, d3);
        dp[c4 + 0] = v[c4 + 0] * (dp[c4 + 0] - d0);
        dp[c4 + 1] = v[c4 + 1] * (dp[c4 + 1] - d1);
        dp[c4 + 2] = v[c4 + 2] * (dp[c4 + 2] - d2);
        dp[c4 + 3] = v[c4 + 3] * (dp[c4 + 3] - d3);
      }
      tmem_st_packed64(tmem_addr(cP, lb, 0), dp);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_ds);
      if (++qi == T) qi = i0;
      if (++s == NS) s = 0;
    }
    // ---- epilogue: WG0 writes dV, WG1 writes dK * (1/sqrt d)
    mbar_wait(&bar_acc, 0);
    tc_fence_after();
    const float scale = wg == 0 ? 1.f : rsqrtf((float)D);
    const uint32_t tacc = wg == 0 ? tdV : tdK;
    __nv_bfloat16* out = (wg == 0 ? p.dv : p.dk) + (((size_t)b * p.N + key) * p.Hkv + kvh) * D;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t o[32];
      tmem_ld32(tmem_addr(tacc, lb, c0), o);
      tmem_wait_ld();
      uint4 o4[4];
      uint32_t* op = reinterpret_cast<uint32_t*>(o4);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        op[k] = pack_bf16(__uint_as_float(o[2 * k]) * scale, __uint_as_float(o[2 * k + 1]) * scale);
      uint4* dst = reinterpret_cast<uint4*>(out + c0);
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[k] = o4[k];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tb);
}

// ---------------------------------------------------------------- B2: dQ
// CTA = (query tile iq, h, b); loop over 128-key blocks j.
// TMEM: dQ [0,D)  S double buffer [D,D+128) [D+128,D+256)  dP [D+256,D+384);
// bf16 dS overwrites dP. MMA order: S(j+1), dQ(j) [needs dS(j)], dP(j+1).
template <int D, bool CAUSAL>
__global__ void __launch_bounds__(320, 1)
    bwd_dq_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapdO,
                  const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                  const BwdParams p) {
  using C = BwdCfg<D>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + C::T128;
  uint8_t* sStage = smem + 2 * C::T128;  // stage s: K_j [T128] V_j [T128]

  __shared__ uint64_t bar_q, bar_full[NS], bar_empty[NS], bar_s[2], bar_dp, bar_ds, bar_acc;
  __shared__ uint32_t tmem_base_s;

  const int warp = warp_id(), lane = lane_id();
  const int T = p.N / 128;
  const int iq = CAUSAL ? (T - 1 - (int)blockIdx.x) : (int)blockIdx.x;  // query tile (heaviest first)
  const int h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (p.Hq / p.Hkv);
  const int n_it = CAUSAL ? iq + 1 : T;  // 128-key blocks

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    mbar_init(&bar_s[0], 1);
    mbar_init(&bar_s[1], 1);
    mbar_init(&bar_dp, 1);
    mbar_init(&bar_ds, 8);
    mbar_init(&bar_acc, 1);
    fence_barrier_init();
  }
  if (warp == 8) {
    tma_prefetch(&mapQ);
    tma_prefetch(&mapdO);
    tma_prefetch(&mapK);
    tma_prefetch(&mapV);
  }
  if (warp == 9) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base_s;
  const uint32_t tdQ = tb, tS0 = tb + D, tP = tb + D + 256;

  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol_keep = policy_evict_last();
      const uint64_t pol_stream = policy_evict_normal();
      mbar_arrive_expect_tx(&bar_q, 2 * C::T128);
      for (int pn = 0; pn < C::PANELS; ++pn) {
        tma_load_4d(&mapQ, &bar_q, sQ + pn * 128 * 128, pn * 64, h, iq * 128, b, pol_stream);
        tma_load_4d(&mapdO, &bar_q, sdO + pn * 128 * 128, pn * 64, h, iq * 128, b, pol_stream);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0; it < n_it; ++it) {
        uint8_t* st = sStage + s * C::STAGE2;
        mbar_wait(&bar_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&bar_full[s], 2 * C::T128);
        for (int pn = 0; pn < C::PANELS; ++pn) {
          tma_load_4d(&mapK, &bar_full[s], st + pn * 128 * 128, pn * 64, kvh, it * 128, b, pol_keep);
          tma_load_4d(&mapV, &bar_full[s], st + C::T128 + pn * 128 * 128, pn * 64, kvh, it * 128, b, pol_keep);
        }
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t idesc_sp = idesc_bf16(128, 128, 0, 0);  // S / dP: M=128 queries, N=128 keys
      constexpr uint32_t idesc_acc = idesc_bf16(128, D, 0, 1);   // dQ += dS K_j: K_j MN-major
      const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO);
      auto stage_k = [&](int it) { return smem_u32(sStage + (it % NS) * C::STAGE2); };
      auto issue_s = [&](int it) {
        const uint32_t k = stage_k(it);
        const uint32_t t = tS0 + 128 * (it & 1);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(t, desc_kmajor(aQ, 128, kk), desc_kmajor(k, 128, kk), idesc_sp, kk > 0);
        tc_commit(&bar_s[it & 1]);
      };
      auto issue_dp = [&](int it) {
        const uint32_t v = stage_k(it) + C::T128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(tP, desc_kmajor(adO, 128, kk), desc_kmajor(v, 128, kk), idesc_sp, kk > 0);
        tc_commit(&bar_dp);
      };
      mbar_wait(&bar_q, 0);
      mbar_wait(&bar_full[0], 0);
      tc_fence_after();
      issue_s(0);
      issue_dp(0);
      for (int it = 0; it < n_it; ++it) {
        const bool more = it + 1 < n_it;
        if (more) {
          mbar_wait(&bar_full[(it + 1) % NS], ((it + 1) / NS) & 1);
          tc_fence_after();
          issue_s(it + 1);
        }
        mbar_wait(&bar_ds, it & 1);
        tc_fence_after();
        const uint32_t k = stage_k(it);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tdQ, tP + packed_col(kk), desc_mnmajor(k, 128, kk), idesc_acc, (it > 0 || kk > 0) ? 1u : 0u);
        if (it + NS < n_it) tc_commit(&bar_empty[it % NS]);
        if (more) issue_dp(it + 1);
      }
      tc_commit(&bar_acc);
    }
  } else {
    const int wg = warp >> 2;              // key columns [64 wg, 64 wg + 64) of each block
    const uint32_t lb = (warp & 3) * 32;
    const int r = (warp & 3) * 32 + lane;  // query row within the tile
    const int q = iq * 128 + r;
    const float c = 1.4426950408889634f / sqrtf((float)D);
    const size_t vrow = ((size_t)b * p.Hq + h) * p.N + q;
    const float l2 = p.lse2[vrow], Dq = p.Dv[vrow];
    const uint32_t cP = tP + 64 * wg;
    for (int it = 0; it < n_it; ++it) {
      const uint32_t cS = tS0 + 128 * (it & 1) + 64 * wg;
      float v[64];
      mbar_wait(&bar_s[it & 1], (it >> 1) & 1);
      tc_fence_after();
      tmem_ld64(tmem_addr(cS, lb, 0), v);
      tmem_wait_ld();
#pragma unroll
      for (int cc = 0; cc < 64; ++cc) v[cc] = ex2(fmaf(v[cc], c, -l2));
      if (CAUSAL && it == iq) {
        const int k0 = it * 128 + 64 * wg;
#pragma unroll
        for (int cc = 0; cc < 64; ++cc)
          if (k0 + cc > q) v[cc] = 0.f;
      }
      mbar_wait(&bar_dp, it & 1);
      tc_fence_after();
      float dp[64];
      tmem_ld64(tmem_addr(cP, lb, 0), dp);
      tmem_wait_ld();
#pragma unroll
      for (int cc = 0; cc < 64; ++cc) dp[cc] = v[cc] * (dp[cc] - Dq);
      tmem_st_packed64(tmem_addr(cP, lb, 0), dp);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_ds);
    }
    // ---- epilogue: dQ * (1/sqrt d); WG0 writes columns [0, D/2), WG1 [D/2, D)
    mbar_wait(&bar_acc, 0);
    tc_fence_after();
    const float scale = rsqrtf((float)D);
    __nv_bfloat16* out = p.dq + (((size_t)b * p.N + q) * p.Hq + h) * D;
#pragma unroll
    for (int c0 = wg * (D / 2); c0 < (wg + 1) * (D / 2); c0 += 32) {
      uint32_t o[32];
      tmem_ld32(tmem_addr(tdQ, lb, c0), o);
      tmem_wait_ld();
      uint4 o4[4];
      uint32_t* op = reinterpret_cast<uint32_t*>(o4);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        op[k] = pack_bf16(__uint_as_float(o[2 * k]) * scale, __uint_as_float(o[2 * k + 1]) * scale);
      uint4* dst = reinterpret_cast<uint4*>(out + c0);
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[k] = o4[k];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tb);
}

// ---------------------------------------------------------------- host launch
template <typename F>
inline bool set_smem(F* fn, uint32_t bytes) {
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)bytes) == cudaSuccess;
}

template <int D, bool CAUSAL>
hk_status launch_bwd_t(const void* Q, const void* K, const void* V, const void* O, const float* LSE, const void* dO,
                       void* dQ, void* dK, void* dV, float* ws, int B, int Hq, int Hkv, int N, cudaStream_t stream,
                       char* err, size_t errlen, int phase) {
  using C = BwdCfg<D>;
  float* Dv = ws;
  float* lse2 = ws + (size_t)B * Hq * N;
  // every operand tile is a 128-row box (two 64-column panels at D=128)
  CUtensorMap mQ, mdO, mK, mV;
  bool ok = encode_bnhd(&mQ, Q, B, N, Hq, D, 128) && encode_bnhd(&mdO, dO, B, N, Hq, D, 128) &&
            encode_bnhd(&mK, K, B, N, Hkv, D, 128) && encode_bnhd(&mV, V, B, N, Hkv, D, 128);
  if (!ok) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled failed");
    return HK_ERR_DEVICE;
  }
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !attr_done[dev]) {
    if (!set_smem(bwd_dkdv_kernel<D, CAUSAL>, C::SMEM1) || !set_smem(bwd_dq_kernel<D, CAUSAL>, C::SMEM2)) {
      snprintf(err, errlen, "cudaFuncSetAttribute(max dynamic smem) failed");
      return HK_ERR_DEVICE;
    }
    if (dev < 64) attr_done[dev] = true;
  }
  BwdParams p{Dv, lse2, reinterpret_cast<__nv_bfloat16*>(dQ), reinterpret_cast<__nv_bfloat16*>(dK),
              reinterpret_cast<__nv_bfloat16*>(dV), B, Hq, Hkv, N};
  // B0
  const size_t rows = (size_t)B * N * Hq;
  const size_t warps_needed = (rows + (32 / (D / 8)) - 1) / (32 / (D / 8));
  size_t blocks = (warps_needed + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (phase < 0 || phase == 0)
    bwd_pre_kernel<D><<<(unsigned)blocks, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(O),
                                                              reinterpret_cast<const __nv_bfloat16*>(dO), LSE, Dv,
                                                              lse2, B, N, Hq);
  // B1, B2
  if (phase < 0 || phase == 1)
    bwd_dkdv_kernel<D, CAUSAL><<<dim3(N / 128, Hkv, B), C::THREADS, C::SMEM1, stream>>>(mQ, mdO, mK, mV, p);
  if (phase < 0 || phase == 2)
    bwd_dq_kernel<D, CAUSAL><<<dim3(N / 128, Hq, B), C::THREADS, C::SMEM2, stream>>>(mQ, mdO, mK, mV, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(err, errlen, "hk_attn_bwd launch failed: %s", cudaGetErrorString(e));
    return HK_ERR_LAUNCH;
  }
  return HK_OK;
}

inline hk_status launch_bwd(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                            const void* dO, void* dQ, void* dK, void* dV, float* ws, int B, int Hq, int Hkv, int N,
                            int d, bool causal, cudaStream_t stream, char* err, size_t errlen, int phase) {
  if (d == 64)
    return causal ? launch_bwd_t<64, true>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, B, Hq, Hkv, N, stream, err, errlen, phase)
                  : launch_bwd_t<64, false>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, B, Hq, Hkv, N, stream, err, errlen, phase);
  return causal ? launch_bwd_t<128, true>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, B, Hq, Hkv, N, stream, err, errlen, phase)
                : launch_bwd_t<128, false>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, B, Hq, Hkv, N, stream, err, errlen, phase);
}

}  // namespace hk
