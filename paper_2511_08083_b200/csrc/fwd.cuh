// Forward fused attention for sm_100a: TMA -> SMEM (128B swizzle) -> tcgen05
// (S = Q K^T and O += P V, accumulators in TMEM) with the online softmax in
// registers between them.
//
// Method: scores with the softmax scale folded into exp2
// (TEMPERATURE_SCALE = (1/sqrt(d)) log2 e), running max / exp2 /
// row sum (col_max, sub_col, exp2, col_sum: P:1338-1340), O
// rescaled by exp2(m_old - m_new) before P V accumulates (mul_col then
// mma_AtB: P:1398-1400), LSE = max ln2 + ln(norm).
//
// B200 design: one CTA = (b, h, two 128-row Q tiles).
//   warps 0-3  softmax WG0: Q tile 0, one thread per query row (TMEM lane)
//   warps 4-7  softmax WG1: Q tile 1
//   warp  8    TMA producer: Q0/Q1 once, then a K ring and a V ring
//   warp  9    MMA issuer (one thread): S_t = Q_t K_j^T, O_t += P_t V_j
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// bf16 P_t is written over S_t's first 64 columns (A operand from TMEM).
// The two Q tiles ping-pong: while WG0 does softmax on S0(j+1) the tensor
// core runs P1(j) V_j and S1(j+1), and vice versa.
// O rescale is lazy: the running max only moves when it grows by more than
// RESCALE_TH (log2 units); l and O always share the same (possibly stale)
// max, which is exact in exact arithmetic (reading #8).
#pragma once
#include "ptx.cuh"

namespace hk {

struct FwdParams {
  float* lse;   // [B][Hq][N]
  __nv_bfloat16* o;  // [B][N][Hq][D]
  int B, Hq, Hkv, N;
  int num_pairs;  // ceil(N / 256)
};

template <int D>
struct FwdCfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int PANELS = D / 64;
  static constexpr uint32_t TILE_BYTES = 128 * D * 2;  // one 128-row tile
  static constexpr int NS = (D == 128) ? 2 : 4;        // K/V ring depth
  static constexpr uint32_t SMEM = 2 * TILE_BYTES + 2 * NS * TILE_BYTES + 1024;
  static constexpr int THREADS = 384;
};

constexpr float RESCALE_TH = 8.0f;

template <int D, bool CAUSAL>
__global__ void __launch_bounds__(384, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
               const __grid_constant__ CUtensorMap mapV, const FwdParams p) {
  using C = FwdCfg<D>;
  constexpr int NS = C::NS;
  constexpr uint32_t TB = C::TILE_BYTES;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // 2 tiles
  uint8_t* sK = smem + 2 * TB;        // NS tiles
  uint8_t* sV = sK + NS * TB;         // NS tiles

  __shared__ uint64_t bar_q, bar_kfull[NS], bar_kempty[NS], bar_vfull[NS], bar_vempty[NS];
  __shared__ uint64_t bar_s[2], bar_p[2], bar_o[2];
  __shared__ uint32_t tmem_base_s;

  const int warp = warp_id();
  const int lane = lane_id();

  // ---- work decomposition: x = Q-tile pair (heaviest first when causal), y = head, z = batch
  const int pair = CAUSAL ? (p.num_pairs - 1 - (int)blockIdx.x) : (int)blockIdx.x;
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int kvh = h / (p.Hq / p.Hkv);
  const int T = p.N / 128;             // 128-row tiles along the sequence
  const int qt0 = 2 * pair, qt1 = 2 * pair + 1;
  const bool has1 = qt1 < T;
  const int nkv0 = CAUSAL ? qt0 + 1 : T;
  const int nkv1 = has1 ? (CAUSAL ? qt1 + 1 : T) : 0;
  const int nkv = nkv1 > nkv0 ? nkv1 : nkv0;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bar_kfull[s], 1);
      mbar_init(&bar_kempty[s], 1);
      mbar_init(&bar_vfull[s], 1);
      mbar_init(&bar_vempty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t], 1);
      mbar_init(&bar_p[t], 4);
      mbar_init(&bar_o[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 8) {
    tma_prefetch(&mapQ);
    tma_prefetch(&mapK);
    tma_prefetch(&mapV);
  }
  if (warp == 9) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  const uint32_t tS[2] = {tbase, tbase + 128};
  const uint32_t tO[2] = {tbase + 256, tbase + 256 + D};

  if (warp == 8) {
    // ================= TMA producer =================
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      mbar_arrive_expect_tx(&bar_q, (has1 ? 2 : 1) * TB);
      for (int pnl = 0; pnl < C::PANELS; ++pnl) {
        tma_load_4d(&mapQ, &bar_q, sQ + pnl * 128 * 128, pnl * 64, h, qt0 * 128, b, pol_q);
        if (has1) tma_load_4d(&mapQ, &bar_q, sQ + TB + pnl * 128 * 128, pnl * 64, h, qt1 * 128, b, pol_q);
      }
      for (int j = 0; j < nkv; ++j) {
        const int s = j % NS;
        const uint32_t ph = (j / NS) & 1;
        mbar_wait(&bar_kempty[s], ph ^ 1);
        mbar_arrive_expect_tx(&bar_kfull[s], TB);
        for (int pnl = 0; pnl < C::PANELS; ++pnl)
          tma_load_4d(&mapK, &bar_kfull[s], sK + s * TB + pnl * 128 * 128, pnl * 64, kvh, j * 128, b, pol_kv);
        mbar_wait(&bar_vempty[s], ph ^ 1);
        mbar_arrive_expect_tx(&bar_vfull[s], TB);
        for (int pnl = 0; pnl < C::PANELS; ++pnl)
          tma_load_4d(&mapV, &bar_vfull[s], sV + s * TB + pnl * 128 * 128, pnl * 64, kvh, j * 128, b, pol_kv);
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);  // S = Q K^T: A K-major, B K-major
      constexpr uint32_t idesc_o = idesc_bf16(128, D, 0, 1);    // O += P V: A TMEM, B (V) MN-major
      const int nk[2] = {nkv0, nkv1};
      auto issue_s = [&](int t, int s) {
        const uint32_t qa = smem_u32(sQ + t * TB);
        const uint32_t ka = smem_u32(sK + s * TB);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * 128 * 128 + (kk % 4) * 32;
          umma_ss(tS[t], sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(ka + off, 16, 1024), idesc_s, kk > 0);
        }
      };
      auto issue_pv = [&](int t, int s, int j) {
        const uint32_t va = smem_u32(sV + s * TB);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          umma_ts(tO[t], tS[t] + kk * 8, sdesc_sw128(va + kk * 16 * 128, 128 * 128, 1024), idesc_o,
                  (j > 0 || kk > 0) ? 1u : 0u);
      };
      mbar_wait(&bar_q, 0);
      mbar_wait(&bar_kfull[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      tc_commit(&bar_s[0]);
      if (nk[1] > 0) {
        issue_s(1, 0);
        tc_commit(&bar_s[1]);
      }
      tc_commit(&bar_kempty[0]);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % NS;
        const uint32_t ph = (j / NS) & 1;
        const int s1 = (j + 1) % NS;
        const uint32_t ph1 = ((j + 1) / NS) & 1;
        mbar_wait(&bar_vfull[s], ph);
        bool k_next_waited = false;
        for (int t = 0; t < 2; ++t) {
          if (j >= nk[t]) continue;
          mbar_wait(&bar_p[t], j & 1);
          tc_fence_after();
          issue_pv(t, s, j);
          if (j + 1 < nk[t]) {
            if (!k_next_waited) {
              mbar_wait(&bar_kfull[s1], ph1);
              tc_fence_after();
              k_next_waited = true;
            }
            issue_s(t, s1);
            tc_commit(&bar_s[t]);
          } else {
            tc_commit(&bar_o[t]);
          }
        }
        tc_commit(&bar_vempty[s]);
        if (k_next_waited) tc_commit(&bar_kempty[s1]);
      }
    }
  } else if (warp < 8) {
    // ================= softmax warpgroups =================
    const int t = warp >> 2;  // Q tile of this warpgroup
    const int nk = t == 0 ? nkv0 : nkv1;
    if (nk > 0) {
      const int qt = t == 0 ? qt0 : qt1;
      const uint32_t lane_base = (warp & 3) * 32;
      const int r = (warp & 3) * 32 + lane;  // row within the Q tile == TMEM lane
      const float c = 1.4426950408889634f / sqrtf((float)D);  // (1/sqrt d) log2 e
      float m = -INFINITY;  // running max, log2-scaled units
      float l = 0.f;        // running row sum
      for (int j = 0; j < nk; ++j) {
        mbar_wait(&bar_s[t], j & 1);
        tc_fence_after();
        uint32_t sr[128];
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32)
          tmem_ld32(tmem_addr(tS[t], lane_base, c0), *reinterpret_cast<uint32_t(*)[32]>(&sr[c0]));
        tmem_wait_ld();
        float* s = reinterpret_cast<float*>(sr);
        if (CAUSAL && j == qt) {
#pragma unroll
          for (int cc = 0; cc < 128; ++cc)
            if (cc > r) s[cc] = -INFINITY;  // key j*128+cc > query qt*128+r
        }
        float mx = s[0];
#pragma unroll
        for (int cc = 1; cc < 128; ++cc) mx = fmaxf(mx, s[cc]);
        const float mxs = mx * c;
        float m_use = m, alpha = 1.f;
        if (mxs > m + RESCALE_TH) {  // also taken on the first tile (m = -inf)
          m_use = mxs;
          alpha = ex2(m - m_use);
        }
        float rs = 0.f;
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int cc = 0; cc < 32; cc += 2) {
            const float p0 = ex2(fmaf(s[c0 + cc], c, -m_use));
            const float p1 = ex2(fmaf(s[c0 + cc + 1], c, -m_use));
            rs += p0 + p1;
            pk[cc / 2] = pack_bf16(p0, p1);
          }
          tmem_st16(tmem_addr(tS[t], lane_base, c0 / 2), pk);
        }
        l = l * alpha + rs;
        // O_t holds P_t(j-1) V_{j-1}: complete, since bar_s[t] tracked every earlier MMA.
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tmem_addr(tO[t], lane_base, c0), o);
            tmem_wait_ld();
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) o[cc] = __float_as_uint(__uint_as_float(o[cc]) * alpha);
            tmem_st32(tmem_addr(tO[t], lane_base, c0), o);
          }
        }
        m = m_use;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_p[t]);
      }
      // ---- epilogue: O = O_acc / l (bf16), LSE = (m + log2 l) ln 2
      mbar_wait(&bar_o[t], 0);
      tc_fence_after();
      const float inv_l = 1.f / l;
      const int row = qt * 128 + r;
      __nv_bfloat16* orow = p.o + (((size_t)b * p.N + row) * p.Hq + h) * D;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t o[32];
        tmem_ld32(tmem_addr(tO[t], lane_base, c0), o);
        tmem_wait_ld();
        uint4 v[4];
        uint32_t* vp = reinterpret_cast<uint32_t*>(v);
#pragma unroll
        for (int cc = 0; cc < 16; ++cc)
          vp[cc] = pack_bf16(__uint_as_float(o[2 * cc]) * inv_l, __uint_as_float(o[2 * cc + 1]) * inv_l);
        uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = v[q];
      }
      p.lse[((size_t)b * p.Hq + h) * p.N + row] = (m + __log2f(l)) * 0.69314718055994531f;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tbase);
}

}  // namespace hk
