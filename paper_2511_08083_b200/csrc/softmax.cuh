// One online-softmax step of the forward pass for one query row per thread
// (PAPER.md P:1338-1340): read the 128 scores of
// this row from TMEM, row max, P = 2^(c s - m) packed to bf16 back into TMEM
// (over the scores, as the A operand of O += P V), row sum, and the lazy O
// rescale. Shared by fwd_kernel and the softmax_rate micro-benchmark.
#pragma once
#include "ptx.cuh"

namespace hk {

constexpr float RESCALE_TH = 8.0f;
constexpr float EXP_MAGIC = 12582912.f;  // 1.5 * 2^23: x + magic rounds x to an integer in the low mantissa

// P for 32 consecutive scores (16 pairs), packed to bf16 pairs; the row sum is
// accumulated in `acc`. EMU_OF_8 of every 8 pairs are evaluated on the FMA
// pipe: with an integral running max m, j = c s + (magic - m) holds
// n = rint(c s - m) in its mantissa, f = c s - m - n is recovered exactly from
// (magic - m) - j, 2^f comes from a degree-3 minimax polynomial (relative
// error 7.7e-5 < bf16's 3.9e-3) and n is added into the exponent bits. Scores
// are clamped so c s - m >= -125 (the exponent add cannot underflow).
template <bool EMU, int EMU_OF_8, bool ROWSUM = false>
__device__ __forceinline__ void softmax_chunk32(const float* s, float c, float m, float smin, uint32_t (&pk)[16],
                                                float2 (&acc)[2]) {
  const float2 c2 = make_float2(c, c), nm2 = make_float2(-m, -m);
  const float2 bias2 = make_float2(EXP_MAGIC - m, EXP_MAGIC - m);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    float2 e;
    if (EMU && (k % 8) < EMU_OF_8) {
      const float2 sc = make_float2(fmaxf(s[2 * k], smin), fmaxf(s[2 * k + 1], smin));
      const float2 j = fma2(sc, c2, bias2);
      const float2 f = fma2(sc, c2, sub2(bias2, j));
#ifndef HK_FWD_POLY2
#define HK_FWD_POLY2 1  // 1.01-1.03x (profiles/ab_fwd_poly2_r2l.jsonl); reading #27
#endif
      float2 q;
      if (HK_FWD_POLY2) {  // degree 2 (max relative error 1.7e-3, below bf16's half ulp 2^-9)
        q = fma2(make_float2(0.23842824f, 0.23842824f), f, make_float2(0.70344784f, 0.70344784f));
        q = fma2(q, f, make_float2(1.00044318f, 1.00044318f));
      } else {
        q = fma2(make_float2(0.05508885905f, 0.05508885905f), f, make_float2(0.242604658f, 0.242604658f));
        q = fma2(q, f, make_float2(0.6932762861f, 0.6932762861f));
        q = fma2(q, f, make_float2(0.999928891658f, 0.999928891658f));
      }
      e = make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(j.x) << 23)),
                      __int_as_float(__float_as_int(q.y) + (__float_as_int(j.y) << 23)));
    } else {
      const float2 x = fma2(make_float2(s[2 * k], s[2 * k + 1]), c2, nm2);
      e = make_float2(ex2(x.x), ex2(x.y));
    }
    if (!ROWSUM) acc[k & 1] = add2(acc[k & 1], e);  // ROWSUM: the P V MMA sums the row (ones column of V)
    pk[k] = pack_bf16(e.x, e.y);
  }
}

// tS: this tile's score columns (fp32 S in, bf16 P out over its first 64
// columns); tO: its O accumulator (rescaled in place when the max moves).
// m, l: running max (log2 units, always integral) and row sum. `shift`: causal
// limit — key column cc is visible to row r iff cc <= r + shift (a large value
// = no causal limit; 0 on the square diagonal tile); `kvalid` < 128: only the
// first kvalid keys of this block exist (ragged / varlen tail). Masked blocks
// run all exps on the MUFU so a masked P is exactly 0; a row that has seen no
// key so far keeps m = -inf and l = 0 (reading #22). `o_live`: O already
// holds earlier P V products.
// Split-P mode (tP != tS, the d=64 forward): P goes to its own TMEM columns, the
// S columns are released (bar_sfree) as soon as S is in registers so the next
// S = Q K^T can overwrite them while this step runs, and the step waits for the
// previous P V (bar_pv) before it rescales O or overwrites P.
// ROWSUM (d = 64): O carries a 17th 16-column block whose first column accumulates P . 1 (a ones
// column appended to V), so the row sum l comes from the tensor core: the step skips its adds
// (l is left untouched) and the O rescale covers ON = D + 16 columns.
template <int D, int EMU_OF_8, bool ROWSUM = false>
__device__ __forceinline__ void softmax_step(uint32_t tS, uint32_t tO, uint32_t lane_base, int r, float c,
                                             float& m, float& l, int shift, bool o_live, int kvalid = 128,
                                             int trace_ev = -1, uint32_t trace_idx = 0, uint64_t* bar_lo = nullptr,
                                             uint32_t tP = 0, uint64_t* bar_sfree = nullptr,
                                             uint64_t* bar_pv = nullptr, uint32_t* pv_phase = nullptr,
                                             int alt_wait = -1, int alt_arrive = -1) {
  if (tP == 0) tP = tS;
#ifdef HK_TRACE
  const bool tr = trace_ev >= 0 && (threadIdx.x % 128) == 0;
#define HK_SM_TRACE(k) \
  if (tr) hk_trace(trace_ev + (k), trace_idx, 0);
#else
#define HK_SM_TRACE(k)
#endif
  float s[128];
#pragma unroll
  for (int c0 = 0; c0 < 128; c0 += 32)
    tmem_ld32(tmem_addr(tS, lane_base, c0), *reinterpret_cast<uint32_t(*)[32]>(&s[c0]));
  tmem_wait_ld();
  if (bar_sfree != nullptr) {  // S columns free for the next S = Q K^T
    tc_fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar_sfree);
  }
  HK_SM_TRACE(0)  // S in registers
  const bool masked = shift < 127 || kvalid < 128;
  if (masked) {
    const int lim = r + 1 + shift < kvalid ? r + 1 + shift : kvalid;  // keys [0, lim) visible (lim may be <= 0)
#pragma unroll
    for (int cc = 0; cc < 128; ++cc)
      if (cc >= lim) s[cc] = -INFINITY;
  }
  // row max: 8 independent 3-input-max chains, then combine
  float mx8[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) mx8[a] = fmaxf(s[a], s[a + 8]);
#pragma unroll
  for (int k = 16; k < 128; k += 16)
#pragma unroll
    for (int a = 0; a < 8; ++a) mx8[a] = max3f(mx8[a], s[k + a], s[k + 8 + a]);
  const float mx = max3f(max3f(mx8[0], mx8[1], mx8[2]), max3f(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
  const float mxs = mx * c;
  float m_use = m, alpha = 1.f;
  if (mxs > m + RESCALE_TH) {  // also taken on the first tile (m = -inf)
    m_use = ceilf(mxs);        // integral max: exact f in the polynomial exp
    alpha = ex2(m - m_use);
  }
  // scores below smin would take the emulated 2^x under 2^-125; multiply by 1/c (a division
  // here compiled to the IEEE slow path: FCHK + call, every step)
  const float smin = (m_use - 125.f) * __frcp_rn(c);
  HK_SM_TRACE(1)  // row max done
  if (bar_pv != nullptr) {  // split P: the previous P V must be complete (O and P reused)
    mbar_wait(bar_pv, *pv_phase);
    *pv_phase ^= 1;
    tc_fence_after();
  }
  // O holds P(j-1) V_{j-1}, complete: the S barrier (split P: bar_pv) tracked every
  // earlier MMA. The rescale comes before any part of P(j) is published (P V(j)
  // accumulates onto it).
  if (o_live && __any_sync(0xffffffffu, alpha != 1.f)) {
    // 16 columns at a time: the 128 scores are still live here
#pragma unroll 1
    for (int c0 = 0; c0 < (ROWSUM ? D + 16 : D); c0 += 16) {
      float o[16];
      tmem_ld16(tmem_addr(tO, lane_base, c0), reinterpret_cast<uint32_t*>(o));
      tmem_wait_ld();
#pragma unroll
      for (int cc = 0; cc < 16; cc += 2) {
        const float2 v = mul2(make_float2(o[cc], o[cc + 1]), make_float2(alpha, alpha));
        o[cc] = v.x;
        o[cc + 1] = v.y;
      }
      tmem_st16(tmem_addr(tO, lane_base, c0), reinterpret_cast<const uint32_t*>(o));
    }
    tmem_wait_st();
  }
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  // Exponential phases of the two Q tiles' warpgroups take turns (named barriers alt_wait /
  // alt_arrive, 256 threads = both warpgroups): each runs with the SM's MUFU and FMA pipes to
  // itself, in the order the MMA warp consumes P (tile 0, then tile 1).
  if (alt_wait >= 0) named_bar_sync(alt_wait, 256);
#ifndef HK_FWD_STLATE
#define HK_FWD_STLATE 1  // 1.003-1.027x (profiles/ab_fwd_stlate_r2l.jsonl)
#endif
#pragma unroll
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t pk[16];
    if (masked)  // a row with no visible key yet (m_use = -inf) gets P = 2^-inf = 0, not NaN
      softmax_chunk32<false, EMU_OF_8, ROWSUM>(s + c0, c, m_use == -INFINITY ? 0.f : m_use, smin, pk, acc);
    else
      softmax_chunk32<true, EMU_OF_8, ROWSUM>(s + c0, c, m_use, smin, pk, acc);
    // HK_FWD_STLATE: publish the first half of P after the third chunk's exponentials, so the
    // wait for the first two chunks' TMEM stores hides behind that work
    const int pub = HK_FWD_STLATE ? 64 : 32;
    if (HK_FWD_STLATE && bar_lo != nullptr && c0 == pub) {
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(bar_lo);
    }
    tmem_st16(tmem_addr(tP, lane_base, c0 / 2), pk);
    if (!HK_FWD_STLATE && bar_lo != nullptr && c0 == pub) {  // P of keys [0, 64) (and the O rescale) in
      tmem_wait_st();                                         // TMEM: the first half of P V may start
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(bar_lo);
    }
  }
  if (alt_arrive >= 0) named_bar_arrive(alt_arrive, 256);
  HK_SM_TRACE(2)  // exps done, P stores issued
  if (!ROWSUM) {
    const float2 rs2 = add2(acc[0], acc[1]);
    l = l * alpha + (rs2.x + rs2.y);
  }
  m = m_use;
#undef HK_SM_TRACE
}

}  // namespace hk
