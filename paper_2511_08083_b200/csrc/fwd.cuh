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
//   warps 10-11 idle (WG2 = warps 8-11 drops to 112 registers, WG0/WG1 rise to 192:
//   128*112 + 256*192 = 63488 <= 64512, the CTA pool at launch, 384 x 168)
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// bf16 P_t is written over S_t's first 64 columns (A operand from TMEM).
// The two Q tiles ping-pong: while WG0 does softmax on S0(j+1) the tensor
// core runs P1(j) V_j and S1(j+1), and vice versa.
// O rescale is lazy: the running max only moves when it grows by more than
// RESCALE_TH (log2 units); l and O always share the same (possibly stale)
// max, which is exact in exact arithmetic (reading #8).
// Softmax issue economy: 3-input max, packed f32x2 FMA/ADD,
// and EMU_OF_8/8 of the exponentials evaluated by a polynomial on the FMA
// pipe instead of the MUFU (16 ex2/clk/SM, the co-bottleneck at d=128).
#pragma once
#include "ptx.cuh"
#include "sched.cuh"
#include "seq.cuh"
#include "rope.cuh"
#include "softmax.cuh"

namespace hk {

struct FwdParams {
  float* lse;        // dense [B][Hq][Nq]; varlen [Hq][total_q]
  __nv_bfloat16* o;  // dense [B][Nq][Hq][D]; varlen [total_q][Hq][D]
  SeqGeom g;         // dense / varlen geometry (seq.cuh)
  int B, Hq, Hkv;
  int num_pairs;  // ceil(Nq / 256): Q-tile pairs per head (varlen: of the longest sequence)
  int num_items;  // B * Hq * num_pairs work items
  unsigned* sched;  // [2] work counters: dynamic scheduling (varlen with a workspace); nullptr = static snake
  const float* rope_cos;  // ROPE: [N][D/2] fp32 (position = query row), the fused rotary of Q
  const float* rope_sin;
};

template <int D>
struct FwdCfg {
  static constexpr int PANELS = D / 64;
  // d=64: TMEM has room for P next to S (S0 S1 O0 O1 P0 P1 = 128+128+64+64+64+64), so S can be
  // released as soon as it is read and the next Q K^T overlaps the softmax (split P).
#ifndef HK_FWD_SPLIT64
#define HK_FWD_SPLIT64 0  // measured slower (DESIGN.md §8 "did not pay"): off
#endif
  static constexpr bool SPLIT_P = (D == 64) && HK_FWD_SPLIT64;
  static constexpr uint32_t TILE_BYTES = 128 * D * 2;  // one 128-row tile
#ifndef HK_FWD_NS64
#define HK_FWD_NS64 4
#endif
  static constexpr int NS = (D == 128) ? 2 : HK_FWD_NS64;  // K/V ring depth
#ifndef HK_FWD_ROWSUM
#define HK_FWD_ROWSUM 1  // C4 forward 1.05-1.08x (profiles/ab_fwd_rowsum_r2p.jsonl); reading #28
#endif
  // d = 64: the row sum l by the tensor core (softmax.cuh ROWSUM): O_t is ON = D + 16 columns and
  // V gains a second MN-major panel (a constant 16 KB tile whose column 0 is 1), reached through
  // each V slot's descriptor LBO
  static constexpr bool ROWSUM = (D == 64) && HK_FWD_ROWSUM;
  static constexpr int ON = ROWSUM ? D + 16 : D;
  // epilogue staging: one 16 KB SW128 panel [128 rows][64 columns] bf16 per Q tile; O leaves through a TMA
  // store of whole rows instead of per-thread row stores (HK_FWD_OSTAGE)
#ifndef HK_FWD_OSTAGE
#define HK_FWD_OSTAGE 1
#endif
  static constexpr bool OSTAGE = HK_FWD_OSTAGE != 0;
  static constexpr uint32_t STAGE_BYTES = OSTAGE ? 2 * 128 * 128 : 0;
  static constexpr uint32_t SMEM =
      2 * TILE_BYTES + 2 * NS * TILE_BYTES + (ROWSUM ? 128 * 128 : 0) + STAGE_BYTES + 1024;
  static constexpr int THREADS = 384;
#ifndef HK_FWD_EMU128
#define HK_FWD_EMU128 3
#endif
#ifndef HK_FWD_EMU64
#define HK_FWD_EMU64 4  // with the row sum on the tensor core: 1.02x at C4-8192 (profiles/ab_fwd_emu64_r2q.jsonl)
#endif
  static constexpr int EMU_OF_8 = (D == 128) ? HK_FWD_EMU128 : HK_FWD_EMU64;  // exps per 8 on the FMA pipe
#ifndef HK_FWD_ALT
#define HK_FWD_ALT 0
#endif
  static constexpr bool ALT = HK_FWD_ALT != 0;  // the two tiles' exponential phases take turns
};

// One work item = (b, h, pair of 128-row Q tiles). Items are numbered so that
// the items of one (b, kvh) group (its G query heads x all pairs, which share
// K and V) are consecutive, pairs fastest and heaviest first when causal; the
// persistent CTAs take them in snake order (round r: CTA c gets item
// r*G + c for even r, r*G + G-1-c for odd r), which pairs heavy with light
// items across rounds and keeps the concurrently processed items on a few
// K/V heads (L2 reuse).
// nkv_t = key tiles Q tile t visits (0: the tile holds no query row, or none of
// its rows sees a key); nkv = max. An item with nkv == 0 is skipped by the
// producer and the MMA warp; the softmax warps still write O = 0, LSE = -inf
// for any rows it holds (reading #22).
struct FwdItem {
  Seq sq;
  int b, h, kvh, qt0, qt1, nkv0, nkv1, nkv;
};

template <bool CAUSAL>
__device__ __forceinline__ int fwd_item_index(int round, int cta, int ctas) {
  return round * ctas + ((round & 1) ? ctas - 1 - cta : cta);
}

template <bool CAUSAL>
__device__ __forceinline__ FwdItem fwd_decode(const FwdParams& p, int item) {
  const int G = p.Hq / p.Hkv;
  const int pr = item % p.num_pairs;
  int rest = item / p.num_pairs;
  const int hg = rest % G;
  rest /= G;
  FwdItem it;
  it.kvh = rest % p.Hkv;
  it.b = rest / p.Hkv;
  it.h = it.kvh * G + hg;
  const int pair = CAUSAL ? (p.num_pairs - 1 - pr) : pr;
  it.sq = seq_of(p.g, it.b);
  it.qt0 = 2 * pair;
  it.qt1 = 2 * pair + 1;
  it.nkv0 = kv_tiles_for<CAUSAL>(it.sq, it.qt0);
  it.nkv1 = kv_tiles_for<CAUSAL>(it.sq, it.qt1);
  it.nkv = it.nkv1 > it.nkv0 ? it.nkv1 : it.nkv0;
  return it;
}

// First round >= r whose item has work for the producer / MMA warp, or -1.
template <bool CAUSAL>
__device__ __forceinline__ int fwd_next_busy(const FwdParams& p, int r, int cta, int ctas) {
  for (;; ++r) {
    const int item = fwd_item_index<CAUSAL>(r, cta, ctas);
    if (item >= p.num_items) return -1;
    if (fwd_decode<CAUSAL>(p, item).nkv > 0) return r;
  }
}

// ROPE (NEXT #3, hk_attn_fwd_rope): each softmax warpgroup rotates its own Q tile in shared
// memory at the start of an item, one row per thread (rotate-half, rope.cuh: the same arithmetic
// as hk_rope), and publishes it on bar_qr[t], which the MMA warp waits on before S_t = Q_t K^T;
// K arrives pre-rotated (hk_rope into Kr).
template <int D, bool CAUSAL, bool ROPE>
__global__ void __launch_bounds__(384, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
               const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapO,
               const FwdParams p) {
  using C = FwdCfg<D>;
  constexpr int NS = C::NS;
  constexpr uint32_t TB = C::TILE_BYTES;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;           // 2 tiles
  uint8_t* sK = smem + 2 * TB;  // NS tiles
  uint8_t* sV = sK + NS * TB;   // NS tiles
  uint8_t* sOnes = sV + NS * TB;  // ROWSUM: [128 keys][64] bf16 panel, column 0 = 1 (SW128)
  uint8_t* sStage = sOnes + (C::ROWSUM ? 128 * 128 : 0);  // OSTAGE: O staging panel of tile t at t * 16 KB

  __shared__ uint64_t bar_q, bar_qfree, bar_kfull[NS], bar_kempty[NS], bar_vfull[NS], bar_vempty[NS];
  __shared__ uint64_t bar_s[2], bar_p[2], bar_pl[2], bar_o[2], bar_oempty[2], bar_sfree[2], bar_pv[2], bar_qr[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ Sched sched;

  const int warp = warp_id();
  const int lane = lane_id();
  const int cta = blockIdx.x, ctas = gridDim.x;
  const bool dyn = p.sched != nullptr;  // dynamic scheduling: every role takes the producer's draws
  if (threadIdx.x == 0) hk_trace(30, 0, 0);  // CTA start

  if (threadIdx.x == 0) {
    sched_init(sched);
    mbar_init(&bar_q, 1);
    mbar_init(&bar_qr[0], 4);  // ROPE: the tile's warpgroup rotated it
    mbar_init(&bar_qr[1], 4);
    mbar_init(&bar_qfree, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bar_kfull[s], 1);
      mbar_init(&bar_kempty[s], 1);
      mbar_init(&bar_vfull[s], 1);
      mbar_init(&bar_vempty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bar_s[t], 1);
      mbar_init(&bar_p[t], 4);
      mbar_init(&bar_pl[t], 4);  // first half of P_t (keys [0, 64)) published
      mbar_init(&bar_o[t], 1);
      mbar_init(&bar_oempty[t], 4);
      mbar_init(&bar_sfree[t], 4);  // split P: S_t read into registers
      mbar_init(&bar_pv[t], 1);     // split P: P_t V done (P_t and O_t reusable)
    }
    fence_barrier_init();
  }
  if (warp == 8) {
    tma_prefetch(&mapQ);
    tma_prefetch(&mapK);
    tma_prefetch(&mapV);
    if (C::OSTAGE) tma_prefetch(&mapO);
  }
  if (warp == 9) tmem_alloc<512>(&tmem_base_s);
  if (C::ROWSUM && warp >= 10) {  // the ones panel: row r's logical chunk 0 = (1, 0 ... 0), the rest 0
    for (int r = (warp - 10) * 32 + lane; r < 128; r += 64) {
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        sts_v4(smem_u32(sOnes) + r * 128 + ((ch ^ (r & 7)) << 4), ch == 0 ? 0x3F80u : 0u, 0u, 0u, 0u);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base_s, 0);  // warp-uniform for ptxas (UR operands)

  // Every role walks the same item sequence; each barrier keeps its own phase
  // counter, and barriers of a Q tile an item lacks (odd T, last pair) are
  // skipped consistently by both sides.
  if (warp >= 8) {
    reg_dealloc<112>();
    if (warp == 8 && lane == 0) {
      // ================= TMA producer =================
#ifndef HK_FWD_QPOL
#define HK_FWD_QPOL 0
#endif
      const uint64_t pol_q = HK_FWD_QPOL ? policy_evict_last() : policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      int s = 0;
      uint32_t ph = 0, qf_ph = 0;
#ifdef HK_TRACE
      uint32_t nq_tr = 0;
#endif
      auto load_kv = [&](const FwdItem& it, int j) {
        mbar_wait(&bar_kempty[s], ph ^ 1);
#ifdef HK_TRACE
        if (j == 0) hk_trace(22, nq_tr, 0);  // producer: K_0 load issued
#endif
        const int row = it.sq.k0 + j * 128;
        mbar_arrive_expect_tx(&bar_kfull[s], TB);
        for (int pnl = 0; pnl < C::PANELS; ++pnl)
          tma_load_4d(&mapK, &bar_kfull[s], sK + s * TB + pnl * 128 * 128, pnl * 64, it.kvh, row, it.sq.tb, pol_kv);
        mbar_wait(&bar_vempty[s], ph ^ 1);
        mbar_arrive_expect_tx(&bar_vfull[s], TB);
        for (int pnl = 0; pnl < C::PANELS; ++pnl)
          tma_load_4d(&mapV, &bar_vfull[s], sV + s * TB + pnl * 128 * 128, pnl * 64, it.kvh, row, it.sq.tb, pol_kv);
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
      };
      bool first = true;
      int r = dyn ? 0 : fwd_next_busy<CAUSAL>(p, 0, cta, ctas);
      for (;;) {
        int item;
        if (dyn) {  // items without any query row are drawn past; the rest go to every role
          item = sched_publish(sched, p.sched, r++, p.num_items, [&](int i) {
            const FwdItem w = fwd_decode<CAUSAL>(p, i);
            return w.qt0 * 128 >= w.sq.lq;
          });
          if (item >= p.num_items) break;
        } else {
          if (r < 0) break;
          item = fwd_item_index<CAUSAL>(r, cta, ctas);
          r = fwd_next_busy<CAUSAL>(p, r + 1, cta, ctas);
        }
        const FwdItem it = fwd_decode<CAUSAL>(p, item);
        if (it.nkv == 0) continue;
#ifndef HK_FWD_QPREF
#define HK_FWD_QPREF 0
#endif
        if (HK_FWD_QPREF && !dyn && r >= 0) {  // static order: warm L2 with the following item's Q tiles (first touch = HBM)
          const FwdItem nx = fwd_decode<CAUSAL>(p, fwd_item_index<CAUSAL>(r, cta, ctas));
          for (int pnl = 0; pnl < C::PANELS; ++pnl) {
            if (nx.nkv0 > 0) tma_prefetch_4d(&mapQ, pnl * 64, nx.h, nx.sq.q0 + nx.qt0 * 128, nx.sq.tb);
            if (nx.nkv1 > 0) tma_prefetch_4d(&mapQ, pnl * 64, nx.h, nx.sq.q0 + nx.qt1 * 128, nx.sq.tb);
          }
        }
#ifndef HK_FWD_QFIRST
#define HK_FWD_QFIRST 0
#endif
        if (!HK_FWD_QFIRST) load_kv(it, 0);  // K/V of the next item stream in while the previous one finishes
        if (!first) {    // Q buffer is free once the previous item's last S = Q K^T completed
          mbar_wait(&bar_qfree, qf_ph);
          qf_ph ^= 1;
        }
        first = false;
#ifdef HK_TRACE
        hk_trace(17, nq_tr++, 0);  // producer: Q load issued
#endif
        const bool has0 = it.nkv0 > 0, has1 = it.nkv1 > 0;
        mbar_arrive_expect_tx(&bar_q, ((has0 ? 1 : 0) + (has1 ? 1 : 0)) * TB);
        for (int pnl = 0; pnl < C::PANELS; ++pnl) {
          if (has0)
            tma_load_4d(&mapQ, &bar_q, sQ + pnl * 128 * 128, pnl * 64, it.h, it.sq.q0 + it.qt0 * 128, it.sq.tb, pol_q);
          if (has1)
            tma_load_4d(&mapQ, &bar_q, sQ + TB + pnl * 128 * 128, pnl * 64, it.h, it.sq.q0 + it.qt1 * 128, it.sq.tb,
                        pol_q);
        }
        for (int j = HK_FWD_QFIRST ? 0 : 1; j < it.nkv; ++j) load_kv(it, j);
      }
    } else if (warp == 9) {
      // ================= MMA issuer (whole warp, one elected lane issues) =================
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);  // S = Q K^T: A K-major, B K-major
      constexpr uint32_t idesc_o = idesc_bf16(128, C::ON, 0, 1);  // O += P V: A TMEM, B (V) MN-major
      constexpr uint64_t KMAJ = sdesc_sw128_const(16, 1024);
      constexpr uint64_t VMN = sdesc_sw128_const(128 * 128, 1024);
      const uint64_t dq0 = KMAJ | (smem_u32(sQ) >> 4);
      const uint64_t dk0 = KMAJ | (smem_u32(sK) >> 4);
      const uint64_t dv0 = VMN | (smem_u32(sV) >> 4);
      auto issue_s = [&](int t, int s) {
        gemm_ss_kk<D / 16>(tbase + 128 * t, dq0 + ((t * TB) >> 4), dk0 + ((s * TB) >> 4), idesc_s, 0u);
        tc_commit_w(&bar_s[t]);
      };

      int s = 0;
      uint32_t ph = 0, q_ph = 0, qr_ph[2] = {0, 0};
      uint32_t p_ph[2] = {0, 0}, oe_ph[2] = {0, 0};  // bar_pl and bar_p complete in lockstep
      bool o_used[2] = {false, false};  // O_t holds an earlier item's accumulator (wait for its epilogue)
      uint32_t sf_ph[2] = {0, 0};        // split P: bar_sfree phases
#ifdef HK_TRACE
      uint32_t tstep[2] = {0, 0};
#endif
      // static: the last busy item skips its final Q / V releases (nothing waits for them);
      // dynamic: the next draw is unknown, so every release is committed and drained at exit
      int rn = dyn ? 0 : fwd_next_busy<CAUSAL>(p, 0, cta, ctas);
      int uses = 0, busy = 0;  // K/V ring uses and busy items so far (dynamic-mode drain)
      for (;;) {
        int item;
        if (dyn) {
          item = sched_take(sched, rn++);
          if (item >= p.num_items) break;
        } else {
          if (rn < 0) break;
          item = fwd_item_index<CAUSAL>(rn, cta, ctas);
          rn = fwd_next_busy<CAUSAL>(p, rn + 1, cta, ctas);
        }
        const FwdItem it = fwd_decode<CAUSAL>(p, item);
        if (it.nkv == 0) continue;
        const bool last_item = !dyn && rn < 0;
        uses += it.nkv;
        ++busy;
#ifdef HK_TRACE
        hk_trace(12, busy - 1, 0);  // MMA: item start
#endif
        if (!ROPE) mbar_wait(&bar_q, q_ph);
        q_ph ^= 1;
#ifdef HK_TRACE
        hk_trace(13, busy - 1, 0);  // MMA: Q landed
#endif
        mbar_wait(&bar_kfull[s], ph);
        tc_fence_after();
#ifdef HK_TRACE
        hk_trace(24, busy - 1, 0);  // MMA: K_0 landed
#endif
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if ((t == 0 ? it.nkv0 : it.nkv1) == 0) continue;
          if (ROPE) {  // Q tile t landed and rotated by its warpgroup
            mbar_wait(&bar_qr[t], qr_ph[t]);
            qr_ph[t] ^= 1;
            tc_fence_after();
          }
          issue_s(t, s);
#ifdef HK_TRACE
          hk_trace(25 + t, busy - 1, 0);  // MMA: first S_t of the item issued
#endif
        }
        tc_commit_w(&bar_kempty[s]);
#ifdef HK_TRACE
        hk_trace(14, busy - 1, 0);  // MMA: first S of the item issued
#endif
        if (it.nkv == 1 && !last_item) tc_commit_w(&bar_qfree);
        for (int j = 0; j < it.nkv; ++j) {
          const int s1 = s + 1 == NS ? 0 : s + 1;
          const uint32_t ph1 = s + 1 == NS ? ph ^ 1 : ph;
          bool k_next_waited = false;
          if constexpr (C::SPLIT_P) {  // S_t(j+1) as soon as the softmax has read S_t(j)
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const int nk = t == 0 ? it.nkv0 : it.nkv1;
              if (j + 1 < nk) {
                mbar_wait(&bar_sfree[t], sf_ph[t]);
                sf_ph[t] ^= 1;
                if (!k_next_waited) {
                  mbar_wait(&bar_kfull[s1], ph1);
                  k_next_waited = true;
                }
                tc_fence_after();
                issue_s(t, s1);
              }
            }
          }
          mbar_wait(&bar_vfull[s], ph);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int nk = t == 0 ? it.nkv0 : it.nkv1;
            if (j < nk) {
              mbar_wait(&bar_pl[t], p_ph[t]);
              if (j == 0 && o_used[t]) {  // previous item's O_t must be read out before PV overwrites it
                mbar_wait(&bar_oempty[t], oe_ph[t]);
                oe_ph[t] ^= 1;
              }
#ifdef HK_TRACE
              if (j == 0) hk_trace(18 + t, busy - 1, 0);  // MMA: first P V of the item may issue
#endif
              tc_fence_after();
#ifdef HK_TRACE
              hk_trace(10 + t, tstep[t]++, 0);  // MMA: P_t seen, PV issue (running step of tile t)
#endif
              // ROWSUM: the second N panel (columns D ..) is the ones tile, LBO bytes past this slot
              const uint64_t vd = C::ROWSUM ? sdesc_const(smem_u32(sOnes) - smem_u32(sV + s * TB), 1024, 2) |
                                                  (smem_u32(sV + s * TB) >> 4)
                                            : dv0 + ((s * TB) >> 4);
              const uint32_t tPa = C::SPLIT_P ? tbase + 256 + 2 * D + 64 * t : tbase + 128 * t;
              gemm_ts_mn_lo(tbase + 256 + C::ON * t, tPa, vd, idesc_o, j > 0 ? 1u : 0u);
              mbar_wait(&bar_p[t], p_ph[t]);
              p_ph[t] ^= 1;
              tc_fence_after();
              gemm_ts_mn_hi(tbase + 256 + C::ON * t, tPa, vd, idesc_o);
              if (C::SPLIT_P) {
                if (j + 1 < nk) {
                  tc_commit_w(&bar_pv[t]);
                } else {
                  tc_commit_w(&bar_o[t]);
                  o_used[t] = true;
                }
              } else if (j + 1 < nk) {
                if (!k_next_waited) {
                  mbar_wait(&bar_kfull[s1], ph1);
                  tc_fence_after();
                  k_next_waited = true;
                }
                issue_s(t, s1);
              } else {
                tc_commit_w(&bar_o[t]);
                o_used[t] = true;
#ifdef HK_TRACE
                hk_trace(15 + t, busy - 1, 0);  // MMA: last P V of tile t issued
#endif
              }
            }
          }
          // the CTA's very last V release is never waited for: skip it so no
          // arrive can land after the CTA exits
          if (!(last_item && j + 1 == it.nkv)) tc_commit_w(&bar_vempty[s]);
          if (k_next_waited) tc_commit_w(&bar_kempty[s1]);
          if (j + 2 == it.nkv && !last_item) tc_commit_w(&bar_qfree);  // every S of this item issued
          s = s1;
          ph = ph1;
        }
#ifdef HK_TRACE
        hk_trace(20, busy - 1, 0);  // MMA: item loop done
#endif
      }
      if (dyn) {  // let the releases nothing waits for land before the CTA exits
        for (int k = 0; k < NS && k < uses; ++k) {
          const int last = uses - 1 - ((uses - 1 - k) % NS);
          mbar_wait(&bar_kempty[k], (last / NS) & 1);
          mbar_wait(&bar_vempty[k], (last / NS) & 1);
        }
        if (busy > 0) mbar_wait(&bar_qfree, (busy - 1) & 1);
      }

    }
  } else {
    // ================= softmax warpgroups =================
    reg_alloc<192>();
    const int t = warp >> 2;  // Q tile of this warpgroup
    const uint32_t tS = tbase + 128 * t;
    const uint32_t tO = tbase + 256 + C::ON * t;
    const uint32_t tP = C::SPLIT_P ? tbase + 256 + 2 * D + 64 * t : tS;  // bf16 P (split P: own columns)
    uint32_t pv_ph = 0;
    const uint32_t lane_base = (warp & 3) * 32;
    const int r = (warp & 3) * 32 + lane;  // row within the Q tile == TMEM lane
    const float c = 1.4426950408889634f / sqrtf((float)D);  // (1/sqrt d) log2 e
    uint32_t s_ph = 0, o_ph = 0, q_ph = 0;
    int step = 0;  // running KV-step count (trace index only)
    // turn-taking (C::ALT): tile 0 waits on barrier 1 and releases barrier 2, tile 1 the reverse;
    // tile 1 opens the first turn. Only steps both tiles have take turns (the counts agree).
    if (C::ALT && t == 1) named_bar_arrive(1, 256);
    // ROPE: wait for an item's Q tiles and rotate this warpgroup's tile, one row per thread
    auto wait_rotate = [&](const FwdItem& x) {
      mbar_wait(&bar_q, q_ph);  // every busy item loads Q once: keep this warpgroup's phase in step
      q_ph ^= 1;
      if ((t == 0 ? x.nkv0 : x.nkv1) == 0) return;  // tile not loaded: the MMA warp does not wait for it
      const int rowx = (t == 0 ? x.qt0 : x.qt1) * 128 + r;  // position of the query row
      if (rowx < x.sq.lq) {
        constexpr int CP = D / 16;  // chunk pairs per row
        float cs[CP][8], sn[CP][8];  // every cos / sin load of the row in flight at once
#pragma unroll
        for (int c = 0; c < CP; ++c) rope_load_cs(p.rope_cos, p.rope_sin, (size_t)rowx, D / 2, c, 1.f, cs[c], sn[c]);
        const uint32_t tile = smem_u32(sQ) + t * TB + r * 128;
#pragma unroll
        for (int c = 0; c < CP; ++c) {
          // a row's elements i and i + D/2: the same chunk slot of the two panels (D = 128) or
          // chunks c and c + 4 of its 128-B row (D = 64), both at the 128B-swizzled position
          const uint32_t alo = tile + ((c ^ (r & 7)) << 4);
          const uint32_t ahi = D == 128 ? alo + 128 * 128 : tile + (((c + 4) ^ (r & 7)) << 4);
          uint4 va, vb;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(va.x), "=r"(va.y), "=r"(va.z), "=r"(va.w)
                       : "r"(alo));
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(vb.x), "=r"(vb.y), "=r"(vb.z), "=r"(vb.w)
                       : "r"(ahi));
          float a[8], b[8], lo[8], hi[8];
          unpack8(va, a);
          unpack8(vb, b);
          rope_pair8(a, b, cs[c], sn[c], lo, hi);
          const uint4 wa = pack8(lo), wb = pack8(hi);
          sts_v4(alo, wa.x, wa.y, wa.z, wa.w);
          sts_v4(ahi, wb.x, wb.y, wb.z, wb.w);
        }
      }
      fence_proxy_async_smem();  // generic-proxy stores visible to the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_qr[t]);
    };
    // (Rotating the next item's Q before this item's epilogue, while the last P V runs, measured
    // 0.83x of the plain forward at C3 against 0.91x for rotating at the item start: the wait for
    // the next Q tile then delays the epilogue and the O release the next P V needs.)
    for (int rr = 0;; ++rr) {
      const int item = dyn ? sched_take(sched, rr) : fwd_item_index<CAUSAL>(rr, cta, ctas);
      if (item >= p.num_items) break;
      const FwdItem it = fwd_decode<CAUSAL>(p, item);
      const int nk = t == 0 ? it.nkv0 : it.nkv1;
      const int qt = t == 0 ? it.qt0 : it.qt1;
      const int row = qt * 128 + r;
      const bool row_ok = row < it.sq.lq;  // rows of a ragged last tile beyond the sequence are not stored
      if (ROPE && it.nkv > 0) wait_rotate(it);
      if (nk == 0) {  // no row of this tile sees a key: O = 0, LSE = -inf (reading #22)
        if (row_ok) {
          uint4* dst = reinterpret_cast<uint4*>(p.o + ((size_t)(it.sq.gq0 + row) * p.Hq + it.h) * D);
#pragma unroll
          for (int q = 0; q < D / 8; ++q) dst[q] = make_uint4(0u, 0u, 0u, 0u);
          p.lse[lse_index(p.g, it.sq, it.b, p.Hq, it.h, row)] = -INFINITY;
        }
        continue;
      }
      const int off = it.sq.lk - it.sq.lq;  // bottom-right causal alignment
      float m = -INFINITY;  // running max, log2-scaled units
      float l = 0.f;        // running row sum
      for (int j = 0; j < nk; ++j, ++step) {
        if (threadIdx.x % 128 == 0) hk_trace(1 + 4 * t, step, 0);  // softmax: start waiting for S_t(j)
        mbar_wait(&bar_s[t], s_ph);
        s_ph ^= 1;
        tc_fence_after();
        if (threadIdx.x % 128 == 0) hk_trace(2 + 4 * t, step, 0);  // S_t(j) ready
        // row r sees key column cc iff cc <= r + shift (causal) and cc < kvalid
        const int shift = CAUSAL ? qt * 128 + off - j * 128 : (1 << 20);
        const int kleft = it.sq.lk - j * 128;
        const int kvalid = kleft < 128 ? kleft : 128;
        const bool turn = C::ALT && j < min(it.nkv0, it.nkv1);
        softmax_step<D, C::EMU_OF_8, C::ROWSUM>(tS, tO, lane_base, r, c, m, l, shift, j > 0, kvalid, 40 + 4 * t, step,
                                     &bar_pl[t], tP, C::SPLIT_P && j + 1 < nk ? &bar_sfree[t] : nullptr,
                                     C::SPLIT_P && j > 0 ? &bar_pv[t] : nullptr, &pv_ph, turn ? 1 + t : -1,
                                     turn ? 2 - t : -1);
        tmem_wait_st();
        if (threadIdx.x % 128 == 0) hk_trace(43 + 4 * t, step, 0);  // P stores complete
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_p[t]);
        if (threadIdx.x % 128 == 0) hk_trace(3 + 4 * t, step, 0);  // P_t(j) published
      }
      // ---- epilogue: O = O_acc / l (bf16), LSE = (m + log2 l) ln 2
      mbar_wait(&bar_o[t], o_ph);
      o_ph ^= 1;
      tc_fence_after();
      if (threadIdx.x % 128 == 0) hk_trace(33 + t, rr, 0);  // epilogue of tile t: O complete
      if constexpr (C::ROWSUM) {  // l = P . 1, accumulated (and lazily rescaled) with O
        uint32_t lv[16];
        tmem_ld16(tmem_addr(tO, lane_base, D), lv);
        tmem_wait_ld();
        l = __uint_as_float(lv[0]);
      }
      const float inv_l = l > 0.f ? 1.f / l : 0.f;  // l = 0: the row saw no key (O = 0)
      if (C::OSTAGE && !CAUSAL && (qt + 1) * 128 <= it.sq.lq) {
        // non-causal, whole tile inside the sequence: all of O_t into registers (O_t free for the next
        // item's P V at once), then 64-column panels through this tile's SW128 staging panel and a TMA
        // store, so rows leave as full 128-B lines. (Causal: the other tile is still in its last,
        // extra step, which this burst of TMEM reads and stores slows: the interleaved form below
        // measured faster there, profiles/ab_fwd_ostage_r2ac.jsonl.)
        uint32_t o[D];
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32)
          tmem_ld32(tmem_addr(tO, lane_base, c0), *reinterpret_cast<uint32_t(*)[32]>(&o[c0]));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_oempty[t]);
        if (threadIdx.x % 128 == 0) hk_trace(35 + t, rr, 0);  // O read out of TMEM
        const uint32_t stg = smem_u32(sStage) + t * (128 * 128);
#pragma unroll
        for (int pnl = 0; pnl < C::PANELS; ++pnl) {
          if (threadIdx.x % 128 == 0) tma_store_wait_read0();  // the previous store has read the panel
          named_bar_sync(3 + t, 128);
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const int cb = pnl * 64 + ch * 8;
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              w[k] = pack_bf16(__uint_as_float(o[cb + 2 * k]) * inv_l, __uint_as_float(o[cb + 2 * k + 1]) * inv_l);
            sts_v4(stg + r * 128 + ((ch ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
          }
          fence_proxy_async_smem();  // generic-proxy stores visible to the TMA engine
          named_bar_sync(3 + t, 128);
          if (threadIdx.x % 128 == 0) {
            tma_store_4d(&mapO, sStage + t * (128 * 128), pnl * 64, it.h, it.sq.q0 + qt * 128, it.sq.tb);
            tma_store_commit();
          }
        }
      } else {
        __nv_bfloat16* orow = p.o + ((size_t)(it.sq.gq0 + (row_ok ? row : 0)) * p.Hq + it.h) * D;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(tmem_addr(tO, lane_base, c0), o);
          tmem_wait_ld();
          if (c0 + 32 == D) {  // O_t fully read: the next item's P V may overwrite it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_oempty[t]);
            if (threadIdx.x % 128 == 0) hk_trace(35 + t, rr, 0);  // O read out of TMEM
          }
          uint4 v[4];
          uint32_t* vp = reinterpret_cast<uint32_t*>(v);
#pragma unroll
          for (int cc = 0; cc < 16; ++cc)
            vp[cc] = pack_bf16(__uint_as_float(o[2 * cc]) * inv_l, __uint_as_float(o[2 * cc + 1]) * inv_l);
          uint4* dst = reinterpret_cast<uint4*>(orow + c0);
          if (row_ok) {
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = v[q];
          }
        }
      }
      if (row_ok)
        p.lse[lse_index(p.g, it.sq, it.b, p.Hq, it.h, row)] =
            l > 0.f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
      if (threadIdx.x % 128 == 0) hk_trace(31 + t, rr, 0);  // epilogue of tile t done
    }
  }

  if (C::ALT && warp < 4) named_bar_sync(1, 256);  // tile 1's opening arrive (or its last turn's)
  if (C::OSTAGE && warp < 8 && threadIdx.x % 128 == 0) tma_store_wait0();  // O stores done before exit
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tbase);
  if (dyn && threadIdx.x == 0) sched_exit(p.sched);
}

}  // namespace hk
