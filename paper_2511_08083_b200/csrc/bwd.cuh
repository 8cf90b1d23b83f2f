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
#include <map>
#include <mutex>
#include <set>
#include <utility>

#include "../../include/hk_attn.h"
#include "ptx.cuh"
#include "sched.cuh"
#include "seq.cuh"
#include "tma_host.h"

namespace hk {

// ---------------------------------------------------------------- B0
// 16-B vectors per lane and row: 2 at d = 128 (fewer shuffle levels and index ops per byte:
// 1.04-1.16x, profiles/ab_pre_vpl_r2af.jsonl), 1 at d = 64 (2 measured 0.88x there)
#ifndef HK_PRE_VPL128
#define HK_PRE_VPL128 2
#endif
#ifndef HK_PRE_VPL64
#define HK_PRE_VPL64 1
#endif
__host__ __device__ constexpr int pre_vpl(int d) { return d == 128 ? HK_PRE_VPL128 : HK_PRE_VPL64; }
// Grid (x, b): one group of d/8 lanes per (n, h) row of sequence b (16-B loads),
// rows in memory order. Workspace rows n in [lq, Np) of each (b, h) are padding:
// LSE2 = +inf and D = 0, so padded query rows of a last tile give P = 0 and
// dS = 0 in the dK/dV pass. A row that saw no key (LSE = -inf, O = 0) gets
// LSE2 = +inf as well: P = 0, no gradient (reading #22).
template <int D>
__global__ void __launch_bounds__(256) bwd_pre_kernel(const __nv_bfloat16* __restrict__ O,
                                                      const __nv_bfloat16* __restrict__ dO,
                                                      const float* __restrict__ lse, float* __restrict__ Dout,
                                                      float* __restrict__ lse2, SeqGeom g, int H, int hshift,
                                                      int Np, unsigned* __restrict__ sched,
                                                      float* __restrict__ dq_acc) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 4) sched[threadIdx.x] = 0u;
  constexpr int VPL = pre_vpl(D);  // 16-B vectors of O (and of dO) per lane and row
  constexpr int LPR = D / (8 * VPL);  // lanes per row
  constexpr int RPW = 32 / LPR;
  const int b = blockIdx.y;
  const Seq sq = seq_of(g, b);
  const size_t rows = (size_t)sq.lq * H;
  const size_t row0 = (size_t)sq.gq0 * H;  // first (n, h) row of this sequence in O / dO
  const int sub = threadIdx.x % LPR;
  const size_t gwarp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const size_t nwarps = (size_t)gridDim.x * blockDim.x / 32;
  const int lrow = (threadIdx.x % 32) / LPR;
  // U row groups per warp iteration, every load issued before the first reduction
  // (bytes in flight per SM are what an HBM-bound pass needs)
#ifndef HK_PRE_U128
#define HK_PRE_U128 2
#endif
#ifndef HK_PRE_U64
#define HK_PRE_U64 4  // r2: with the fused backward's dQ-accumulator zeroing, 4 is 1.10x at C4-8192 (profiles/ab_pre_u_r2r.jsonl)
#endif
  constexpr int U = D == 128 ? HK_PRE_U128 : HK_PRE_U64;  // measured (scripts/ab.py): 2 for both since the 32-bit (h, n) division
  // One warp iteration's rows: their O / dO vectors, LSE and (h, n).
  struct Grp {
    uint4 a[U][VPL], gv[U][VPL];
    float L[U];        // LSE of the row (lane sub == 0), loaded with O / dO: not a dependent round trip later
    int hh[U], nn[U];  // (h, n) of each row (rows * H < 2^31, validated)
  };
  auto load = [&](size_t base, Grp& q) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t row = base + u * RPW + lrow;
      q.L[u] = 0.f;
      const uint32_t r32 = (uint32_t)row;
      if (hshift >= 0) {  // H a power of two (every BASELINE config): shift and mask
        q.nn[u] = (int)(r32 >> hshift);
        q.hh[u] = (int)(r32 & (uint32_t)(H - 1));
      } else {
        q.nn[u] = (int)(r32 / (uint32_t)H);
        q.hh[u] = (int)(r32 - (uint32_t)q.nn[u] * (uint32_t)H);
      }
      if (row < rows) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          q.a[u][v] = __ldcs(reinterpret_cast<const uint4*>(O + (row0 + row) * D) + sub * VPL + v);
          q.gv[u][v] = __ldcs(reinterpret_cast<const uint4*>(dO + (row0 + row) * D) + sub * VPL + v);
        }
        if (sub == 0) q.L[u] = __ldg(lse + lse_index(g, sq, b, H, q.hh[u], q.nn[u]));
      } else {
#pragma unroll
        for (int v = 0; v < VPL; ++v) q.a[u][v] = q.gv[u][v] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
  };
  auto finish = [&](size_t base, const Grp& q) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t row = base + u * RPW + lrow;
      float acc = 0.f;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const __nv_bfloat162* ap = reinterpret_cast<const __nv_bfloat162*>(&q.a[u][v]);
        const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&q.gv[u][v]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 x = __bfloat1622float2(ap[k]), y = __bfloat1622float2(gp[k]);
          acc = fmaf(x.x, y.x, acc);
          acc = fmaf(x.y, y.y, acc);
        }
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (row < rows) {
        if (sub == 0) {
          const size_t idx = ((size_t)b * H + q.hh[u]) * Np + q.nn[u];  // workspace rows are padded to Np
          Dout[idx] = acc;
          lse2[idx] = q.L[u] == -INFINITY ? INFINITY : q.L[u] * 1.4426950408889634f;
        }
        if (dq_acc != nullptr) {  // fused backward: zero this row's fp32 dQ accumulator (8 VPL floats per lane)
          uint4* z = reinterpret_cast<uint4*>(dq_acc + (row0 + row) * D) + 2 * VPL * sub;
#pragma unroll
          for (int v = 0; v < 2 * VPL; ++v) z[v] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
    }
  };
  const size_t stride = nwarps * RPW * U;
#ifndef HK_PRE_PIPE
#define HK_PRE_PIPE 0  // measured 0.92-1.00x (profiles/ab_pre_pipe_r2j.jsonl): off
#endif
  if (HK_PRE_PIPE) {  // software pipeline: the next iteration's loads are in flight while this one reduces
    size_t base = gwarp * RPW * U;
    Grp cur;
    if (base < rows) load(base, cur);
    for (; base < rows; base += stride) {
      Grp nxt;
      if (base + stride < rows) load(base + stride, nxt);
      finish(base, cur);
      cur = nxt;
    }
  } else {
    for (size_t base = gwarp * RPW * U; base < rows; base += stride) {
      Grp cur;
      load(base, cur);
      finish(base, cur);
    }
  }
  if (Np > sq.lq) {
    const size_t pad = (size_t)Np - sq.lq, npad = (size_t)H * pad;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += (size_t)gridDim.x * blockDim.x) {
      const size_t idx = ((size_t)b * H + i / pad) * Np + sq.lq + i % pad;
      Dout[idx] = 0.f;
      lse2[idx] = INFINITY;
    }
  }
}

// fp32 accumulate mode: dst[0..8) += scale * o[0..8) (one CTA owns each output row: no atomics)
__device__ __forceinline__ void add8_f32(float* dst, const uint32_t* o, float scale) {
  float4* d4 = reinterpret_cast<float4*>(dst);
  float4 a = d4[0], b = d4[1];
  a.x += __uint_as_float(o[0]) * scale, a.y += __uint_as_float(o[1]) * scale;
  a.z += __uint_as_float(o[2]) * scale, a.w += __uint_as_float(o[3]) * scale;
  b.x += __uint_as_float(o[4]) * scale, b.y += __uint_as_float(o[5]) * scale;
  b.z += __uint_as_float(o[6]) * scale, b.w += __uint_as_float(o[7]) * scale;
  d4[0] = a;
  d4[1] = b;
}

// Fused backward epilogue: dQ = bf16(dQ_acc / sqrt(d)) over the query rows of sequence b =
// blockIdx.y (its rows beyond max_seqlen are left untouched, hk_attn.h), 8 elements per thread-step.
template <int D>
__global__ void __launch_bounds__(256) dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                                         SeqGeom g, int H, float scale, bool acc32) {
  const Seq sq = seq_of(g, blockIdx.y);
  const size_t base = (size_t)sq.gq0 * H * (D / 8), n8 = (size_t)sq.lq * H * (D / 8);
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n8; j += (size_t)gridDim.x * blockDim.x) {
    const size_t i = base + j;
    const float4 a = __ldcs(reinterpret_cast<const float4*>(acc) + 2 * i);
    const float4 b = __ldcs(reinterpret_cast<const float4*>(acc) + 2 * i + 1);
    if (acc32) {  // fp32 accumulate mode: dq is the caller's fp32 accumulator
      const uint32_t o[8] = {__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(a.z), __float_as_uint(a.w),
                             __float_as_uint(b.x), __float_as_uint(b.y), __float_as_uint(b.z), __float_as_uint(b.w)};
      add8_f32(reinterpret_cast<float*>(dq) + 8 * i, o, scale);
      continue;
    }
    uint4 o;
    o.x = pack_bf16(a.x * scale, a.y * scale);
    o.y = pack_bf16(a.z * scale, a.w * scale);
    o.z = pack_bf16(b.x * scale, b.y * scale);
    o.w = pack_bf16(b.z * scale, b.w * scale);
    __stcs(reinterpret_cast<uint4*>(dq) + i, o);
  }
}

struct BwdParams {
  const float* Dv;    // [B][Hq][Np], Np = Nq (varlen: max_seqlen_q) rounded up to 128
  const float* lse2;  // [B][Hq][Np]
  __nv_bfloat16* dq;  // dense [B][Nq][Hq][D]; varlen [total_q][Hq][D]
  __nv_bfloat16* dk;  // dense [B][Nk][Hkv][D]; varlen [total_k][Hkv][D]
  __nv_bfloat16* dv;
  unsigned* sched;    // [4] work counters in the workspace: dK/dV draw, done; dQ draw, done
  SeqGeom g;          // dense / varlen geometry (seq.cuh)
  int B, Hq, Hkv, Np, Npk;  // Npk = Nk (varlen: max_seqlen_k) rounded up to 128
  bool acc32;         // HK_BWD_ACCUMULATE_F32: dq / dk / dv are fp32 accumulators the results add into
  // Stored-dS backward (d = 128, dense; ds_block_index): the dK/dV pass also writes each block's bf16
  // dS^T tile here, 32 KB in the shared-memory image of the MN-major SW128 A operand of dQ = dS K, and
  // the dQ pass (bwd_dqds_kernel) is one GEMM per block reading it back. nullptr: the two-pass dQ.
  __nv_bfloat16* ds;
  int ds_tri;  // 1: causal with Nq == Nk, blocks (qi, jt <= qi) packed per head as a triangle
};

// 32-byte streaming store (sm_100: STG.256)
__device__ __forceinline__ void st_global_cs_v8(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// Block (b, h, qi, jt) of the stored dS: per (b, h) either the triangle jt <= qi (causal, Nq == Nk:
// the only blocks the dK/dV pass visits) or the whole Tq x Tk rectangle.
__device__ __forceinline__ size_t ds_block_index(const BwdParams& p, int b, int h, int qi, int jt) {
  const int Tq = p.Np / 128, Tk = p.Npk / 128;
  const size_t per_head = p.ds_tri ? (size_t)Tq * (Tq + 1) / 2 : (size_t)Tq * Tk;
  const size_t in_head = p.ds_tri ? (size_t)qi * (qi + 1) / 2 + jt : (size_t)qi * Tk + jt;
  return ((size_t)b * p.Hq + h) * per_head + in_head;
}
constexpr uint32_t DS_BLOCK_ELEMS = 128 * 128;  // one bf16 dS tile: [2 panels of 64 queries][128 keys][64]


// 128 x 128 tiles throughout: tcgen05.mma with N=64 paces at 48 cycles per
// K=16 step instead of 32 (measured, scripts/rates.py), N=128 at full rate.
// Each per-iteration operand has its own ring, released right after its last
// MMA, so the next load starts as early as possible (a 64 KB stage needs
// ~1450 cycles to land).
template <int D>
struct BwdCfg {
  static constexpr int PANELS = D / 64;
  static constexpr uint32_t T128 = 128 * D * 2;  // a 128-row [rows][D] bf16 tile
#ifndef HK_DKDV_NSA128
#define HK_DKDV_NSA128 3
#endif
  static constexpr int NSA = (D == 128) ? HK_DKDV_NSA128 : 4;  // ring A depth
  static constexpr int NSB = (D == 128) ? 2 : 4;  // ring B depth
  // B1: K_j, V_j resident; ring A = {Q_i}, ring B = {dO_i, lse2_i, D_i} (both freed after dK).
  // At D=128 this is 224 KB + barriers: no room for alignment slack, so the
  // barriers live at the end of the dynamic region (no static shared memory)
  // and the kernel checks that the dynamic base is 1024-aligned.
  static constexpr uint32_t SLOT_B1 = T128 + 1024;
  static constexpr uint32_t BAR_BYTES = 256;
  static constexpr uint32_t SLACK1 = (D == 128) ? 0 : 1024;
  static constexpr uint32_t SMEM1 = 2 * T128 + NSA * T128 + NSB * SLOT_B1 + BAR_BYTES + SLACK1;
  // B2: ring A = {K_j}, ring B = {Q_i, dO_i, V_j ...} (NSB + 2 slots)
  static constexpr uint32_t SMEM2 = 2 * T128 + (NSA + NSB) * T128 + 1024;
  static constexpr int THREADS = 320;  // 8 elementwise warps + TMA warp + MMA warp
  // dK/dV pass: elementwise warpgroups (HK_DKDV_4WG: 4 at d=64, 32 query columns each, to hide
  // the per-phase latency that bounds the d=64 pass; 2 otherwise)
#ifndef HK_DKDV_4WG
#define HK_DKDV_4WG 1
#endif
#ifndef HK_BWD_4WG128
#define HK_BWD_4WG128 0  // the same at d=128 (experiment)
#endif
  static constexpr int NWG1 = ((D == 64 && HK_DKDV_4WG) || (D == 128 && HK_BWD_4WG128)) ? 4 : 2;
  static constexpr int THREADS1 = 32 * (4 * NWG1 + 2);
  // dQ pass: the same at d=64 (HK_DQ_4WG): 4 elementwise warpgroups of 32 key columns
#ifndef HK_DQ_4WG
#define HK_DQ_4WG 1
#endif
  static constexpr int NWG2 = ((D == 64 && HK_DQ_4WG) || (D == 128 && HK_BWD_4WG128)) ? 4 : 2;
  static constexpr int THREADS2 = 32 * (4 * NWG2 + 2);
  // Fused single pass (d = 64 only): the dK/dV pass also forms
  // dQ_partial = dS K_j per block on the tensor core (dS staged in shared memory as the MN-major A
  // operand, accumulator in TMEM columns [384, 512), double-buffered) and a dQ warpgroup adds it
  // into an fp32 dQ accumulator with the bulk-async tensor reduce (cp.reduce.async.bulk.tensor
  // .add.f32, from a shared-memory staging tile); a convert pass scales and rounds it to bf16.
  // d = 128 (round 2): TMEM has no free columns (dV, dK, S^T, dP^T fill all 512), so dQ_partial
  // accumulates in the S^T columns once dV has consumed P^T, and S^T of the next block waits for its
  // read-out; shared memory has no room for a separate staging tile, so the dS tile is reused as
  // the staging of the two 64-column halves of dQ_partial (rings 2 + 2 deep: 226.5 KB).
  static constexpr uint32_t DS_TILE = 128 * 128 * 2;  // dS [128 keys][128 queries] bf16, two SW128 panels
  static constexpr uint32_t DQ_STAGE = D == 64 ? 128 * 64 * 4 : 0;  // dQ_partial [128][64] fp32 (d=128: in DS_TILE)
  static constexpr int NSA_F = D == 64 ? 4 : 2, NSB_F = D == 64 ? 3 : 2;
  static constexpr uint32_t BAR_BYTES_F = 512;
  static constexpr uint32_t SLACK_F = D == 64 ? 1024 : 0;
  static constexpr uint32_t SMEM1F = 2 * T128 + NSA_F * T128 + NSB_F * SLOT_B1 + DS_TILE + DQ_STAGE + BAR_BYTES_F +
                                     SLACK_F;
  static_assert(SMEM1F <= 232448, "fused dK/dV shared memory");
  // 16 warps: two elementwise warpgroups (64 query columns per thread), TMA, MMA, two idle warps,
  // four dQ warps — every SM sub-partition gets two elementwise warps and two others, so after
  // setmaxnreg (elementwise 160, others 96) each holds exactly its 4 x 128 launch registers.
  // (Four elementwise warpgroups, the two-pass d = 64 choice, would leave 80 registers each.)
  static constexpr int NWG1F = 2;
  static constexpr int THREADS1F = 512;
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

// P = 2^x for a pair of backward scores (x = c s - LSE2 <= ~0): BWD_EMU_OF_8
// of every 8 pairs on the FMA pipe (ex2_poly2), the rest on the MUFU, which
// otherwise needs 1024 of each block's 1536-2048 tensor cycles.
#ifndef HK_BWD_EMU
#define HK_BWD_EMU 3
#endif
constexpr int BWD_EMU_OF_8 = HK_BWD_EMU;
template <int EMU_OF_8>
__device__ __forceinline__ float2 bwd_exp2_pair(float2 x, int k) {
  if ((k % 8) < EMU_OF_8) return ex2_poly2(x);
  return make_float2(ex2(x.x), ex2(x.y));
}

__device__ __forceinline__ float2 lds_v2(const void* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(smem_u32(p)));
  return v;
}
// HK_DKDV_SHFL: the dK/dV elementwise warps read LSE2 / D of their query columns with one
// conflict-free ld.shared.v2 per lane and broadcast them by shuffles, instead of 16 broadcast
// ld.shared.v4 per phase (2 wavefronts each on a shared-memory port the pass saturates)
#ifndef HK_DKDV_SHFL
#define HK_DKDV_SHFL 0
#endif
// HK_DKDV_LDG: the same per-query vectors read with ld.global.nc.v4 (all lanes one address, an
// L1 hit after the first warp) from the workspace, off the shared-memory port
#ifndef HK_DKDV_LDG
#define HK_DKDV_LDG 0
#endif
__device__ __forceinline__ void ldg_nc_v4(const float* p, float& a, float& b, float& c, float& d) {
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(p));
}
__device__ __forceinline__ float shfl_col(float2 v, int c) {
  return __shfl_sync(0xffffffffu, (c & 1) ? v.y : v.x, c >> 1);
}
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

// CW fp32 TMEM columns of this thread's lane -> registers, and CW values packed to bf16 pairs
// back into CW/2 columns (CW = 64: two warpgroups per block, 32: four).
template <int CW>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[CW]) {
  if constexpr (CW == 64)
    tmem_ld64(taddr, v);
  else
    tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
}
template <int CW>
__device__ __forceinline__ void tmem_st_packed_cols(uint32_t taddr, const float (&v)[CW]) {
  if constexpr (CW == 64) {
    tmem_st_packed64(taddr, v);
  } else {
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) pk[c] = pack_bf16(v[2 * c], v[2 * c + 1]);
    tmem_st16(taddr, pk);
  }
}

// ---------------------------------------------------------------- B1: dK, dV
// Persistent: one CTA per SM draws work items (key tile jt, kvh, b) from the
// dynamic scheduler (items numbered tiles fastest, heaviest first when causal;
// consecutive items share the Q/dO of their (b, kvh) group in L2). Per item: loop h in the GQA group x
// 128-row query blocks qi. K_j, V_j are resident; once the item's last S^T and
// dP^T completed (bar_kvfree) the next item's K, V load into the same tiles
// while this item finishes; the Q and dO rings run on across items.
// TMEM: dV [0,D)  dK [D,2D)  S^T [2D,2D+128)  dP^T [2D+128,2D+256); bf16 P^T / dS^T
// overwrite the first half of each warpgroup's columns of S^T / dP^T.
// MMA order per block: dV(i) [needs P^T(i)], S^T(i+1), dK(i) [needs dS^T(i)],
// dP^T(i+1): the exponentials of block i+1 overlap dK(i)/dP^T(i+1) and the dS
// work overlaps dV(i+1)/S^T(i+2). The next item's first dV/dK (which overwrite
// the accumulators) need its first P^T/dS^T, which the elementwise warps
// publish only after reading this item's dV/dK out.
// n_it == 0: no query sees this key tile (or it holds no key); the producer and
// the MMA warp skip the item, the elementwise warps write dK = dV = 0 for its keys.
struct KvItem {
  Seq sq;
  int jt, kvh, b, i0, nqt, n_it;
};
template <bool CAUSAL>
__device__ __forceinline__ KvItem kv_decode(const BwdParams& p, int item) {
  const int T = p.Npk / 128;
  const int tr = item % T;
  const int rest = item / T;
  KvItem it;
  it.kvh = rest % p.Hkv;
  it.b = rest / p.Hkv;
  it.sq = seq_of(p.g, it.b);
  it.jt = tr;  // heaviest first when causal: key tile jt is seen by the query tiles i >= jt
  it.i0 = first_q_tile_for<CAUSAL>(it.sq, it.jt);  // first query block that sees key tile jt
  it.nqt = (it.sq.lq + 127) / 128;
  const bool live = it.jt * 128 < it.sq.lk && it.i0 < it.nqt;
  it.n_it = live ? (p.Hq / p.Hkv) * (it.nqt - it.i0) : 0;
  return it;
}

template <int D, bool CAUSAL, bool FQ, bool DS = false>
__global__ void __launch_bounds__(FQ ? BwdCfg<D>::THREADS1F : BwdCfg<D>::THREADS1, 1)
    bwd_dkdv_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapdO,
                    const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                    const __grid_constant__ CUtensorMap mapDQ, const BwdParams p) {
  using C = BwdCfg<D>;
  static_assert(!DS || (D == 128 && !FQ), "stored-dS dK/dV pass: d = 128, two-pass");
  constexpr bool FQ128 = FQ && D == 128;  // fused, d = 128: dQ_partial in the S^T columns (BwdCfg)
  // DS: ring A one slot shallower, its 32 KB the staging tile of the dS^T stores
  constexpr int NSA = FQ ? C::NSA_F : (DS ? C::NSA - 1 : C::NSA), NSB = FQ ? C::NSB_F : C::NSB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if ((FQ ? C::SLACK_F : C::SLACK1) == 0 && smem != smem_raw) __trap();  // layouts without alignment slack
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::T128;
  uint8_t* sA = smem + 2 * C::T128;   // ring A slot s: Q [T128]
  uint8_t* sB = sA + NSA * C::T128;   // ring B slot s: dO [T128] lse2 [512 B] D [512 B]
  uint8_t* sDS = sB + NSB * C::SLOT_B1;                 // FQ: dS tile (MN-major A of dQ_partial = dS K); DS: staging
  uint8_t* sDQ = FQ128 ? sDS : sDS + (FQ ? C::DS_TILE : 0);  // FQ: dQ_partial staging (d=128: the dS tile)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sDS + (FQ ? C::DS_TILE + C::DQ_STAGE : (DS ? C::T128 : 0)));
  uint64_t* fullA = bars;             // [NSA]
  uint64_t* emptyA = bars + NSA;      // [NSA]
  uint64_t* fullB = bars + 2 * NSA;   // [NSB]
  uint64_t* emptyB = fullB + NSB;     // [NSB]
  uint64_t& bar_kv = emptyB[NSB];
  uint64_t& bar_s = emptyB[NSB + 1];
  uint64_t& bar_dp = emptyB[NSB + 2];
  uint64_t& bar_p = emptyB[NSB + 3];
  uint64_t& bar_ds = emptyB[NSB + 4];
  uint64_t& bar_acc = emptyB[NSB + 5];
  uint64_t& bar_kvfree = emptyB[NSB + 6];
  uint32_t& tmem_base_s = *reinterpret_cast<uint32_t*>(emptyB + NSB + 7);
  Sched& sched = *reinterpret_cast<Sched*>(emptyB + NSB + 8);
  uint64_t* fq_bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(&sched) + sizeof(Sched));
  uint64_t& bar_dsfree = fq_bars[0];  // FQ: dQ_partial(u) MMA done reading the dS tile
  uint64_t* bar_dqfull = fq_bars + 1;   // FQ [2]: dQ_partial in TMEM buffer b complete
  uint64_t* bar_dqempty = fq_bars + 3;  // FQ [2]: TMEM buffer b read out by the dQ warpgroup
  static_assert((2 * NSA + 2 * NSB + 8) * 8 + sizeof(Sched) + (FQ ? 5 * 8 : 0) <=
                    (FQ ? C::BAR_BYTES_F : C::BAR_BYTES), "barrier area");

  const int warp = warp_id(), lane = lane_id();
  constexpr int NWG = FQ ? C::NWG1F : C::NWG1;  // elementwise warpgroups
  constexpr int CW = 128 / NWG;           // query columns per elementwise thread
  constexpr int WTMA = 4 * NWG, WMMA = 4 * NWG + 1;
  constexpr int WDQ = 12;                 // FQ: the four dQ warps 12-15 (one per TMEM lane quadrant)
  const int G = p.Hq / p.Hkv;
  const int num_items = p.B * p.Hkv * (p.Npk / 128);

  if (threadIdx.x == 0) {
    sched_init(sched, 1 + 4 * NWG + (FQ ? 4 : 0));
    if (FQ) {
      mbar_init(&bar_dsfree, 1);
      for (int b2 = 0; b2 < 2; ++b2) {
        mbar_init(&bar_dqfull[b2], 1);
        mbar_init(&bar_dqempty[b2], 4);
      }
    }
    mbar_init(&bar_kv, 1);
    mbar_init(&bar_kvfree, 1);
    for (int s = 0; s < NSA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < NSB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    mbar_init(&bar_s, 1);
    mbar_init(&bar_dp, 1);
    mbar_init(&bar_p, 4 * NWG);
    mbar_init(&bar_ds, 4 * NWG);
    mbar_init(&bar_acc, 1);
    fence_barrier_init();
  }
  if (warp == WTMA) {
    tma_prefetch(&mapQ);
    tma_prefetch(&mapdO);
    tma_prefetch(&mapK);
    tma_prefetch(&mapV);
    if (FQ) tma_prefetch(&mapDQ);
  }
  if (warp == WMMA) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base_s, 0);  // warp-uniform for ptxas (UR operands)
  const uint32_t tdV = tb, tdK = tb + D, tS = tb + 2 * D, tP = tb + 2 * D + 128;
  const uint32_t tdQ = FQ128 ? tS : tb + 2 * D + 256;  // FQ: d = 64 two 64-column buffers; d = 128 the S^T columns
  // FQ: 512 threads launch at 128 registers; each role re-sizes at the top of its branch (ptxas
  // allocates per region): per sub-partition 2 x 160 (elementwise) + 2 x 96 = 4 x 128.

  // All roles walk the same items; ring uses and barrier phases run on across items.
  if (warp == WTMA) {
    // ================= TMA producer =================
    if constexpr (FQ) reg_dealloc<96>();
    if (lane == 0) {
      const uint64_t pol_keep = policy_evict_last();
      const uint64_t pol_stream = policy_evict_normal();
      int u = 0;  // ring uses so far (rings A and B advance together, one use per block)
      uint32_t kvf_ph = 0;
      bool first = true;
      for (int r = 0;; ++r) {
        const int item = sched_publish(sched, p.sched, r);
        if (item >= num_items) break;
        const KvItem w = kv_decode<CAUSAL>(p, item);
        if (w.n_it == 0) continue;
        if (!first) {  // K, V tiles free once the previous item's last S^T / dP^T completed
          mbar_wait(&bar_kvfree, kvf_ph);
          kvf_ph ^= 1;
        }
        first = false;
        const int krow = w.sq.k0 + w.jt * 128;
        mbar_arrive_expect_tx(&bar_kv, 2 * C::T128);
        for (int pn = 0; pn < C::PANELS; ++pn) {
          tma_load_4d(&mapK, &bar_kv, sK + pn * 128 * 128, pn * 64, w.kvh, krow, w.sq.tb, pol_stream);
          tma_load_4d(&mapV, &bar_kv, sV + pn * 128 * 128, pn * 64, w.kvh, krow, w.sq.tb, pol_stream);
        }
        // blocking waits (the hardware suspends the warp: no issue slots taken
        // from the elementwise warps sharing its SM sub-partition)
        int h = w.kvh * G, qi = w.i0;
        for (int it = 0; it < w.n_it; ++it, ++u) {
          const int sa = u % NSA, sb = u % NSB;
          mbar_wait(&emptyA[sa], ((u / NSA) & 1) ^ 1);
          hk_trace(20, u, 0);  // producer: ring A slot free, loads for it issued
          mbar_arrive_expect_tx(&fullA[sa], C::T128);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_4d(&mapQ, &fullA[sa], sA + sa * C::T128 + pn * 128 * 128, pn * 64, h, w.sq.q0 + qi * 128,
                        w.sq.tb, pol_keep);
          mbar_wait(&emptyB[sb], ((u / NSB) & 1) ^ 1);
          uint8_t* st = sB + sb * C::SLOT_B1;
          mbar_arrive_expect_tx(&fullB[sb], C::T128 + 1024);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_4d(&mapdO, &fullB[sb], st + pn * 128 * 128, pn * 64, h, w.sq.q0 + qi * 128, w.sq.tb, pol_keep);
          const size_t off = ((size_t)w.b * p.Hq + h) * p.Np + (size_t)qi * 128;
          bulk_load(st + C::T128, p.lse2 + off, 512, &fullB[sb]);
          bulk_load(st + C::T128 + 512, p.Dv + off, 512, &fullB[sb]);
          if (++qi == w.nqt) {
            qi = w.i0;
            ++h;
          }
        }
      }
    }
  } else if (warp == WMMA) {
    // ================= MMA issuer (whole warp, one elected lane issues) =================
    if constexpr (FQ) reg_dealloc<96>();
    constexpr uint32_t idesc_sp = idesc_bf16(128, 128, 0, 0);  // S^T / dP^T: M=128 keys, N=128 queries
    constexpr uint32_t idesc_acc = idesc_bf16(128, D, 0, 1);   // dV / dK: B = dO_i / Q_i MN-major
    constexpr uint64_t KMAJ = sdesc_sw128_const(16, 1024);
    constexpr uint64_t MNMAJ = sdesc_sw128_const(128 * 128, 1024);
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aA = smem_u32(sA), aB = smem_u32(sB);
    auto kmaj = [&](uint32_t base, int kk) { return KMAJ | ((base + (kk / 4) * 128 * 128 + (kk % 4) * 32) >> 4); };
    auto mnmaj = [&](uint32_t base, int kk) { return MNMAJ | ((base + kk * 16 * 128) >> 4); };
    auto slotQ = [&](int u) { return aA + (u % NSA) * C::T128; };
    auto slotO = [&](int u) { return aB + (u % NSB) * C::SLOT_B1; };
    auto issue_s = [&](int u) {
      gemm_ss_kk<D / 16>(tS, kmaj(aK, 0), kmaj(slotQ(u), 0), idesc_sp, 0u);
      tc_commit_w(&bar_s);
    };
    auto issue_dp = [&](int u) {
      hk_trace(14, u, 0);  // MMA: dP^T(u) issue
      gemm_ss_kk<D / 16>(tP, kmaj(aV, 0), kmaj(slotO(u), 0), idesc_sp, 0u);
      tc_commit_w(&bar_dp);
    };
    int u0 = 0;  // ring uses before this item == blocks before this item
    uint32_t kv_ph = 0;
    int busy = 0;  // items with work so far (one bar_kv / bar_kvfree phase each)
    if constexpr (FQ128) {
      // d = 128 fused order per block u: dV(u) [P^T in the S^T columns], dK(u) [dS^T in the dP^T
      // columns], dQ_partial(u) = dS K_j into the S^T columns, dP^T(u+1) (fills the tensor pipe while
      // the dQ warps read dQ_partial(u) out), then S^T(u+1) once the S^T columns are free again.
      constexpr uint32_t idesc_dq = idesc_bf16(128, D, 1, 1);  // M = 128 queries, A = dS MN-major
      auto issue_s_free = [&](int u) {  // S^T(u) into columns dQ_partial(u - 1) may still occupy
        if (u > 0) {
          mbar_wait(&bar_dqempty[0], (u - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&fullA[u % NSA], (u / NSA) & 1);
        tc_fence_after();
        issue_s(u);
      };
      for (int r = 0;; ++r) {
        const int item = sched_take(sched, r);
        if (item >= num_items) break;
        const KvItem w = kv_decode<CAUSAL>(p, item);
        const int n = w.n_it;
        if (n == 0) continue;
        ++busy;
        mbar_wait(&bar_kv, kv_ph);
        kv_ph ^= 1;
        mbar_wait(&fullB[u0 % NSB], (u0 / NSB) & 1);
        tc_fence_after();
        issue_dp(u0);
        issue_s_free(u0);
        for (int it = 0; it < n; ++it) {
          const int u = u0 + it;
          const uint32_t q = slotQ(u), dO = slotO(u);
          const uint32_t acc = it > 0 ? 1u : 0u;
          const bool more = it + 1 < n;
          mbar_wait(&bar_p, u & 1);
          tc_fence_after();
          gemm_tsp_mn(tdV, tS, mnmaj(dO, 0), idesc_acc, acc);
          mbar_wait(&bar_ds, u & 1);
          tc_fence_after();
          gemm_tsp_mn(tdK, tP, mnmaj(q, 0), idesc_acc, acc);
          gemm_ss_mnmn(tdQ, mnmaj(smem_u32(sDS), 0), mnmaj(aK, 0), idesc_dq, 0u);
          tc_commit_w(&bar_dqfull[0]);
          tc_commit_w(&emptyA[u % NSA]);
          tc_commit_w(&emptyB[u % NSB]);
          if (more) {
            mbar_wait(&fullB[(u + 1) % NSB], ((u + 1) / NSB) & 1);
            tc_fence_after();
            issue_dp(u + 1);
            issue_s_free(u + 1);
          } else {
            tc_commit_w(&bar_kvfree);  // K_j's last use (dQ_partial), V_j's (dP^T) before it
          }
        }
        tc_commit_w(&bar_acc);
        u0 += n;
      }
    } else {
    for (int r = 0;; ++r) {
      const int item = sched_take(sched, r);
      if (item >= num_items) break;
      const KvItem w = kv_decode<CAUSAL>(p, item);
      const int n = w.n_it;
      if (n == 0) continue;
      ++busy;
      mbar_wait(&bar_kv, kv_ph);
      kv_ph ^= 1;
      mbar_wait(&fullA[u0 % NSA], (u0 / NSA) & 1);
      tc_fence_after();
      issue_s(u0);
      mbar_wait(&fullB[u0 % NSB], (u0 / NSB) & 1);
      tc_fence_after();
      issue_dp(u0);
      if (!FQ && n == 1) tc_commit_w(&bar_kvfree);
      for (int it = 0; it < n; ++it) {
        const int u = u0 + it;
        const uint32_t q = slotQ(u), dO = slotO(u);
        const uint32_t acc = it > 0 ? 1u : 0u;
        const bool more = it + 1 < n;
        mbar_wait(&bar_p, u & 1);
        tc_fence_after();
        hk_trace(10, u, 0);  // MMA: P^T(it) seen, dV issue
        if constexpr (NWG == 4)
          gemm_tsp4_mn(tdV, tS, mnmaj(dO, 0), idesc_acc, acc);
        else
          gemm_tsp_mn(tdV, tS, mnmaj(dO, 0), idesc_acc, acc);
        if (more) {
          mbar_wait(&fullA[(u + 1) % NSA], ((u + 1) / NSA) & 1);
          tc_fence_after();
          hk_trace(13, u + 1, 0);  // ring A slot u+1 landed, S^T issue
          issue_s(u + 1);
        }
        mbar_wait(&bar_ds, u & 1);
        tc_fence_after();
        hk_trace(11, u, 0);  // MMA: dS^T(it) seen, dK issue
        if constexpr (NWG == 4)
          gemm_tsp4_mn(tdK, tP, mnmaj(q, 0), idesc_acc, acc);
        else
          gemm_tsp_mn(tdK, tP, mnmaj(q, 0), idesc_acc, acc);
        // Q(it) (last use dK) and dO/lse2/D(it) (last uses dV, the dS phase): free both
        tc_commit_w(&emptyA[u % NSA]);
        tc_commit_w(&emptyB[u % NSB]);
        if (more) {  // dP^T(it+1) overwrites dS^T(it): after dK(it) in issue order
          mbar_wait(&fullB[(u + 1) % NSB], ((u + 1) / NSB) & 1);
          tc_fence_after();
          issue_dp(u + 1);
          if (!FQ && it + 2 == n) tc_commit_w(&bar_kvfree);  // last S^T and dP^T issued
        }
        if constexpr (FQ && !FQ128) {  // dQ_partial(it) = dS(it) K_j into TMEM buffer u % 2 (drained by the dQ warps)
          constexpr uint32_t idesc_dq = idesc_bf16(128, D, 1, 1);  // M = 128 queries, A = dS MN-major
          mbar_wait(&bar_dqempty[u & 1], ((u >> 1) & 1) ^ 1);
          tc_fence_after();
          gemm_ss_mnmn(tdQ + 64 * (u & 1), mnmaj(smem_u32(sDS), 0), mnmaj(aK, 0), idesc_dq, 0u);
          tc_commit_w(&bar_dqfull[u & 1]);
          tc_commit_w(&bar_dsfree);
          if (it + 1 == n) tc_commit_w(&bar_kvfree);  // K_j's last use
        }
      }
      tc_commit_w(&bar_acc);
      u0 += n;
    }
    }
    // the releases of the final uses are never waited for by the producer: let them land
    drain_ring(emptyA, NSA, u0);
    drain_ring(emptyB, NSB, u0);
    if (busy > 0) mbar_wait(&bar_kvfree, (busy - 1) & 1);
    if (FQ && u0 > 0) mbar_wait(&bar_dsfree, (u0 - 1) & 1);  // the last dS-tile release
  } else if (FQ && warp >= WDQ) {
    // ================= dQ warpgroup (FQ): TMEM dQ_partial -> staging -> bulk tensor reduce-add =================
    reg_dealloc<96>();
    const int qd = warp & 3;                // TMEM lane quadrant of this warp
    const int r = qd * 32 + lane;           // query row within the 128-row tile
    const bool issuer = warp == WDQ && lane == 0;
    int u = 0;
    for (int rr = 0;; ++rr) {
      const int item = sched_take(sched, rr);
      if (item >= num_items) break;
      const KvItem w = kv_decode<CAUSAL>(p, item);
      if (w.n_it == 0) continue;
      int h = w.kvh * G, qi = w.i0;
      if constexpr (FQ128) {
        // d = 128: dQ_partial (128 columns, in the S^T columns) leaves in two 64-column halves through
        // the dS tile (two [128][32] fp32 SW128 boxes per half); the S^T columns are released after
        // the second half is read, the dS tile after the TMA has read the second half's staging
        for (int it = 0; it < w.n_it; ++it, ++u) {
          mbar_wait(&bar_dqfull[0], u & 1);
          tc_fence_after();
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            if (half == 1 && issuer) tma_store_wait_read0();  // the first half's staging has been read
            named_bar_sync(3, 128);
#pragma unroll
            for (int bx = 0; bx < 2; ++bx) {
              uint32_t v[32];
              tmem_ld32(tmem_addr(tdQ, qd * 32, 64 * half + 32 * bx), v);
              tmem_wait_ld();
              if (half == 1 && bx == 1) {  // every column read: S^T(u + 1) may overwrite them
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_dqempty[0]);
              }
              const uint32_t rowp = smem_u32(sDQ) + bx * (128 * 128) + r * 128;
#pragma unroll
              for (int c8 = 0; c8 < 8; ++c8)
                sts_v4(rowp + ((c8 ^ (r & 7)) << 4), v[4 * c8], v[4 * c8 + 1], v[4 * c8 + 2], v[4 * c8 + 3]);
            }
            fence_proxy_async_smem();
            named_bar_sync(3, 128);
            if (issuer) {
              for (int bx = 0; bx < 2; ++bx)
                tma_reduce_add_4d(&mapDQ, sDQ + bx * (128 * 128), 64 * half + 32 * bx, h, w.sq.q0 + qi * 128,
                                  w.sq.tb);
              tma_store_commit();
            }
          }
          if (issuer) {  // the dS tile is free for the next block's dS once the TMA has read it
            tma_store_wait_read0();
            mbar_arrive(&bar_dsfree);
          }
          if (++qi == w.nqt) {
            qi = w.i0;
            ++h;
          }
        }
        continue;
      }
      for (int it = 0; it < w.n_it; ++it, ++u) {
        const uint32_t b2 = u & 1;
        mbar_wait(&bar_dqfull[b2], (u >> 1) & 1);
        tc_fence_after();
        if (issuer) tma_store_wait_read0();  // the previous reduce has read the staging tile
        named_bar_sync(3, 128);
        // 32 columns at a time (704 threads leave 88 registers each): row r of the [128][32] fp32
        // box bx, SWIZZLE_128B (16-B chunk c at c ^ (r % 8))
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
          uint32_t v[32];
          tmem_ld32(tmem_addr(tdQ + 64 * b2, qd * 32, 32 * bx), v);
          tmem_wait_ld();
          if (bx == 1) {  // TMEM buffer read out: the next-but-one dQ_partial may overwrite it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_dqempty[b2]);
          }
          const uint32_t rowp = smem_u32(sDQ) + bx * (128 * 128) + r * 128;
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8)
            sts_v4(rowp + ((c8 ^ (r & 7)) << 4), v[4 * c8], v[4 * c8 + 1], v[4 * c8 + 2], v[4 * c8 + 3]);
        }
        fence_proxy_async_smem();
        named_bar_sync(3, 128);
        if (issuer) {
          for (int bx = 0; bx < 2; ++bx)
            tma_reduce_add_4d(&mapDQ, sDQ + bx * (128 * 128), 32 * bx, h, w.sq.q0 + qi * 128, w.sq.tb);
          tma_store_commit();
        }
        if (++qi == w.nqt) {
          qi = w.i0;
          ++h;
        }
      }
    }
    if (issuer) tma_store_wait0();  // every reduce complete before the CTA exits
  } else if (warp < 4 * NWG) {
    // ================= elementwise warpgroups (warps 0 .. 4 NWG - 1) =================
    if constexpr (FQ) reg_alloc<160>();
    const int wg = warp >> 2;              // query columns [CW wg, CW wg + CW) of each block
    const uint32_t lb = (warp & 3) * 32;   // TMEM lane base
    const int r = (warp & 3) * 32 + lane;  // key row within the tile
    const float c = 1.4426950408889634f / sqrtf((float)D);
    const uint32_t cS = tS + CW * wg, cP = tP + CW * wg;
    // epilogue columns: the first half of the warpgroups write dV, the second dK
    constexpr int HALF = NWG / 2, ECOLS = D / HALF;
    const bool is_dk = wg >= HALF;
    const int ecol0 = (wg % HALF) * ECOLS;
    int u = 0, s = 0;  // blocks so far; ring B slot of block u
    uint32_t acc_ph = 0;
    for (int rr = 0;; ++rr) {
      const int item = sched_take(sched, rr);
      if (item >= num_items) break;
      const KvItem w = kv_decode<CAUSAL>(p, item);
      const int key = w.jt * 128 + r;
      const bool key_ok = key < w.sq.lk;  // key rows of a ragged last tile beyond the sequence are not stored
      __nv_bfloat16* out =
          (is_dk ? p.dk : p.dv) + ((size_t)(w.sq.gk0 + (key_ok ? key : 0)) * p.Hkv + w.kvh) * D + ecol0;
      if (w.n_it == 0) {  // no query sees these keys: dK = dV = 0 (accumulate mode: nothing to add)
        if (key_ok && !p.acc32) {
#pragma unroll
          for (int k = 0; k < ECOLS / 8; ++k) reinterpret_cast<uint4*>(out)[k] = make_uint4(0u, 0u, 0u, 0u);
        }
        continue;
      }
      const int off = w.sq.lk - w.sq.lq;  // bottom-right causal alignment
      int qi = w.i0;
      int hq = w.kvh * G;  // query head of block u (HK_DKDV_LDG)
      for (int it = 0; it < w.n_it; ++it, ++u) {
        const uint8_t* vec = sB + s * C::SLOT_B1 + C::T128;  // lse2 [128], then D [128]
        const size_t goff = ((size_t)w.b * p.Hq + hq) * p.Np + (size_t)qi * 128 + CW * wg;  // HK_DKDV_LDG
        (void)goff;
        const uint32_t par = u & 1;
        float v[CW];
        // ---- phase 1: P^T = exp2(c S^T - LSE2) (masked), bf16 into TMEM for dV += P^T dO
        if (threadIdx.x == 0) hk_trace(1, u, 0);
        mbar_wait(&fullB[s], (u / NSB) & 1);  // lse2/D ride with dO in ring B: landed?
        mbar_wait(&bar_s, par);
        tc_fence_after();
        if (threadIdx.x == 0) hk_trace(2, u, 0);
        tmem_ld_cols<CW>(tmem_addr(cS, lb, 0), v);
        tmem_wait_ld();
        const int q0 = qi * 128 + CW * wg;
#if HK_DKDV_SHFL
        const float2 lsp = lds_v2(vec + 4 * (CW * wg) + 8 * (lane % (CW / 2)));
#endif
#pragma unroll
        for (int c4 = 0; c4 < CW; c4 += 4) {
          float l0, l1, l2, l3;
#if HK_DKDV_SHFL
          l0 = shfl_col(lsp, c4);
          l1 = shfl_col(lsp, c4 + 1);
          l2 = shfl_col(lsp, c4 + 2);
          l3 = shfl_col(lsp, c4 + 3);
#elif HK_DKDV_LDG
          ldg_nc_v4(p.lse2 + goff + c4, l0, l1, l2, l3);
#else
          lds_v4(vec + 4 * (CW * wg + c4), l0, l1, l2, l3);
#endif
          const float2 xa = fma2(make_float2(v[c4], v[c4 + 1]), make_float2(c, c), make_float2(-l0, -l1));
          const float2 xb = fma2(make_float2(v[c4 + 2], v[c4 + 3]), make_float2(c, c), make_float2(-l2, -l3));
          const float2 ea = bwd_exp2_pair<BWD_EMU_OF_8>(xa, c4 / 2);
          const float2 eb = bwd_exp2_pair<BWD_EMU_OF_8>(xb, c4 / 2 + 1);
          v[c4] = ea.x;
          v[c4 + 1] = ea.y;
          v[c4 + 2] = eb.x;
          v[c4 + 3] = eb.y;
        }
        if (CAUSAL && qi * 128 + off < w.jt * 128 + 127) {
#pragma unroll
          for (int cc = 0; cc < CW; ++cc)
            if (q0 + cc + off < key) v[cc] = 0.f;  // key > query + (lk - lq) is masked
        }
        tmem_st_packed_cols<CW>(tmem_addr(cS, lb, 0), v);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_p);
        if (threadIdx.x == 0) hk_trace(3, u, 0);
        // ---- phase 2: dS^T = P^T (dP^T - D), bf16 into TMEM for dK += dS^T Q
        mbar_wait(&bar_dp, par);
        tc_fence_after();
        if (threadIdx.x == 0) hk_trace(4, u, 0);
        float dp[CW];
        uint32_t dsk[DS ? 32 : 1];  // stored-dS (DS): this row's packed bf16 dS^T
        tmem_ld_cols<CW>(tmem_addr(cP, lb, 0), dp);
        tmem_wait_ld();
#if HK_DKDV_SHFL
        const float2 dsp = lds_v2(vec + 512 + 4 * (CW * wg) + 8 * (lane % (CW / 2)));
#endif
#pragma unroll
        for (int c4 = 0; c4 < CW; c4 += 4) {  // packed f32x2: half the issue slots of scalar FADD + FMUL
          float d0, d1, d2, d3;
#if HK_DKDV_SHFL
          d0 = shfl_col(dsp, c4);
          d1 = shfl_col(dsp, c4 + 1);
          d2 = shfl_col(dsp, c4 + 2);
          d3 = shfl_col(dsp, c4 + 3);
#elif HK_DKDV_LDG
          ldg_nc_v4(p.Dv + goff + c4, d0, d1, d2, d3);
#else
          lds_v4(vec + 512 + 4 * (CW * wg + c4), d0, d1, d2, d3);
#endif
          const float2 a = mul2(make_float2(v[c4], v[c4 + 1]),
                                sub2(make_float2(dp[c4], dp[c4 + 1]), make_float2(d0, d1)));
          const float2 b = mul2(make_float2(v[c4 + 2], v[c4 + 3]),
                                sub2(make_float2(dp[c4 + 2], dp[c4 + 3]), make_float2(d2, d3)));
          dp[c4] = a.x;
          dp[c4 + 1] = a.y;
          dp[c4 + 2] = b.x;
          dp[c4 + 3] = b.y;
        }
        if constexpr (FQ) {
          // a key row beyond the sequence (varlen: the next sequence's keys in this tile) must add
          // nothing to dQ: its dS row is zeroed (its dK, dV rows are never stored)
          if (!key_ok) {
#pragma unroll
            for (int cc = 0; cc < CW; ++cc) dp[cc] = 0.f;
          }
          uint32_t pk[CW / 2];
#pragma unroll
          for (int c2 = 0; c2 < CW / 2; ++c2) pk[c2] = pack_bf16(dp[2 * c2], dp[2 * c2 + 1]);
          if constexpr (CW == 64)
            tmem_st32(tmem_addr(cP, lb, 0), *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
          else
            tmem_st16(tmem_addr(cP, lb, 0), pk);
          // dS row r (a key) = the K-row r of the MN-major A operand: queries [CW wg, CW wg + CW) sit
          // in panel CW wg / 64, 16-B chunks from (CW wg % 64) / 8, SWIZZLE_128B (chunk c at c ^ (r % 8))
          if (u > 0) mbar_wait(&bar_dsfree, (u & 1) ^ 1);  // dQ_partial(u - 1) has read the tile
          const uint32_t rowp = smem_u32(sDS) + ((CW * wg) >> 6) * (128 * 128) + r * 128;
          const int c0 = ((CW * wg) & 63) >> 3;
#pragma unroll
          for (int k = 0; k < CW / 8; ++k)
            sts_v4(rowp + (((c0 + k) ^ (r & 7)) << 4), pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
          fence_proxy_async_smem();  // generic-proxy stores visible to the tensor core
        } else if constexpr (DS) {
          // stored-dS backward: the same bf16 dS^T into TMEM (dK) and — after bar_ds is published,
          // off the MMA's critical path — to the workspace for the dQ pass (below)
#pragma unroll
          for (int c2 = 0; c2 < 32; ++c2) dsk[c2] = pack_bf16(dp[2 * c2], dp[2 * c2 + 1]);
          tmem_st32(tmem_addr(cP, lb, 0), dsk);
        } else {
          tmem_st_packed_cols<CW>(tmem_addr(cP, lb, 0), dp);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_ds);
        if (threadIdx.x == 0) hk_trace(5, u, 0);
        if constexpr (DS) {
          {
          // key row r of panel wg of the block's MN-major SW128 A-operand image (16-B chunk c at
          // c ^ (r % 8)) in 32-byte streaming stores (whole sectors): chunks 2m, 2m + 1 sit at positions
          // (2m) ^ x, (2m + 1) ^ x, x = r % 8, i.e. in the 32-B slot m ^ (x / 2), swapped when x is odd
          // through this warp's 4 KB of the staging tile (its 32 key rows of panel wg, contiguous in
          // the block image too) and one bulk copy by lane 0: whole 128-B lines issued by the TMA
          // engine (global stores from 256 threads would queue in the load/store unit ahead of the
          // LSE2/D broadcasts the next phases need), and no barrier wider than the warp
          const uint32_t stg = smem_u32(sDS) + wg * (C::T128 / 2) + lb * 128;
          if (lane == 0) tma_store_wait_read0();  // this warp's previous copy has read its rows
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 8; ++k)
            sts_v4(stg + lane * 128 + ((k ^ (r & 7)) << 4), dsk[4 * k], dsk[4 * k + 1], dsk[4 * k + 2], dsk[4 * k + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            bulk_store_hint(p.ds + ds_block_index(p, w.b, hq, qi, w.jt) * DS_BLOCK_ELEMS + wg * (DS_BLOCK_ELEMS / 2) +
                                lb * 64,
                            sDS + wg * (C::T128 / 2) + lb * 128, 32 * 128, policy_evict_first());
            tma_store_commit();
          }
          }
        }
        if (++qi == w.nqt) {
          qi = w.i0;
          ++hq;
        }
        if (++s == NSB) s = 0;
      }
      // ---- epilogue: WG0 writes dV, WG1 writes dK * (1/sqrt d)
      mbar_wait(&bar_acc, acc_ph);
      acc_ph ^= 1;
      tc_fence_after();
      const float scale = is_dk ? rsqrtf((float)D) : 1.f;
      const uint32_t tacc = (is_dk ? tdK : tdV) + ecol0;
#pragma unroll
      for (int c0 = 0; c0 < ECOLS; c0 += 32) {
        uint32_t o[32];
        tmem_ld32(tmem_addr(tacc, lb, c0), o);
        tmem_wait_ld();
        if (p.acc32) {  // fp32 accumulate mode: add into the caller's fp32 dK / dV
          float* outf = reinterpret_cast<float*>(is_dk ? p.dk : p.dv) +
                        ((size_t)(w.sq.gk0 + (key_ok ? key : 0)) * p.Hkv + w.kvh) * D + ecol0 + c0;
          if (key_ok) {
#pragma unroll
            for (int k = 0; k < 4; ++k) add8_f32(outf + 8 * k, o + 8 * k, scale);
          }
          continue;
        }
        uint4 o4[4];
        uint32_t* op = reinterpret_cast<uint32_t*>(o4);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          op[k] = pack_bf16(__uint_as_float(o[2 * k]) * scale, __uint_as_float(o[2 * k + 1]) * scale);
        uint4* dst = reinterpret_cast<uint4*>(out + c0);
        if (key_ok) {
#pragma unroll
          for (int k = 0; k < 4; ++k) dst[k] = o4[k];
        }
      }
    }
    if constexpr (DS) {
      if (lane == 0) tma_store_wait0();  // this warp's dS copies complete
    }
  } else if constexpr (FQ) {
    reg_dealloc<96>();  // the two idle warps (10, 11) give their share to the elementwise warps
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WMMA) tmem_dealloc<512>(tb);
  if (threadIdx.x == 0) sched_exit(p.sched);
}

// ---------------------------------------------------------------- B2: dQ
// Persistent: one CTA per SM draws work items (query tile iq, h, b) from the
// dynamic scheduler, numbered like the forward's (the G heads x tiles of one
// (b, kvh) group consecutive, tiles fastest, heaviest first when causal).
// Per item, loop over 128-key blocks j. Q_i and dO_i land (TMA) in two staging
// tiles and the elementwise warps copy them into TMEM, so S = Q_i K_j^T and
// dP = dO_i V_j^T run with A from TMEM: per block the tensor core then reads
// only K_j (twice) and V_j from SMEM (96 KB instead of 160 KB), which with the
// 64 KB of TMA traffic keeps the pass under the 128 B/clk shared-memory
// bandwidth. The staging tiles are free again right after the
// copy, so the next item's Q/dO stream in during the current item, and at the
// item boundary the copy for the next item is done between reading dQ out of
// TMEM and storing it.
// TMEM: dQ [0,D)  S [D,D+128)  dP [D+128,D+256)  Q_A [D+256,D+256+D/2)  dO_A [+D/2);
// bf16 dS overwrites dP. S is single-buffered but released as soon as the
// elementwise warps have loaded it (bar_sfree), so S(j+1) still overlaps the
// exponentials of block j. MMA order: S(j+1), dQ(j) [needs dS(j)], dP(j+1).
// n_it == 0: the tile holds no query row, or none of its rows sees a key; the
// producer and the MMA warp skip the item, the elementwise warps write dQ = 0.
struct DqItem {
  Seq sq;
  int iq, h, kvh, b, n_it;
};
template <bool CAUSAL>
__device__ __forceinline__ DqItem dq_decode(const BwdParams& p, int item) {
  const int T = p.Np / 128;
  const int G = p.Hq / p.Hkv;
  const int tr = item % T;
  int rest = item / T;
  const int hg = rest % G;
  rest /= G;
  DqItem it;
  it.kvh = rest % p.Hkv;
  it.b = rest / p.Hkv;
  it.h = it.kvh * G + hg;
  it.iq = CAUSAL ? T - 1 - tr : tr;  // heaviest first
  it.sq = seq_of(p.g, it.b);
  it.n_it = kv_tiles_for<CAUSAL>(it.sq, it.iq);  // 128-key blocks
  return it;
}

template <int D, bool CAUSAL>
__global__ void __launch_bounds__(BwdCfg<D>::THREADS2, 1)
    bwd_dq_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapdO,
                  const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                  const BwdParams p) {
  using C = BwdCfg<D>;
  // ring A = K_j; ring B (NSB + 2 slots) carries, per item, Q_i, dO_i, then V_0 .. V_{n-1}:
  // the Q_i/dO_i slots are released once copied into TMEM, so V keeps a deep ring
  // and the next item's Q_i/dO_i queue behind the current item's last V blocks.
  constexpr int NSA = C::NSA, NB = C::NSB + 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // ring A slot s: K_j [T128]
  uint8_t* sB = sA + NSA * C::T128;   // ring B slot s: Q_i | dO_i | V_j [T128]

  __shared__ uint64_t bar_qa, fullA[NSA], emptyA[NSA], fullB[NB], emptyB[NB], bar_s, bar_sfree, bar_dp, bar_ds,
      bar_acc;
  __shared__ Sched sched;
  __shared__ uint32_t tmem_base_s;

  const int warp = warp_id(), lane = lane_id();
  constexpr int NWG = C::NWG2;            // elementwise warpgroups
  constexpr int CW = 128 / NWG;           // key columns per elementwise thread
  constexpr int WTMA = 4 * NWG, WMMA = 4 * NWG + 1;
  const int num_items = p.B * p.Hq * (p.Np / 128);
  unsigned* const ctr = p.sched + 2;

  if (threadIdx.x == 0) {
    sched_init(sched, 1 + 4 * NWG);
    mbar_init(&bar_qa, 8);
    for (int s = 0; s < NSA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    mbar_init(&bar_s, 1);
    mbar_init(&bar_sfree, 4 * NWG);
    mbar_init(&bar_dp, 1);
    mbar_init(&bar_ds, 4 * NWG);
    mbar_init(&bar_acc, 1);
    fence_barrier_init();
  }
  if (warp == WTMA) {
    tma_prefetch(&mapQ);
    tma_prefetch(&mapdO);
    tma_prefetch(&mapK);
    tma_prefetch(&mapV);
  }
  if (warp == WMMA) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base_s, 0);  // warp-uniform for ptxas (UR operands)
  const uint32_t tdQ = tb, tS = tb + D, tP = tb + D + 128, tQa = tb + D + 256, tdOa = tQa + D / 2;

  // All roles walk the same items; ring uses and barrier phases run on across items.
  if (warp == WTMA) {
    if (lane == 0) {
      const uint64_t pol_keep = policy_evict_last();
      const uint64_t pol_stream = policy_evict_normal();
      int ua = 0, ub = 0;  // ring A / ring B uses so far
      auto load_k = [&](const DqItem& w, int j) {
        const int sa = ua % NSA;
        mbar_wait(&emptyA[sa], ((ua / NSA) & 1) ^ 1);
        mbar_arrive_expect_tx(&fullA[sa], C::T128);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_4d(&mapK, &fullA[sa], sA + sa * C::T128 + pn * 128 * 128, pn * 64, w.kvh, w.sq.k0 + j * 128,
                      w.sq.tb, pol_keep);
        ++ua;
      };
      auto load_b = [&](const CUtensorMap* map, int head, int row0, int b, uint64_t pol) {
        const int sb = ub % NB;
        mbar_wait(&emptyB[sb], ((ub / NB) & 1) ^ 1);
        mbar_arrive_expect_tx(&fullB[sb], C::T128);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_4d(map, &fullB[sb], sB + sb * C::T128 + pn * 128 * 128, pn * 64, head, row0, b, pol);
        ++ub;
      };
      for (int r = 0;; ++r) {
        const int item = sched_publish(sched, ctr, r);
        if (item >= num_items) break;
        const DqItem w = dq_decode<CAUSAL>(p, item);
        if (w.n_it == 0) continue;
        load_b(&mapQ, w.h, w.sq.q0 + w.iq * 128, w.sq.tb, pol_stream);
        load_b(&mapdO, w.h, w.sq.q0 + w.iq * 128, w.sq.tb, pol_stream);
        // K (ring A, freed after dQ) for block it+1 goes out right after V (ring B,
        // freed after dP) for block it, keeping K one block ahead.
        load_k(w, 0);
        for (int it = 0; it < w.n_it; ++it) {
          load_b(&mapV, w.kvh, w.sq.k0 + it * 128, w.sq.tb, pol_keep);
          if (it + 1 < w.n_it) load_k(w, it + 1);
        }
      }
    }
  } else if (warp == WMMA) {
    // ================= MMA issuer (whole warp, one elected lane issues) =================
    constexpr uint32_t idesc_sp = idesc_bf16(128, 128, 0, 0);  // S / dP: A (Q/dO) from TMEM, B K-major
    constexpr uint32_t idesc_acc = idesc_bf16(128, D, 0, 1);   // dQ += dS K_j: K_j MN-major
    constexpr uint64_t KMAJ = sdesc_sw128_const(16, 1024);
    constexpr uint64_t MNMAJ = sdesc_sw128_const(128 * 128, 1024);
    const uint32_t aA = smem_u32(sA), aB = smem_u32(sB);
    auto kmaj = [&](uint32_t base, int kk) { return KMAJ | ((base + (kk / 4) * 128 * 128 + (kk % 4) * 32) >> 4); };
    auto mnmaj = [&](uint32_t base, int kk) { return MNMAJ | ((base + kk * 16 * 128) >> 4); };
    int ua = 0, ub = 0;  // ring A / ring B uses so far
    uint32_t g = 0;      // blocks so far (phase of bar_s, bar_sfree, bar_dp, bar_ds)
    uint32_t qa_ph = 0;
    auto issue_s = [&](int u) {
      gemm_ts_kk<D / 16>(tS, tQa, kmaj(aA + (u % NSA) * C::T128, 0), idesc_sp, 0u);
      tc_commit_w(&bar_s);
    };
    auto issue_dp = [&](int u) {
      gemm_ts_kk<D / 16>(tP, tdOa, kmaj(aB + (u % NB) * C::T128, 0), idesc_sp, 0u);
      tc_commit_w(&bar_dp);
      tc_commit_w(&emptyB[u % NB]);  // V: dP is its only use
    };
    for (int r = 0;; ++r) {
      const int item = sched_take(sched, r);
      if (item >= num_items) break;
      const DqItem w = dq_decode<CAUSAL>(p, item);
      const int n = w.n_it;
      if (n == 0) continue;
      const int a0 = ua, v0 = ub + 2;  // ring B: Q_i at ub, dO_i at ub + 1, V_j at v0 + j
      mbar_wait(&bar_qa, qa_ph);        // Q_A, dO_A of this item in TMEM
      qa_ph ^= 1;
      if (lane == 0) {  // their staging slots are free
        mbar_arrive(&emptyB[ub % NB]);
        mbar_arrive(&emptyB[(ub + 1) % NB]);
      }
      mbar_wait(&fullA[a0 % NSA], (a0 / NSA) & 1);
      tc_fence_after();
      issue_s(a0);
      mbar_wait(&fullB[v0 % NB], (v0 / NB) & 1);
      tc_fence_after();
      issue_dp(v0);
      for (int it = 0; it < n; ++it, ++g) {
        const bool more = it + 1 < n;
        mbar_wait(&bar_sfree, g & 1);  // S(it) loaded by the elementwise warps
        if (more) {
          const int u = a0 + it + 1;
          mbar_wait(&fullA[u % NSA], (u / NSA) & 1);
          tc_fence_after();
          issue_s(u);
        }
        mbar_wait(&bar_ds, g & 1);
        tc_fence_after();
        hk_trace(11, g, 1);  // MMA: dS(it) seen, dQ issue
        if constexpr (NWG == 4)
          gemm_tsp4_mn(tdQ, tP, mnmaj(aA + ((a0 + it) % NSA) * C::T128, 0), idesc_acc, it > 0 ? 1u : 0u);
        else
          gemm_tsp_mn(tdQ, tP, mnmaj(aA + ((a0 + it) % NSA) * C::T128, 0), idesc_acc, it > 0 ? 1u : 0u);
        tc_commit_w(&emptyA[(a0 + it) % NSA]);  // K(it): last use dQ(it)
        if (more) {  // dP(it+1) overwrites dS(it): after dQ(it) in issue order
          const int u = v0 + it + 1;
          mbar_wait(&fullB[u % NB], (u / NB) & 1);
          tc_fence_after();
          issue_dp(u);
        }
      }
      tc_commit_w(&bar_acc);
      ua += n;
      ub += n + 2;
    }
    // the releases of the final uses are never waited for by the producer: let them land
    drain_ring(emptyA, NSA, ua);
    drain_ring(emptyB, NB, ub);
  } else {
    const int wg = warp >> 2;              // key columns [CW wg, CW wg + CW) of each block
    const uint32_t lb = (warp & 3) * 32;
    const int r = (warp & 3) * 32 + lane;  // query row within the tile
    const float c = 1.4426950408889634f / sqrtf((float)D);
    const uint32_t cP = tP + CW * wg, cS = tS + CW * wg;
    constexpr int QC = D / NWG;  // dQ columns each warpgroup stores
    uint32_t g = 0, acc_ph = 0;
    int ub = 0;  // ring B uses so far (Q_i of the current item sits at ub, dO_i at ub + 1)
    // WG0 copies Q_i, WG1 dO_i from swizzled SMEM rows into TMEM (A operands)
    auto copy_in = [&]() {
      if (wg >= 2) return;  // WG0 copies Q_i, WG1 dO_i; the others have no copy
      const int u = ub + wg;
      mbar_wait(&fullB[u % NB], (u / NB) & 1);
      const uint8_t* src = sB + (u % NB) * C::T128;
      const uint32_t dst = wg == 0 ? tQa : tdOa;
#pragma unroll
      for (int pn = 0; pn < C::PANELS; ++pn) {
        uint32_t w[32];
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {  // 16-B chunk ch of the row sits at chunk ch ^ (r % 8) (128B swizzle)
          const uint32_t a = smem_u32(src + pn * 128 * 128 + r * 128 + ((ch ^ (r & 7)) * 16));
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w[4 * ch]), "=r"(w[4 * ch + 1]), "=r"(w[4 * ch + 2]), "=r"(w[4 * ch + 3])
                       : "r"(a));
        }
        tmem_st32(tmem_addr(dst + 32 * pn, lb, 0), w);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_qa);
    };
    auto busy = [&](int it) { return it < num_items && dq_decode<CAUSAL>(p, it).n_it > 0; };
    int item = sched_take(sched, 0);
    if (busy(item)) copy_in();
    for (int rr = 1; item < num_items; ++rr) {
      const DqItem w = dq_decode<CAUSAL>(p, item);
      const int q = w.iq * 128 + r;
      const bool q_ok = q < w.sq.lq;  // query rows of a ragged last tile beyond the sequence are not stored
      __nv_bfloat16* out = p.dq + ((size_t)(w.sq.gq0 + (q_ok ? q : 0)) * p.Hq + w.h) * D + wg * QC;
      if (w.n_it == 0) {  // no key visible to these rows: dQ = 0 (accumulate mode: nothing to add)
        if (q_ok && !p.acc32) {
#pragma unroll
          for (int k = 0; k < QC / 8; ++k) reinterpret_cast<uint4*>(out)[k] = make_uint4(0u, 0u, 0u, 0u);
        }
        item = sched_take(sched, rr);
        if (busy(item)) copy_in();
        continue;
      }
      const int off = w.sq.lk - w.sq.lq;  // bottom-right causal alignment
      const size_t vrow = ((size_t)w.b * p.Hq + w.h) * p.Np + q;
      const float l2 = p.lse2[vrow], Dq = p.Dv[vrow];
      for (int it = 0; it < w.n_it; ++it, ++g) {
        float v[CW];
        if (threadIdx.x == 0) hk_trace(1, g, 1);
        mbar_wait(&bar_s, g & 1);
        tc_fence_after();
        if (threadIdx.x == 0) hk_trace(2, g, 1);
        tmem_ld_cols<CW>(tmem_addr(cS, lb, 0), v);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_sfree);  // S buffer free for S(it+1)
#pragma unroll
        for (int k = 0; k < CW / 2; ++k) {
          const float2 e = bwd_exp2_pair<BWD_EMU_OF_8>(
              fma2(make_float2(v[2 * k], v[2 * k + 1]), make_float2(c, c), make_float2(-l2, -l2)), k);
          v[2 * k] = e.x;
          v[2 * k + 1] = e.y;
        }
        // keys beyond the sequence (ragged / varlen tail: K may hold the next
        // sequence's rows) and, when causal, keys > query + (lk - lq) are masked
        if ((it + 1) * 128 > w.sq.lk || (CAUSAL && it * 128 + 127 > w.iq * 128 + off)) {
          const int k0 = it * 128 + CW * wg;
          const int klim = CAUSAL ? min(q + off, w.sq.lk - 1) : w.sq.lk - 1;
#pragma unroll
          for (int cc = 0; cc < CW; ++cc)
            if (k0 + cc > klim) v[cc] = 0.f;
        }
        if (threadIdx.x == 0) hk_trace(3, g, 1);
        mbar_wait(&bar_dp, g & 1);
        tc_fence_after();
        if (threadIdx.x == 0) hk_trace(4, g, 1);
        float dp[CW];
        tmem_ld_cols<CW>(tmem_addr(cP, lb, 0), dp);
        tmem_wait_ld();
#pragma unroll
        for (int cc = 0; cc < CW; cc += 2) {  // packed f32x2: half the issue slots of scalar FADD + FMUL
          const float2 r2 = mul2(make_float2(v[cc], v[cc + 1]),
                                 sub2(make_float2(dp[cc], dp[cc + 1]), make_float2(Dq, Dq)));
          dp[cc] = r2.x;
          dp[cc + 1] = r2.y;
        }
        tmem_st_packed_cols<CW>(tmem_addr(cP, lb, 0), dp);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_ds);
        if (threadIdx.x == 0) hk_trace(5, g, 1);
      }
      ub += w.n_it + 2;
      // ---- epilogue: dQ * (1/sqrt d); warpgroup wg writes columns [QC wg, QC wg + QC)
      mbar_wait(&bar_acc, acc_ph);
      acc_ph ^= 1;
      tc_fence_after();
      uint32_t o[QC];
      if constexpr (QC % 32 == 0) {
#pragma unroll
        for (int c0 = 0; c0 < QC; c0 += 32)
          tmem_ld32(tmem_addr(tdQ, lb, wg * QC + c0), *reinterpret_cast<uint32_t(*)[32]>(&o[c0]));
      } else {
        tmem_ld16(tmem_addr(tdQ, lb, wg * QC), o);
      }
      tmem_wait_ld();
      // the next item's Q/dO go into TMEM before dQ is stored: its S/dP start now.
      // (Its dQ MMAs, which overwrite this accumulator, follow this WG's reads.)
      item = sched_take(sched, rr);  // look ahead: is there a next item?
      if (busy(item)) copy_in();
      const float scale = rsqrtf((float)D);
      if (p.acc32) {  // fp32 accumulate mode: add into the caller's fp32 dQ
        float* outf = reinterpret_cast<float*>(p.dq) + ((size_t)(w.sq.gq0 + (q_ok ? q : 0)) * p.Hq + w.h) * D + wg * QC;
        if (q_ok) {
#pragma unroll
          for (int c0 = 0; c0 < QC; c0 += 8) add8_f32(outf + c0, o + c0, scale);
        }
        continue;
      }
#pragma unroll
      for (int c0 = 0; c0 < QC; c0 += 8) {
        uint4 o4;
        o4.x = pack_bf16(__uint_as_float(o[c0 + 0]) * scale, __uint_as_float(o[c0 + 1]) * scale);
        o4.y = pack_bf16(__uint_as_float(o[c0 + 2]) * scale, __uint_as_float(o[c0 + 3]) * scale);
        o4.z = pack_bf16(__uint_as_float(o[c0 + 4]) * scale, __uint_as_float(o[c0 + 5]) * scale);
        o4.w = pack_bf16(__uint_as_float(o[c0 + 6]) * scale, __uint_as_float(o[c0 + 7]) * scale);
        if (q_ok) *reinterpret_cast<uint4*>(out + c0) = o4;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WMMA) tmem_dealloc<512>(tb);
  if (threadIdx.x == 0) sched_exit(ctr);
}

// ---------------------------------------------------------------- B2 from the stored dS
// dQ(qi) = (1/sqrt d) sum_j dS(qi, j) K_j with dS read back from the workspace (written by the dK/dV
// pass, bwd_dkdv_kernel with p.ds): one 128 x 128 x 128 GEMM per block instead of the three of
// bwd_dq_kernel (S and dP recomputed there). The pass is HBM-bound (32 KB of dS per 512 tensor
// cycles). Persistent, dynamic schedule (items as dq_decode: heaviest first). Roles: warp 0 producer
// (1-D bulk copy of the 32 KB dS image + TMA of K_j into a 3-stage ring), warp 1 MMA (dQ += dS K_j into
// one of two TMEM accumulators), warps 2-5 epilogue (TMEM -> bf16 rows, or added into fp32 dQ).
struct DqdsCfg {
  static constexpr int NS = 3;
  static constexpr uint32_t TILE = 128 * 128 * 2;  // 32 KB
  static constexpr uint32_t STAGE = 2 * TILE;      // dS block | K_j
  static constexpr uint32_t SMEM = NS * STAGE + 1024;
  static constexpr int THREADS = 192;
};

template <bool CAUSAL>
__global__ void __launch_bounds__(DqdsCfg::THREADS, 1)
    bwd_dqds_kernel(const __grid_constant__ CUtensorMap mapK, const BwdParams p) {
  using C = DqdsCfg;
  constexpr int D = 128, NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[NS], empty[NS], tfull[2], tempty[2];
  __shared__ Sched sched;
  __shared__ uint32_t tmem_base_s;
  const int warp = warp_id(), lane = lane_id();
  const int num_items = p.B * p.Hq * (p.Np / 128);
  unsigned* const ctr = p.sched + 2;
  if (threadIdx.x == 0) {
    sched_init(sched, 5);  // MMA warp + 4 epilogue warps
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0) tma_prefetch(&mapK);
  if (warp == 1) tmem_alloc<256>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base_s, 0);

  if (warp == 0) {
    // ================= producer =================
    if (lane == 0) {
      const uint64_t pol_k = policy_evict_last();
      const uint64_t pol_ds = policy_evict_first();  // each dS tile is read once
      int u = 0;
      for (int r = 0;; ++r) {
        const int item = sched_publish(sched, ctr, r);
        if (item >= num_items) break;
        const DqItem w = dq_decode<CAUSAL>(p, item);
        for (int j = 0; j < w.n_it; ++j, ++u) {
          const int s = u % NS;
          mbar_wait(&empty[s], ((u / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], C::STAGE);
          uint8_t* st = smem + s * C::STAGE;
          bulk_load_hint(st, p.ds + ds_block_index(p, w.b, w.h, w.iq, j) * DS_BLOCK_ELEMS, C::TILE, &full[s], pol_ds);
          for (int pn = 0; pn < 2; ++pn)
            tma_load_4d(&mapK, &full[s], st + C::TILE + pn * 128 * 128, pn * 64, w.kvh, w.sq.k0 + j * 128, w.sq.tb,
                        pol_k);
        }
      }
      drain_ring(empty, NS, u);
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    constexpr uint32_t idesc = idesc_bf16(128, D, 1, 1);  // M = 128 queries, A = dS and B = K MN-major
    constexpr uint64_t MNMAJ = sdesc_sw128_const(128 * 128, 1024);
    const uint32_t a0 = smem_u32(smem);
    int u = 0, n_items = 0;
    for (int r = 0;; ++r) {
      const int item = sched_take(sched, r);
      if (item >= num_items) break;
      const DqItem w = dq_decode<CAUSAL>(p, item);
      const int a = n_items & 1;
      // every item takes a turn of its accumulator (an item without keys commits no MMA: its tfull
      // completes at once and the epilogue writes zeros), so both sides count phases per item
      mbar_wait(&tempty[a], ((n_items >> 1) & 1) ^ 1);  // the epilogue has read this accumulator out
      for (int j = 0; j < w.n_it; ++j, ++u) {
        const int s = u % NS;
        mbar_wait(&full[s], (u / NS) & 1);
        tc_fence_after();
        const uint32_t st = a0 + s * C::STAGE;
        gemm_ss_mnmn(tb + 128 * a, MNMAJ | (st >> 4), MNMAJ | ((st + C::TILE) >> 4), idesc, j > 0 ? 1u : 0u);
        tc_commit_w(&empty[s]);
      }
      tc_commit_w(&tfull[a]);
      ++n_items;
    }
  } else {
    // ================= epilogue (warps 2-5: TMEM lane quadrant warp % 4) =================
    const uint32_t lb = (warp & 3) * 32;
    const int r = (warp & 3) * 32 + lane;  // query row within the tile
    const float scale = rsqrtf((float)D);
    int n_items = 0;
    for (int rr = 0;; ++rr) {
      const int item = sched_take(sched, rr);
      if (item >= num_items) break;
      const DqItem w = dq_decode<CAUSAL>(p, item);
      const int a = n_items & 1;
      const int row = w.iq * 128 + r;
      const bool row_ok = row < w.sq.lq;
      const size_t base = ((size_t)(w.sq.gq0 + (row_ok ? row : 0)) * p.Hq + w.h) * D;
      mbar_wait(&tfull[a], (n_items >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t o[32];
        if (w.n_it > 0) {
          tmem_ld32(tmem_addr(tb + 128 * a, lb, c0), o);
          tmem_wait_ld();
          if (c0 + 32 == D) {  // accumulator read out: the item after next may overwrite it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[a]);
          }
        } else {  // no key visible to this tile: dQ = 0
#pragma unroll
          for (int k = 0; k < 32; ++k) o[k] = 0u;
          if (c0 + 32 == D) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[a]);
          }
        }
        if (p.acc32 && w.n_it == 0) continue;  // accumulate mode: nothing to add
        if (!row_ok) continue;
        if (p.acc32) {
          float* dst = reinterpret_cast<float*>(p.dq) + base + c0;
#pragma unroll
          for (int k = 0; k < 4; ++k) add8_f32(dst + 8 * k, o + 8 * k, scale);
        } else {
          uint4 v[4];
          uint32_t* vp = reinterpret_cast<uint32_t*>(v);
#pragma unroll
          for (int k = 0; k < 16; ++k)
            vp[k] = pack_bf16(__uint_as_float(o[2 * k]) * scale, __uint_as_float(o[2 * k + 1]) * scale);
          uint4* dst = reinterpret_cast<uint4*>(p.dq + base + c0);
#pragma unroll
          for (int k = 0; k < 4; ++k) dst[k] = v[k];
        }
      }
      ++n_items;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tb);
  if (threadIdx.x == 0) sched_exit(ctr);
}

// ---------------------------------------------------------------- host launch
#ifndef HK_BWD_FORK
#define HK_BWD_FORK 1
#endif
// One non-blocking side stream per (device, caller stream) for the forked dQ pass, created on
// first use with the caller stream's priority and never destroyed. Keying by the caller's
// stream keeps concurrent backward calls on different streams independent (no false
// cross-stream dependencies, and a graph capture on one stream never pulls in another
// caller's work). Beyond 256 distinct caller streams the call runs serially on `stream`.
inline cudaStream_t side_stream(cudaStream_t caller) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, cudaStream_t> streams;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(dev, caller);
  const auto it = streams.find(key);
  if (it != streams.end()) return it->second;
  if (streams.size() >= 256) return nullptr;
  int prio = 0;
  if (cudaStreamGetPriority(caller, &prio) != cudaSuccess) prio = 0;
  cudaStream_t s2 = nullptr;
  if (cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, prio) != cudaSuccess) {
    (void)cudaGetLastError();  // fall back to serial launches without leaving a sticky error behind
    return nullptr;
  }
  streams.emplace(key, s2);
  return s2;
}

template <typename F>
inline bool set_smem(F* fn, uint32_t bytes) {
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)bytes) == cudaSuccess;
}

// Geometry of one backward call: dense (cu_q == nullptr: Q [B][Nq][Hq][d],
// K [B][Nk][Hkv][d]) or varlen (Q [total_q][Hq][d], K [total_k][Hkv][d]).
struct BwdShape {
  const int* cu_q;
  const int* cu_k;
  int B, Hq, Hkv, Nq, Nk;  // varlen: Nq, Nk = max_seqlen_q, max_seqlen_k
  int total_q, total_k;    // varlen only
  bool fused;              // d = 64: single-pass dQ (bulk reduce-add into the fp32 accumulator) — not bitwise
  bool acc32;              // HK_BWD_ACCUMULATE_F32: dQ, dK, dV are fp32 accumulators
  bool ds;                 // stored-dS backward (bwd_ds_bytes > 0 and the workspace holds it)
};

// Workspace layout of one backward call (hk_attn.h): D and LSE2 [B][Hq][Np] fp32, 256 bytes of work
// counters, then the fused backward's fp32 dQ accumulator: B * Np * Hq * d floats, which covers
// [B][Nq][Hq][d] (dense) and [total_q][Hq][d] (varlen: total_q <= B * max_seqlen_q).
// The fused single pass at d = 128 (1 CTA per key tile, dQ_partial in the S^T columns, staging in
// the dS tile) is correct but measured 0.64-0.83x of the two-pass backward (its 64 KB
// of dQ partials per block need ~26 B/clk/SM of L2 reduce bandwidth, the chip's whole measured
// rate, on the S^T critical path): built only with -DHK_FUSED128=1.
#ifndef HK_FUSED128
#define HK_FUSED128 0
#endif
constexpr bool bwd_fused_default(int d) { return d == 64 || HK_FUSED128; }

// Stored-dS backward (d = 128, dense, not the fused pass): bf16 dS tiles of every visited block after
// the workspace's first part, at a 1024-byte aligned offset; 0 where the path does not apply.
inline size_t bwd_ds_bytes(int B, int Hq, int Nq, int Nk, int d, bool causal, bool varlen) {
  if (d != 128 || varlen || bwd_fused_default(d) || B <= 0 || Hq <= 0 || Nq <= 0 || Nk <= 0) return 0;
  const size_t Tq = ((size_t)Nq + 127) / 128, Tk = ((size_t)Nk + 127) / 128;
  const size_t per_head = (causal && Nq == Nk) ? Tq * (Tq + 1) / 2 : Tq * Tk;
  return (size_t)B * Hq * per_head * DS_BLOCK_ELEMS * 2;
}
inline size_t bwd_ds_offset(size_t ws) { return (ws + 1023) / 1024 * 1024; }

inline size_t bwd_ws_bytes(int B, int Hq, int Nq, int d) {
  if (B <= 0 || Hq <= 0 || Nq <= 0) return 0;
  const size_t Np = ((size_t)Nq + 127) / 128 * 128;
  return (size_t)2 * B * Hq * Np * sizeof(float) + 256 +
         (bwd_fused_default(d) ? (size_t)B * Np * Hq * d * sizeof(float) : 0);
}

template <int D, bool CAUSAL>
hk_status launch_bwd_t(const void* Q, const void* K, const void* V, const void* O, const float* LSE, const void* dO,
                       void* dQ, void* dK, void* dV, float* ws, const BwdShape& sh, cudaStream_t stream, char* err,
                       size_t errlen, int phase, int num_sms) {
  using C = BwdCfg<D>;
  const int B = sh.B, Hq = sh.Hq, Hkv = sh.Hkv;
  const int Np = (sh.Nq + 127) / 128 * 128;   // workspace rows padded to whole tiles
  const int Npk = (sh.Nk + 127) / 128 * 128;  // key tiles
  float* Dv = ws;
  float* lse2 = ws + (size_t)B * Hq * Np;
  // every operand tile is a 128-row box (two 64-column panels at D=128)
  const bool varlen = sh.cu_q != nullptr;
  const int mb = varlen ? 1 : B, mnq = varlen ? sh.total_q : sh.Nq, mnk = varlen ? sh.total_k : sh.Nk;
  CUtensorMap mQ, mdO, mK, mV;
  bool ok = encode_bnhd(&mQ, Q, mb, mnq, Hq, D, 128) && encode_bnhd(&mdO, dO, mb, mnq, Hq, D, 128) &&
            encode_bnhd(&mK, K, mb, mnk, Hkv, D, 128) && encode_bnhd(&mV, V, mb, mnk, Hkv, D, 128);
  if (!ok) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled failed (CUresult %d)", last_encode_result());
    return HK_ERR_DEVICE;
  }
  {  // max dynamic smem, once per (instantiation, device), under a lock (concurrent first calls)
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!done.count(dev)) {
      bool ok2 = set_smem(bwd_dkdv_kernel<D, CAUSAL, false>, C::SMEM1) && set_smem(bwd_dq_kernel<D, CAUSAL>, C::SMEM2);
      ok2 = ok2 && set_smem(bwd_dkdv_kernel<D, CAUSAL, true>, C::SMEM1F);
      if (D == 128)
        ok2 = ok2 && set_smem(bwd_dqds_kernel<CAUSAL>, DqdsCfg::SMEM) &&
              set_smem(bwd_dkdv_kernel<D, CAUSAL, false, D == 128>, C::SMEM1);
      if (!ok2) {
        snprintf(err, errlen, "cudaFuncSetAttribute(max dynamic smem) failed");
        return HK_ERR_DEVICE;
      }
      done.insert(dev);
    }
  }
  unsigned* sched = reinterpret_cast<unsigned*>(ws + (size_t)2 * B * Hq * Np);  // 4 counters after D, LSE2
  const bool fq = sh.fused;
  float* dq_acc = fq ? ws + (size_t)2 * B * Hq * Np + 64 : nullptr;  // after the 256-byte counter block
  CUtensorMap mDQ = mK;  // unused by the two-pass kernels
  if (fq && !encode_bnhd_f32(&mDQ, dq_acc, mb, mnq, Hq, D)) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled (dQ accumulator) failed (CUresult %d)", last_encode_result());
    return HK_ERR_DEVICE;
  }
  SeqGeom g{sh.cu_q, sh.cu_k, sh.Nq, sh.Nk, sh.total_q};
  BwdParams p{Dv,
              lse2,
              reinterpret_cast<__nv_bfloat16*>(dQ),
              reinterpret_cast<__nv_bfloat16*>(dK),
              reinterpret_cast<__nv_bfloat16*>(dV),
              sched,
              g,
              B,
              Hq,
              Hkv,
              Np,
              Npk,
              sh.acc32,
              sh.ds ? reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(ws) +
                                                      bwd_ds_offset(bwd_ws_bytes(B, Hq, sh.Nq, D)))
                    : nullptr,
              CAUSAL && sh.Nq == sh.Nk ? 1 : 0};
  // B0: grid (x, b), x sized for the longest sequence and capped at ~16 blocks per SM overall
  const size_t rows = (size_t)sh.Nq * Hq;
  constexpr int RPW0 = 32 / (D / (8 * pre_vpl(D)));  // rows per warp pass of the preprocess
  const size_t warps_needed = (rows + RPW0 - 1) / RPW0;
  size_t bx = (warps_needed + 7) / 8;
  size_t cap = (size_t)num_sms * 16 / (size_t)B;
  if (cap < 1) cap = 1;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  if (phase < 0 || phase == 0)
    bwd_pre_kernel<D><<<dim3((unsigned)bx, (unsigned)B), 256, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(O), reinterpret_cast<const __nv_bfloat16*>(dO), LSE, Dv, lse2, g, Hq,
        (Hq & (Hq - 1)) == 0 ? __builtin_ctz((unsigned)Hq) : -1, Np, sched, dq_acc);
  // B1, B2. They are independent (both only read the preprocess output): with HK_BWD_FORK the dQ
  // pass goes on a side stream forked from `stream` after B0 and joined back after it, so its
  // CTAs take the SMs the dK/dV pass's last CTAs free instead of waiting for the whole pass.
  cudaStream_t s2 = stream;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (HK_BWD_FORK && phase < 0 && !fq && !sh.ds) {  // (the stored-dS dQ pass reads the dK/dV pass's dS)
    s2 = side_stream(stream);
    if (s2 && cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventRecord(ev_fork, stream) == cudaSuccess && cudaStreamWaitEvent(s2, ev_fork, 0) == cudaSuccess) {
    } else {
      s2 = stream;  // no side stream: serial launches on `stream`
      (void)cudaGetLastError();
    }
  }
  if (phase < 0 || phase == 1) {
    const int items = B * Hkv * (Npk / 128);  // persistent: one CTA per SM
    const int grid = items < num_sms ? items : num_sms;
    if (fq)
      bwd_dkdv_kernel<D, CAUSAL, true><<<grid, C::THREADS1F, C::SMEM1F, stream>>>(mQ, mdO, mK, mV, mDQ, p);
    else if (D == 128 && sh.ds)
      bwd_dkdv_kernel<D, CAUSAL, false, D == 128><<<grid, C::THREADS1, C::SMEM1, stream>>>(mQ, mdO, mK, mV, mDQ, p);
    else
      bwd_dkdv_kernel<D, CAUSAL, false><<<grid, C::THREADS1, C::SMEM1, stream>>>(mQ, mdO, mK, mV, mDQ, p);
  }
  if (fq && (phase < 0 || phase == 2)) {  // dQ = bf16(dQ_acc / sqrt(d)), grid (x, sequence) like B0
    dq_convert_kernel<D><<<dim3((unsigned)bx, (unsigned)B), 256, 0, stream>>>(
        dq_acc, reinterpret_cast<__nv_bfloat16*>(dQ), g, Hq, rsqrtf((float)D), sh.acc32);
  }
  if (D == 128 && sh.ds && (phase < 0 || phase == 2)) {
    const int items = B * Hq * (Np / 128);
    bwd_dqds_kernel<CAUSAL><<<items < num_sms ? items : num_sms, DqdsCfg::THREADS, DqdsCfg::SMEM, stream>>>(mK, p);
  } else if (!fq && (phase < 0 || phase == 2)) {
    const int items = B * Hq * (Np / 128);  // persistent: one CTA per SM
    bwd_dq_kernel<D, CAUSAL><<<items < num_sms ? items : num_sms, C::THREADS2, C::SMEM2, s2>>>(mQ, mdO, mK, mV,
                                                                                             p);
  }
  if (s2 != stream) {
    cudaEventRecord(ev_join, s2);
    cudaStreamWaitEvent(stream, ev_join, 0);
  }
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(err, errlen, "hk_attn_bwd launch failed: %s", cudaGetErrorString(e));
    return HK_ERR_LAUNCH;
  }
  return HK_OK;
}

inline hk_status launch_bwd(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                            const void* dO, void* dQ, void* dK, void* dV, float* ws, const BwdShape& sh, int d,
                            bool causal, cudaStream_t stream, char* err, size_t errlen, int phase, int num_sms) {
  if (d == 64)
    return causal ? launch_bwd_t<64, true>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, sh, stream, err, errlen, phase, num_sms)
                  : launch_bwd_t<64, false>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, sh, stream, err, errlen, phase, num_sms);
  return causal ? launch_bwd_t<128, true>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, sh, stream, err, errlen, phase, num_sms)
                : launch_bwd_t<128, false>(Q, K, V, O, LSE, dO, dQ, dK, dV, ws, sh, stream, err, errlen, phase, num_sms);
}

}  // namespace hk
