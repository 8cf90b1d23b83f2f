// BF16 GEMM C = A B^T on sm_100a (the paper's GEMM
// listing accumulates mma_ABt over K_STEP slices of row-major A [M,K] and
// B [N,K]: P:1160-1193, 256x256 output tile per block P:1044, benchmarked at
// M = N = K = 8192 with N(0,1) inputs; the B200 bars it prints are
// TK 1538 and CUTLASS 1570 TFLOP/s).
//
// B200 design: a persistent kernel of CTA PAIRS (cluster of 2
// on one TPC). A pair computes one 256x256 C tile per item with
// tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16): CTA r holds rows
// 128r.. of the A slice and rows 128r.. of the B slice, so each SM reads only
// half of B from its own shared memory (the 1-CTA 128x256 shape would need
// 192 B/clk of shared-memory traffic against 128 available).
//   warp 0      TMA producer (both CTAs): per 64-wide K stage, its A and B
//               halves (2 x 16 KB), completing on the LEADER's full barrier
//   warp 1      MMA issuer (leader CTA only): 4 MMAs per stage, stage release
//               and accumulator-ready commits multicast to both CTAs
//   warps 2-5   epilogue (both CTAs): TMEM -> registers -> bf16 -> global
// TMEM: two 256-column fp32 accumulators (512 columns), so the epilogue of
// one tile overlaps the MMAs of the next. SMEM: 6 stages x 32 KB.
#pragma once
#include "ptx.cuh"

namespace hk {

struct GemmParams {
  __nv_bfloat16* c;  // [M][N] row-major
  int M, N, K;
  int tiles_m, tiles_n;  // M / 256, N / BNP
};

constexpr int GEMM_BK = 64;                           // K per stage: one 128-B swizzle panel
constexpr uint32_t GEMM_HALF = 128 * GEMM_BK * 2;     // 16 KB: 128 rows x 64 bf16
constexpr int GEMM_THREADS = 192;
// BNP = N extent of a pair tile: 256 (one 256-column accumulator per CTA, two
// buffers) or 512 (two 256-column accumulators per CTA covering N = 512: each
// stage moves A-half + 2 B-halves = 48 KB per CTA for twice the MMA work, 25%
// fewer operand bytes per FLOP through L2 -- the kernel is power-capped and
// that traffic costs clock).
template <int BNP>
struct GemmCfg {
  static constexpr int NB = BNP / 256;                         // B halves per CTA per stage
  static constexpr uint32_t STAGE = (1 + NB) * GEMM_HALF;      // A half + NB B halves
  static constexpr int STAGES = BNP == 256 ? 6 : 4;
  static constexpr uint32_t SMEM = STAGES * STAGE + 1024;
};
constexpr int GEMM_GROUP_M = 8;                       // tile raster: 8 M-tiles share B tiles in L2

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address -> shared::cluster address of the same variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(saddr), "r"(rank));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive on another CTA's barrier with the default .release.cta semantics (as CUTLASS's
// ClusterBarrier::arrive(cta_id)): enough where tcgen05 fences order the work being signalled
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
// 2-D TMA tile load into this CTA's shared memory whose completion (bytes) is
// signalled on the leader CTA's barrier (cluster address).
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t bar_cluster, void* dst, int c0,
                                                 int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
// Commit of this thread's earlier MMAs to the barrier at the same offset in both CTAs.
__device__ __forceinline__ void tc_commit_pair_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::
          "r"(smem_u32(bar))
      : "memory");
}
// One K stage (4 x K=16) of the pair GEMM: both operands K-major SW128, 128-row tiles
// per CTA; descriptors step 32 B (2 units) per K=16.
__device__ __forceinline__ void gemm_pair_stage(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e, t;\n\t.reg .b64 a, b;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, %4, %4;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "add.s64 a, %1, 2;\n\tadd.s64 b, %2, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, t;\n\t"
      "add.s64 a, %1, 4;\n\tadd.s64 b, %2, 4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, t;\n\t"
      "add.s64 a, %1, 6;\n\tadd.s64 b, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, t;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// Grouped raster: GEMM_GROUP_M consecutive M tiles walk the N tiles together.
__device__ __forceinline__ void gemm_tile_coords(const GemmParams& p, int t, int& mt, int& nt) {
  const int per_group = GEMM_GROUP_M * p.tiles_n;
  const int first_m = (t / per_group) * GEMM_GROUP_M;
  const int gsz = min(p.tiles_m - first_m, GEMM_GROUP_M);
  const int r = t % per_group;
  mt = first_m + r % gsz;
  nt = r / gsz;
}

template <int BNP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const GemmParams p) {
  using C = GemmCfg<BNP>;
  constexpr int GEMM_STAGES = C::STAGES;
  constexpr uint32_t GEMM_STAGE = C::STAGE;
  constexpr int NB = C::NB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // tfull: accumulator(s) of a tile complete; tempty[a]: TMEM columns [256a, 256a+256)
  // free again (BNP = 256: two alternating accumulators; BNP = 512: the two halves
  // of one accumulator, released half by half by the epilogue)
  __shared__ uint64_t full[GEMM_STAGES], empty[GEMM_STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_s;

  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int warp = warp_id(), lane = lane_id();
  const int ktiles = p.K / GEMM_BK;
  const int ntiles = p.tiles_m * p.tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < GEMM_STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive + both CTAs' bytes
      mbar_init(&empty[s], 1);  // multicast MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);   // multicast MMA commit
      mbar_init(&tempty[a], 8);  // leader: 4 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    tmem_alloc_pair<512>(&tmem_base_s);
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits and the TMEM allocation visible to both CTAs
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base_s, 0);

  if (warp == 0) {
    // ================= TMA producer (both CTAs) =================
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      const uint32_t full_leader = mapa_shared(smem_u32(&full[0]), 0);
      int it = 0;  // K stages so far (ring position)
      for (int t = pair; t < ntiles; t += npairs) {
        int mt, nt;
        gemm_tile_coords(p, t, mt, nt);
        for (int kt = 0; kt < ktiles; ++kt, ++it) {
          const int s = it % GEMM_STAGES;
          mbar_wait(&empty[s], ((it / GEMM_STAGES) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * GEMM_STAGE);  // both CTAs' halves
          uint8_t* st = smem + s * GEMM_STAGE;
          tma_load_2d_pair(&mapA, full_leader + 8 * s, st, kt * GEMM_BK, mt * 256 + rank * 128, pol);
#pragma unroll
          for (int h = 0; h < NB; ++h)  // B rows [256h + 128 rank, +128) of this tile's BNP
            tma_load_2d_pair(&mapB, full_leader + 8 * s, st + (1 + h) * GEMM_HALF, kt * GEMM_BK,
                             nt * BNP + 256 * h + rank * 128, pol);
        }
      }
      // let the final (never awaited) stage releases land before exit
      for (int s = 0; s < GEMM_STAGES && s < it; ++s) {
        const int last = it - 1 - ((it - 1 - s) % GEMM_STAGES);
        mbar_wait(&empty[s], (last / GEMM_STAGES) & 1);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA, whole warp) =================
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(256, 256, 0, 0);  // A, B K-major
      constexpr uint64_t KMAJ = sdesc_sw128_const(16, 1024);
      const uint32_t a0 = smem_u32(smem);
      int it = 0, tc = 0;
      for (int t = pair; t < ntiles; t += npairs, ++tc) {
        const int acc = NB == 1 ? (tc & 1) : 0;
        // both epilogues done with the TMEM columns this tile accumulates into
        const uint32_t te_ph = NB == 1 ? (((tc >> 1) & 1) ^ 1) : ((tc & 1) ^ 1);
        for (int kt = 0; kt < ktiles; ++kt, ++it) {
          const int s = it % GEMM_STAGES;
          mbar_wait(&full[s], (it / GEMM_STAGES) & 1);
          const uint32_t sa = a0 + s * GEMM_STAGE;
#pragma unroll
          for (int h = 0; h < NB; ++h) {
            if (kt == 0) mbar_wait(&tempty[NB == 1 ? acc : h], te_ph);
            tc_fence_after();
            gemm_pair_stage(tbase + (NB == 1 ? acc : h) * 256, KMAJ | (sa >> 4),
                            KMAJ | ((sa + (1 + h) * GEMM_HALF) >> 4), idesc, kt > 0 ? 1u : 0u);
          }
          tc_commit_pair_w(&empty[s]);
        }
        tc_commit_pair_w(&tfull[acc]);
      }
    }
  } else {
    // ================= epilogue (both CTAs): warps 2-5 =================
    const uint32_t lane_base = (warp & 3) * 32;  // TMEM lanes this warp may access
    const int r = lane_base + lane;              // row within this CTA's 128 rows
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    int tc = 0;
    for (int t = pair; t < ntiles; t += npairs, ++tc) {
      int mt, nt;
      gemm_tile_coords(p, t, mt, nt);
      const int acc = NB == 1 ? (tc & 1) : 0;
      mbar_wait(&tfull[acc], NB == 1 ? ((tc >> 1) & 1) : (tc & 1));
      tc_fence_after();
      const int row = mt * 256 + rank * 128 + r;
      __nv_bfloat16* crow = p.c + (size_t)row * p.N + nt * BNP;
#ifndef HK_GEMM_EPI_EARLY
#define HK_GEMM_EPI_EARLY 1
#endif
      if (HK_GEMM_EPI_EARLY) {
        // each 256-column half: read all of it out of TMEM (packed to bf16 as it arrives), release it to
        // the MMA warp, then store — the release no longer waits behind this half's global stores, and
        // it uses the .release.cta form of the remote arrive (the .release.cluster form compiles to a
        // full memory barrier, which would wait for the previous half's stores to complete)
#pragma unroll 1
        for (int h = 0; h < NB; ++h) {
          uint32_t pk[128];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint32_t v[32];
            tmem_ld32(tmem_addr(tbase + acc * 256, lane_base, 256 * h + 32 * c), v);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 16; ++k) pk[16 * c + k] = pack_bf16(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(tempty_leader + 8 * (NB == 1 ? acc : h));
          uint4* dst = reinterpret_cast<uint4*>(crow + 256 * h);
#pragma unroll
          for (int k = 0; k < 32; ++k) dst[k] = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
        }
      } else {
#pragma unroll 1
      for (int c0 = 0; c0 < BNP; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_addr(tbase + acc * 256, lane_base, c0), v);
        tmem_wait_ld();
        if ((c0 & 255) == 256 - 32) {  // 256 columns fully read: the MMA may reuse them
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader + 8 * (NB == 1 ? acc : c0 / 256));
        }
        uint4 o[4];
        uint32_t* op = reinterpret_cast<uint32_t*>(o);
#pragma unroll
        for (int k = 0; k < 16; ++k) op[k] = pack_bf16(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
        uint4* dst = reinterpret_cast<uint4*>(crow + c0);
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[k] = o[k];
      }
      }
    }
  }

  tc_fence_before();
  cluster_sync_all();  // both CTAs done (MMAs, epilogue reads, remote arrivals) before TMEM is freed
  if (warp == 0) tmem_dealloc_pair<512>(tbase);
}

}  // namespace hk
