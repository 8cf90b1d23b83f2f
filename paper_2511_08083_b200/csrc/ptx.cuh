// Thin inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05 (UMMA/TMEM).
// Bit layouts follow the PTX ISA (tcgen05 instruction / shared-memory
// descriptors); nothing here is specific to attention.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>

namespace hk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------------ tracing (HK_TRACE builds only)
// hk_trace(ev, a, b): one traced CTA stores clock64 at slot (ev, a) of a device
// table, a < 1024 (later indices are dropped; a plain store: no atomics on the hot
// path), read back by hk_diag_trace_read (include/hk_attn_diag.h). `b` is unused.
#ifdef HK_TRACE
__device__ unsigned long long g_hk_trace[64 * 1024];
__device__ __forceinline__ bool hk_trace_cta() {
  return blockIdx.x == gridDim.x / 2 && blockIdx.y == 0 && blockIdx.z == 0;
}
__device__ __forceinline__ void hk_trace(uint32_t ev, uint32_t a, uint32_t) {
  if (hk_trace_cta() && a < 1024) g_hk_trace[(ev & 63) * 1024 + a] = (unsigned long long)clock64();
}
#else
__device__ __forceinline__ void hk_trace(uint32_t, uint32_t, uint32_t) {}
#endif

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
#ifdef HK_DEBUG_HANG
// Debug build: bounded spin, then report the barrier and trap (turns a hang into an error).
__device__ __forceinline__ void mbar_wait_dbg(uint64_t* bar, uint32_t parity, int line) {
  for (long long i = 0; i < (1ll << 28); ++i) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
  }
  printf("HK hang: line %d block (%d,%d,%d) thread %d bar smem 0x%x parity %u\n", line, blockIdx.x, blockIdx.y,
         blockIdx.z, threadIdx.x, smem_u32(bar), parity);
  __trap();
}
#define mbar_wait(bar, parity) mbar_wait_dbg((bar), (parity), __LINE__)
#else
// HK_WAIT_HINT (ns): suspend-time hint of try_wait. Without it the hardware returns after
// a short, system-dependent time and the retry loop (try_wait, branch, yield) issued ~18% of
// all forward instructions (ncu r1g), taking issue slots from the softmax warps of the same
// sub-partition; the warp is woken when the phase completes either way.
#ifndef HK_WAIT_HINT
#define HK_WAIT_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if HK_WAIT_HINT
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"((uint32_t)HK_WAIT_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
#endif

// Non-blocking probe of a phase (all lanes of a converged warp call it; the
// result is OR-ed across the warp so the warp never diverges on it).
__device__ __forceinline__ bool mbar_test_warp(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return __any_sync(0xffffffffu, ok != 0);
}

// Non-blocking probe from a single thread.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 4-D tiled load (coords innermost first) completing on `bar`.
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                            int c1, int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (bytes % 16 == 0, both 16-B aligned) completing on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// Bulk-async reduce-add of a shared-memory tile into global memory through a 4-D tensor map
// (fp32 add; the dQ accumulator of the fused backward).
__device__ __forceinline__ void tma_reduce_add_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                  int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// L2 prefetch of one 4-D tile (no shared memory, no completion): warms L2 for a later tma_load_4d.
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
// 1-D bulk copy shared -> global (bytes % 16 == 0, both 16-B aligned), in the current bulk group
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(dst)),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// the same with an L2 cache-policy hint (e.g. evict_first for data read once, much later)
__device__ __forceinline__ void bulk_store_hint(void* dst, const void* src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                   reinterpret_cast<uint64_t>(dst)),
               "r"(smem_u32(src)), "r"(bytes), "l"(policy)
               : "memory");
}
// 1-D bulk copy global -> shared with an L2 cache-policy hint
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 16-byte shared-memory store at a 32-bit shared address (a generic-pointer store through a
// computed address compiles to ST.E with a 64-bit address per chunk)
__device__ __forceinline__ void sts_v4(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ------------------------------------------------------------------ named barriers
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ register reallocation
template <uint32_t N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

// ------------------------------------------------------------------ tcgen05: TMEM
// Allocation is warp-collective; the TMEM base address is written to smem.
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrive (once) on `bar` when all prior tcgen05.mma of this thread complete.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// TMEM address: lane in bits [31:16], column in [15:0].
__device__ __forceinline__ uint32_t tmem_addr(uint32_t base, uint32_t lane, uint32_t col) {
  return base + (lane << 16) + col;
}

// 32 lanes x 32 bit, 32 consecutive columns per thread (thread t <- lane 32*(warp%4)+t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ tcgen05: MMA
// Instruction descriptor for kind::f16 with bf16 A/B and fp32 accumulate.
//   [4,6) D format (1 = f32)  [7,10) A format (1 = bf16)  [10,13) B format (1 = bf16)
//   bit 15 A major (0 = K, 1 = MN)  bit 16 B major  [17,23) N >> 3  [24,29) M >> 4
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn_major,
                                                  uint32_t b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn_major << 15) | (b_mn_major << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), version 1.
//   [0,14) start >> 4   [16,30) LBO >> 4   [32,46) SBO >> 4   [46,48) version = 1
//   [49,52) base offset = 0 (tiles are 1024-B aligned)   [61,64) layout = 2 (128B swizzle)
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Constant part of a SWIZZLE_128B descriptor (LBO, SBO, version, layout); OR in
// (smem address >> 4) for the start field. Shared-memory addresses are < 2^18,
// so adding byte offsets >> 4 to a descriptor never carries out of the field.
__host__ __device__ constexpr uint64_t sdesc_sw128_const(uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Constant part of a descriptor of any layout type (0 none, 2 SW128, 4 SW64, 6 SW32).
__host__ __device__ constexpr uint64_t sdesc_const(uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
  return ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// D[tmem] (+)= A[smem] * B[smem]
__device__ __forceinline__ void umma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-collective forms: called by all 32 lanes of a converged warp with
// warp-uniform operands (kept in uniform registers); one elected lane issues.
__device__ __forceinline__ void umma_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// ---- whole-GEMM issue: one elect.sync, then the NK k-steps of one 128 x N x 16NK
// GEMM with the operand descriptors / TMEM columns advanced by immediates inside
// the asm (one instruction each instead of per-step descriptor math + elect).
// Offsets in 16-byte units (descriptor start-address field) or TMEM columns:
//   K-major SW128, 128-row tile: k-step kk at (kk/4)*1024 + (kk%4)*2
//   MN-major SW128:              k-step kk at kk*128 (16 rows of 128 B)
//   TMEM A, contiguous bf16:     kk*8 columns;  packed by two warpgroups: packed_col(kk)
#define HK_MMA_HEAD                                   \
  "{\n\t.reg .pred p, e, t;\n\t.reg .b64 a, b;\n\t"  \
  ".reg .b32 ta;\n\t"                                  \
  "setp.ne.b32 p, %4, 0;\n\t"                          \
  "setp.eq.b32 t, %4, %4;\n\t"                         \
  "elect.sync _|e, 0xffffffff;\n\t"
#define HK_SS_FIRST "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
#define HK_SS_STEP(AO, BO)                                          \
  "add.s64 a, %1, " #AO ";\n\tadd.s64 b, %2, " #BO ";\n\t"          \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
#define HK_TS_FIRST "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
#define HK_TS_STEP(AO, BO)                                          \
  "add.s32 ta, %1, " #AO ";\n\tadd.s64 b, %2, " #BO ";\n\t"         \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, t;\n\t"

// A, B both K-major SW128 128-row tiles (S = Q K^T, S^T = K Q^T, dP^T = V dO^T)
template <int NK>
__device__ __forceinline__ void gemm_ss_kk(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  static_assert(NK == 4 || NK == 8, "k-steps");
  if constexpr (NK == 4) {
    asm volatile(HK_MMA_HEAD HK_SS_FIRST HK_SS_STEP(2, 2) HK_SS_STEP(4, 4) HK_SS_STEP(6, 6) "}" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  } else {
    asm volatile(HK_MMA_HEAD HK_SS_FIRST HK_SS_STEP(2, 2) HK_SS_STEP(4, 4) HK_SS_STEP(6, 6) HK_SS_STEP(1024, 1024)
                     HK_SS_STEP(1026, 1026) HK_SS_STEP(1028, 1028) HK_SS_STEP(1030, 1030) "}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  }
}
// A from TMEM (contiguous bf16 columns), B K-major SW128 (dQ pass: S = Q_A K^T, dP = dO_A V^T)
template <int NK>
__device__ __forceinline__ void gemm_ts_kk(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  static_assert(NK == 4 || NK == 8, "k-steps");
  if constexpr (NK == 4) {
    asm volatile(HK_MMA_HEAD HK_TS_FIRST HK_TS_STEP(8, 2) HK_TS_STEP(16, 4) HK_TS_STEP(24, 6) "}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  } else {
    asm volatile(HK_MMA_HEAD HK_TS_FIRST HK_TS_STEP(8, 2) HK_TS_STEP(16, 4) HK_TS_STEP(24, 6) HK_TS_STEP(32, 1024)
                     HK_TS_STEP(40, 1026) HK_TS_STEP(48, 1028) HK_TS_STEP(56, 1030) "}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  }
}
// A from TMEM (contiguous bf16 columns), B MN-major SW128, K = 128 (forward O += P V)
__device__ __forceinline__ void gemm_ts_mn(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(HK_MMA_HEAD HK_TS_FIRST HK_TS_STEP(8, 128) HK_TS_STEP(16, 256) HK_TS_STEP(24, 384)
                   HK_TS_STEP(32, 512) HK_TS_STEP(40, 640) HK_TS_STEP(48, 768) HK_TS_STEP(56, 896) "}" ::"r"(d),
               "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
// The two K halves of gemm_ts_mn (keys [0,64) then [64,128)): the forward publishes P
// in two halves so the first half of O += P V overlaps the second half's exponentials.
__device__ __forceinline__ void gemm_ts_mn_lo(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(HK_MMA_HEAD HK_TS_FIRST HK_TS_STEP(8, 128) HK_TS_STEP(16, 256) HK_TS_STEP(24, 384) "}" ::"r"(d),
               "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void gemm_ts_mn_hi(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc) {
  asm volatile(HK_MMA_HEAD HK_TS_FIRST HK_TS_STEP(8, 128) HK_TS_STEP(16, 256) HK_TS_STEP(24, 384) "}" ::"r"(d),
               "r"(a_tmem + 32), "l"(b + 512), "r"(idesc), "r"(1u)
               : "memory");
}
// A from TMEM packed by four warpgroups (warpgroup w owns score columns [32w, 32w+32) and packs
// its 32 queries into the first 16 of them: queries 16kk.. at column 32(kk/2) + 8(kk%2)),
// B MN-major SW128, K = 128 (the d=64 dK/dV pass with 4 elementwise warpgroups)
__device__ __forceinline__ void gemm_tsp4_mn(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(HK_MMA_HEAD HK_TS_FIRST HK_TS_STEP(8, 128) HK_TS_STEP(32, 256) HK_TS_STEP(40, 384)
                   HK_TS_STEP(64, 512) HK_TS_STEP(72, 640) HK_TS_STEP(96, 768) HK_TS_STEP(104, 896) "}" ::"r"(d),
               "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
// A from TMEM packed by two warpgroups (columns 16kk.. at kk*8 for kk<4, 64+(kk-4)*8 after),
// B MN-major SW128, K = 128 (dV += P^T dO, dK += dS^T Q, dQ += dS K)
__device__ __forceinline__ void gemm_tsp_mn(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(HK_MMA_HEAD HK_TS_FIRST HK_TS_STEP(8, 128) HK_TS_STEP(16, 256) HK_TS_STEP(24, 384)
                   HK_TS_STEP(64, 512) HK_TS_STEP(72, 640) HK_TS_STEP(80, 768) HK_TS_STEP(88, 896) "}" ::"r"(d),
               "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}

// A and B both MN-major SW128 128-row-per-K-step tiles, K = 128 (8 k-steps of 16 rows x 128 B):
// the fused backward's dQ_partial = dS K_j (dS stored [keys][queries], K_j [keys][d]).
__device__ __forceinline__ void gemm_ss_mnmn(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(HK_MMA_HEAD HK_SS_FIRST HK_SS_STEP(128, 128) HK_SS_STEP(256, 256) HK_SS_STEP(384, 384)
                   HK_SS_STEP(512, 512) HK_SS_STEP(640, 640) HK_SS_STEP(768, 768) HK_SS_STEP(896, 896) "}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}

__device__ __forceinline__ void tc_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------ packed fp32x2 (sm_100 FFMA2/FADD2/FMUL2)
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// 2^x for a pair on the FMA pipe (offloads the MUFU): x = n + f, n = rint(x) via the
// 1.5*2^23 magic add, f in [-1/2, 1/2], 2^f by a degree-3 minimax polynomial
// (max relative error 7.7e-5, below bf16's 3.9e-3), 2^n added into the exponent bits.
// Valid for x <= 127; x is clamped at -125 (result ~2e-38, not 0) so that the
// exponent-field add cannot underflow for 2^f < 1.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  const float2 magic = make_float2(12582912.f, 12582912.f);
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 j = add2(x, magic);
  const float2 f = sub2(x, sub2(j, magic));
  float2 p = fma2(make_float2(0.05508885905f, 0.05508885905f), f, make_float2(0.242604658f, 0.242604658f));
  p = fma2(p, f, make_float2(0.6932762861f, 0.6932762861f));
  p = fma2(p, f, make_float2(0.999928891658f, 0.999928891658f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

// ------------------------------------------------------------------ math
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

}  // namespace hk
