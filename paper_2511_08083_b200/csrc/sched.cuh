// Dynamic work distribution for the persistent kernels (backward passes; the
// varlen forward when given a workspace): a producer lane draws item indices
// from a global counter and hands each draw to the 9 consumer warps (the MMA
// warp + 8 softmax / elementwise warps) through a 2-entry ring in shared memory.
#pragma once
#include "ptx.cuh"

namespace hk {

// The TMA lane
// draws item indices from a global counter (so the CTAs work through one
// contiguous, heaviest-first window of items: balanced, and the items in
// flight share their Q/dO or K/V in L2) and hands each draw to the MMA warp and
// the 8 elementwise warps through a 2-entry ring in shared memory. A draw
// >= the item count ends every role. The CTA that finishes last resets the
// counters for the next launch; the pre-kernel zeroes them too.
constexpr int SCHED_NQ = 2;
struct Sched {
  uint64_t full[SCHED_NQ], empty[SCHED_NQ];
  int item[SCHED_NQ];
};
__device__ __forceinline__ void sched_init(Sched& q, int consumers = 9) {  // default: MMA warp + 8 warps
  for (int i = 0; i < SCHED_NQ; ++i) {
    mbar_init(&q.full[i], 1);
    mbar_init(&q.empty[i], consumers);
  }
}
// producer lane: draw number k. `skip(item)` (optional) marks items no role has any
// work for: they are drawn past without being handed to the consumers.
__device__ __forceinline__ int sched_publish(Sched& q, unsigned* ctr, int k) {
  const int i = k % SCHED_NQ;
  mbar_wait(&q.empty[i], ((k / SCHED_NQ) & 1) ^ 1);
  const int item = (int)atomicAdd(ctr, 1u);
  *reinterpret_cast<volatile int*>(&q.item[i]) = item;
  mbar_arrive(&q.full[i]);
  return item;
}
template <typename Skip>
__device__ __forceinline__ int sched_publish(Sched& q, unsigned* ctr, int k, int num_items, Skip skip) {
  const int i = k % SCHED_NQ;
  mbar_wait(&q.empty[i], ((k / SCHED_NQ) & 1) ^ 1);
  int item = (int)atomicAdd(ctr, 1u);
  while (item < num_items && skip(item)) item = (int)atomicAdd(ctr, 1u);
  *reinterpret_cast<volatile int*>(&q.item[i]) = item;
  mbar_arrive(&q.full[i]);
  return item;
}
// consumer (whole warp): draw number k
__device__ __forceinline__ int sched_take(Sched& q, int k) {
  const int i = k % SCHED_NQ;
  mbar_wait(&q.full[i], (k / SCHED_NQ) & 1);
  // Lane 0 alone reads the slot and releases it (its arrive orders its own read
  // before the producer's next write); the other lanes get the value by shfl,
  // which also makes the index (and everything the MMA warp derives from it)
  // warp-uniform for ptxas, keeping descriptors in uniform registers.
  int v = 0;
  if (lane_id() == 0) v = *reinterpret_cast<volatile int*>(&q.item[i]);
  const int item = __shfl_sync(0xffffffffu, v, 0);
  if (lane_id() == 0) mbar_arrive(&q.empty[i]);
  return item;
}
// last CTA out resets the draw counter (ctr[0]) and the exit counter (ctr[1])
__device__ __forceinline__ void sched_exit(unsigned* ctr) {
  __threadfence();
  if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
    atomicExch(ctr, 0u);
    atomicExch(ctr + 1, 0u);
  }
}
// Wait until the last release committed on each slot of a ring (U uses so far)
// has landed, so no asynchronous arrive is still in flight when the CTA exits.
__device__ __forceinline__ void drain_ring(uint64_t* empty, int ns, int U) {
  for (int s = 0; s < ns && s < U; ++s) {
    const int last = U - 1 - ((U - 1 - s) % ns);
    mbar_wait(&empty[s], (last / ns) & 1);
  }
}

}  // namespace hk
