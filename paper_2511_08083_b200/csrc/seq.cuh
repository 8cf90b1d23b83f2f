// Sequence geometry shared by the attention kernels: dense [B][N][H][d]
// batches (Nq may differ from Nk) and packed variable-length batches
// [total][H][d] with per-sequence offsets.
//
// Mask (readings #3, #22): key j of a sequence is visible to its
// query i iff j < lk and, when causal, j <= i + (lk - lq) (bottom-right
// aligned; j <= i when lq == lk). A query row that sees no key gets O = 0 and
// LSE = -inf; the backward treats it as contributing nothing.
#pragma once
#include <cstddef>

namespace hk {

struct SeqGeom {
  const int* cu_q;  // [B+1] packed row offsets into Q/O/dO/dQ; nullptr = dense
  const int* cu_k;  // [B+1] packed row offsets into K/V/dK/dV
  int Nq, Nk;       // dense: the lengths; varlen: the maximum lengths (tile counts derive from them)
  int total_q;      // varlen: row count of the packed Q (LSE is [Hq][total_q])
};

struct Seq {
  int tb;        // TMA coordinate along the batch dimension (dense: b; varlen: 0)
  int q0, k0;    // TMA row coordinate of the sequence's row 0 (dense: 0; varlen: cu[b])
  int gq0, gk0;  // global row index of row 0 in the [rows][H][d] tensors
  int lq, lk;    // lengths
};

__device__ __forceinline__ Seq seq_of(const SeqGeom& g, int b) {
  Seq s;
  if (g.cu_q == nullptr) {
    s.tb = b;
    s.q0 = s.k0 = 0;
    s.gq0 = b * g.Nq;
    s.gk0 = b * g.Nk;
    s.lq = g.Nq;
    s.lk = g.Nk;
  } else {
    s.tb = 0;
    s.q0 = s.gq0 = __ldg(g.cu_q + b);
    s.k0 = s.gk0 = __ldg(g.cu_k + b);
    // lengths clamped to [0, max_seqlen]: rows beyond a sequence's max_seqlen are not computed
    // (hk_attn.h), and offsets that break the contract cannot index past the padded workspace
    s.lq = min(max(__ldg(g.cu_q + b + 1) - s.q0, 0), g.Nq);
    s.lk = min(max(__ldg(g.cu_k + b + 1) - s.k0, 0), g.Nk);
  }
  return s;
}

// Index of LSE[b, h, row]: dense [B][Hq][Nq], varlen [Hq][total_q].
__device__ __forceinline__ size_t lse_index(const SeqGeom& g, const Seq& s, int b, int Hq, int h, int row) {
  if (g.cu_q == nullptr) return ((size_t)b * Hq + h) * g.Nq + row;
  return (size_t)h * g.total_q + s.gq0 + row;
}

// Number of 128-key tiles query tile qt must visit (0 when none of its rows
// sees a key or the tile holds no query row).
template <bool CAUSAL>
__device__ __forceinline__ int kv_tiles_for(const Seq& s, int qt) {
  if (qt * 128 >= s.lq || s.lk <= 0) return 0;
  const int ntk = (s.lk + 127) / 128;
  if (!CAUSAL) return ntk;
  const int last_row = min(qt * 128 + 127, s.lq - 1);
  const int kmax = min(last_row + s.lk - s.lq, s.lk - 1);
  return kmax < 0 ? 0 : kmax / 128 + 1;
}

// First query tile that sees key tile jt (causal), 0 otherwise.
template <bool CAUSAL>
__device__ __forceinline__ int first_q_tile_for(const Seq& s, int jt) {
  if (!CAUSAL) return 0;
  const int i_min = jt * 128 - (s.lk - s.lq);  // smallest query row that sees key jt*128
  return i_min <= 0 ? 0 : i_min / 128;
}

}  // namespace hk
