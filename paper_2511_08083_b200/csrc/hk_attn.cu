// libhkattn.so: C ABI (include/hk_attn.h, hk_gemm.h, hk_membound.h, hk_ring.h) over the
// sm_100a kernels. Host side only validates, encodes TMA maps and launches; every step of
// the computation runs in the kernels. Diagnostics (hk_attn_diag.h) live in
// libhkattn_diag.so (hk_diag.cu), not here.
//
// Built with -fvisibility=hidden: only the C ABI below is exported. (Template
// statics such as per-kernel "attribute set" flags would otherwise become
// process-wide GNU-unique symbols shared between two loaded copies of the library.)
#include "host.cuh"
#pragma GCC visibility push(default)
#include "../../include/hk_gemm.h"
#include "../../include/hk_membound.h"
#include "../../include/hk_ring.h"
#pragma GCC visibility pop
#include "gemm.cuh"
#include "membound.cuh"
#include "ring.cuh"

// Rotary launch shared by hk_rope(_ex) and hk_attn_fwd_rope (arguments validated by the caller).
static hk_status rope_launch(const void* x, const float* cos, const float* sin, void* out, int B, int N, int H, int d,
                             float sgn, int num_sms, cudaStream_t stream) {
  const size_t bytes = (size_t)B * N * H * d * 2;
  hk::RopeParams q;
  q.x = reinterpret_cast<const __nv_bfloat16*>(x);
  q.cos = cos;
  q.sin = sin;
  q.out = reinterpret_cast<__nv_bfloat16*>(out);
  q.rows = (size_t)B * N * H;
  q.N = N;
  q.H = H;
  q.d = d;
  q.sgn = sgn;
  // inputs beyond L2 (126 MB): the head-loop form loads each position's cos/sin once for all H
  // heads (1.08-1.13x at 268 MB / 1 GB); smaller ones stay with one thread per (row, chunk)
  // (the head loop leaves too few threads there: 0.91x at 67 MB). Same results either way.
  if (bytes > ((size_t)126 << 20)) {
    const size_t threads = (size_t)B * N * (d / 16);
    size_t blocks = (threads + 255) / 256;
    if (blocks > (size_t)num_sms * 16) blocks = (size_t)num_sms * 16;
    if (threads < ((size_t)1 << 31))
      hk::rope_hloop_kernel<uint32_t><<<(unsigned)blocks, 256, 0, stream>>>(q);
    else
      hk::rope_hloop_kernel<size_t><<<(unsigned)blocks, 256, 0, stream>>>(q);
    return launched("hk_rope");
  }
  const size_t threads = q.rows * (d / 16);
  size_t blocks = (threads + 255) / 256;
  if (blocks > (size_t)num_sms * 16) blocks = (size_t)num_sms * 16;
  if (threads < ((size_t)1 << 31))
    hk::rope_kernel<uint32_t><<<(unsigned)blocks, 256, 0, stream>>>(q);
  else
    hk::rope_kernel<size_t><<<(unsigned)blocks, 256, 0, stream>>>(q);
  return launched("hk_rope");
}

extern "C" {

const char* hk_attn_last_error(void) { return g_err; }

const char* hk_status_string(hk_status s) {
  switch (s) {
    case HK_OK: return "HK_OK";
    case HK_ERR_INVALID_ARGUMENT: return "HK_ERR_INVALID_ARGUMENT";
    case HK_ERR_UNSUPPORTED: return "HK_ERR_UNSUPPORTED";
    case HK_ERR_DEVICE: return "HK_ERR_DEVICE";
    case HK_ERR_LAUNCH: return "HK_ERR_LAUNCH";
  }
  return "HK_ERR_UNKNOWN";
}

int hk_attn_abi_version(void) { return 6; }  // 2: + Nq != Nk and varlen; 4: + _ex (flags), fused d=64 bwd, rope;
                                              // 5: + hk_set_max_ctas / hk_get_max_ctas, hk_accum_f32
                                              // 6: + stored-dS backward (hk_attn_bwd_ds_workspace_bytes)
void hk_set_max_ctas(int max_ctas) { g_max_ctas.store(max_ctas > 0 ? max_ctas : 0); }
int hk_get_max_ctas(void) { return g_max_ctas.load(); }

hk_status hk_attn_fwd(const void* Q, const void* K, const void* V, void* O, float* LSE, int B, int Hq, int Hkv,
                      int N, int d, int causal, cudaStream_t stream) {
  if (N <= 0) {
    g_err[0] = 0;
    return fail(HK_ERR_INVALID_ARGUMENT, "N must be positive (got %d)", N);
  }
  return fwd_impl(Q, K, V, O, LSE, dense(B, Hq, Hkv, N, N), d, causal, stream);
}
size_t hk_attn_bwd_workspace_bytes(int B, int Hq, int Hkv, int N, int d) {
  (void)Hkv;
  return ws_bytes(B, Hq, N, d);
}
size_t hk_attn_bwd_ds_workspace_bytes(int B, int Hq, int Hkv, int Nq, int Nk, int d, int causal) {
  (void)Hkv;
  const size_t ws = ws_bytes(B, Hq, Nq, d);
  const size_t ds = hk::bwd_ds_bytes(B, Hq, Nq, Nk, d, causal != 0, false);
  return ds ? hk::bwd_ds_offset(ws) + ds : ws;
}
hk_status hk_attn_bwd(const void* Q, const void* K, const void* V, const void* O, const float* LSE, const void* dO,
                      void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes, int B, int Hq, int Hkv,
                      int N, int d, int causal, cudaStream_t stream) {
  return bwd_impl(-1, Q, K, V, O, LSE, dO, dQ, dK, dV, workspace, workspace_bytes, dense(B, Hq, Hkv, N, N), d, causal,
                  stream);
}
hk_status hk_attn_fwd_qk(const void* Q, const void* K, const void* V, void* O, float* LSE, int B, int Hq, int Hkv,
                         int Nq, int Nk, int d, int causal, cudaStream_t stream) {
  return fwd_impl(Q, K, V, O, LSE, dense(B, Hq, Hkv, Nq, Nk), d, causal, stream);
}
size_t hk_attn_bwd_qk_workspace_bytes(int B, int Hq, int Hkv, int Nq, int Nk, int d) {
  (void)Hkv;
  (void)Nk;
  return ws_bytes(B, Hq, Nq, d);
}
hk_status hk_attn_bwd_qk(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                         const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes, int B,
                         int Hq, int Hkv, int Nq, int Nk, int d, int causal, cudaStream_t stream) {
  return bwd_impl(-1, Q, K, V, O, LSE, dO, dQ, dK, dV, workspace, workspace_bytes, dense(B, Hq, Hkv, Nq, Nk), d,
                  causal, stream);
}
hk_status hk_attn_fwd_varlen(const void* Q, const void* K, const void* V, void* O, float* LSE,
                             const int* cu_seqlens_q, const int* cu_seqlens_k, int B, int Hq, int Hkv, int total_q,
                             int total_k, int max_seqlen_q, int max_seqlen_k, int d, int causal, void* workspace,
                             size_t workspace_bytes, cudaStream_t stream) {
  if (!cu_seqlens_q || !cu_seqlens_k) {
    g_err[0] = 0;
    return fail(HK_ERR_INVALID_ARGUMENT, "null cu_seqlens");
  }
  return fwd_impl(Q, K, V, O, LSE,
                  packed(cu_seqlens_q, cu_seqlens_k, B, Hq, Hkv, total_q, total_k, max_seqlen_q, max_seqlen_k), d,
                  causal, stream, workspace, workspace_bytes);
}
size_t hk_attn_bwd_varlen_workspace_bytes(int B, int Hq, int Hkv, int max_seqlen_q, int max_seqlen_k, int d) {
  (void)Hkv;
  (void)max_seqlen_k;
  return ws_bytes(B, Hq, max_seqlen_q, d);
}
hk_status hk_attn_bwd_varlen(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                             const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                             const int* cu_seqlens_q, const int* cu_seqlens_k, int B, int Hq, int Hkv, int total_q,
                             int total_k, int max_seqlen_q, int max_seqlen_k, int d, int causal,
                             cudaStream_t stream) {
  if (!cu_seqlens_q || !cu_seqlens_k) {
    g_err[0] = 0;
    return fail(HK_ERR_INVALID_ARGUMENT, "null cu_seqlens");
  }
  return bwd_impl(-1, Q, K, V, O, LSE, dO, dQ, dK, dV, workspace, workspace_bytes,
                  packed(cu_seqlens_q, cu_seqlens_k, B, Hq, Hkv, total_q, total_k, max_seqlen_q, max_seqlen_k), d,
                  causal, stream);
}
hk_status hk_attn_bwd_ex(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                         const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes, int B,
                         int Hq, int Hkv, int Nq, int Nk, int d, int causal, unsigned flags, cudaStream_t stream) {
  return bwd_impl(-1, Q, K, V, O, LSE, dO, dQ, dK, dV, workspace, workspace_bytes, dense(B, Hq, Hkv, Nq, Nk), d,
                  causal, stream, flags);
}
hk_status hk_attn_bwd_varlen_ex(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                                const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                                const int* cu_seqlens_q, const int* cu_seqlens_k, int B, int Hq, int Hkv, int total_q,
                                int total_k, int max_seqlen_q, int max_seqlen_k, int d, int causal, unsigned flags,
                                cudaStream_t stream) {
  if (!cu_seqlens_q || !cu_seqlens_k) {
    g_err[0] = 0;
    return fail(HK_ERR_INVALID_ARGUMENT, "null cu_seqlens");
  }
  return bwd_impl(-1, Q, K, V, O, LSE, dO, dQ, dK, dV, workspace, workspace_bytes,
                  packed(cu_seqlens_q, cu_seqlens_k, B, Hq, Hkv, total_q, total_k, max_seqlen_q, max_seqlen_k), d,
                  causal, stream, flags);
}

hk_status hk_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, cudaStream_t stream) {
  g_err[0] = 0;
  if (M <= 0 || N <= 0 || K <= 0) return fail(HK_ERR_INVALID_ARGUMENT, "M, N, K must be positive (%d, %d, %d)", M, N, K);
  if (!A || !B || !C) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!aligned16(A) || !aligned16(B) || !aligned16(C))
    return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  if (M % 256 || N % 256 || K % 64)
    return fail(HK_ERR_UNSUPPORTED, "need M %% 256 == 0, N %% 256 == 0, K %% 64 == 0 (got %d, %d, %d)", M, N, K);
  const size_t a_bytes = (size_t)M * K * 2, b_bytes = (size_t)N * K * 2, c_bytes = (size_t)M * N * 2;
  if (overlaps(C, c_bytes, A, a_bytes) || overlaps(C, c_bytes, B, b_bytes))
    return fail(HK_ERR_INVALID_ARGUMENT, "C must not overlap A or B");
  int num_sms = 0;
  hk_status s = check_device(&num_sms);
  if (s != HK_OK) return s;
  CUtensorMap ma, mb;
  if (!hk::encode_rowmajor(&ma, A, M, K, 128) || !hk::encode_rowmajor(&mb, B, N, K, 128))
    return fail(HK_ERR_DEVICE, "cuTensorMapEncodeTiled failed (CUresult %d)", hk::last_encode_result());
  hk::GemmParams p;
  p.c = reinterpret_cast<__nv_bfloat16*>(C);
  p.M = M;
  p.N = N;
  p.K = K;
  p.tiles_m = M / 256;
  const bool wide = N % 512 == 0 && getenv("HK_GEMM_NARROW") == nullptr;  // 256x512 pair tiles when N allows
  p.tiles_n = wide ? N / 512 : N / 256;
  const int tiles = p.tiles_m * p.tiles_n;
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;  // persistent: one CTA pair per TPC
  if (wide) {
    s = ensure_smem(hk::gemm_bf16_kernel<512>, hk::GemmCfg<512>::SMEM);
    if (s != HK_OK) return s;
    hk::gemm_bf16_kernel<512><<<2 * pairs, hk::GEMM_THREADS, hk::GemmCfg<512>::SMEM, stream>>>(ma, mb, p);
  } else {
    s = ensure_smem(hk::gemm_bf16_kernel<256>, hk::GemmCfg<256>::SMEM);
    if (s != HK_OK) return s;
    hk::gemm_bf16_kernel<256><<<2 * pairs, hk::GEMM_THREADS, hk::GemmCfg<256>::SMEM, stream>>>(ma, mb, p);
  }
  return launched("hk_gemm_bf16");
}

hk_status hk_ln_dropout_residual(const void* x, const void* residual, const void* weight, const void* bias, void* out,
                                 void* out_resid, int rows, int D, float p, unsigned int seed, float eps,
                                 cudaStream_t stream) {
  g_err[0] = 0;
  if (rows <= 0 || D <= 0) return fail(HK_ERR_INVALID_ARGUMENT, "rows and D must be positive (%d, %d)", rows, D);
  if (!x || !residual || !weight || !bias || !out || !out_resid)
    return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!aligned16(x) || !aligned16(residual) || !aligned16(weight) || !aligned16(bias) || !aligned16(out) ||
      !aligned16(out_resid))
    return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  if (!(p >= 0.f && p < 1.f) || !(eps > 0.f)) return fail(HK_ERR_INVALID_ARGUMENT, "need 0 <= p < 1 and eps > 0");
  if (D % 8 || D > 8192) return fail(HK_ERR_UNSUPPORTED, "need D %% 8 == 0 and D <= 8192 (got %d)", D);
  if ((long long)rows * D >= (1ll << 32)) return fail(HK_ERR_UNSUPPORTED, "rows * D must be < 2^32");
  const size_t bytes = (size_t)rows * D * 2;
  if (overlaps(out, bytes, out_resid, bytes) || overlaps(out, bytes, x, bytes) ||
      overlaps(out, bytes, residual, bytes) || overlaps(out_resid, bytes, x, bytes) ||
      overlaps(out_resid, bytes, residual, bytes))
    return fail(HK_ERR_INVALID_ARGUMENT, "outputs must not overlap each other or the inputs");
  int num_sms = 0;
  hk_status s = check_device(&num_sms);
  if (s != HK_OK) return s;
  hk::LnParams q;
  q.x = reinterpret_cast<const __nv_bfloat16*>(x);
  q.residual = reinterpret_cast<const __nv_bfloat16*>(residual);
  q.weight = reinterpret_cast<const __nv_bfloat16*>(weight);
  q.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
  q.out = reinterpret_cast<__nv_bfloat16*>(out);
  q.out_resid = reinterpret_cast<__nv_bfloat16*>(out_resid);
  q.rows = rows;
  q.D = D;
  q.thresh = p > 0.f ? (uint32_t)fmin((double)p * 4294967296.0, 4294967295.0) : 0u;
  q.seed = seed;
  q.scale = 1.f / (1.f - p);
  q.eps = eps;
  const int warps = 8, blocks_needed = (rows + warps - 1) / warps;
  const int blocks = blocks_needed < num_sms * 8 ? blocks_needed : num_sms * 8;
  const int vpl = (D / 8 + 31) / 32;  // 8-element vectors per lane
#define HK_LN(V) hk::ln_dropout_residual_kernel<V><<<blocks, 256, 0, stream>>>(q)
  if (vpl <= 1) HK_LN(1);
  else if (vpl <= 2) HK_LN(2);
  else if (vpl <= 4) HK_LN(4);
  else if (vpl <= 8) HK_LN(8);
  else if (vpl <= 16) HK_LN(16);
  else HK_LN(32);
#undef HK_LN
  return launched("hk_ln_dropout_residual");
}

hk_status hk_rope_ex(const void* x, const float* cos, const float* sin, void* out, int B, int N, int H, int d,
                     int inverse, cudaStream_t stream) {
  g_err[0] = 0;
  if (B <= 0 || N <= 0 || H <= 0 || d <= 0) return fail(HK_ERR_INVALID_ARGUMENT, "B, N, H, d must be positive");
  if (!x || !cos || !sin || !out) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!aligned16(x) || !aligned16(cos) || !aligned16(sin) || !aligned16(out))
    return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  if (d % 16 || d > 512) return fail(HK_ERR_UNSUPPORTED, "need d %% 16 == 0 and d <= 512 (got %d)", d);
  const size_t bytes = (size_t)B * N * H * d * 2;
  if (out != x && overlaps(out, bytes, x, bytes)) return fail(HK_ERR_INVALID_ARGUMENT, "out partially overlaps x");
  int num_sms = 0;
  hk_status s = check_device(&num_sms);
  if (s != HK_OK) return s;
  return rope_launch(x, cos, sin, out, B, N, H, d, inverse ? -1.f : 1.f, num_sms, stream);
}

hk_status hk_rope(const void* x, const float* cos, const float* sin, void* out, int B, int N, int H, int d,
                  cudaStream_t stream) {
  return hk_rope_ex(x, cos, sin, out, B, N, H, d, 0, stream);
}

hk_status hk_attn_fwd_rope(const void* Q, const void* K, const void* V, const float* cos, const float* sin, void* O,
                           float* LSE, void* Kr, int B, int Hq, int Hkv, int N, int d, int causal,
                           cudaStream_t stream) {
  g_err[0] = 0;
  if (N <= 0) return fail(HK_ERR_INVALID_ARGUMENT, "N must be positive (got %d)", N);
  if (!cos || !sin || !Kr || !K) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!aligned16(cos) || !aligned16(sin) || !aligned16(Kr))
    return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  if (B <= 0 || Hkv <= 0) return fail(HK_ERR_INVALID_ARGUMENT, "B, Hkv must be positive");
  const size_t kv_bytes = (size_t)B * N * Hkv * d * 2, q_bytes = (size_t)B * N * Hq * d * 2;
  if (overlaps(Kr, kv_bytes, K, kv_bytes) || (V && overlaps(Kr, kv_bytes, V, kv_bytes)) ||
      (Q && overlaps(Kr, kv_bytes, Q, q_bytes)) || (O && overlaps(Kr, kv_bytes, O, q_bytes)) ||
      (LSE && overlaps(Kr, kv_bytes, LSE, (size_t)B * Hq * N * 4)))
    return fail(HK_ERR_INVALID_ARGUMENT, "Kr must not alias the other tensors");
  hk_status s = validate_common(dense(B, Hq, Hkv, N, N), d);  // d in {64, 128} before anything runs
  if (s != HK_OK) return s;
  int num_sms = 0;
  s = check_device(&num_sms);
  if (s != HK_OK) return s;
  // K is read by every query tile of its group: rotate it once, into Kr; Q tiles are rotated in
  // shared memory by the forward kernel itself (read once per CTA)
  s = rope_launch(K, cos, sin, Kr, B, N, Hkv, d, 1.f, num_sms, stream);
  if (s != HK_OK) return s;
  return fwd_impl(Q, Kr, V, O, LSE, dense(B, Hq, Hkv, N, N), d, causal, stream, nullptr, 0, cos, sin);
}

hk_status hk_attn_merge(float* O_acc, float* LSE_acc, const void* O_part, const float* LSE_part, void* O_out, int B,
                        int N, int H, int d, int init, cudaStream_t stream) {
  g_err[0] = 0;
  if (B <= 0 || N <= 0 || H <= 0) return fail(HK_ERR_INVALID_ARGUMENT, "B, N, H must be positive");
  if (!O_acc || !LSE_acc || !O_part || !LSE_part) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!aligned16(O_acc) || !aligned16(O_part) || (O_out && !aligned16(O_out)) ||
      (reinterpret_cast<uintptr_t>(LSE_acc) & 3u) || (reinterpret_cast<uintptr_t>(LSE_part) & 3u))
    return fail(HK_ERR_INVALID_ARGUMENT, "O pointers must be 16-byte aligned, LSE pointers 4-byte aligned");
  if (d < 8 || d > 256 || (d & (d - 1))) return fail(HK_ERR_UNSUPPORTED, "d must be a power of two in [8, 256]");
  const size_t rows = (size_t)B * N * H;
  const size_t ob = rows * d * 2, ab = rows * d * 4, lb = rows * 4;
  if (overlaps(O_acc, ab, O_part, ob) || overlaps(O_acc, ab, LSE_part, lb) || overlaps(LSE_acc, lb, O_part, ob) ||
      overlaps(LSE_acc, lb, LSE_part, lb) || overlaps(O_acc, ab, LSE_acc, lb) ||
      (O_out && (overlaps(O_out, ob, O_acc, ab) || overlaps(O_out, ob, LSE_acc, lb) || overlaps(O_out, ob, O_part, ob))))
    return fail(HK_ERR_INVALID_ARGUMENT, "buffers must not overlap");
  int num_sms = 0;
  hk_status s = check_device(&num_sms);
  if (s != HK_OK) return s;
  hk::MergeParams q{O_acc, LSE_acc, reinterpret_cast<const __nv_bfloat16*>(O_part), LSE_part,
                    reinterpret_cast<__nv_bfloat16*>(O_out), B, N, H, d, init != 0};
  const size_t warps = (rows + (32 / (d / 8)) - 1) / (32 / (d / 8));
  size_t blocks = (warps + 7) / 8;
  if (blocks > (size_t)num_sms * 16) blocks = (size_t)num_sms * 16;
  hk::attn_merge_kernel<<<(unsigned)blocks, 256, 0, stream>>>(q);
  return launched("hk_attn_merge");
}
hk_status hk_accum_bf16(float* acc, const void* x, void* out, size_t n, int init, cudaStream_t stream) {
  g_err[0] = 0;
  if (n == 0 || n % 8) return fail(HK_ERR_INVALID_ARGUMENT, "n must be a positive multiple of 8");
  if (!x && !(out && acc && !init)) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!acc && !(out && init)) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if ((acc && !aligned16(acc)) || (x && !aligned16(x)) || (out && !aligned16(out)))
    return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  if ((acc && x && overlaps(acc, n * 4, x, n * 2)) ||
      (out && ((x && overlaps(out, n * 2, x, n * 2)) || (acc && overlaps(out, n * 2, acc, n * 4)))))
    return fail(HK_ERR_INVALID_ARGUMENT, "buffers must not overlap");
  int num_sms = 0;
  hk_status s = check_device(&num_sms);
  if (s != HK_OK) return s;
  const size_t n8 = n / 8;
  size_t blocks = (n8 + 255) / 256;
  if (blocks > (size_t)num_sms * 16) blocks = (size_t)num_sms * 16;
  hk::accum_bf16_kernel<<<(unsigned)blocks, 256, 0, stream>>>(acc, reinterpret_cast<const __nv_bfloat16*>(x),
                                                               reinterpret_cast<__nv_bfloat16*>(out), n8, init != 0);
  return launched("hk_accum_bf16");
}
hk_status hk_accum_f32(float* acc, const float* x, size_t n, cudaStream_t stream) {
  g_err[0] = 0;
  if (n == 0 || n % 4) return fail(HK_ERR_INVALID_ARGUMENT, "n must be a positive multiple of 4");
  if (!acc || !x) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!aligned16(acc) || !aligned16(x)) return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  if (overlaps(acc, n * 4, x, n * 4)) return fail(HK_ERR_INVALID_ARGUMENT, "buffers must not overlap");
  int num_sms = 0;
  hk_status s = check_device(&num_sms);
  if (s != HK_OK) return s;
  size_t blocks = (n / 4 + 255) / 256;
  if (blocks > (size_t)num_sms * 16) blocks = (size_t)num_sms * 16;
  hk::accum_f32_kernel<<<(unsigned)blocks, 256, 0, stream>>>(acc, x, n / 4);
  return launched("hk_accum_f32");
}
}  // extern "C"
