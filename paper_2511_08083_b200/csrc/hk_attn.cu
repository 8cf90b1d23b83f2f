// libhkattn.so: C ABI (include/hk_attn.h) over the sm_100a attention kernels.
// Host side only validates, encodes TMA maps and launches; every step of the
// computation runs in the kernels below.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

// Built with -fvisibility=hidden: only the C ABI below is exported. (Template
// statics such as per-kernel "attribute set" flags would otherwise become
// process-wide GNU-unique symbols shared between two loaded copies of the library.)
#pragma GCC visibility push(default)
#include "../../include/hk_attn.h"
#include "../../include/hk_attn_diag.h"
#include "../../include/hk_gemm.h"
#include "../../include/hk_membound.h"
#include "../../include/hk_ring.h"
#pragma GCC visibility pop
#include "bwd.cuh"
#include "fwd.cuh"
#include "gemm.cuh"
#include "membound.cuh"
#include "ring.cuh"
#include "tma_host.h"
#include "rates_diag.cuh"
#include "umma_diag.cuh"

namespace {

thread_local char g_err[512] = "";

hk_status fail(hk_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
hk_status fail(hk_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

hk_status check_device(int* num_sms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(HK_ERR_DEVICE, "cudaGetDevice failed");
  // Bind the device's primary context to this host thread: the driver-API tensor-map
  // encoder needs a current context, and a fresh thread (e.g. autograd's backward
  // thread) has none until a runtime call makes it current.
  if (cudaSetDevice(dev) != cudaSuccess) return fail(HK_ERR_DEVICE, "cudaSetDevice(%d) failed", dev);
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(HK_ERR_DEVICE, "device %d is sm_%d%d; libhkattn is built for sm_100a only", dev, major, minor);
  if (num_sms) cudaDeviceGetAttribute(num_sms, cudaDevAttrMultiProcessorCount, dev);
  return HK_OK;
}

// cudaFuncSetAttribute(max dynamic smem) once per (kernel, device).
hk_status ensure_smem_impl(const void* fn, uint32_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({fn, dev})) return HK_OK;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return fail(HK_ERR_DEVICE, "cudaFuncSetAttribute(max dynamic smem = %u) failed", bytes);
  done.insert({fn, dev});
  return HK_OK;
}
template <typename F>
hk_status ensure_smem(F* fn, uint32_t bytes) {
  return ensure_smem_impl(reinterpret_cast<const void*>(fn), bytes);
}

hk_status launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HK_ERR_LAUNCH, "%s launch failed: %s", what, cudaGetErrorString(e));
  return HK_OK;
}

// Shape of one call (dense when cu_q == nullptr; varlen: Nq, Nk are the max lengths).
struct Shape {
  const int* cu_q;
  const int* cu_k;
  int B, Hq, Hkv, Nq, Nk, total_q, total_k;
  size_t q_rows() const { return cu_q ? (size_t)total_q : (size_t)B * Nq; }
  size_t k_rows() const { return cu_q ? (size_t)total_k : (size_t)B * Nk; }
};

hk_status validate_common(const Shape& sh, int d) {
  const int B = sh.B, Hq = sh.Hq, Hkv = sh.Hkv;
  if (B <= 0 || Hq <= 0 || Hkv <= 0 || sh.Nq <= 0 || sh.Nk <= 0)
    return fail(HK_ERR_INVALID_ARGUMENT, "B, Hq, Hkv, Nq, Nk must be positive (got %d, %d, %d, %d, %d)", B, Hq, Hkv,
                sh.Nq, sh.Nk);
  if (Hq % Hkv != 0) return fail(HK_ERR_INVALID_ARGUMENT, "Hq (%d) must be a multiple of Hkv (%d)", Hq, Hkv);
  if (d != 64 && d != 128) return fail(HK_ERR_UNSUPPORTED, "head dim d=%d unsupported (need 64 or 128)", d);
  if (Hq > 65535 || B > 65535) return fail(HK_ERR_UNSUPPORTED, "Hq and B must be <= 65535");
  const long long tq = (sh.Nq + 127) / 128, tk = (sh.Nk + 127) / 128;
  if ((long long)B * Hq * tq > 0x7fffffffLL || (long long)B * Hkv * tk > 0x7fffffffLL)
    return fail(HK_ERR_UNSUPPORTED, "B * H * ceil(N/128) must fit in int32");
  if (sh.cu_q) {
    if (!sh.cu_k) return fail(HK_ERR_INVALID_ARGUMENT, "cu_seqlens_k is null");
    if (sh.total_q <= 0 || sh.total_k <= 0)
      return fail(HK_ERR_INVALID_ARGUMENT, "total_q, total_k must be positive (got %d, %d)", sh.total_q, sh.total_k);
    if ((reinterpret_cast<uintptr_t>(sh.cu_q) | reinterpret_cast<uintptr_t>(sh.cu_k)) & 3u)
      return fail(HK_ERR_INVALID_ARGUMENT, "cu_seqlens must be 4-byte aligned");
  }
  if (sh.q_rows() * Hq > 0x7fffffffULL || sh.k_rows() * Hkv > 0x7fffffffULL)
    return fail(HK_ERR_UNSUPPORTED, "rows * H must fit in int32");
  return HK_OK;
}

size_t ws_bytes(int B, int Hq, int Nq) {
  if (B <= 0 || Hq <= 0 || Nq <= 0) return 0;
  const size_t Np = ((size_t)Nq + 127) / 128 * 128;  // rows padded to whole 128-row tiles
  return (size_t)2 * B * Hq * Np * sizeof(float) + 256;  // + the persistent kernels' work counters
}

template <int D, bool CAUSAL>
hk_status launch_fwd(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const hk::FwdParams& p,
                     int num_sms, cudaStream_t stream) {
  using C = hk::FwdCfg<D>;
  auto* fn = hk::fwd_kernel<D, CAUSAL>;
  hk_status s = ensure_smem(fn, C::SMEM);
  if (s != HK_OK) return s;
  // persistent: one CTA per SM (the SMEM footprint allows one), items in snake order
  dim3 grid(p.num_items < num_sms ? p.num_items : num_sms);
  fn<<<grid, C::THREADS, C::SMEM, stream>>>(mq, mk, mv, p);
  return launched("hk_attn_fwd");
}

}  // namespace

static hk_status bwd_impl(int phase, const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                          const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                          const Shape& sh, int d, int causal, cudaStream_t stream) {
  g_err[0] = 0;
  hk_status s = validate_common(sh, d);
  if (s != HK_OK) return s;
  if (!Q || !K || !V || !O || !LSE || !dO || !dQ || !dK || !dV || !workspace)
    return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  const void* ptrs[] = {Q, K, V, O, LSE, dO, dQ, dK, dV, workspace};
  for (const void* ptr : ptrs)
    if (!aligned16(ptr)) return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  const size_t need = ws_bytes(sh.B, sh.Hq, sh.Nq);
  if (workspace_bytes < need)
    return fail(HK_ERR_INVALID_ARGUMENT, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  const size_t q_bytes = sh.q_rows() * sh.Hq * d * 2, kv_bytes = sh.k_rows() * sh.Hkv * d * 2;
  const size_t lse_bytes = sh.q_rows() * sh.Hq * 4;
  const void* ins[] = {Q, K, V, O, LSE, dO};
  const size_t in_sz[] = {q_bytes, kv_bytes, kv_bytes, q_bytes, lse_bytes, q_bytes};
  void* outs[] = {dQ, dK, dV, workspace};
  const size_t out_sz[] = {q_bytes, kv_bytes, kv_bytes, workspace_bytes};
  for (int i = 0; i < 4; ++i) {
    for (int k = 0; k < 6; ++k)
      if (overlaps(outs[i], out_sz[i], ins[k], in_sz[k]))
        return fail(HK_ERR_INVALID_ARGUMENT, "outputs/workspace must not alias inputs");
    for (int k = i + 1; k < 4; ++k)
      if (overlaps(outs[i], out_sz[i], outs[k], out_sz[k]))
        return fail(HK_ERR_INVALID_ARGUMENT, "outputs/workspace must not alias each other");
  }
  int num_sms = 0;
  s = check_device(&num_sms);
  if (s != HK_OK) return s;
  const hk::BwdShape bs{sh.cu_q, sh.cu_k, sh.B, sh.Hq, sh.Hkv, sh.Nq, sh.Nk, sh.total_q, sh.total_k};
  return hk::launch_bwd(Q, K, V, O, LSE, dO, dQ, dK, dV, reinterpret_cast<float*>(workspace), bs, d, causal != 0,
                        stream, g_err, sizeof(g_err), phase, num_sms);
}

static hk_status fwd_impl(const void* Q, const void* K, const void* V, void* O, float* LSE, const Shape& sh, int d,
                          int causal, cudaStream_t stream, void* workspace = nullptr, size_t workspace_bytes = 0) {
  g_err[0] = 0;
  hk_status s = validate_common(sh, d);
  if (s != HK_OK) return s;
  if (!Q || !K || !V || !O || !LSE) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || !aligned16(O) || !aligned16(LSE))
    return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  const size_t q_bytes = sh.q_rows() * sh.Hq * d * 2, kv_bytes = sh.k_rows() * sh.Hkv * d * 2;
  const size_t lse_bytes = sh.q_rows() * sh.Hq * 4;
  if (overlaps(O, q_bytes, Q, q_bytes) || overlaps(O, q_bytes, K, kv_bytes) || overlaps(O, q_bytes, V, kv_bytes) ||
      overlaps(LSE, lse_bytes, O, q_bytes) || overlaps(LSE, lse_bytes, Q, q_bytes) ||
      overlaps(LSE, lse_bytes, K, kv_bytes) || overlaps(LSE, lse_bytes, V, kv_bytes))
    return fail(HK_ERR_INVALID_ARGUMENT, "outputs O/LSE must not alias inputs or each other");
  if (workspace && (workspace_bytes < 256 || !aligned16(workspace)))
    return fail(HK_ERR_INVALID_ARGUMENT, "forward workspace must be >= 256 bytes and 16-byte aligned");
  if (workspace && (overlaps(workspace, 256, O, q_bytes) || overlaps(workspace, 256, LSE, lse_bytes) ||
                    overlaps(workspace, 256, Q, q_bytes) || overlaps(workspace, 256, K, kv_bytes) ||
                    overlaps(workspace, 256, V, kv_bytes)))
    return fail(HK_ERR_INVALID_ARGUMENT, "workspace must not alias the inputs or outputs");
  int num_sms = 0;
  s = check_device(&num_sms);
  if (s != HK_OK) return s;

  const bool varlen = sh.cu_q != nullptr;
  const int mb = varlen ? 1 : sh.B, mnq = varlen ? sh.total_q : sh.Nq, mnk = varlen ? sh.total_k : sh.Nk;
  CUtensorMap mq, mk, mv;
  if (!hk::encode_bnhd(&mq, Q, mb, mnq, sh.Hq, d, 128) || !hk::encode_bnhd(&mk, K, mb, mnk, sh.Hkv, d, 128) ||
      !hk::encode_bnhd(&mv, V, mb, mnk, sh.Hkv, d, 128))
    return fail(HK_ERR_DEVICE, "cuTensorMapEncodeTiled failed (CUresult %d)", hk::last_encode_result());
  hk::FwdParams p;
  p.lse = LSE;
  p.o = reinterpret_cast<__nv_bfloat16*>(O);
  p.g = hk::SeqGeom{sh.cu_q, sh.cu_k, sh.Nq, sh.Nk, sh.total_q};
  p.B = sh.B;
  p.Hq = sh.Hq;
  p.Hkv = sh.Hkv;
  p.num_pairs = ((sh.Nq + 127) / 128 + 1) / 2;
  p.num_items = sh.B * sh.Hq * p.num_pairs;
  p.sched = reinterpret_cast<unsigned*>(workspace);  // dynamic scheduling when given a workspace
  if (workspace && cudaMemsetAsync(workspace, 0, 8, stream) != cudaSuccess)
    return fail(HK_ERR_LAUNCH, "cudaMemsetAsync(workspace counters) failed");
  if (d == 64)
    return causal ? launch_fwd<64, true>(mq, mk, mv, p, num_sms, stream)
                  : launch_fwd<64, false>(mq, mk, mv, p, num_sms, stream);
  return causal ? launch_fwd<128, true>(mq, mk, mv, p, num_sms, stream)
                : launch_fwd<128, false>(mq, mk, mv, p, num_sms, stream);
}

static Shape dense(int B, int Hq, int Hkv, int Nq, int Nk) { return Shape{nullptr, nullptr, B, Hq, Hkv, Nq, Nk, 0, 0}; }
static Shape packed(const int* cu_q, const int* cu_k, int B, int Hq, int Hkv, int total_q, int total_k, int max_q,
                    int max_k) {
  return Shape{cu_q, cu_k, B, Hq, Hkv, max_q, max_k, total_q, total_k};
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

int hk_attn_abi_version(void) { return 3; }  // 2: + Nq != Nk and varlen entry points

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
  (void)d;
  return ws_bytes(B, Hq, N);
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
  (void)d;
  return ws_bytes(B, Hq, Nq);
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
  (void)d;
  return ws_bytes(B, Hq, max_seqlen_q);
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
hk_status hk_diag_bwd_phase(int phase, const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                            const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                            int B, int Hq, int Hkv, int N, int d, int causal, cudaStream_t stream) {
  g_err[0] = 0;
  if (phase < 0 || phase > 2) return fail(HK_ERR_INVALID_ARGUMENT, "phase must be 0, 1 or 2");
  return bwd_impl(phase, Q, K, V, O, LSE, dO, dQ, dK, dV, workspace, workspace_bytes, dense(B, Hq, Hkv, N, N), d,
                  causal, stream);
}

hk_status hk_diag_umma(const void* A, const void* Bm, float* D, int N, int K, int a_tmem, int b_mn,
                       cudaStream_t stream) {
  g_err[0] = 0;
  if (!A || !Bm || !D) return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  if ((N != 64 && N != 128) || (K != 64 && K != 128)) return fail(HK_ERR_UNSUPPORTED, "N, K must be 64 or 128");
  hk_status s = check_device(nullptr);
  if (s != HK_OK) return s;
  CUtensorMap ma, mb;
  // A: [128][K] as (d=K, H=1, N=128, B=1); B: [N][K] (K-major) or [K][N] (MN-major).
  bool ok = hk::encode_bnhd(&ma, A, 1, 128, 1, K, 128);
  ok = ok && (b_mn ? hk::encode_bnhd(&mb, Bm, 1, K, 1, N, K) : hk::encode_bnhd(&mb, Bm, 1, N, 1, K, N));
  if (!ok) return fail(HK_ERR_DEVICE, "cuTensorMapEncodeTiled failed (CUresult %d)", hk::last_encode_result());
  const uint32_t smem = 128 * K * 2 + N * K * 2 + 1024;
  auto* A16 = reinterpret_cast<const __nv_bfloat16*>(A);
#define HK_DIAG(NN, KK, AT, BMN)                                                   \
  if (N == NN && K == KK && (a_tmem != 0) == AT && (b_mn != 0) == BMN) {           \
    auto* fn = hk::umma_diag_kernel<NN, KK, AT, BMN>;                              \
    if ((s = ensure_smem(fn, smem)) != HK_OK) return s;                            \
    fn<<<1, 128, smem, stream>>>(ma, mb, A16, D);                                  \
    return launched("hk_diag_umma");                                               \
  }
  HK_DIAG(64, 64, false, false) HK_DIAG(64, 64, false, true) HK_DIAG(64, 64, true, false) HK_DIAG(64, 64, true, true)
  HK_DIAG(64, 128, false, false) HK_DIAG(64, 128, false, true) HK_DIAG(64, 128, true, false)
  HK_DIAG(64, 128, true, true) HK_DIAG(128, 64, false, false) HK_DIAG(128, 64, false, true)
  HK_DIAG(128, 64, true, false) HK_DIAG(128, 64, true, true) HK_DIAG(128, 128, false, false)
  HK_DIAG(128, 128, false, true) HK_DIAG(128, 128, true, false) HK_DIAG(128, 128, true, true)
#undef HK_DIAG
  return fail(HK_ERR_UNSUPPORTED, "unsupported diag configuration");
}

hk_status hk_diag_rates(int kind, int param, int iters, float* out, cudaStream_t stream) {
  g_err[0] = 0;
  if (!out || iters <= 0) return fail(HK_ERR_INVALID_ARGUMENT, "bad arguments");
  hk_status s = check_device(nullptr);
  if (s != HK_OK) return s;
  static float* sink = nullptr;
  if (!sink && cudaMalloc(&sink, 16) != cudaSuccess) return fail(HK_ERR_DEVICE, "cudaMalloc failed");
  if (kind == 0) {
    const int threads = param >= 100 ? 128 : 512;  // param + 100: one warp per SMSP
    param %= 100;
    switch (param) {
      case 0: hk::pipe_rate_kernel<0><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 1: hk::pipe_rate_kernel<1><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 2: hk::pipe_rate_kernel<2><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 3: hk::pipe_rate_kernel<3><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 4: hk::pipe_rate_kernel<4><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 5: hk::pipe_rate_kernel<5><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 6: hk::pipe_rate_kernel<6><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 7: hk::pipe_rate_kernel<7><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 8: hk::pipe_rate_kernel<8><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 9: hk::pipe_rate_kernel<9><<<148, threads, 0, stream>>>(iters, out, sink); break;
      case 10: hk::pipe_rate_kernel<10><<<148, threads, 0, stream>>>(iters, out, sink); break;
      default: return fail(HK_ERR_UNSUPPORTED, "unknown op");
    }
    return launched("hk_diag_rates");
  }
  if (kind == 2) {  // TMEM load bandwidth: param = number of warps (4, 8 or 16), 128 columns each
    if (param != 4 && param != 8 && param != 16) return fail(HK_ERR_UNSUPPORTED, "warps must be 4, 8 or 16");
    hk::tmem_ld_rate_kernel<128><<<148, 32 * param, 0, stream>>>(iters, out, sink);
    return launched("hk_diag_rates");
  }
  if (kind == 5) {  // L2 fp32 reduce-add: param = region size in 64 KB tiles
    static float* dst = nullptr;
    static int have = 0;
    if (have < param) {
      if (dst) cudaFree(dst);
      if (cudaMalloc(&dst, (size_t)param * 65536) != cudaSuccess) return fail(HK_ERR_DEVICE, "cudaMalloc");
      cudaMemset(dst, 0, (size_t)param * 65536);
      have = param;
    }
    hk::red_rate_kernel<<<148, 256, 0, stream>>>(dst, param, iters, out);
    return launched("hk_diag_rates");
  }
  if (kind == 4) {  // TMA throughput: param = rows per box (64, 128 or 256); 64 MB source buffer
    static void* src = nullptr;
    const int total_rows = 64 * 1024 * 1024 / 128;
    if (!src && cudaMalloc(&src, (size_t)total_rows * 128) != cudaSuccess) return fail(HK_ERR_DEVICE, "cudaMalloc");
    CUtensorMap m;
    if (!hk::encode_bnhd(&m, src, 1, total_rows, 1, 64, param)) return fail(HK_ERR_DEVICE, "encode");
    const uint32_t smem = 8 * param * 128 + 1024;
#define HK_TMA_RATE(R)                                                        \
  if (param == R) {                                                           \
    auto* fn = hk::tma_rate_kernel<R>;                                        \
    if ((s = ensure_smem(fn, smem)) != HK_OK) return s;                       \
    fn<<<148, 64, smem, stream>>>(m, iters, total_rows, out);                 \
    return launched("hk_diag_rates");                                         \
  }
    HK_TMA_RATE(64) HK_TMA_RATE(128) HK_TMA_RATE(256)
#undef HK_TMA_RATE
    return fail(HK_ERR_UNSUPPORTED, "rows must be 64, 128 or 256");
  }
  if (kind == 3) {  // softmax step: param = 10 * EMU_OF_8 + warpgroups (1 or 2)
    const int nwg = param % 10, emu = param / 10;
    if (nwg < 1 || nwg > 2) return fail(HK_ERR_UNSUPPORTED, "1 or 2 warpgroups");
    dim3 g(148), blk(128 * nwg);
    switch (emu) {
      case 0: hk::softmax_rate_kernel<0><<<g, blk, 0, stream>>>(iters, out, sink); break;
      case 2: hk::softmax_rate_kernel<2><<<g, blk, 0, stream>>>(iters, out, sink); break;
      case 3: hk::softmax_rate_kernel<3><<<g, blk, 0, stream>>>(iters, out, sink); break;
      case 4: hk::softmax_rate_kernel<4><<<g, blk, 0, stream>>>(iters, out, sink); break;
      case 5: hk::softmax_rate_kernel<5><<<g, blk, 0, stream>>>(iters, out, sink); break;
      default: return fail(HK_ERR_UNSUPPORTED, "emu must be 0, 2, 3, 4 or 5");
    }
    return launched("hk_diag_rates");
  }
  const uint32_t smem = 128 * 128 * 2 + 256 * 128 * 2 + 1024;
#define HK_RATE(MODE, NN)                                          \
  if (param == MODE * 1000 + NN) {                                 \
    auto* fn = hk::mma_rate_kernel<MODE, NN>;                      \
    if ((s = ensure_smem(fn, smem)) != HK_OK) return s;            \
    fn<<<148, 128, smem, stream>>>(iters, out);                    \
    return launched("hk_diag_rates");                              \
  }
  HK_RATE(0, 64) HK_RATE(0, 128) HK_RATE(0, 256) HK_RATE(1, 64) HK_RATE(1, 128) HK_RATE(1, 256)
  HK_RATE(2, 64) HK_RATE(2, 128) HK_RATE(2, 256)
#undef HK_RATE
  return fail(HK_ERR_UNSUPPORTED, "unknown mma mode");
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

hk_status hk_rope(const void* x, const float* cos, const float* sin, void* out, int B, int N, int H, int d,
                  cudaStream_t stream) {
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
  hk::RopeParams q;
  q.x = reinterpret_cast<const __nv_bfloat16*>(x);
  q.cos = cos;
  q.sin = sin;
  q.out = reinterpret_cast<__nv_bfloat16*>(out);
  q.rows = (size_t)B * N * H;
  q.N = N;
  q.H = H;
  q.d = d;
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
hk_status hk_diag_trace_read(void* dst, size_t bytes, int reset) {
  g_err[0] = 0;
#ifdef HK_TRACE
  const size_t n = 64 * 1024 * sizeof(unsigned long long);
  if (dst && bytes >= n && cudaMemcpyFromSymbol(dst, hk::g_hk_trace, n) != cudaSuccess)
    return fail(HK_ERR_DEVICE, "trace read failed");
  if (reset && cudaMemset(nullptr, 0, 0) == cudaSuccess) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, hk::g_hk_trace) == cudaSuccess) cudaMemset(p, 0, n);
  }
#else
  (void)reset;
  if (dst && bytes) memset(dst, 0, bytes);
#endif
  return HK_OK;
}

}  // extern "C"
