// Host-side helpers shared by libhkattn.so (hk_attn.cu) and libhkattn_diag.so (hk_diag.cu):
// argument validation, thread-local error text, TMA-map encoding and the launch wrappers of
// the attention kernels. Each library compiles its own copy (built with -fvisibility=hidden).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <set>
#include <utility>

#pragma GCC visibility push(default)
#include "../../include/hk_attn.h"
#pragma GCC visibility pop
#include "bwd.cuh"
#include "fwd.cuh"
#include "tma_host.h"

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

// hk_set_max_ctas: SM budget of the persistent kernels (0 = all SMs)
std::atomic<int> g_max_ctas{0};

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
  if (num_sms) {
    cudaDeviceGetAttribute(num_sms, cudaDevAttrMultiProcessorCount, dev);
    const int cap = g_max_ctas.load();
    if (cap > 0 && cap < *num_sms) *num_sms = cap < 2 ? 2 : cap;  // the GEMM needs one CTA pair
  }
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

size_t ws_bytes(int B, int Hq, int Nq, int d) { return hk::bwd_ws_bytes(B, Hq, Nq, d); }

template <int D, bool CAUSAL, bool ROPE = false>
hk_status launch_fwd(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mo,
                     const hk::FwdParams& p,
                     int num_sms, cudaStream_t stream) {
  using C = hk::FwdCfg<D>;
  auto* fn = hk::fwd_kernel<D, CAUSAL, ROPE>;
  hk_status s = ensure_smem(fn, C::SMEM);
  if (s != HK_OK) return s;
  // persistent: one CTA per SM (the SMEM footprint allows one), items in snake order
  dim3 grid(p.num_items < num_sms ? p.num_items : num_sms);
  fn<<<grid, C::THREADS, C::SMEM, stream>>>(mq, mk, mv, mo, p);
  return launched("hk_attn_fwd");
}

}  // namespace

static hk_status bwd_impl(int phase, const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                          const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                          const Shape& sh, int d, int causal, cudaStream_t stream,
                          unsigned flags = 0) {
  g_err[0] = 0;
  if (flags & ~(unsigned)(HK_BWD_DETERMINISTIC | HK_BWD_ACCUMULATE_F32))
    return fail(HK_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", flags);
  const bool acc32 = (flags & HK_BWD_ACCUMULATE_F32) != 0;
  hk_status s = validate_common(sh, d);
  if (s != HK_OK) return s;
  if (!Q || !K || !V || !O || !LSE || !dO || !dQ || !dK || !dV || !workspace)
    return fail(HK_ERR_INVALID_ARGUMENT, "null pointer argument");
  const void* ptrs[] = {Q, K, V, O, LSE, dO, dQ, dK, dV, workspace};
  for (const void* ptr : ptrs)
    if (!aligned16(ptr)) return fail(HK_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  const size_t need = ws_bytes(sh.B, sh.Hq, sh.Nq, d);
  if (workspace_bytes < need)
    return fail(HK_ERR_INVALID_ARGUMENT, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  const size_t q_bytes = sh.q_rows() * sh.Hq * d * 2, kv_bytes = sh.k_rows() * sh.Hkv * d * 2;
  const size_t lse_bytes = sh.q_rows() * sh.Hq * 4;
  const void* ins[] = {Q, K, V, O, LSE, dO};
  const size_t in_sz[] = {q_bytes, kv_bytes, kv_bytes, q_bytes, lse_bytes, q_bytes};
  void* outs[] = {dQ, dK, dV, workspace};
  const size_t osc = acc32 ? 2 : 1;  // fp32 accumulators are twice the bf16 outputs
  const size_t out_sz[] = {q_bytes * osc, kv_bytes * osc, kv_bytes * osc, workspace_bytes};
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
  // NEXT #1 single pass: d = 64 (d = 128 only in -DHK_FUSED128=1 builds, bwd.cuh)
  const bool fused = hk::bwd_fused_default(d) && !(flags & HK_BWD_DETERMINISTIC);
  // stored-dS backward: whenever the caller's workspace has room for the dS tiles
  // (hk_attn_bwd_ds_workspace_bytes)
  const size_t ds_need = hk::bwd_ds_bytes(sh.B, sh.Hq, sh.Nq, sh.Nk, d, causal != 0, sh.cu_q != nullptr);
  const bool ds = !fused && ds_need > 0 && workspace_bytes >= hk::bwd_ds_offset(need) + ds_need;
  const hk::BwdShape bs{sh.cu_q, sh.cu_k, sh.B,        sh.Hq, sh.Hkv, sh.Nq, sh.Nk,
                        sh.total_q, sh.total_k, fused, acc32, ds};
  return hk::launch_bwd(Q, K, V, O, LSE, dO, dQ, dK, dV, reinterpret_cast<float*>(workspace), bs, d, causal != 0,
                        stream, g_err, sizeof(g_err), phase, num_sms);
}

static hk_status fwd_impl(const void* Q, const void* K, const void* V, void* O, float* LSE, const Shape& sh, int d,
                          int causal, cudaStream_t stream, void* workspace = nullptr, size_t workspace_bytes = 0,
                          const float* rope_cos = nullptr, const float* rope_sin = nullptr) {
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
  CUtensorMap mq, mk, mv, mo;
  if (!hk::encode_bnhd(&mq, Q, mb, mnq, sh.Hq, d, 128) || !hk::encode_bnhd(&mk, K, mb, mnk, sh.Hkv, d, 128) ||
      !hk::encode_bnhd(&mv, V, mb, mnk, sh.Hkv, d, 128) || !hk::encode_bnhd(&mo, O, mb, mnq, sh.Hq, d, 128))
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
  p.rope_cos = rope_cos;
  p.rope_sin = rope_sin;
  if (workspace && cudaMemsetAsync(workspace, 0, 8, stream) != cudaSuccess)
    return fail(HK_ERR_LAUNCH, "cudaMemsetAsync(workspace counters) failed");
  if (rope_cos) {
    if (d == 64)
      return causal ? launch_fwd<64, true, true>(mq, mk, mv, mo, p, num_sms, stream)
                    : launch_fwd<64, false, true>(mq, mk, mv, mo, p, num_sms, stream);
    return causal ? launch_fwd<128, true, true>(mq, mk, mv, mo, p, num_sms, stream)
                  : launch_fwd<128, false, true>(mq, mk, mv, mo, p, num_sms, stream);
  }
  if (d == 64)
    return causal ? launch_fwd<64, true>(mq, mk, mv, mo, p, num_sms, stream)
                  : launch_fwd<64, false>(mq, mk, mv, mo, p, num_sms, stream);
  return causal ? launch_fwd<128, true>(mq, mk, mv, mo, p, num_sms, stream)
                : launch_fwd<128, false>(mq, mk, mv, mo, p, num_sms, stream);
}

static Shape dense(int B, int Hq, int Hkv, int Nq, int Nk) { return Shape{nullptr, nullptr, B, Hq, Hkv, Nq, Nk, 0, 0}; }
static Shape packed(const int* cu_q, const int* cu_k, int B, int Hq, int Hkv, int total_q, int total_k, int max_q,
                    int max_k) {
  return Shape{cu_q, cu_k, B, Hq, Hkv, max_q, max_k, total_q, total_k};
}

