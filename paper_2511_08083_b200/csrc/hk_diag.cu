// libhkattn_diag.so: diagnostic entry points (include/hk_attn_diag.h) — not the hot path.
// Kept out of libhkattn.so: the micro-benchmarks allocate scratch memory of their own, which
// the product library never does. Links its own copy of the attention kernels (one-phase
// backward launches for per-kernel timing) and the micro-benchmark kernels.
#include "host.cuh"
#pragma GCC visibility push(default)
#include "../../include/hk_attn_diag.h"
#pragma GCC visibility pop
#include "rates_diag.cuh"
#include "umma_diag.cuh"

extern "C" {

const char* hk_diag_last_error(void) { return g_err; }

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
  if (kind == 6) {  // bulk-async fp32 reduce of 128x128 tiles: param = mode * 100000 + row tiles (H = 32 heads)
    const int mode = param / 100000, row_tiles = param % 100000, H = 32;
    if (mode > 1 || row_tiles < 1) return fail(HK_ERR_UNSUPPORTED, "mode 0/1, row tiles >= 1");
    static float* dst = nullptr;
    static size_t have = 0;
    const size_t bytes = (size_t)row_tiles * 128 * H * 128 * 4;
    if (have < bytes) {
      if (dst) cudaFree(dst);
      if (cudaMalloc(&dst, bytes) != cudaSuccess) return fail(HK_ERR_DEVICE, "cudaMalloc");
      cudaMemset(dst, 0, bytes);
      have = bytes;
    }
    auto fn_enc = hk::get_encode_fn();
    if (!fn_enc) return fail(HK_ERR_DEVICE, "no cuTensorMapEncodeTiled");
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)H * 128, (cuuint64_t)row_tiles * 128};
    cuuint64_t strides[1] = {(cuuint64_t)H * 128 * 4};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    if (fn_enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dst, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(HK_ERR_DEVICE, "encode fp32 map");
    const uint32_t smem = 65536 + 1024;
    if (mode == 0) {
      if ((s = ensure_smem(hk::bulk_red_rate_kernel<0>, smem)) != HK_OK) return s;
      hk::bulk_red_rate_kernel<0><<<148, 128, smem, stream>>>(m, dst, row_tiles, H, iters, out);
    } else {
      if ((s = ensure_smem(hk::bulk_red_rate_kernel<1>, smem)) != HK_OK) return s;
      hk::bulk_red_rate_kernel<1><<<148, 128, smem, stream>>>(m, dst, row_tiles, H, iters, out);
    }
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
