/* hk_attn.h — C ABI of the B200 (sm_100a) fused attention library libhkattn.so.
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, arXiv 2511.08083):
 *   S_ij  = (1/sqrt(d)) <Q[b,i,h,:], K[b,j,kvh,:]>,  kvh = h / (Hq/Hkv)
 *   LSE_i = ln sum_{j in A(i)} exp(S_ij)     (natural log)
 *   O_i   = sum_{j in A(i)} exp(S_ij - LSE_i) V[b,j,kvh,:]
 *   A(i)  = {j <= i} if causal else all keys                                  P:571 (reading #3)
 * The backward is the analytic gradient of that forward (P:577-580 give no
 * algorithm; DESIGN.md "Readings" #11): dQ, dK, dV of L = sum(O * dO), with
 * dK/dV summed over the G = Hq/Hkv query heads of each KV head.
 *
 * Layouts (index order of the paper's globals):
 *   Q, O, dO, dQ : [B][N][Hq][d]  bf16, contiguous, d fastest ("BNHD")
 *   K, V, dK, dV : [B][N][Hkv][d] bf16, contiguous
 *   LSE          : [B][Hq][N]     fp32
 * Supported: d in {64, 128}; any N >= 1 (a ragged last 128-row tile is masked,
 * never read past N in the caller's buffers); Hq % Hkv == 0.
 *
 * Ownership: every pointer is a CUDA device pointer owned by the caller; the
 * library allocates no device memory and keeps no per-call state. All work is
 * enqueued on `stream` (no host synchronisation). Outputs are fully
 * overwritten (no pre-zeroing needed) and bitwise reproducible for fixed
 * inputs (no atomics).
 *
 * Errors: arguments are validated before anything is enqueued; on a non-OK
 * status nothing is launched and outputs are untouched. No exceptions cross
 * the ABI, nothing is printed, nothing aborts. hk_attn_last_error() returns a
 * thread-local description of the last non-OK status. Asynchronous device
 * faults surface at the caller's next synchronisation, as usual in CUDA.
 */
#ifndef HK_ATTN_H_
#define HK_ATTN_H_

#include <stddef.h>
#include <cuda_runtime_api.h> /* cudaStream_t */

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HK_OK = 0,
  HK_ERR_INVALID_ARGUMENT = 1, /* null / misaligned (16 B) pointer; B,Hq,Hkv,N <= 0; Hq % Hkv != 0;
                                  an output aliases an input; workspace too small             */
  HK_ERR_UNSUPPORTED = 2,      /* d not in {64,128}; a dimension too large                     */
  HK_ERR_DEVICE = 3,           /* current device is not CC 10.0 (sm_100) or setup failed       */
  HK_ERR_LAUNCH = 4            /* the launch itself failed (cudaGetLastError after enqueue)    */
} hk_status;

/* Forward: O = softmax(Q K^T / sqrt(d)) V and LSE, per head (GQA via kvh = h / (Hq/Hkv)).
 * causal != 0 masks key j > query i. */
hk_status hk_attn_fwd(const void* Q, const void* K, const void* V, void* O, float* LSE, int B, int Hq,
                      int Hkv, int N, int d, int causal, cudaStream_t stream);

/* Bytes of workspace hk_attn_bwd needs: D = rowsum(dO * O) and LSE*log2(e),
 * each [B][Hq][Np] fp32 with Np = N rounded up to a multiple of 128, then 256 bytes
 * of work counters for the persistent kernels: 2*B*Hq*Np*4 + 256. The call
 * initialises all of it (no zeroing needed); calls sharing one workspace must be
 * stream-ordered. */
size_t hk_attn_bwd_workspace_bytes(int B, int Hq, int Hkv, int N, int d);

/* Backward: given Q, K, V, the forward's O and LSE, and dO, writes dQ, dK, dV
 * (bf16, fully overwritten). Runs three stream-ordered kernels:
 * D-preprocess, dK/dV pass (GQA group reduced inside the kernel), dQ pass. */
hk_status hk_attn_bwd(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                      const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                      int B, int Hq, int Hkv, int N, int d, int causal, cudaStream_t stream);

const char* hk_attn_last_error(void);
const char* hk_status_string(hk_status s);
int hk_attn_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HK_ATTN_H_ */
