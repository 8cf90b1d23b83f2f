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
 * of work counters for the persistent kernels, then for d = 64 the fused backward's fp32 dQ
 * accumulator (B*Np*Hq*64 floats): 2*B*Hq*Np*4 + 256 (+ B*Np*Hq*256 when d == 64). The call
 * initialises all of it (no zeroing needed); calls sharing one workspace must be
 * stream-ordered. */
size_t hk_attn_bwd_workspace_bytes(int B, int Hq, int Hkv, int N, int d);

/* Backward: given Q, K, V, the forward's O and LSE, and dO, writes dQ, dK, dV
 * (bf16, fully overwritten). Runs three kernels: D-preprocess, then the dK/dV pass
 * (GQA group reduced inside the kernel) on `stream` and the dQ pass, which is
 * independent of it, on a library-owned non-blocking side stream forked from `stream`
 * after the preprocess and joined back into `stream` with events. There is one side
 * stream per (device, caller stream), created on first use with the caller stream's
 * priority, so concurrent backward calls on different streams stay independent — make
 * the first backward call on a given stream outside CUDA-graph capture; if the side
 * stream cannot be created (or more than 256 caller streams were seen) the kernels
 * run serially on `stream`. Work enqueued on `stream` afterwards sees all three; the
 * fork/join is CUDA-graph capturable. */
hk_status hk_attn_bwd(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                      const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                      int B, int Hq, int Hkv, int N, int d, int causal, cudaStream_t stream);

/* ---- Sequence-length variants (reading #22).
 * The paper's problem has Nq == Nk (P:1292 `num_tiles = ATTN_N / KV_BLOCK_SIZE`);
 * these entry points take the baselines' API features (AITER flash_attn_func /
 * varlen; SDPA) with the same kernels.
 * Mask: key j is visible to query i iff j < Nk and, when causal,
 *   j <= i + (Nk - Nq)         (bottom-right aligned; j <= i when Nq == Nk).
 * A query row that sees no key (causal with Nq > Nk, or a varlen sequence with
 * no keys) gets O = 0 and LSE = -inf, and adds nothing to the gradients
 * (its dQ row is 0). */

/* Dense, Nq != Nk. Q, O, dO, dQ: [B][Nq][Hq][d]; K, V, dK, dV: [B][Nk][Hkv][d];
 * LSE: [B][Hq][Nq] fp32. Nq, Nk >= 1. Errors and ownership as above. */
hk_status hk_attn_fwd_qk(const void* Q, const void* K, const void* V, void* O, float* LSE, int B, int Hq,
                         int Hkv, int Nq, int Nk, int d, int causal, cudaStream_t stream);
/* = 2*B*Hq*Nqp*4 + 256 (+ B*Nqp*Hq*256 when d == 64), Nqp = Nq rounded up to a multiple of 128. */
size_t hk_attn_bwd_qk_workspace_bytes(int B, int Hq, int Hkv, int Nq, int Nk, int d);
hk_status hk_attn_bwd_qk(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                         const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                         int B, int Hq, int Hkv, int Nq, int Nk, int d, int causal, cudaStream_t stream);

/* Packed variable-length batch of B sequences.
 *   Q, O, dO, dQ : [total_q][Hq][d] bf16;  K, V, dK, dV : [total_k][Hkv][d] bf16
 *   LSE          : [Hq][total_q] fp32
 *   cu_seqlens_q, cu_seqlens_k : DEVICE int32 [B+1], cu[0] = 0, non-decreasing,
 *     cu_q[B] = total_q, cu_k[B] = total_k; sequence b is Q rows
 *     cu_q[b] .. cu_q[b+1]-1 against K/V rows cu_k[b] .. cu_k[b+1]-1
 *     (lengths may differ per sequence and between Q and K, and may be 0).
 *   max_seqlen_q / max_seqlen_k : >= every sequence's length (sizes the grid).
 * total_q, total_k, max_seqlen_* >= 1. The cu_seqlens contents live on the
 * device and are NOT validated (that would need a host sync): offsets that
 * break the contract give undefined results. Each sequence's lengths are
 * clamped to [0, max_seqlen] on the device, so query rows / keys beyond a
 * sequence's max_seqlen are not computed (their output rows are left
 * untouched) and the backward never indexes past its padded workspace. A query sequence with no keys gets O = 0,
 * LSE = -inf, dQ = 0; keys no query sees get dK = dV = 0. */
/* workspace: NULL (the forward's CTAs take work items in a static order) or >= 256 bytes of
 * device memory, 16-B aligned, for the dynamic scheduler's counters (CTAs draw items from a
 * counter: balanced when sequence lengths differ). Calls sharing a workspace must be
 * stream-ordered; the call initialises it (no zeroing needed). */
hk_status hk_attn_fwd_varlen(const void* Q, const void* K, const void* V, void* O, float* LSE,
                             const int* cu_seqlens_q, const int* cu_seqlens_k, int B, int Hq, int Hkv,
                             int total_q, int total_k, int max_seqlen_q, int max_seqlen_k, int d, int causal,
                             void* workspace, size_t workspace_bytes, cudaStream_t stream);
/* = 2*B*Hq*Mp*4 + 256 (+ B*Mp*Hq*256 when d == 64), Mp = max_seqlen_q rounded up to 128. */
size_t hk_attn_bwd_varlen_workspace_bytes(int B, int Hq, int Hkv, int max_seqlen_q, int max_seqlen_k, int d);
hk_status hk_attn_bwd_varlen(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                             const void* dO, void* dQ, void* dK, void* dV, void* workspace,
                             size_t workspace_bytes, const int* cu_seqlens_q, const int* cu_seqlens_k, int B,
                             int Hq, int Hkv, int total_q, int total_k, int max_seqlen_q, int max_seqlen_k, int d,
                             int causal, cudaStream_t stream);

/* ---- Backward with flags (ABI 4).
 * At d = 64 the default backward is the fused single pass (DESIGN.md
 * §6 "Fused backward"): the dK/dV pass also forms dQ_partial = dS K_j per 128 x 128 block on the
 * tensor core and adds it into an fp32 accumulator in the workspace with the bulk-async tensor
 * reduce (cp.reduce.async.bulk.tensor .add.f32), then one pass scales and rounds it to bf16; the
 * separate dQ pass (which recomputes S and dP) is not run. The fp32 additions of the
 * partials land in L2 in whatever order the CTAs reach them, so dQ is reproducible only up to
 * fp32 reordering (dK, dV stay bitwise reproducible). HK_BWD_DETERMINISTIC selects the two-pass
 * backward (bitwise reproducible dQ, the d = 128 path) at d = 64; at d = 128 flags change nothing.
 * hk_attn_bwd* without _ex use flags = 0. Unknown flag bits: HK_ERR_INVALID_ARGUMENT. */
#define HK_BWD_DETERMINISTIC 1u
/* HK_BWD_ACCUMULATE_F32: dQ, dK, dV point to fp32 tensors of the same shapes, and the call ADDS
 * its (scaled, unrounded) results into them instead of writing bf16 — for callers that sum the
 * gradients of several calls (context-parallel ring attention: one call per visible chunk pair)
 * without rounding each part to bf16. Rows no query / key sees add nothing. Each output row is
 * owned by one CTA (no atomics); concurrent calls adding into the same accumulator must be
 * stream-ordered. */
#define HK_BWD_ACCUMULATE_F32 2u
hk_status hk_attn_bwd_ex(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                         const void* dO, void* dQ, void* dK, void* dV, void* workspace, size_t workspace_bytes,
                         int B, int Hq, int Hkv, int Nq, int Nk, int d, int causal, unsigned flags,
                         cudaStream_t stream);
hk_status hk_attn_bwd_varlen_ex(const void* Q, const void* K, const void* V, const void* O, const float* LSE,
                                const void* dO, void* dQ, void* dK, void* dV, void* workspace,
                                size_t workspace_bytes, const int* cu_seqlens_q, const int* cu_seqlens_k, int B,
                                int Hq, int Hkv, int total_q, int total_k, int max_seqlen_q, int max_seqlen_k,
                                int d, int causal, unsigned flags, cudaStream_t stream);

/* ---- Stored-dS backward (ABI 6; d = 128, dense calls: hk_attn_bwd, _qk, _ex).
 * A workspace of at least hk_attn_bwd_ds_workspace_bytes(...) bytes (> the plain size exactly when the
 * path applies) selects it: the dK/dV pass also writes every visited 128 x 128 block's bf16 dS^T
 * into the workspace (after the plain part, 1024-byte aligned), and the dQ pass is then ONE GEMM per
 * block, dQ = (1/sqrt d) dS K, reading those tiles back, instead of re-computing S and dP (three
 * GEMMs). The extra workspace is B * Hq * blocks * 32 KB, blocks = T(T+1)/2 (causal, Nq == Nk) or
 * Tq * Tk, T = ceil(N / 128): 35 GB for B = 16, Hq = 32, N = 8192 causal. Results: dK, dV bitwise the
 * two-pass ones; dQ is formed from the dK/dV pass's bf16 dS (computed from S^T = K Q^T) and differs
 * from the two-pass dQ by that rounding (reading #29); bitwise reproducible run to run.
 * Returns the plain workspace size where the path does not apply (d = 64, varlen is separate API). */
size_t hk_attn_bwd_ds_workspace_bytes(int B, int Hq, int Hkv, int Nq, int Nk, int d, int causal);

/* ---- SM budget for the persistent kernels (ABI 5).
 * Every kernel of this library that runs one CTA per SM (forward, backward passes, GEMM) and the
 * grid-stride helpers launch on at most max_ctas SMs' worth of CTAs (max_ctas <= 0: all SMs, the
 * default). Purpose: leave SMs to a concurrent kernel on another stream — the copy kernels NCCL
 * runs for a context-parallel ring step's K/V and dK/dV transfers (ring.py) — so
 * that communication overlaps the attention kernels instead of queueing behind CTAs that hold
 * every SM. A process-wide setting (atomic; read at each launch, so it applies to later calls on
 * any thread); results do not depend on it (work order is fixed per output tile, reading #19).
 * hk_get_max_ctas returns the current value (0 = all SMs). */
void hk_set_max_ctas(int max_ctas);
int hk_get_max_ctas(void);

const char* hk_attn_last_error(void);
const char* hk_status_string(hk_status s);
int hk_attn_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HK_ATTN_H_ */
