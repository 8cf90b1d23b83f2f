"""Plain fp64 BF16-GEMM oracle: C = A B^T — the parity oracle for NEXT #2.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Never imported by the
product package.

What is computed (PAPER.md lines cited as P:L):

    C[m, n] = sum_k A[m, k] * B[n, k]

  * The paper's GEMM listing accumulates `mma_ABt(C_accum, A_tile, B_tile, C_accum)`
    over K_STEP slices of row-major A [M, K] and B [N, K] (P:1160, P:1172,
    P:1183, P:1193 [App. Kernel listings > Matrix Multiply]), i.e. C = A B^T
    with both operands K-contiguous.
  * BF16 inputs with fp32 accumulation; the benchmarked shape is
    M = N = K = 8192 with inputs drawn from N(0, 1) (P:284 [Tab. "Producer
    consumer comparisons"]). The epilogue (output dtype) is not shown in the
    listing; the product path stores bf16 (reading #18). The oracle
    returns the exact fp64 product of the given (bf16-valued) inputs.

The definition is written out as one library matmul (numpy, fp64), which is
the plain definition; `gemm_loops` is the same sum as explicit Python loops
for tiny inputs (used to pin the library call).
"""
from __future__ import annotations

import numpy as np


def gemm_abt(A, B) -> np.ndarray:
    """C = A @ B^T in fp64. A: [M, K], B: [N, K] (any float dtype, e.g. bf16 values
    held in float32). Returns fp64 [M, N]."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[1]:
        raise ValueError(f"need A [M, K] and B [N, K]; got {A.shape} and {B.shape}")
    return A @ B.T


def gemm_abt_rows(A, B, rows) -> np.ndarray:
    """Rows `rows` of C = A B^T only (full-size sampled checks)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    return A[np.asarray(rows)] @ B.T


def gemm_loops(A, B) -> np.ndarray:
    """The same sum, term by term (tiny inputs only)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    M, K = A.shape
    N = B.shape[0]
    C = np.zeros((M, N))
    for m in range(M):
        for n in range(N):
            s = 0.0
            for k in range(K):
                s += A[m, k] * B[n, k]
            C[m, n] = s
    return C
