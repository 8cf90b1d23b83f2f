"""GPU parity of the tcgen05 CTA-pair BF16 GEMM (include/hk_gemm.h) against the
fp64 oracle (oracle/gemm.py), through the C ABI.

Tolerance (reading #18): C is the fp32-accumulated product rounded
once to bf16, so |C_gpu - C_ref| <= 2^-9 |C_ref| + (fp32 summation error);
the test allows 2^-8 |C_ref| + 1e-2 (the absolute term covers entries near 0,
whose fp32 summation-order error is ~1e-4 at K = 8192)."""
import numpy as np
import pytest
import torch

from oracle import gemm_abt, gemm_abt_rows
from paper_2511_08083_b200 import HKError, gemm
from paper_2511_08083_b200.inputs import make_gemm_inputs

pytestmark = pytest.mark.gpu


def check(c_gpu, ref):
    c = c_gpu.float().cpu().numpy().astype(np.float64)
    err = np.abs(c - ref)
    bound = 2.0 ** -8 * np.abs(ref) + 1e-2
    bad = err > bound
    assert not bad.any(), f"{bad.sum()} entries out of tolerance; worst {err.max():.4g} at ref {ref.flat[err.argmax()]:.4g}"


@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (256, 512, 128), (512, 256, 192), (768, 1024, 320),
                                   (2048, 1536, 1024)])
def test_gemm_parity(M, N, K):
    x = make_gemm_inputs(M, N, K, seed=M + N + K, device="cuda")
    c = gemm(x["A"], x["B"])
    torch.cuda.synchronize()
    ref = gemm_abt(x["A"].float().cpu().numpy(), x["B"].float().cpu().numpy())
    check(c, ref)


def test_gemm_full_size_sampled_rows():
    """M = N = K = 8192 (the paper's shape): rows sampled from every 256-row
    tile position class (first/last rows of both CTA halves) checked against the oracle."""
    M = N = K = 8192
    x = make_gemm_inputs(M, N, K, seed=7, device="cuda")
    c = gemm(x["A"], x["B"])
    torch.cuda.synchronize()
    rows = [0, 127, 128, 255, 256 * 17 + 5, 256 * 17 + 200, M - 129, M - 1]
    A, B = x["A"].float().cpu().numpy(), x["B"].float().cpu().numpy()
    ref = gemm_abt_rows(A, B, rows)
    check(c[rows], ref)
    # and a column block through every M tile (columns of the last N tile)
    cols = list(range(N - 256, N, 37))
    ref_c = A @ B[cols].T.astype(np.float64)
    check(c[:, cols], ref_c)


def test_gemm_deterministic():
    x = make_gemm_inputs(1024, 1024, 2048, seed=3, device="cuda")
    c1 = gemm(x["A"], x["B"])
    c2 = gemm(x["A"], x["B"])
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)


def test_gemm_special_values():
    """Identity B gives C = A exactly (every product exact, one nonzero term per sum)."""
    M, K = 512, 256
    x = make_gemm_inputs(M, 256, K, seed=11, device="cuda")
    eye = torch.eye(K, dtype=torch.bfloat16, device="cuda")
    c = gemm(x["A"], eye.contiguous())
    torch.cuda.synchronize()
    assert torch.equal(c, x["A"])


def test_gemm_rejects_unsupported_shapes():
    a = torch.zeros(300, 64, dtype=torch.bfloat16, device="cuda")
    b = torch.zeros(256, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(HKError):
        gemm(a, b)
