"""GPU parity of the memory-bound kernels (include/hk_membound.h) against the fp64
oracles (oracle/membound.py), through the C ABI.

Tolerances (readings #20, #21): every output is one bf16 rounding of an
fp32 computation, so it may sit one bf16 ulp (<= 2^-7 relative) from the rounded
fp64 value: |gpu - ref| <= 2^-7 |ref| + atol, with atol 1e-2 for the LayerNorm
output (fp32 vs fp64 statistics, values O(1); plus, element by element, the
propagated effect |dr| rstd |w| of any one-ulp difference in r), 1e-6 for out_resid (a
single rounding of residual + dropout(x); the absolute term covers cancellation to ~0,
where the fp32 rounding of x / (1 - p), ~1e-7, is the whole result) and 2e-3 for rotary (cancellation in
x_i cos - x_j sin near zero). The dropout zero pattern matches the oracle's hash
exactly (the oracle gets the fp32 p the ABI receives)."""
import numpy as np
import pytest
import torch

from oracle import dropout_keep, layernorm_dropout_residual, rope as rope_ref, rope_tables
from paper_2511_08083_b200 import HKError, ln_dropout_residual, rope
from paper_2511_08083_b200.inputs import make_ln_inputs, make_rope_inputs

pytestmark = pytest.mark.gpu


def np64(t):
    return t.float().cpu().numpy().astype(np.float64)


def within(gpu, ref, atol):
    err = np.abs(np64(gpu) - ref)
    bound = 2.0 ** -7 * np.abs(ref) + atol
    assert (err <= bound).all(), f"{(err > bound).sum()} out of tolerance, worst {err.max():.4g}"


@pytest.mark.parametrize("rows,D,p", [(64, 128, 0.0), (37, 2048, 0.0), (37, 2048, 0.1), (16, 264, 0.5),
                                      (8, 8192, 0.25), (300, 1024, 0.0)])
def test_ln_dropout_residual_parity(rows, D, p):
    x = make_ln_inputs(rows, D, seed=rows + D, device="cuda")
    seed = 1234
    out, res = ln_dropout_residual(x["x"], x["residual"], x["weight"], x["bias"], p=p, seed=seed)
    torch.cuda.synchronize()
    p32 = float(np.float32(p))  # the ABI takes p as fp32
    o_ref, r_ref = layernorm_dropout_residual(np64(x["x"]), np64(x["residual"]), np64(x["weight"]),
                                              np64(x["bias"]), p=p32, seed=seed)
    within(res, r_ref, 1e-6)
    # where the GPU's r sits one ulp from the oracle's (a rounding straddle), that
    # difference propagates through (r - mean) * rstd * w into out: widen by exactly it
    r64 = r_ref
    rstd = 1.0 / np.sqrt(((r64 - r64.mean(axis=1, keepdims=True)) ** 2).mean(axis=1, keepdims=True) + 1e-5)
    dr = np.abs(np64(res) - r_ref) * rstd * np.abs(np64(x["weight"]))
    err = np.abs(np64(out) - o_ref)
    bound = 2.0 ** -7 * np.abs(o_ref) + 1e-2 + 1.01 * dr
    assert (err <= bound).all(), f"{(err > bound).sum()} out of tolerance, worst {err.max():.4g}"
    if p > 0:  # dropped elements: out_resid == residual exactly
        keep = dropout_keep(rows * D, p32, seed).reshape(rows, D)
        np.testing.assert_array_equal(np64(res)[~keep], np64(x["residual"])[~keep])


def test_ln_rejects_unsupported():
    x = make_ln_inputs(4, 100, device="cuda")
    with pytest.raises(HKError):
        ln_dropout_residual(x["x"], x["residual"], x["weight"], x["bias"])


@pytest.mark.parametrize("B,N,H,d", [(2, 33, 3, 64), (1, 100, 4, 128), (2, 17, 2, 256)])
def test_rope_parity(B, N, H, d):
    x = make_rope_inputs(B, N, H, d, seed=d, device="cuda")["x"]
    c, s = rope_tables(N, d)
    cf, sf = c.astype(np.float32), s.astype(np.float32)
    out = rope(x, torch.from_numpy(cf).cuda(), torch.from_numpy(sf).cuda())
    torch.cuda.synchronize()
    within(out, rope_ref(np64(x), cf, sf), 2e-3)


def test_rope_in_place_and_position_zero():
    B, N, H, d = 1, 9, 2, 128
    x = make_rope_inputs(B, N, H, d, seed=5, device="cuda")["x"]
    x0 = x.clone()
    c, s = rope_tables(N, d)
    rope(x, torch.from_numpy(c.astype(np.float32)).cuda(), torch.from_numpy(s.astype(np.float32)).cuda(), out=x)
    torch.cuda.synchronize()
    assert torch.equal(x[:, 0], x0[:, 0])  # theta = 0: exact identity
    within(x, rope_ref(np64(x0), c.astype(np.float32), s.astype(np.float32)), 2e-3)
