"""Backward parity: CUDA path (through the C ABI) vs the fp64 oracle on the
same bf16 inputs: relative L2 <= 1e-2 for dQ, dK, dV (BASELINE.json), plus the
D = rowsum(dO * O) preprocess output in the workspace (diagnostic, 1e-2)."""
import numpy as np
import pytest
import torch

import oracle
from util import TOL_MAXABS, TOL_RELL2, gen, np64, rel_l2

pytestmark = pytest.mark.gpu

CASES = [
    # B, N, Hq, Hkv, d
    (1, 128, 2, 2, 64),     # C1
    (2, 384, 4, 2, 128),    # 3 tiles, G=2
    (1, 640, 8, 1, 64),     # 5 tiles, G=8
    (1, 512, 2, 2, 128),
    (2, 256, 6, 3, 64),
    (1, 256, 8, 1, 128),    # G=8, d=128 (the 70B head geometry at small N)
    (1, 200, 4, 2, 128),    # ragged: N % 128 != 0
    (2, 333, 2, 1, 64),     # ragged, 3 tiles
    (1, 77, 2, 2, 128),     # a single partial tile
    (1, 1, 2, 1, 64),       # N = 1
]


def run(B, N, Hq, Hkv, d, causal, seed, std_qk=None):
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    x = gen(B, N, Hq, Hkv, d, seed=seed, std_qk=std_qk)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    from paper_2511_08083_b200 import bwd_workspace_bytes
    Np = (N + 127) // 128 * 128
    ws = torch.empty(bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4, dtype=torch.float32, device="cuda")
    dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=ws)
    torch.cuda.synchronize()
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), causal)
    errs = {}
    for n, t in (("dQ", dq), ("dK", dk), ("dV", dv)):
        got = np64(t)
        if np.linalg.norm(ref[n]) < 1e-9 * np.sqrt(ref[n].size):
            # Identically zero gradient (N = 1: dS = P (dP - D) = 0 exactly). Relative L2 is
            # undefined; what the GPU returns is the usual FlashAttention rounding noise: P is
            # rounded to bf16 inside O while l sums the fp32 P (reading #6), and D is taken from
            # the bf16 O (reading #11), so dP - D carries ~2^-9 |dO.V| — for N = 1 that noise is
            # the whole signal. Bound it absolutely at 2 x the O tolerance (scaled into the
            # rel-L2 slot so one threshold applies).
            errs[n] = float(np.abs(got).max()) * (TOL_RELL2 / (2 * TOL_MAXABS))
        else:
            errs[n] = rel_l2(got, ref[n])
    errs["D"] = rel_l2(np64(ws[: B * Hq * Np]).reshape(B, Hq, Np)[:, :, :N], ref["D"])
    return errs


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("B,N,Hq,Hkv,d", CASES)
def test_bwd_parity(B, N, Hq, Hkv, d, causal):
    errs = run(B, N, Hq, Hkv, d, causal, seed=7 * N + d)
    assert all(e <= TOL_RELL2 for e in errs.values()), errs


@pytest.mark.parametrize("causal", [False, True])
def test_bwd_stress_std4(causal):
    errs = run(1, 512, 4, 2, 128, causal, seed=5, std_qk=4.0)
    assert all(e <= TOL_RELL2 for e in errs.values()), errs


@pytest.mark.parametrize("d", [64, 128])
def test_bwd_deterministic(d):
    """Bitwise run-to-run reproducibility of the deterministic backward (no atomics, fixed
    reduction order). Also the race canary: a pipeline hazard shows up as a run that differs."""
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    x = gen(2, 640, 8, 2, d, seed=11)
    outs = []
    for _ in range(4):
        o, lse = attn_fwd(x["Q"], x["K"], x["V"], True)
        outs.append((o, lse) + attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], True, deterministic=True))
    torch.cuda.synchronize()
    for run in outs[1:]:
        for a, b in zip(outs[0], run):
            assert torch.equal(a, b)


@pytest.mark.parametrize("d", [64, 128])  # d = 128 runs the two-pass backward unless built with HK_FUSED128=1
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("B,N,Hq,Hkv", [(2, 640, 8, 2), (1, 1024, 4, 4), (2, 333, 6, 3), (1, 128, 2, 1)])
def test_bwd_fused(B, N, Hq, Hkv, causal, d):
    """The default backward is the fused single pass (NEXT #1, hk_attn.h): dK, dV bitwise equal
    to the deterministic two-pass backward (same kernel arithmetic for them) and bitwise run to run;
    dQ — fp32 partials added in L2 in arrival order — within the BASELINE tolerance of the oracle,
    of itself across runs up to the bf16 rounding flips fp32 reordering causes (a flip moves an
    element by one bf16 ulp, 2^-8 relative; rel-L2 <= 2^-8 sqrt(1%) = 4e-4), and within bf16 rounding of the
    two-pass dQ (which rounds its own dS = P (dP - D), from S = Q K^T instead of S^T = K Q^T, to
    bf16: rel-L2 <= 4e-3 = one bf16 ulp 2^-8)."""
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    x = gen(B, N, Hq, Hkv, d, seed=N + Hq)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    det = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, deterministic=True)
    runs = [attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal) for _ in range(3)]
    torch.cuda.synchronize()
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), causal)
    for dq, dk, dv in runs:
        assert torch.equal(dk, det[1]) and torch.equal(dv, det[2])
        assert rel_l2(np64(dq), np64(det[0])) <= 4e-3
        assert rel_l2(np64(dq), np64(runs[0][0])) <= 4e-4
        assert rel_l2(np64(dq), ref["dQ"]) <= TOL_RELL2


@pytest.mark.parametrize("det", [True, False])
@pytest.mark.parametrize("d,causal", [(128, True), (64, False), (64, True)])
def test_bwd_accumulate_f32(d, causal, det):
    """HK_BWD_ACCUMULATE_F32 adds the (scaled, unrounded) gradients into caller fp32 tensors: two
    calls on the same inputs from a start value A give A + 2 g, with g within fp32 rounding of the
    bf16 call's result (which rounds g once) and within the BASELINE tolerance of the oracle."""
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    B, N, Hq, Hkv = 2, 333, 4, 2
    x = gen(B, N, Hq, Hkv, d, seed=40 + d)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    bf = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, deterministic=True)
    start = [torch.full(t.shape, 0.5, dtype=torch.float32, device="cuda") for t in bf]
    acc = [t.clone() for t in start]
    for _ in range(2):
        attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, dq=acc[0], dk=acc[1], dv=acc[2],
                 deterministic=det, accumulate=True)
    torch.cuda.synchronize()
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), causal)
    for name, a, s0, b in zip(("dQ", "dK", "dV"), acc, start, bf):
        g = (np64(a) - np64(s0)) / 2
        assert rel_l2(g, np64(b)) <= 4e-3, name          # bf16 rounding of the bf16 call
        assert rel_l2(g, ref[name]) <= TOL_RELL2, name
    with pytest.raises(ValueError):
        attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, accumulate=True)
