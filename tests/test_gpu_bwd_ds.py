"""Stored-dS backward (d = 128, dense; include/hk_attn.h hk_attn_bwd_ds_workspace_bytes, DESIGN.md
§6 and reading #29): parity with the fp64 oracle at the BASELINE tolerance, dK and dV bitwise equal
to the two-pass backward, dQ within the bf16 rounding of dS of it, bitwise run-to-run, the public
API's automatic choice (and its budget), and the fp32-accumulate mode."""
import numpy as np
import pytest
import torch

import oracle
from util import TOL_RELL2, np64, rel_l2

pytestmark = pytest.mark.gpu

CASES = [
    # B, Nq, Nk, Hq, Hkv, causal
    (1, 256, 256, 2, 1, True),
    (2, 384, 384, 4, 2, False),
    (1, 640, 640, 8, 2, True),      # 5 tiles, G = 4
    (2, 200, 200, 4, 4, True),      # ragged: N % 128 != 0
    (1, 77, 77, 2, 1, False),       # a single partial tile
    (2, 300, 700, 4, 2, True),      # Nq < Nk (bottom-right causal, rectangle layout)
    (1, 500, 260, 6, 3, True),      # Nq > Nk: key-less query rows
    (1, 777, 333, 6, 3, False),
    (2, 2048, 2048, 16, 4, True),   # 256 query items on 148 CTAs: several items per CTA in both passes
    (1, 512, 512, 16, 2, True),     # G = 8 (the 70B head geometry)
    (3, 1000, 1000, 8, 8, True),    # MHA, ragged, 3 sequences
    (2, 640, 640, 4, 1, False),     # MQA (Hkv = 1), non-causal
]


def _inputs(B, Nq, Nk, Hq, Hkv, seed):
    from paper_2511_08083_b200.inputs import make_qk_inputs
    return make_qk_inputs(B, Nq, Nk, Hq, Hkv, 128, seed=seed, device="cuda")


def _ws(nbytes):
    return torch.zeros((nbytes + 3) // 4, dtype=torch.float32, device="cuda")


@pytest.mark.parametrize("case", CASES)
def test_stored_ds_parity(case):
    from paper_2511_08083_b200 import api
    B, Nq, Nk, Hq, Hkv, causal = case
    x = _inputs(B, Nq, Nk, Hq, Hkv, seed=11)
    o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
    plain = api.bwd_workspace_bytes(B, Hq, Hkv, Nq, 128, Nk)
    big = api.bwd_ds_workspace_bytes(B, Hq, Hkv, Nq, 128, Nk, causal)
    assert big > plain  # the path applies to every dense d = 128 shape
    g2 = api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=_ws(plain))
    gs = api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=_ws(big))
    gr = api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=_ws(big))
    torch.cuda.synchronize()
    # dK, dV: the same kernel arithmetic as the two-pass backward
    assert torch.equal(gs[1], g2[1]) and torch.equal(gs[2], g2[2])
    # dQ from the dK/dV pass's bf16 dS (S^T = K Q^T) vs the dQ pass's own (S = Q K^T): bf16 rounding
    # of dS only (reading #29)
    assert rel_l2(np64(gs[0]), np64(g2[0])) <= 4e-3
    assert all(torch.equal(a, b) for a, b in zip(gs, gr))  # no atomics: bitwise run to run
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), causal)
    for n, t in zip(("dQ", "dK", "dV"), gs):
        r = ref[n]
        if np.linalg.norm(r) == 0:
            assert np.abs(np64(t)).max() == 0
        else:
            assert rel_l2(np64(t), r) <= TOL_RELL2, n


def test_stored_ds_default_and_budget():
    """attn_bwd without a workspace takes the stored-dS path when it fits the budget, the two-pass
    backward otherwise (budget 0), each bitwise equal to an explicit workspace of that size."""
    from paper_2511_08083_b200 import api
    B, N, Hq, Hkv, causal = 2, 640, 8, 2, True
    x = _inputs(B, N, N, Hq, Hkv, seed=3)
    o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
    args = (x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
    auto = api.attn_bwd(*args)
    ds = api.attn_bwd(*args, workspace=_ws(api.bwd_ds_workspace_bytes(B, Hq, Hkv, N, 128, None, causal)))
    old = api.DS_WORKSPACE_BUDGET
    try:
        api.DS_WORKSPACE_BUDGET = 0
        auto2 = api.attn_bwd(*args)
    finally:
        api.DS_WORKSPACE_BUDGET = old
    two = api.attn_bwd(*args, workspace=_ws(api.bwd_workspace_bytes(B, Hq, Hkv, N, 128)))
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(auto, ds))
    assert all(torch.equal(a, b) for a, b in zip(auto2, two))
    assert not torch.equal(auto[0], two[0])  # the two dQ paths round dS from S^T vs S


@pytest.mark.parametrize("causal", [False, True])
def test_stored_ds_accumulate_f32(causal):
    """HK_BWD_ACCUMULATE_F32 through the stored-dS path: the fp32 results added into nonzero
    accumulators equal the bf16 call's results to bf16 rounding."""
    from paper_2511_08083_b200 import api
    B, N, Hq, Hkv = 1, 384, 4, 2
    x = _inputs(B, N, N, Hq, Hkv, seed=5)
    o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
    wsb = api.bwd_ds_workspace_bytes(B, Hq, Hkv, N, 128, None, causal)
    g = api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=_ws(wsb))
    base = [torch.full(t.shape, 0.25, dtype=torch.float32, device="cuda") for t in g]
    acc = [b.clone() for b in base]
    api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=_ws(wsb), dq=acc[0], dk=acc[1],
                 dv=acc[2], accumulate=True)
    torch.cuda.synchronize()
    for a, b, t in zip(acc, base, g):
        assert rel_l2(np64(a - b), np64(t)) <= 4e-3
