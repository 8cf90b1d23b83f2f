"""Parity at BASELINE.json's full sizes (SURVEY §8(c).5 ROW mode), in the
launch configuration bench.py times (B=16, all heads, one call each).

The oracle checks one unit — the last (b, kvh), exercising the largest
offsets — on sampled rows it can compute one by one:
  * query rows R (first/last 8, tile edges, random) of every head of the unit:
    O and LSE (max-abs 2e-2), dQ (relative L2 1e-2 over the sampled rows);
  * key rows J of the unit: dK, dV (relative L2 1e-2), from the oracle's own
    LSE and D of every row of the unit's heads (configs up to N = 16384).
Every config also checks properties that hold at any size:
sum_j dK_j = 0, sum_j dV_j = sum_{h in group} sum_i dO_i, and
sum <Q, dQ> = sum <K, dK> per unit.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_08083_b200.inputs import sample_rows
from util import TOL_MAXABS, TOL_RELL2, gen, np64, rel_l2

pytestmark = pytest.mark.gpu

# name: B, N, Hq, Hkv, d, causal, check dK/dV key rows with the oracle
CONFIGS = {
    "C2-nc": (16, 4096, 16, 16, 128, False, True),
    "C2-c": (16, 4096, 16, 16, 128, True, True),
    "C3": (16, 8192, 32, 8, 128, True, True),
    "C4-2048": (16, 2048, 32, 32, 64, True, True),
    "C4-16384": (16, 16384, 32, 32, 64, True, True),
    "C5-1024-nc": (16, 1024, 64, 8, 128, False, True),
    "C5-1024-c": (16, 1024, 64, 8, 128, True, True),
    "C5-16384-c": (16, 16384, 64, 8, 128, True, True),
    "C5-32768-c": (16, 32768, 64, 8, 128, True, False),
}


def _oracle_lse_d(Q, K, V, dO, causal, b, h, N, block=2048):
    """Oracle LSE and D for every row of head (b, h), one row block at a time."""
    lse, D = np.empty(N), np.empty(N)
    for r0 in range(0, N, block):
        rows = np.arange(r0, min(N, r0 + block))
        r = oracle.attn_rows(Q, K, V, dO, causal, b, h, rows)
        lse[rows], D[rows] = r["LSE"], r["D"]
    return lse, D


@pytest.mark.parametrize("name", list(CONFIGS))
def test_fullsize(name):
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    B, N, Hq, Hkv, d, causal, check_keys = CONFIGS[name]
    G = Hq // Hkv
    x = gen(B, N, Hq, Hkv, d, seed=101)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
    torch.cuda.synchronize()

    # ---- properties at full size, every unit
    f32 = lambda t: t.float()
    sdk = f32(dk).sum(dim=1)                                      # [B, Hkv, d]
    assert (sdk.norm() / (f32(dk).norm() + 1e-30)).item() < 1e-2
    sdv = f32(dv).sum(dim=1)
    sdo = f32(x["dO"]).sum(dim=1).reshape(B, Hkv, G, d).sum(dim=2)
    assert ((sdv - sdo).norm() / sdo.norm()).item() < 1e-2
    qdq = (f32(x["Q"]) * f32(dq)).sum(dim=(1, 3)).reshape(B, Hkv, G).sum(dim=2)
    kdk = (f32(x["K"]) * f32(dk)).sum(dim=(1, 3))
    # a cancelling sum of N*G*d bf16-rounded products: compare as relative L2 over units
    assert ((qdq - kdk).norm() / kdk.norm()).item() < 1e-2
    assert torch.isfinite(lse).all()

    # ---- oracle on sampled rows of the last unit
    b, kvh = B - 1, Hkv - 1
    ub = lambda t, heads: np64(t[b:b + 1, :, heads])  # one batch, the unit's heads
    hs = slice(kvh * G, (kvh + 1) * G)
    Q, dO = ub(x["Q"], hs), ub(x["dO"], hs)
    K, V = ub(x["K"], slice(kvh, kvh + 1)), ub(x["V"], slice(kvh, kvh + 1))
    rows = sample_rows(N, 64, seed=N)
    o_np, lse_np, dq_np = np64(o[b, rows][:, hs]), np64(lse[b, hs][:, rows]), np64(dq[b, rows][:, hs])
    ref_dq, got_dq = [], []
    for g in range(G):
        r = oracle.attn_rows(Q, K, V, dO, causal, 0, g, rows)
        assert np.abs(o_np[:, g] - r["O"]).max() <= TOL_MAXABS
        assert np.abs(lse_np[g] - r["LSE"]).max() <= TOL_MAXABS
        ref_dq.append(r["dQ"])
        got_dq.append(dq_np[:, g])
    assert rel_l2(np.stack(got_dq), np.stack(ref_dq)) <= TOL_RELL2
    if check_keys:
        keys = sample_rows(N, 32, seed=N + 1)
        LSE = np.empty((1, G, N))
        Dv = np.empty((1, G, N))
        for g in range(G):
            LSE[0, g], Dv[0, g] = _oracle_lse_d(Q, K, V, dO, causal, 0, g, N)
        kr = oracle.attn_key_rows(Q, K, V, dO, causal, 0, 0, keys, LSE, Dv)
        assert rel_l2(np64(dk[b, keys, kvh]), kr["dK"]) <= TOL_RELL2
        assert rel_l2(np64(dv[b, keys, kvh]), kr["dV"]) <= TOL_RELL2


def test_causal_future_perturbation_bitwise():
    """Changing K, V at keys > i must leave O_i, LSE_i bitwise unchanged."""
    from paper_2511_08083_b200 import attn_fwd
    B, N, Hq, Hkv, d = 2, 1024, 8, 2, 128
    x = gen(B, N, Hq, Hkv, d, seed=5)
    o1, l1 = attn_fwd(x["Q"], x["K"], x["V"], True)
    cut = 517
    k2, v2 = x["K"].clone(), x["V"].clone()
    k2[:, cut + 1:] = torch.randn_like(k2[:, cut + 1:].float()).to(k2.dtype)
    v2[:, cut + 1:] = 0
    o2, l2 = attn_fwd(x["Q"], k2, v2, True)
    torch.cuda.synchronize()
    assert torch.equal(o1[:, :cut + 1], o2[:, :cut + 1])
    assert torch.equal(l1[:, :, :cut + 1], l2[:, :, :cut + 1])
    assert not torch.equal(o1[:, cut + 1:], o2[:, cut + 1:])
