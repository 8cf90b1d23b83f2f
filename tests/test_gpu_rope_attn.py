"""Rotary fused into the attention forward (hk_attn_fwd_rope): bitwise equal to
hk_rope on Q and K followed by hk_attn_fwd, and the whole chain (rotary -> attention -> gradients
mapped back through the inverse rotation) against the fp64 oracle at the BASELINE tolerances."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_08083_b200.inputs import make_inputs
from util import TOL_MAXABS, TOL_RELL2, np64, rel_l2

pytestmark = pytest.mark.gpu

CASES = [  # B, N, Hq, Hkv, d
    (2, 384, 4, 2, 128),
    (1, 200, 8, 1, 64),     # ragged last tile, G = 8
    (2, 256, 4, 4, 64),
    (1, 1024, 8, 2, 128),
]


def tables(N, d):
    c, s = oracle.rope_tables(N, d)
    return c.astype(np.float32), s.astype(np.float32)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("case", CASES)
def test_fwd_rope_bitwise_equals_unfused(case, causal):
    from paper_2511_08083_b200 import attn_fwd, attn_fwd_rope, rope
    B, N, Hq, Hkv, d = case
    x = make_inputs(B, N, Hq, Hkv, d, seed=N + d, device="cuda")
    cf, sf = tables(N, d)
    c, s = torch.from_numpy(cf).cuda(), torch.from_numpy(sf).cuda()
    o, lse, kr = attn_fwd_rope(x["Q"], x["K"], x["V"], c, s, causal)
    qr2, kr2 = rope(x["Q"], c, s), rope(x["K"], c, s)
    o2, lse2 = attn_fwd(qr2, kr2, x["V"], causal)
    torch.cuda.synchronize()
    assert torch.equal(kr, kr2)
    assert torch.equal(o, o2) and torch.equal(lse, lse2)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("case", CASES[:3])
def test_rope_attention_parity(case, causal):
    """O, LSE and the gradients w.r.t. the unrotated q, k, v (autograd AttentionRope) vs the oracle:
    rope (fp64) -> attention fwd/bwd -> dQ, dK mapped back through rope(., cos, -sin)."""
    from paper_2511_08083_b200 import AttentionRope, attn_fwd_rope
    B, N, Hq, Hkv, d = case
    x = make_inputs(B, N, Hq, Hkv, d, seed=3 * N + d, device="cuda")
    cf, sf = tables(N, d)
    c, s = torch.from_numpy(cf).cuda(), torch.from_numpy(sf).cuda()
    q, k, v = (x[n].clone().requires_grad_() for n in ("Q", "K", "V"))
    o = AttentionRope.apply(q, k, v, c, s, causal)
    o.backward(x["dO"])
    _, lse, _ = attn_fwd_rope(x["Q"], x["K"], x["V"], c, s, causal)
    torch.cuda.synchronize()
    Q, K, V, dO = np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"])
    ref = oracle.attn_fwd_bwd(oracle.rope(Q, cf, sf), oracle.rope(K, cf, sf), V, dO, causal)
    assert np.abs(np64(o) - ref["O"]).max() <= TOL_MAXABS
    assert np.abs(np64(lse) - ref["LSE"]).max() <= TOL_MAXABS
    want = {"dQ": oracle.rope(ref["dQ"], cf, -sf), "dK": oracle.rope(ref["dK"], cf, -sf), "dV": ref["dV"]}
    for n, t in (("dQ", q.grad), ("dK", k.grad), ("dV", v.grad)):
        assert rel_l2(np64(t), want[n]) <= TOL_RELL2, n
