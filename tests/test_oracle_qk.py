"""Pins for the oracle's sequence-length variants:
Nq != Nk with bottom-right-aligned causal masking, rows that see no key, and
packed variable-length batches (reading #22). Every check is against
something other than the code under test: the triple-loop brute force, the
square (Nq == Nk) oracle already pinned in test_oracle.py via exact
suffix / prefix identities, closed forms, finite differences, and torch SDPA
in fp64 with an explicit boolean mask."""
import math

import numpy as np
import pytest

from oracle import attn_fwd, attn_fwd_bwd, attn_naive, attn_varlen_fwd_bwd, attn_rows, attn_key_rows

OUTS = ("O", "LSE", "D", "dQ", "dK", "dV")


def rand(shape, seed, std=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * std


def qk_problem(B, Nq, Nk, Hq, Hkv, d, seed=0):
    return (rand((B, Nq, Hq, d), seed), rand((B, Nk, Hkv, d), seed + 1),
            rand((B, Nk, Hkv, d), seed + 2), rand((B, Nq, Hq, d), seed + 3))


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("Nq,Nk", [(3, 7), (7, 3), (1, 5), (5, 1), (6, 6)])
def test_naive_matches_blocked_qk(causal, Nq, Nk):
    Q, K, V, dO = qk_problem(2, Nq, Nk, 4, 2, 5, seed=3)
    a = attn_naive(Q, K, V, dO, causal)
    b = attn_fwd_bwd(Q, K, V, dO, causal)
    for k in OUTS:
        np.testing.assert_allclose(b[k], a[k], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("Nq,Nk", [(5, 12), (12, 12), (1, 9)])
def test_bottom_right_is_suffix_of_square(Nq, Nk):
    """Nq <= Nk: causal attention of the last Nq queries of an Nk x Nk causal
    problem, whatever the first Nk - Nq query rows hold. With dO = 0 on those
    prefix rows the square problem's dK, dV equal the Nq x Nk ones."""
    Q, K, V, dO = qk_problem(1, Nq, Nk, 2, 1, 8, seed=7)
    pre = rand((1, Nk - Nq, 2, 8), 99)
    Qs = np.concatenate([pre, Q], axis=1)
    dOs = np.concatenate([np.zeros_like(pre), dO], axis=1)
    sq = attn_fwd_bwd(Qs, K, V, dOs, True)
    r = attn_fwd_bwd(Q, K, V, dO, True)
    np.testing.assert_allclose(r["O"], sq["O"][:, Nk - Nq:], atol=1e-13)
    np.testing.assert_allclose(r["LSE"], sq["LSE"][:, :, Nk - Nq:], atol=1e-13)
    np.testing.assert_allclose(r["dQ"], sq["dQ"][:, Nk - Nq:], atol=1e-13)
    np.testing.assert_allclose(r["dK"], sq["dK"], atol=1e-12)
    np.testing.assert_allclose(r["dV"], sq["dV"], atol=1e-12)


def test_more_queries_than_keys():
    """Nq > Nk: rows i < Nq - Nk see no key (O = 0, LSE = -inf, dQ = 0); the
    last Nk rows are the square Nk x Nk causal problem."""
    Nq, Nk = 11, 4
    Q, K, V, dO = qk_problem(1, Nq, Nk, 2, 2, 8, seed=17)
    r = attn_fwd_bwd(Q, K, V, dO, True)
    e = Nq - Nk
    assert np.all(r["O"][:, :e] == 0) and np.all(r["dQ"][:, :e] == 0) and np.all(r["D"][:, :, :e] == 0)
    assert np.all(np.isneginf(r["LSE"][:, :, :e]))
    sq = attn_fwd_bwd(Q[:, e:], K, V, dO[:, e:], True)
    for k in ("O", "dQ"):
        np.testing.assert_allclose(r[k][:, e:], sq[k], atol=1e-13)
    for k in ("LSE", "D"):
        np.testing.assert_allclose(r[k][:, :, e:], sq[k], atol=1e-13)
    for k in ("dK", "dV"):
        np.testing.assert_allclose(r[k], sq[k], atol=1e-13)
    O, L = attn_fwd(Q, K, V, True)
    np.testing.assert_allclose(O, r["O"], atol=1e-13)
    np.testing.assert_array_equal(np.isneginf(L), np.isneginf(r["LSE"]))


def test_single_query_sees_all_keys():
    """Nq = 1, causal: the only query is the last row, which sees every key,
    so the result equals the non-causal one; the last row of any Nq <= Nk
    causal problem likewise equals its non-causal row."""
    Q, K, V, dO = qk_problem(2, 1, 9, 2, 1, 4, seed=23)
    a, b = attn_fwd_bwd(Q, K, V, dO, True), attn_fwd_bwd(Q, K, V, dO, False)
    for k in OUTS:
        np.testing.assert_allclose(a[k], b[k], atol=1e-14)
    Q, K, V, dO = qk_problem(1, 4, 9, 2, 1, 4, seed=29)
    a, b = attn_fwd_bwd(Q, K, V, dO, True), attn_fwd_bwd(Q, K, V, dO, False)
    np.testing.assert_allclose(a["O"][:, -1], b["O"][:, -1], atol=1e-14)


def test_q_zero_closed_form_qk():
    """Q = 0, causal, Nq < Nk: row i sees keys 0..i+Nk-Nq, O_i = their mean V,
    LSE_i = ln(i + Nk - Nq + 1)."""
    Nq, Nk, d = 3, 8, 4
    _, K, V, _ = qk_problem(1, Nq, Nk, 1, 1, d, seed=31)
    O, L = attn_fwd(np.zeros((1, Nq, 1, d)), K, V, True)
    for i in range(Nq):
        n = i + Nk - Nq + 1
        np.testing.assert_allclose(O[0, i, 0], V[0, :n, 0].mean(axis=0), atol=1e-14)
        assert abs(L[0, 0, i] - math.log(n)) < 1e-14


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("Nq,Nk", [(2, 5), (5, 2)])
def test_finite_differences_qk(causal, Nq, Nk):
    Q, K, V, dO = qk_problem(1, Nq, Nk, 2, 1, 4, seed=41)
    r = attn_fwd_bwd(Q, K, V, dO, causal)
    loss = lambda q, k, v: (attn_fwd(q, k, v, causal)[0] * dO).sum()
    eps = 1e-6
    for name, X, idx in (("dQ", Q, 0), ("dK", K, 1), ("dV", V, 2)):
        g = np.zeros_like(X)
        for pos in np.ndindex(*X.shape):
            args = [Q, K, V]
            Xp, Xm = X.copy(), X.copy()
            Xp[pos] += eps
            Xm[pos] -= eps
            args[idx] = Xp
            fp = loss(*args)
            args[idx] = Xm
            fm = loss(*args)
            g[pos] = (fp - fm) / (2 * eps)
        np.testing.assert_allclose(r[name], g, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("Nq,Nk", [(40, 100), (100, 40), (1, 33)])
def test_matches_torch_sdpa_bottom_right(Nq, Nk):
    """torch SDPA (fp64, CPU, autograd) with a boolean attn_mask: for Nq <= Nk
    the mask is torch's own lower-triangular matrix shifted by Nk - Nq via
    torch.ones(...).tril(diagonal=Nk - Nq); rows that see nothing (Nq > Nk) are
    compared on the rows that do."""
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    B, Hq, Hkv, d = 2, 4, 2, 16
    Q, K, V, dO = qk_problem(B, Nq, Nk, Hq, Hkv, d, seed=51)
    G = Hq // Hkv
    mask = torch.ones(Nq, Nk, dtype=torch.bool).tril(diagonal=Nk - Nq)
    live = mask.any(dim=1).numpy()
    q = torch.tensor(Q).permute(0, 2, 1, 3).requires_grad_()
    k = torch.tensor(K).permute(0, 2, 1, 3).requires_grad_()
    v = torch.tensor(V).permute(0, 2, 1, 3).requires_grad_()
    m = mask.clone()
    m[~mask.any(dim=1)] = True  # SDPA needs a key per row; those rows are excluded below
    o = F.scaled_dot_product_attention(q, k.repeat_interleave(G, 1), v.repeat_interleave(G, 1), attn_mask=m)
    go = torch.tensor(dO).permute(0, 2, 1, 3) * torch.tensor(live, dtype=torch.float64)[None, None, :, None]
    o.backward(go)
    r = attn_fwd_bwd(Q, K, V, dO, True)
    perm = lambda t: t.detach().permute(0, 2, 1, 3).numpy()
    np.testing.assert_allclose(r["O"][:, live], perm(o)[:, live], atol=1e-10)
    np.testing.assert_allclose(r["dQ"][:, live], perm(q.grad)[:, live], atol=1e-10)
    np.testing.assert_allclose(r["dK"], perm(k.grad), atol=1e-10)
    np.testing.assert_allclose(r["dV"], perm(v.grad), atol=1e-10)


def test_row_samplers_qk():
    """attn_rows / attn_key_rows at Nq != Nk equal the full computation."""
    for Nq, Nk in ((20, 50), (50, 20)):
        Q, K, V, dO = qk_problem(1, Nq, Nk, 4, 2, 8, seed=61)
        full = attn_fwd_bwd(Q, K, V, dO, True)
        rows = [0, Nq // 2, Nq - 1]
        r = attn_rows(Q, K, V, dO, True, 0, 3, rows)
        np.testing.assert_allclose(r["O"], full["O"][0, rows, 3], atol=1e-12)
        np.testing.assert_allclose(r["LSE"], full["LSE"][0, 3, rows], atol=1e-12)
        np.testing.assert_allclose(r["dQ"], full["dQ"][0, rows, 3], atol=1e-12)
        keys = [0, Nk // 2, Nk - 1]
        kr = attn_key_rows(Q, K, V, dO, True, 0, 1, keys, full["LSE"], full["D"])
        np.testing.assert_allclose(kr["dK"], full["dK"][0, keys, 1], atol=1e-11)
        np.testing.assert_allclose(kr["dV"], full["dV"][0, keys, 1], atol=1e-11)


@pytest.mark.parametrize("causal", [False, True])
def test_varlen_is_concatenation_of_dense(causal):
    """A packed batch equals independent dense problems on each sequence;
    zero-length query or key sequences give nothing / O = 0, LSE = -inf."""
    lq = [5, 0, 9, 3, 4]
    lk = [7, 4, 9, 0, 2]
    cu_q, cu_k = np.concatenate([[0], np.cumsum(lq)]), np.concatenate([[0], np.cumsum(lk)])
    Hq, Hkv, d = 4, 2, 8
    Q, K = rand((cu_q[-1], Hq, d), 1), rand((cu_k[-1], Hkv, d), 2)
    V, dO = rand((cu_k[-1], Hkv, d), 3), rand((cu_q[-1], Hq, d), 4)
    r = attn_varlen_fwd_bwd(Q, K, V, dO, cu_q, cu_k, causal)
    for b in range(len(lq)):
        qs, ks = slice(cu_q[b], cu_q[b + 1]), slice(cu_k[b], cu_k[b + 1])
        if lq[b] == 0:
            np.testing.assert_array_equal(r["dK"][ks], 0)
            np.testing.assert_array_equal(r["dV"][ks], 0)
            continue
        if lk[b] == 0:
            np.testing.assert_array_equal(r["O"][qs], 0)
            assert np.all(np.isneginf(r["LSE"][:, qs]))
            continue
        n = attn_naive(Q[None, qs], K[None, ks], V[None, ks], dO[None, qs], causal)
        for k in ("O", "dQ"):
            np.testing.assert_allclose(r[k][qs], n[k][0], atol=1e-12)
        for k in ("dK", "dV"):
            np.testing.assert_allclose(r[k][ks], n[k][0], atol=1e-12)
        for k in ("LSE", "D"):
            np.testing.assert_allclose(r[k][:, qs], n[k][0], atol=1e-12)


def test_varlen_rejects_bad_offsets():
    Q, K = rand((5, 2, 4), 1), rand((5, 2, 4), 2)
    with pytest.raises(ValueError):
        attn_varlen_fwd_bwd(Q, K, K, Q, [0, 3, 2, 5], [0, 1, 2, 5], False)
    with pytest.raises(ValueError):
        attn_varlen_fwd_bwd(Q, K, K, Q, [0, 4], [0, 5], False)
