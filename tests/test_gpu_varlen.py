"""Parity of the sequence-length variants through the C ABI:
Nq != Nk with the bottom-right causal mask (hk_attn_fwd_qk / hk_attn_bwd_qk) and
packed variable-length batches (hk_attn_fwd_varlen / hk_attn_bwd_varlen), vs the
fp64 oracle on the same bf16 inputs at the BASELINE tolerances (max-abs 2e-2 on
O and LSE, relative L2 1e-2 on dQ, dK, dV). Rows that see no key must come
back exactly as O = 0, LSE = -inf, dQ = 0 (reading #22)."""
import numpy as np
import pytest
import torch

import oracle
from util import TOL_MAXABS, TOL_RELL2, np64, rel_l2

pytestmark = pytest.mark.gpu


def grad_err(got, ref, n_terms=2):
    """Relative L2, or — for an identically zero exact gradient (one visible key:
    dS = P (dP - D) = 0) — max-abs against the rounding-noise bound of DESIGN.md
    reading #16: each of the n_terms (query, head) pairs summed into one output
    row adds an independent ~2^-9 |dO.V| residue (bf16 P inside O vs fp32 l), so
    the bound 2 x TOL_MAXABS of the single-pair case grows like sqrt(n_terms / 2).
    Returned scaled into the rel-L2 slot so one threshold applies."""
    if np.linalg.norm(ref) < 1e-9 * np.sqrt(max(ref.size, 1)):
        bound = 2 * TOL_MAXABS * np.sqrt(max(n_terms, 2) / 2)
        return float(np.abs(got).max(initial=0.0)) * (TOL_RELL2 / bound)
    return rel_l2(got, ref)


def check_fwd(o, lse, ref_o, ref_lse):
    dead = np.isneginf(ref_lse)
    assert np.array_equal(np.isneginf(lse), dead), "key-less rows must have LSE = -inf, and only those"
    live = ~dead
    assert np.abs(lse[live] - ref_lse[live]).max(initial=0.0) <= TOL_MAXABS
    assert np.abs(o - ref_o).max(initial=0.0) <= TOL_MAXABS
    return dead


QK_CASES = [
    # B, Nq, Nk, Hq, Hkv, d
    (1, 128, 384, 4, 2, 128),
    (2, 384, 128, 4, 2, 64),    # Nq > Nk: the first Nq - Nk rows see no key when causal
    (1, 77, 300, 2, 1, 128),    # ragged both
    (1, 300, 77, 2, 2, 64),
    (2, 1, 257, 4, 1, 128),     # one query (decode-like)
    (1, 256, 1, 2, 1, 64),      # one key
    (1, 200, 520, 8, 1, 128),   # G = 8, offsets not multiples of 128
]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("case", QK_CASES)
def test_qk_parity(case, causal):
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    from paper_2511_08083_b200.inputs import make_qk_inputs
    B, Nq, Nk, Hq, Hkv, d = case
    x = make_qk_inputs(B, Nq, Nk, Hq, Hkv, d, seed=3, device="cuda")
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
    torch.cuda.synchronize()
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), causal)
    dead = check_fwd(np64(o), np64(lse), ref["O"], ref["LSE"])
    if dead.any():  # key-less rows: exactly zero output and gradient
        rows = dead.any(axis=(0, 1))
        assert np.all(np64(o)[:, rows] == 0) and np.all(np64(dq)[:, rows] == 0)
    for n, t in (("dQ", dq), ("dK", dk), ("dV", dv)):
        e = grad_err(np64(t), ref[n], 2 if n == "dQ" else Nq * (Hq // Hkv))
        assert e <= TOL_RELL2, (n, e)


VARLEN_CASES = [
    # lens_q, lens_k, Hq, Hkv, d
    ([128, 256, 384], [128, 256, 384], 4, 2, 128),          # whole tiles, Nq == Nk per sequence
    ([77, 300, 1, 129], [77, 300, 1, 129], 2, 1, 64),        # ragged, equal lengths
    ([100, 0, 260, 33], [50, 70, 0, 400], 4, 4, 128),        # zero-length sequences, Nq != Nk
    ([500, 17, 130], [260, 300, 130], 8, 2, 64),
    ([1, 1, 1, 1, 1], [300, 5, 129, 1, 64], 4, 1, 128),      # decode-like batch
]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("case", VARLEN_CASES)
def test_varlen_parity(case, causal):
    from paper_2511_08083_b200 import attn_bwd_varlen, attn_fwd_varlen
    from paper_2511_08083_b200.inputs import make_varlen_inputs
    lq, lk, Hq, Hkv, d = case
    x = make_varlen_inputs(lq, lk, Hq, Hkv, d, seed=5, device="cuda")
    mq, mk = max(lq), max(lk)
    o, lse = attn_fwd_varlen(x["Q"], x["K"], x["V"], x["cu_q"], x["cu_k"], mq, mk, causal)
    dq, dk, dv = attn_bwd_varlen(x["Q"], x["K"], x["V"], o, lse, x["dO"], x["cu_q"], x["cu_k"], mq, mk, causal)
    torch.cuda.synchronize()
    ref = oracle.attn_varlen_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]),
                                     x["cu_q"].cpu().numpy(), x["cu_k"].cpu().numpy(), causal)
    dead = check_fwd(np64(o), np64(lse), ref["O"], ref["LSE"])
    rows = dead.any(axis=0)
    assert np.all(np64(dq)[rows] == 0)
    for n, t in (("dQ", dq), ("dK", dk), ("dV", dv)):
        e = grad_err(np64(t), ref[n], 2 if n == "dQ" else mq * (Hq // Hkv))
        assert e <= TOL_RELL2, (n, e)
    # keys of a sequence with no queries: dK = dV = 0 exactly
    cu_q, cu_k = x["cu_q"].tolist(), x["cu_k"].tolist()
    for b in range(len(lq)):
        if lq[b] == 0:
            assert torch.all(dk[cu_k[b]:cu_k[b + 1]] == 0) and torch.all(dv[cu_k[b]:cu_k[b + 1]] == 0)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(256, 128), (333, 64)])
def test_varlen_uniform_equals_dense_bitwise(N, d, causal):
    """A packed batch of equal-length sequences runs the same arithmetic as the
    dense call on the same data: results must be bitwise equal."""
    from paper_2511_08083_b200 import attn_bwd, attn_bwd_varlen, attn_fwd, attn_fwd_varlen
    from paper_2511_08083_b200.inputs import make_inputs
    B, Hq, Hkv = 3, 4, 2
    x = make_inputs(B, N, Hq, Hkv, d, seed=9, device="cuda")
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    # the plain workspace: the two-pass backward the varlen entry runs (without one, a dense d = 128
    # call takes the stored-dS path, whose dQ rounds dS from S^T: reading #29)
    from paper_2511_08083_b200 import bwd_workspace_bytes
    ws = torch.empty(bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4, dtype=torch.float32, device="cuda")
    dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, deterministic=True, workspace=ws)
    cu = torch.arange(0, (B + 1) * N, N, dtype=torch.int32, device="cuda")
    flat = lambda t: t.reshape(B * N, t.shape[2], d)
    ov, lv = attn_fwd_varlen(flat(x["Q"]), flat(x["K"]), flat(x["V"]), cu, cu, N, N, causal)
    dqv, dkv, dvv = attn_bwd_varlen(flat(x["Q"]), flat(x["K"]), flat(x["V"]), ov, lv, flat(x["dO"]), cu, cu, N, N,
                                    causal, deterministic=True)
    torch.cuda.synchronize()
    assert torch.equal(ov, flat(o))
    assert torch.equal(lv, lse.permute(1, 0, 2).reshape(Hq, B * N))
    for a, b in ((dqv, dq), (dkv, dk), (dvv, dv)):
        assert torch.equal(a, flat(b))


def test_qk_full_size_sampled():
    """A long-context shape (Nq = 1024 queries against Nk = 16384 keys, the
    chunked-prefill / ring-step shape) checked on sampled rows (ROW mode)."""
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    from paper_2511_08083_b200.inputs import make_qk_inputs
    B, Nq, Nk, Hq, Hkv, d = 2, 1024, 16384, 8, 2, 128
    x = make_qk_inputs(B, Nq, Nk, Hq, Hkv, d, seed=13, device="cuda")
    for causal in (False, True):
        o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
        dq, _, _ = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
        torch.cuda.synchronize()
        Q, K, V, dO = (np64(x[n]) for n in ("Q", "K", "V", "dO"))
        rows = [0, 1, 127, 128, 511, 1000, 1023]
        for b, h in ((0, 0), (1, 7)):
            r = oracle.attn_rows(Q, K, V, dO, causal, b, h, rows)
            assert np.abs(np64(o)[b, rows, h] - r["O"]).max() <= TOL_MAXABS
            assert np.abs(np64(lse)[b, h, rows] - r["LSE"]).max() <= TOL_MAXABS
            assert rel_l2(np64(dq)[b, rows, h], r["dQ"]) <= TOL_RELL2


def test_varlen_full_size_sampled():
    """The packed-document workload scripts/bench_varlen.py times (C3 heads, 131072
    tokens, document lengths uniform in [1, 16383]) checked per document on
    sampled query rows (O, LSE, dQ) and key rows (dK, dV) against the oracle run
    on that document alone, plus the any-size invariants per document and KV head:
    sum_j dK_j = 0 and sum_j dV_j = sum over the group's heads and rows of dO."""
    from paper_2511_08083_b200 import attn_bwd_varlen, attn_fwd_varlen
    from paper_2511_08083_b200.inputs import make_varlen_inputs, sample_rows, varlen_lengths
    Hq, Hkv, d, causal, total = 32, 8, 128, True, 16 * 8192
    lens, s = [], 0
    for L in varlen_lengths(64, 8192, seed=7):
        L = min(L, total - s)
        lens.append(L)
        s += L
        if s == total:
            break
    x = make_varlen_inputs(lens, lens, Hq, Hkv, d, seed=1, device="cuda")
    mx = max(lens)
    o, lse = attn_fwd_varlen(x["Q"], x["K"], x["V"], x["cu_q"], x["cu_k"], mx, mx, causal)
    dq, dk, dv = attn_bwd_varlen(x["Q"], x["K"], x["V"], o, lse, x["dO"], x["cu_q"], x["cu_k"], mx, mx, causal)
    torch.cuda.synchronize()
    cu = x["cu_q"].tolist()
    G = Hq // Hkv
    for b in (0, len(lens) // 2, len(lens) - 1):
        a, e = cu[b], cu[b + 1]
        n = e - a
        Q, K, V, dO = (np64(x[k][a:e])[None] for k in ("Q", "K", "V", "dO"))
        # ROW mode: 256 rows — first/last 8, tile edges, random. Relative L2 is
        # over the sample (reading #16); per-row errors are a logged diagnostic (reading #24: rows
        # with few visible keys carry the D-from-bf16-O residue of reading #11).
        rows = sample_rows(n, 256, seed=b)
        kvh = 3
        for h in (kvh * G, kvh * G + G - 1):
            r = oracle.attn_rows(Q, K, V, dO, causal, 0, h, rows)
            assert np.abs(np64(o)[a:e][rows, h] - r["O"]).max() <= TOL_MAXABS
            assert np.abs(np64(lse)[h, a:e][rows] - r["LSE"]).max() <= TOL_MAXABS
            got = np64(dq)[a:e][rows, h]
            row_rel = np.linalg.norm(got - r["dQ"], axis=1) / np.maximum(np.linalg.norm(r["dQ"], axis=1), 1e-30)
            worst = np.argsort(row_rel)[::-1][:3]
            print({"doc": b, "len": n, "head": h, "dQ_rel_l2": rel_l2(got, r["dQ"]),
                   "worst_rows_dQ_rel": [[int(rows[i]), float(row_rel[i])] for i in worst]})
            assert rel_l2(got, r["dQ"]) <= TOL_RELL2
        LSEf = np.zeros((1, Hq, n))
        Df = np.zeros((1, Hq, n))
        for h in range(kvh * G, kvh * G + G):
            rr = oracle.attn_rows(Q, K, V, dO, causal, 0, h, np.arange(n))
            LSEf[0, h], Df[0, h] = rr["LSE"], rr["D"]
        kr = oracle.attn_key_rows(Q, K, V, dO, causal, 0, kvh, rows, LSEf, Df)
        assert rel_l2(np64(dk)[a:e][rows, kvh], kr["dK"]) <= TOL_RELL2
        assert rel_l2(np64(dv)[a:e][rows, kvh], kr["dV"]) <= TOL_RELL2
        sdk = dk[a:e].float().sum(dim=0)
        sdv = dv[a:e].float().sum(dim=0)
        want = x["dO"][a:e].float().reshape(n, Hkv, G, d).sum(dim=(0, 2))
        assert float(sdk.abs().max()) <= 0.05 * float(dk[a:e].float().abs().max()) * np.sqrt(n) / 8 + 1e-3
        assert torch.allclose(sdv, want, rtol=2e-2, atol=0.05 * np.sqrt(n))


@pytest.mark.parametrize("causal", [False, True])
def test_varlen_dynamic_schedule_equals_static_bitwise(causal):
    """The forward's dynamic scheduler (workspace counter) changes only which CTA takes
    which item: O and LSE must be bitwise those of the static order, across repeats."""
    from paper_2511_08083_b200 import attn_fwd_varlen
    from paper_2511_08083_b200.inputs import make_varlen_inputs
    lens = [900, 3, 0, 2049, 640, 1, 1500]
    x = make_varlen_inputs(lens, lens, 8, 2, 128, seed=21, device="cuda")
    args = (x["Q"], x["K"], x["V"], x["cu_q"], x["cu_k"], max(lens), max(lens), causal)
    o0, l0 = attn_fwd_varlen(*args, dynamic=False)
    ws = torch.empty(64, dtype=torch.int32, device="cuda")
    for _ in range(3):
        o1, l1 = attn_fwd_varlen(*args, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(o0, o1) and torch.equal(l0, l1)


def test_varlen_lengths_beyond_max_seqlen_are_clamped():
    """a sequence longer than max_seqlen (a broken offset contract) must not write
    past the padded workspace; per hk_attn.h its lengths are clamped to max_seqlen, so its
    first max_seqlen rows equal the oracle on the truncated sequence and the others are exact."""
    from paper_2511_08083_b200 import attn_bwd_varlen, attn_fwd_varlen
    from paper_2511_08083_b200.inputs import make_varlen_inputs
    lens = [300, 130, 64]
    mx = 256  # < lens[0]
    Hq, Hkv, d = 4, 2, 64
    v = make_varlen_inputs(lens, lens, Hq, Hkv, d, seed=7, device="cuda")
    tq = sum(lens)
    o = torch.zeros_like(v["Q"])
    lse = torch.zeros((Hq, tq), dtype=torch.float32, device="cuda")
    o, lse = attn_fwd_varlen(v["Q"], v["K"], v["V"], v["cu_q"], v["cu_k"], mx, mx, True, out=o, lse=lse)
    from paper_2511_08083_b200 import _lib
    nbytes = int(_lib.lib().hk_attn_bwd_varlen_workspace_bytes(len(lens), Hq, Hkv, mx, mx, d))
    ws_and_guard = torch.full((nbytes // 4 + 4096,), 7.0, dtype=torch.float32, device="cuda")
    dq = torch.zeros_like(v["Q"]); dk = torch.zeros_like(v["K"]); dv = torch.zeros_like(v["V"])
    attn_bwd_varlen(v["Q"], v["K"], v["V"], o, lse, v["dO"], v["cu_q"], v["cu_k"], mx, mx, True,
                    workspace=ws_and_guard[: nbytes // 4], dq=dq, dk=dk, dv=dv)
    torch.cuda.synchronize()
    assert torch.all(ws_and_guard[nbytes // 4:] == 7.0), "backward wrote past its workspace"
    cut = [min(n, mx) for n in lens]
    offs = np.concatenate([[0], np.cumsum(lens)])
    for b, n in enumerate(cut):
        s0 = offs[b]
        sl = slice(s0, s0 + n)
        ref = oracle.attn_fwd_bwd(np64(v["Q"][sl])[None], np64(v["K"][sl])[None], np64(v["V"][sl])[None],
                                  np64(v["dO"][sl])[None], True)
        assert np.abs(np64(o[sl]) - ref["O"][0]).max() <= TOL_MAXABS
        assert np.abs(np64(lse[:, sl]) - ref["LSE"][0]).max() <= TOL_MAXABS
        for nm, t in (("dQ", dq), ("dK", dk), ("dV", dv)):
            assert rel_l2(np64(t[sl]), ref[nm][0]) <= TOL_RELL2, (b, nm)
        if lens[b] > n:  # rows beyond max_seqlen are left untouched
            tail = slice(s0 + n, s0 + lens[b])
            assert torch.all(dq[tail] == 0) and torch.all(dk[tail] == 0)
