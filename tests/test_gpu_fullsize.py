"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (B=16, all heads, one hk_attn_fwd + one hk_attn_bwd call), following the
sampling policy of SURVEY §8(c).5:

  * UNIT mode (C2, C3, C4 at every N, C5 N <= 8192): three seeded units —
    (0, 0), (B-1, Hkv-1) and one drawn from the seed — every element of O, LSE
    (max-abs 2e-2), dQ, dK, dV (relative L2 1e-2 per tensor over the unit), the
    oracle run on the whole unit (oracle.attn_fwd_bwd).
  * ROW mode (C5 N in {16384, 32768}): for the same three units the oracle's
    per-row outputs for EVERY query row of every head of the unit (O, LSE, D,
    dQ: oracle.attn_rows, so O/LSE/dQ are checked on all rows here too), then
    dK, dV on a 256-key-row sample J (first/last 8, tile edges, random:
    inputs.sample_rows) from the oracle's own LSE and D (oracle.attn_key_rows).

Every config also checks, on every unit, the properties that hold at any size
(SURVEY §8(c).4): sum_j dK_j = 0, sum_j dV_j = sum_{h in group} sum_i dO_i,
sum <Q, dQ> = sum <K, dK>, and bitwise run-to-run determinism of the backward.

Per-unit errors and the worst rows are reported as a diagnostic (§8(c).3 #16):
printed, and appended as JSON lines to $HK_PARITY_LOG when that is set.
The oracle work runs in a thread pool on the host's cores (numpy releases the
GIL in BLAS and ufuncs); the oracle itself is unchanged.
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
from paper_2511_08083_b200.inputs import sample_rows, splitmix64
from util import TOL_MAXABS, TOL_RELL2, gen, np64, rel_l2

pytestmark = pytest.mark.gpu

# every BASELINE.json config at full size: name -> B, N, Hq, Hkv, d, causal
CONFIGS = {
    "C2-nc": (16, 4096, 16, 16, 128, False),
    "C2-c": (16, 4096, 16, 16, 128, True),
    "C3": (16, 8192, 32, 8, 128, True),
}
for _n in (2048, 4096, 8192, 16384):
    CONFIGS[f"C4-{_n}"] = (16, _n, 32, 32, 64, True)
for _n in (1024, 2048, 4096, 8192, 16384, 32768):
    for _c in (False, True):
        CONFIGS[f"C5-{_n}-{'c' if _c else 'nc'}"] = (16, _n, 64, 8, 128, _c)

SEED = 101
CORES = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def mode_of(name):
    return "ROW" if name in ("C5-16384-nc", "C5-16384-c", "C5-32768-nc", "C5-32768-c") else "UNIT"


def sampled_units(B, Hkv, seed):
    """(0, 0), (B-1, Hkv-1) and one unit drawn from the seed."""
    u = splitmix64(seed, 77) % (B * Hkv)
    units = [(0, 0), (B - 1, Hkv - 1), (u // Hkv, u % Hkv)]
    return list(dict.fromkeys(units))


def _log(rec):
    print(json.dumps(rec))
    path = os.environ.get("HK_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _worst_rows(err_rows, rows, k=3, valid=None):
    """The k rows with the largest error: a per-row diagnostic, not a bound. `valid` masks out
    rows whose reference is ~0 (causal row 0: one visible key, dQ = 0 exactly), where a
    relative error is undefined."""
    e = np.where(valid, err_rows, -1.0) if valid is not None else err_rows
    idx = np.argsort(e)[::-1][:k]
    return [[int(rows[i]), float(err_rows[i])] for i in idx]


def _blas_threads(n):
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=max(1, n), user_api="blas")


def _unit_inputs(x, b, kvh, G):
    hs = slice(kvh * G, (kvh + 1) * G)
    Q, dO = np64(x["Q"][b:b + 1, :, hs]), np64(x["dO"][b:b + 1, :, hs])
    K, V = np64(x["K"][b:b + 1, :, kvh:kvh + 1]), np64(x["V"][b:b + 1, :, kvh:kvh + 1])
    return Q, K, V, dO


def check_unit_mode(name, x, outs, units, G, causal):
    """All elements of each sampled unit against oracle.attn_fwd_bwd on that unit."""
    o, lse, dq, dk, dv = outs
    ins = [_unit_inputs(x, b, kvh, G) for b, kvh in units]
    with _blas_threads(CORES // len(units)):
        with ThreadPoolExecutor(len(units)) as ex:
            refs = list(ex.map(lambda a: oracle.attn_fwd_bwd(*a, causal), ins))
    failures = []
    for (b, kvh), ref in zip(units, refs):
        hs = slice(kvh * G, (kvh + 1) * G)
        got = {"O": np64(o[b:b + 1, :, hs]), "LSE": np64(lse[b:b + 1, hs]), "dQ": np64(dq[b:b + 1, :, hs]),
               "dK": np64(dk[b:b + 1, :, kvh:kvh + 1]), "dV": np64(dv[b:b + 1, :, kvh:kvh + 1])}
        e_o = np.abs(got["O"] - ref["O"])
        rec = {"config": name, "mode": "UNIT", "unit": [b, kvh],
               "O_maxabs": float(e_o.max()), "LSE_maxabs": float(np.abs(got["LSE"] - ref["LSE"]).max()),
               "dQ_rel_l2": rel_l2(got["dQ"], ref["dQ"]), "dK_rel_l2": rel_l2(got["dK"], ref["dK"]),
               "dV_rel_l2": rel_l2(got["dV"], ref["dV"])}
        # per-row diagnostics: O max-abs and dQ relative error of the worst query rows
        rows = np.arange(e_o.shape[1])
        rn = np.linalg.norm(ref["dQ"][0], axis=(1, 2))
        dq_row = np.linalg.norm((got["dQ"] - ref["dQ"])[0], axis=(1, 2)) / np.maximum(rn, 1e-30)
        rec["worst_rows_O"] = _worst_rows(e_o[0].max(axis=(1, 2)), rows)
        rec["worst_rows_dQ_rel"] = _worst_rows(dq_row, rows, valid=rn > 1e-6 * rn.max())
        _log(rec)
        if rec["O_maxabs"] > TOL_MAXABS or rec["LSE_maxabs"] > TOL_MAXABS:
            failures.append(rec)
        if max(rec["dQ_rel_l2"], rec["dK_rel_l2"], rec["dV_rel_l2"]) > TOL_RELL2:
            failures.append(rec)
    assert not failures, failures


def check_row_mode(name, x, outs, units, G, causal, N):
    """Every query row of each sampled unit via oracle.attn_rows (O, LSE, D, dQ), then dK/dV
    on 256 sampled key rows from the oracle's own LSE and D (oracle.attn_key_rows)."""
    o, lse, dq, dk, dv = outs
    block = 256  # query rows per oracle call: bounds each worker's fp64 temporaries to ~5 x 256 x N
    failures = []
    with _blas_threads(1):
        for b, kvh in units:
            Q, K, V, dO = _unit_inputs(x, b, kvh, G)
            jobs = [(g, r0) for g in range(G) for r0 in range(0, N, block)]
            with ThreadPoolExecutor(CORES) as ex:
                res = list(ex.map(lambda j: oracle.attn_rows(Q, K, V, dO, causal, 0, j[0],
                                                             np.arange(j[1], min(N, j[1] + block))), jobs))
            ref = {k: np.empty((G, N) + ((Q.shape[3],) if k in ("O", "dQ") else ())) for k in ("O", "LSE", "D", "dQ")}
            for (g, r0), r in zip(jobs, res):
                for k in ref:
                    ref[k][g, r0:r0 + block] = r[k]
            hs = slice(kvh * G, (kvh + 1) * G)
            go = np64(o[b, :, hs]).transpose(1, 0, 2)   # [G, N, d]
            gdq = np64(dq[b, :, hs]).transpose(1, 0, 2)
            gl = np64(lse[b, hs])
            keys = sample_rows(N, 256, seed=SEED + b * 131 + kvh)
            kparts = [keys[i::CORES] for i in range(CORES) if keys[i::CORES]]
            with ThreadPoolExecutor(len(kparts)) as ex:
                kres = list(ex.map(lambda ks: oracle.attn_key_rows(Q, K, V, dO, causal, 0, 0, ks, ref["LSE"][None],
                                                                   ref["D"][None]), kparts))
            rdk = np.empty((len(keys), Q.shape[3]))
            rdv = np.empty_like(rdk)
            pos = {k: i for i, k in enumerate(keys)}
            for ks, r in zip(kparts, kres):
                for i, k in enumerate(ks):
                    rdk[pos[k]], rdv[pos[k]] = r["dK"][i], r["dV"][i]
            e_o = np.abs(go - ref["O"])
            rec = {"config": name, "mode": "ROW", "unit": [b, kvh], "query_rows": "all", "key_rows": len(keys),
                   "O_maxabs": float(e_o.max()), "LSE_maxabs": float(np.abs(gl - ref["LSE"]).max()),
                   "dQ_rel_l2": rel_l2(gdq, ref["dQ"]),
                   "dK_rel_l2": rel_l2(np64(dk[b, keys, kvh]), rdk), "dV_rel_l2": rel_l2(np64(dv[b, keys, kvh]), rdv)}
            rows = np.arange(N)
            rec["worst_rows_O"] = _worst_rows(e_o.max(axis=(0, 2)), rows)
            rn = np.linalg.norm(ref["dQ"], axis=(0, 2))
            dq_row = np.linalg.norm(gdq - ref["dQ"], axis=(0, 2)) / np.maximum(rn, 1e-30)
            rec["worst_rows_dQ_rel"] = _worst_rows(dq_row, rows, valid=rn > 1e-6 * rn.max())
            _log(rec)
            if rec["O_maxabs"] > TOL_MAXABS or rec["LSE_maxabs"] > TOL_MAXABS:
                failures.append(rec)
            if max(rec["dQ_rel_l2"], rec["dK_rel_l2"], rec["dV_rel_l2"]) > TOL_RELL2:
                failures.append(rec)
    assert not failures, failures


def check_invariants(x, outs, B, Hq, Hkv, G):
    """Properties that hold at any size, on every unit."""
    o, lse, dq, dk, dv = outs
    f32 = lambda t: t.float()
    sdk = f32(dk).sum(dim=1)                                      # [B, Hkv, d]
    assert (sdk.norm() / (f32(dk).norm() + 1e-30)).item() < 1e-2
    sdv = f32(dv).sum(dim=1)
    sdo = f32(x["dO"]).sum(dim=1).reshape(B, Hkv, G, -1).sum(dim=2)
    assert ((sdv - sdo).norm() / sdo.norm()).item() < 1e-2
    qdq = (f32(x["Q"]) * f32(dq)).sum(dim=(1, 3)).reshape(B, Hkv, G).sum(dim=2)
    kdk = (f32(x["K"]) * f32(dk)).sum(dim=(1, 3))
    # a cancelling sum of N*G*d bf16-rounded products: compare as relative L2 over units
    assert ((qdq - kdk).norm() / kdk.norm()).item() < 1e-2
    assert torch.isfinite(lse).all() and torch.isfinite(f32(o)).all()


@pytest.mark.parametrize("name", list(CONFIGS))
def test_fullsize(name):
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    B, N, Hq, Hkv, d, causal = CONFIGS[name]
    G = Hq // Hkv
    x = gen(B, N, Hq, Hkv, d, seed=SEED)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
    # run-to-run determinism: bitwise for dK, dV (fixed reduction order, no atomics) and, at d = 128,
    # dQ; the d = 64 fused backward adds fp32 dQ partials in L2 arrival order (hk_attn.h)
    dq2, dk2, dv2 = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
    torch.cuda.synchronize()
    assert torch.equal(dk, dk2) and torch.equal(dv, dv2)
    assert torch.equal(dq, dq2) if d == 128 else rel_l2(np64(dq2), np64(dq)) <= 4e-4  # bf16 flips (test_gpu_bwd)
    del dq2, dk2, dv2
    outs = (o, lse, dq, dk, dv)
    check_invariants(x, outs, B, Hq, Hkv, G)
    units = sampled_units(B, Hkv, SEED)
    if mode_of(name) == "UNIT":
        check_unit_mode(name, x, outs, units, G, causal)
    else:
        check_row_mode(name, x, outs, units, G, causal, N)


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
