"""Plain fp64 attention forward + analytic backward — the parity oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Never imported by the
product package.

What is computed (PAPER.md lines cited as P:L):

    S_ij   = (1/sqrt(d)) * sum_k Q[b,i,h,k] K[b,j,kvh,k]   j in A(i), else -inf
    LSE_i  = ln sum_{j in A(i)} exp(S_ij)
    P_ij   = exp(S_ij - LSE_i)
    O_i    = sum_j P_ij V[b,j,kvh,:]
    dP_ij  = sum_k dO[b,i,h,k] V[b,j,kvh,k]
    D_i    = sum_k dO[b,i,h,k] O[b,i,h,k]
    dS_ij  = P_ij (dP_ij - D_i)
    dQ_i   = (1/sqrt(d)) sum_j dS_ij K_j
    dK_j   = (1/sqrt(d)) sum_{h in group(kvh)} sum_i dS^(h)_ij Q^(h)_i
    dV_j   =              sum_{h in group(kvh)} sum_i P^(h)_ij  dO^(h)_i

Sources:
  * softmax scale 1/sqrt(d) (with log2(e) folded in for exp2):
    P:1293 [App. Kernel listings > Attention, `TEMPERATURE_SCALE`].
  * scores / running max / exp2 / row sum / PV accumulate:
    P:1335-1340, P:1372-1378, P:1398-1405 [same listing].
  * LSE = max*ln2 + ln(norm) stored per (batch, head, row): P:1496-1500.
    With max in log2 units, max*ln2 + ln(sum 2^(x-max)) == ln sum e^S,
    i.e. the natural-log logsumexp (SURVEY §8(c).3 reading #2).
  * GQA head map head_idx_kv = head_idx / GROUP_SIZE: P:1287.
  * Tensor index order {batch, seq, head, d} (BNHD) for Q/K/V/O: P:1307,
    P:1313; L indexed {batch, head, 0, seq}: P:1500.
  * Causal: key j visible to query i iff j <= i (reading #3; P:571 names
    causal attention without fixing alignment; Nq == Nk so it is unique).
    With Nq != Nk the mask is bottom-right aligned:
    key j visible to query i iff j <= i + (Nk - Nq) (reading #22).
    A query row that sees no key has O = 0, LSE = -inf (the logsumexp of an
    empty set), D = 0 and dQ = 0; it adds nothing to dK, dV (reading #22).
  * Backward: the analytic gradient of the forward (reading #11); the paper
    gives no algorithm.

Layout conventions (all numpy, any float dtype accepted, converted to fp64):
  Q, dO: [B, Nq, Hq, d]   K, V: [B, Nk, Hkv, d]   LSE, D: [B, Hq, Nq]
  (Nq == Nk == N for the paper's problem; Nq != Nk is NEXT #4.)
Packed variable-length batches (NEXT #4, `attn_varlen_fwd_bwd`):
  Q, dO: [total_q, Hq, d]   K, V: [total_k, Hkv, d]   LSE, D: [Hq, total_q]
  sequence b = rows cu_q[b]..cu_q[b+1]-1 of Q and cu_k[b]..cu_k[b+1]-1 of K.
"""
from __future__ import annotations

import math

import numpy as np

# Printed constants, P:1293 and P:1497 (used verbatim; pinned in tests/golden).
LOG2E = 1.44269504089
LN2 = 0.69314718056

_ROW_BLOCK = 1024  # query rows per block: bounds the fp64 S block to 1024 x N


def softmax_scale(d: int) -> float:
    """1/sqrt(d); P:1293 prints 0.08838834764 (d=128) and 0.125 (d=64)."""
    return 1.0 / math.sqrt(d)


def _check(Q, K, V):
    """Shapes; returns B, Nq, Hq, Hkv, d, G (K, V may have Nk != Nq rows)."""
    B, N, Hq, d = Q.shape
    Bk, Nk, Hkv, dk = K.shape
    if K.shape != V.shape or (Bk, dk) != (B, d):
        raise ValueError("K, V must be [B, Nk, Hkv, d] matching Q [B, Nq, Hq, d]")
    if Hq % Hkv != 0:
        raise ValueError("Hq must be a multiple of Hkv (P:1287 GROUP_SIZE)")
    return B, N, Hq, Hkv, d, Hq // Hkv


def _allowed(rows: np.ndarray, Nq: int, Nk: int, causal: bool) -> np.ndarray:
    """Boolean mask [len(rows), Nk]: key j visible to query i (readings #3, #22:
    j <= i + Nk - Nq, which is j <= i when Nq == Nk)."""
    cols = np.arange(Nk)
    if causal:
        return cols[None, :] <= rows[:, None] + (Nk - Nq)
    return np.ones((len(rows), Nk), dtype=bool)


def _scores(q_rows, k, rows, Nq, causal, scale):
    """S = scale * q k^T with -inf outside A(i). q_rows [r, d], k [Nk, d]."""
    S = (q_rows @ k.T) * scale
    S[~_allowed(rows, Nq, k.shape[0], causal)] = -np.inf
    return S


def _lse(S):
    """Stable natural-log logsumexp per row: m + ln sum exp(S - m); -inf for a
    row with no visible key (reading #22)."""
    m = S.max(axis=1, keepdims=True) if S.shape[1] else np.full((S.shape[0], 1), -np.inf)
    empty = ~np.isfinite(m)
    m0 = np.where(empty, 0.0, m)
    with np.errstate(divide="ignore"):
        out = m0 + np.log(np.exp(S - m0).sum(axis=1, keepdims=True))
    return np.where(empty, -np.inf, out)[:, 0]


def _probs(S, lse):
    """P_ij = exp(S_ij - LSE_i); 0 on a row with no visible key (reading #22)."""
    live = np.isfinite(lse)
    return np.exp(S - np.where(live, lse, 0.0)[:, None]) * live[:, None]


def attn_fwd(Q, K, V, causal: bool):
    """Forward. Returns O [B,N,Hq,d] fp64 and LSE [B,Hq,N] fp64."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    B, N, Hq, Hkv, d, G = _check(Q, K, V)
    scale = softmax_scale(d)
    O = np.zeros((B, N, Hq, d))
    LSE = np.zeros((B, Hq, N))
    for b in range(B):
        for h in range(Hq):
            kvh = h // G
            k, v = K[b, :, kvh, :], V[b, :, kvh, :]
            for r0 in range(0, N, _ROW_BLOCK):
                rows = np.arange(r0, min(N, r0 + _ROW_BLOCK))
                S = _scores(Q[b, rows, h, :], k, rows, N, causal, scale)
                lse = _lse(S)
                P = _probs(S, lse)
                O[b, rows, h, :] = P @ v
                LSE[b, h, rows] = lse
    return O, LSE


def attn_fwd_bwd(Q, K, V, dO, causal: bool):
    """Forward + analytic backward, row-blocked per (b, h).

    Returns dict with O, LSE, D, dQ, dK, dV (all fp64).
    D is computed from the oracle's own fp64 O (reading #11).
    """
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    dO = np.asarray(dO, dtype=np.float64)
    B, N, Hq, Hkv, d, G = _check(Q, K, V)
    if dO.shape != Q.shape:
        raise ValueError("dO must have Q's shape")
    scale = softmax_scale(d)
    O = np.zeros((B, N, Hq, d))
    LSE = np.zeros((B, Hq, N))
    Dv = np.zeros((B, Hq, N))
    Nk = K.shape[1]
    dQ = np.zeros((B, N, Hq, d))
    dK = np.zeros((B, Nk, Hkv, d))
    dV = np.zeros((B, Nk, Hkv, d))
    for b in range(B):
        for h in range(Hq):
            kvh = h // G
            k, v = K[b, :, kvh, :], V[b, :, kvh, :]
            for r0 in range(0, N, _ROW_BLOCK):
                rows = np.arange(r0, min(N, r0 + _ROW_BLOCK))
                q = Q[b, rows, h, :]
                do = dO[b, rows, h, :]
                S = _scores(q, k, rows, N, causal, scale)
                lse = _lse(S)
                P = _probs(S, lse)
                o = P @ v
                D = (do * o).sum(axis=1)
                dP = do @ v.T
                dS = P * (dP - D[:, None])
                O[b, rows, h, :] = o
                LSE[b, h, rows] = lse
                Dv[b, h, rows] = D
                dQ[b, rows, h, :] = (dS @ k) * scale
                dK[b, :, kvh, :] += (dS.T @ q) * scale
                dV[b, :, kvh, :] += P.T @ do
    return {"O": O, "LSE": LSE, "D": Dv, "dQ": dQ, "dK": dK, "dV": dV}


def attn_rows(Q, K, V, dO, causal: bool, b: int, h: int, rows):
    """Per-query-row outputs for head (b, h): O, LSE, D and dQ at `rows`.

    Each query row is independent: its LSE_i and D_i come from the row itself
    (sampling mode ROW). Cost O(N d) per row.
    Returns dict of arrays indexed like `rows`.
    """
    rows = np.asarray(rows)
    Hq, Hkv = np.shape(Q)[2], np.shape(K)[2]
    kvh = h // (Hq // Hkv)
    q = np.asarray(Q[b, rows, h, :], dtype=np.float64)
    k = np.asarray(K[b, :, kvh, :], dtype=np.float64)
    v = np.asarray(V[b, :, kvh, :], dtype=np.float64)
    do = np.asarray(dO[b, rows, h, :], dtype=np.float64)
    scale = softmax_scale(k.shape[1])
    S = _scores(q, k, rows, np.shape(Q)[1], causal, scale)
    lse = _lse(S)
    P = _probs(S, lse)
    o = P @ v
    D = (do * o).sum(axis=1)
    dP = do @ v.T
    dS = P * (dP - D[:, None])
    return {"O": o, "LSE": lse, "D": D, "dQ": (dS @ k) * scale}


def attn_key_rows(Q, K, V, dO, causal: bool, b: int, kvh: int, keys, LSE, D):
    """dK, dV at key rows `keys` of unit (b, kvh), given LSE and D [B,Hq,N].

    dK_j = scale * sum_{h in group} sum_i dS_ij Q_i ; dV_j = sum_h sum_i P_ij dO_i.
    Cost O(G N d) per key row. LSE and D must be the oracle's (fp64) for the
    whole unit (ROW mode).
    """
    keys = np.asarray(keys)
    B, N, Hq, d = np.shape(Q)
    Nk, Hkv = K.shape[1], K.shape[2]
    G = Hq // Hkv
    scale = softmax_scale(d)
    kj = np.asarray(K[b, keys, kvh, :], dtype=np.float64)  # [r, d]
    vj = np.asarray(V[b, keys, kvh, :], dtype=np.float64)
    dK = np.zeros((len(keys), d))
    dV = np.zeros((len(keys), d))
    rows = np.arange(N)
    for h in range(kvh * G, (kvh + 1) * G):
        q = np.asarray(Q[b, :, h, :], dtype=np.float64)      # [N, d]
        do = np.asarray(dO[b, :, h, :], dtype=np.float64)
        # S^T for the sampled keys: [r, N] = scale * k_j q_i
        ST = (kj @ q.T) * scale
        mask = _allowed(rows, N, Nk, causal)[:, keys].T       # [r, N]: query i sees key j
        ST[~mask] = -np.inf
        PT = _probs(ST.T, np.asarray(LSE[b, h], dtype=np.float64)).T
        dPT = vj @ do.T
        dST = PT * (dPT - np.asarray(D[b, h], dtype=np.float64)[None, :])
        dV += PT @ do
        dK += (dST @ q) * scale
    return {"dK": dK, "dV": dV}


def attn_naive(Q, K, V, dO, causal: bool):
    """Triple-loop version for tiny shapes (N <= 64), written straight from
    the definitions above with no blocking; cross-checks attn_fwd_bwd."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    dO = np.asarray(dO, dtype=np.float64)
    B, N, Hq, Hkv, d, G = _check(Q, K, V)
    Nk = K.shape[1]
    scale = softmax_scale(d)
    O = np.zeros((B, N, Hq, d))
    LSE = np.zeros((B, Hq, N))
    Dv = np.zeros((B, Hq, N))
    dQ = np.zeros((B, N, Hq, d))
    dK = np.zeros((B, Nk, Hkv, d))
    dV = np.zeros((B, Nk, Hkv, d))
    for b in range(B):
        for h in range(Hq):
            kvh = h // G
            for i in range(N):
                js = [j for j in range(Nk) if (not causal) or j <= i + (Nk - N)]
                if not js:  # no visible key: O = 0, LSE = -inf, no gradient (reading #22)
                    LSE[b, h, i] = -math.inf
                    continue
                s = {j: scale * sum(Q[b, i, h, x] * K[b, j, kvh, x] for x in range(d)) for j in js}
                mx = max(s.values())
                lse = mx + math.log(sum(math.exp(s[j] - mx) for j in js))
                p = {j: math.exp(s[j] - lse) for j in js}
                for x in range(d):
                    O[b, i, h, x] = sum(p[j] * V[b, j, kvh, x] for j in js)
                LSE[b, h, i] = lse
                D = sum(dO[b, i, h, x] * O[b, i, h, x] for x in range(d))
                Dv[b, h, i] = D
                for j in js:
                    dp = sum(dO[b, i, h, x] * V[b, j, kvh, x] for x in range(d))
                    ds = p[j] * (dp - D)
                    for x in range(d):
                        dQ[b, i, h, x] += scale * ds * K[b, j, kvh, x]
                        dK[b, j, kvh, x] += scale * ds * Q[b, i, h, x]
                        dV[b, j, kvh, x] += p[j] * dO[b, i, h, x]
    return {"O": O, "LSE": LSE, "D": Dv, "dQ": dQ, "dK": dK, "dV": dV}


def attn_varlen_fwd_bwd(Q, K, V, dO, cu_q, cu_k, causal: bool):
    """Packed variable-length batch (NEXT #4): sequence b is the dense problem
    on Q rows cu_q[b]:cu_q[b+1] and K/V rows cu_k[b]:cu_k[b+1] (lengths may
    differ; causal is bottom-right aligned per sequence, reading #22).

    Q, dO [total_q, Hq, d]; K, V [total_k, Hkv, d]. Returns O, dQ like Q,
    dK, dV like K, LSE and D [Hq, total_q]; a sequence with no keys gives
    O = 0, LSE = -inf, dQ = 0.
    """
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    dO = np.asarray(dO, dtype=np.float64)
    cu_q = [int(x) for x in cu_q]
    cu_k = [int(x) for x in cu_k]
    if len(cu_q) != len(cu_k) or cu_q[0] != 0 or cu_k[0] != 0 or cu_q[-1] != Q.shape[0] \
            or cu_k[-1] != K.shape[0] or any(b < a for a, b in zip(cu_q, cu_q[1:])) \
            or any(b < a for a, b in zip(cu_k, cu_k[1:])):
        raise ValueError("cu_q / cu_k must be monotone offsets from 0 to total_q / total_k")
    Hq, d = Q.shape[1], Q.shape[2]
    out = {"O": np.zeros_like(Q), "dQ": np.zeros_like(Q), "dK": np.zeros_like(K), "dV": np.zeros_like(K),
           "LSE": np.zeros((Hq, Q.shape[0])), "D": np.zeros((Hq, Q.shape[0]))}
    for b in range(len(cu_q) - 1):
        qs, ks = slice(cu_q[b], cu_q[b + 1]), slice(cu_k[b], cu_k[b + 1])
        if cu_q[b + 1] == cu_q[b]:
            continue  # no queries: nothing to compute, dK = dV = 0 for this sequence
        if cu_k[b + 1] == cu_k[b]:  # no keys: every row sees nothing (reading #22)
            out["LSE"][:, qs] = -np.inf
            continue
        r = attn_fwd_bwd(Q[None, qs], K[None, ks], V[None, ks], dO[None, qs], causal)
        for k in ("O", "dQ"):
            out[k][qs] = r[k][0]
        for k in ("dK", "dV"):
            out[k][ks] = r[k][0]
        for k in ("LSE", "D"):
            out[k][:, qs] = r[k][0]
    return out
