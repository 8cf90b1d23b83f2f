"""Host logic of context-parallel ring attention (paper_2511_08083_b200/ring.py) on
CPU: the zigzag layout, the per-rank schedule (every (query chunk, key chunk) pair
visible under the mask is computed exactly once, with the right mask, and causal
work is balanced across ranks), the forward schedule composed with the fp64
oracle (attention + LSE merge) against the oracle on the whole sequence, and the
DistRing exchange over gloo at world sizes 2 and 3."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2511_08083_b200 import ring


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_zigzag_roundtrip(P):
    x = torch.arange(2 * 4 * P * 3, dtype=torch.float32).reshape(2, 4 * P, 3)
    parts = [ring.zigzag_shard(x, P, r) for r in range(P)]
    assert all(a.shape == (2, 2, 3) and a.is_contiguous() for p in parts for a in p)
    assert torch.equal(ring.zigzag_unshard(parts), x)
    with pytest.raises(ValueError):
        ring.zigzag_shard(torch.zeros(1, 2 * P + 1, 1), P, 0)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("causal", [False, True])
def test_plan_covers_mask_once_and_balances(P, causal):
    work = []
    for r in range(P):
        seen = {}
        for s, qh, kh, mode in ring.plan(P, r, causal):
            src = (r - s) % P
            qc, kc = ring.zigzag_chunks(P, r)[qh], ring.zigzag_chunks(P, src)[kh]
            assert (qc, kc) not in seen
            seen[(qc, kc)] = mode
        for qc in ring.zigzag_chunks(P, r):
            for kc in range(2 * P):
                want = "full" if (not causal or kc < qc) else ("causal" if kc == qc else None)
                assert seen.get((qc, kc)) == want, (r, qc, kc)
        work.append(sum(1.0 if m == "full" else 0.5 for m in seen.values()))
    assert max(work) == min(work)  # zigzag: every rank does the same amount of attention


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("causal", [False, True])
def test_forward_schedule_with_oracle_equals_whole_sequence(P, causal):
    """The ring forward's composition (plan + LSE merge), evaluated with the fp64
    oracle in place of the kernels, reproduces attention over the whole sequence."""
    B, c, Hq, Hkv, d = 1, 5, 4, 2, 8
    N = 2 * P * c
    g = np.random.default_rng(3)
    Q, K, V = (g.standard_normal((B, N, h, d)) for h in (Hq, Hkv, Hkv))
    O, L = oracle.attn_fwd(Q, K, V, causal)
    sl = lambda x, i: x[:, i * c:(i + 1) * c]
    for r in range(P):
        acc = [None, None]
        for s, qh, kh, mode in ring.plan(P, r, causal):
            qc, kc = ring.zigzag_chunks(P, r)[qh], ring.zigzag_chunks(P, (r - s) % P)[kh]
            part = oracle.attn_fwd(sl(Q, qc), sl(K, kc), sl(V, kc), mode == "causal")
            acc[qh] = part if acc[qh] is None else oracle.attn_merge(*acc[qh], *part)
        for qh, qc in enumerate(ring.zigzag_chunks(P, r)):
            np.testing.assert_allclose(acc[qh][0], sl(O, qc), atol=1e-12)
            np.testing.assert_allclose(acc[qh][1], L[:, :, qc * c:(qc + 1) * c], atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = ring.DistRing()
    ok = comm.world == world and comm.ranks == [rank]
    cur = [torch.full((3,), float(rank)), torch.full((2, 2), 10.0 + rank)]
    for step in range(1, world + 1):  # world rotations bring every tensor home
        cur = comm.finish(comm.start([cur]))[0]
        src = (rank - step) % world
        ok = ok and torch.equal(cur[0], torch.full((3,), float(src))) and torch.equal(
            cur[1], torch.full((2, 2), 10.0 + src))
    out.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distring_gloo_rotation(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(res[r] for r in range(world)), res


# ---------------------------------------------------------------- backward schedule on CPU
def _share_bwd(q, k, v, o, lse, do, causal, workspace=None, dq=None, dk=None, dv=None, deterministic=True,
               accumulate=True):
    """Stand-in for the kernel call the ring backward makes (hk_attn_bwd with the final O, LSE, adding into
    fp32 accumulators): the gradient share of one (query chunk, key chunk) pair, written out from the
    analytic backward with the GLOBAL O and LSE — P = exp(S - LSE), D = rowsum(dO O), dS = P (dP - D)."""
    assert accumulate
    B, c, Hq, d = q.shape
    Hkv = k.shape[2]
    G = Hq // Hkv
    sc = 1.0 / np.sqrt(d)
    for h in range(Hq):
        kh = h // G
        S = torch.einsum("bid,bjd->bij", q[:, :, h], k[:, :, kh]) * sc
        if causal:
            S = S.masked_fill(torch.triu(torch.ones(c, c, dtype=torch.bool), 1), float("-inf"))
        P = torch.exp(S - lse[:, h, :, None])
        dP = torch.einsum("bid,bjd->bij", do[:, :, h], v[:, :, kh])
        D = (do[:, :, h] * o[:, :, h]).sum(-1, keepdim=True)
        dS = P * (dP - D)
        dq[:, :, h] += (torch.einsum("bij,bjd->bid", dS, k[:, :, kh]) * sc).to(dq.dtype)
        dk[:, :, kh] += (torch.einsum("bij,bid->bjd", dS, q[:, :, h]) * sc).to(dk.dtype)
        dv[:, :, kh] += torch.einsum("bij,bid->bjd", P, do[:, :, h]).to(dv.dtype)
    return dq, dk, dv


def _cpu_kernels(monkeypatch):
    from paper_2511_08083_b200 import api
    import contextlib

    def accum(acc, x, out=None, init=False):
        if acc is not None and x is not None:
            acc.copy_((0 if init else acc) + x.to(acc.dtype))
        if out is not None:
            out.copy_(acc)

    monkeypatch.setattr(api, "attn_bwd", _share_bwd)
    monkeypatch.setattr(api, "accum_f32", lambda acc, x: acc.add_(x))
    monkeypatch.setattr(api, "sm_budget", lambda n: contextlib.nullcontext())
    monkeypatch.setattr(ring, "_accum", accum)


def _bwd_case(P, causal, seed=4):
    B, c, Hq, Hkv, d = 1, 4, 4, 2, 8
    N = 2 * P * c
    g = np.random.default_rng(seed)
    Q, K, V, dO = (g.standard_normal((B, N, h, d)) for h in (Hq, Hkv, Hkv, Hq))
    ref = oracle.attn_fwd_bwd(Q, K, V, dO, causal)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    O, LSE = t(ref["O"]), t(ref["LSE"])
    shard = lambda x, r: ring.zigzag_shard(t(x), P, r)
    lse_sh = lambda r: tuple(x.transpose(1, 2).contiguous() for x in ring.zigzag_shard(LSE.transpose(1, 2), P, r))
    return ref, shard, lse_sh, Q, K, V, dO, O


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("causal", [False, True])
def test_backward_schedule_loopback_equals_whole_sequence(P, causal, monkeypatch):
    """ring_attn_bwd's schedule — K/V one step ahead, the fp32 dK/dV accumulators one step behind the
    compute (each rank's contributions formed while the previous rank's sums travel, then added and
    sent on, the last send bringing every chunk home) — with the kernels replaced by the analytic
    share of each chunk pair: the whole-sequence gradients of the fp64 oracle."""
    _cpu_kernels(monkeypatch)
    ref, shard, lse_sh, Q, K, V, dO, O = _bwd_case(P, causal)
    qs = [shard(Q, r) for r in range(P)]
    ks = [shard(K, r) for r in range(P)]
    vs = [shard(V, r) for r in range(P)]
    dos = [shard(dO, r) for r in range(P)]
    os_ = [ring.zigzag_shard(O, P, r) for r in range(P)]
    lses = [lse_sh(r) for r in range(P)]
    res = ring.ring_attn_bwd(qs, ks, vs, os_, lses, dos, causal, ring.LoopbackRing(P))
    for i, n in enumerate(("dQ", "dK", "dV")):
        got = ring.zigzag_unshard([r[i] for r in res]).numpy()
        np.testing.assert_allclose(got, ref[n], atol=2e-5, rtol=1e-4, err_msg=n)


def _bwd_worker(rank, world, port, causal, out):
    import contextlib
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_08083_b200 import api

    def accum(acc, x, out_=None, init=False):
        if acc is not None and x is not None:
            acc.copy_((0 if init else acc) + x.to(acc.dtype))
        if out_ is not None:
            out_.copy_(acc)
    api.attn_bwd = _share_bwd
    api.accum_f32 = lambda acc, x: acc.add_(x)
    api.sm_budget = lambda n: contextlib.nullcontext()
    ring._accum = accum
    ref, shard, lse_sh, Q, K, V, dO, O = _bwd_case(world, causal)
    (dq, dk, dv), = ring.ring_attn_bwd([shard(Q, rank)], [shard(K, rank)], [shard(V, rank)],
                                       [ring.zigzag_shard(O, world, rank)], [lse_sh(rank)], [shard(dO, rank)],
                                       causal, ring.DistRing())
    ok = True
    for n, got in (("dQ", dq), ("dK", dk), ("dV", dv)):
        want = ring.zigzag_shard(torch.from_numpy(np.ascontiguousarray(ref[n])), world, rank)
        ok = ok and all(np.allclose(a.numpy(), b.numpy(), atol=2e-5, rtol=1e-4) for a, b in zip(got, want))
    out.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("causal", [False, True])
def test_backward_schedule_gloo_two_ranks(causal):
    """The same backward schedule over torch.distributed (gloo, 2 processes, DistRing)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bwd_worker, args=(r, 2, port, causal, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(res.values()), res
