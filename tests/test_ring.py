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
