"""Multi-rank host logic on CPU with gloo (world size 2): unit partitioning,
per-rank input generation equal to the 1-rank run, and max-over-ranks timing."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_08083_b200.inputs import make_inputs
from paper_2511_08083_b200.shard import strong_shard, weak_shard


def test_partitions_cover_units_exactly_once():
    for B, Hq, Hkv, world in [(16, 32, 8, 1), (16, 32, 8, 2), (16, 32, 8, 8), (16, 64, 8, 4), (2, 64, 8, 8),
                              (1, 8, 8, 8), (4, 16, 4, 8)]:
        seen = set()
        for r in range(world):
            s = strong_shard(r, world, B, Hq, Hkv)
            for b in s.batches:
                for k in s.kv_heads:
                    assert (b, k) not in seen
                    seen.add((b, k))
            G = Hq // Hkv
            assert s.q_heads == tuple(h for k in s.kv_heads for h in range(k * G, (k + 1) * G))
        assert seen == {(b, k) for b in range(B) for k in range(Hkv)}
    with pytest.raises(ValueError):
        strong_shard(0, 3, 16, 32, 8)
    w = [weak_shard(r, 4, 16, 32, 8) for r in range(4)]
    assert [s.batches[0] for s in w] == [0, 16, 32, 48] and all(s.units == 16 * 8 for s in w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, N, Hq, Hkv, d = 4, 32, 4, 2, 8
    sh = strong_shard(rank, world, B, Hq, Hkv)
    x = make_inputs(B, N, Hq, Hkv, d, seed=3, batches=sh.batches)
    gathered = [torch.empty_like(x["Q"]) for _ in range(world)]
    dist.all_gather(gathered, x["Q"])
    t = torch.tensor([1.5 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = make_inputs(B, N, Hq, Hkv, d, seed=3)
        out.put((bool(torch.equal(torch.cat(gathered), full["Q"])), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_inputs_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    same, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert same and tmax == 2.5
