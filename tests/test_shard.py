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


def _fake_outputs(x, B, Hq, N):
    """Stand-ins for a rank's outputs with the real shapes (the checks only move bits)."""
    lse = x["Q"].float().sum(dim=3).transpose(1, 2).contiguous()  # [B', Hq', N]
    return {"O": x["Q"], "LSE": lse, "dQ": x["dO"], "dK": x["K"], "dV": x["V"]}


def _check_worker(rank, world, port, out, B, Hq, Hkv):
    from paper_2511_08083_b200.shard import (gather_checksums, gather_unit_to_rank0, owner_of, unit_checksums,
                                             unit_slices)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, d = 32, 8
    G = Hq // Hkv
    sh = strong_shard(rank, world, B, Hq, Hkv)
    x = make_inputs(B, N, Hq, Hkv, d, seed=4, batches=sh.batches, kv_heads=sh.kv_heads)
    outs = _fake_outputs(x, B, Hq, N)
    ids, sums = unit_checksums(outs, sh, G)
    got = gather_checksums(ids, sums, world)
    unit = (B - 1, Hkv - 1)
    owner, bi, ki = owner_of(unit, world, B, Hq, Hkv)
    like = [(t.shape, t.dtype, "cpu") for t in unit_slices(outs, bi, ki, G)] if rank == owner else None
    # rank 0 needs the shapes: every unit slice has the same shapes, take its own first unit's
    like0 = [(t.shape, t.dtype, "cpu") for t in unit_slices(outs, 0, 0, G)]
    recv = gather_unit_to_rank0(unit_slices(outs, bi, ki, G) if rank == owner else None, owner, rank, like0)
    if rank == 0:
        # the same checks from a 1-rank run of the whole problem
        full = make_inputs(B, N, Hq, Hkv, d, seed=4)
        fo = _fake_outputs(full, B, Hq, N)
        fs = strong_shard(0, 1, B, Hq, Hkv)
        want = gather_checksums(*unit_checksums(fo, fs, G), 1)
        ref_unit = unit_slices(fo, unit[0], unit[1], G)
        same_unit = all(torch.equal(a, b) for a, b in zip(recv, ref_unit))
        out.put((got == want, len(got) == B * Hkv, same_unit, owner))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B,Hq,Hkv", [(4, 4, 2), (1, 8, 2)])  # batch split; KV-head split (B < world)
def test_gloo_world2_checksums_and_unit_gather(B, Hq, Hkv):
    """bench.py's multi-GPU checking: per-unit checksums all-gathered from the
    ranks equal those of the 1-rank run, and the sampled unit reaches rank 0 intact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_check_worker, args=(r, 2, port, q, B, Hq, Hkv)) for r in range(2)]
    for p in procs:
        p.start()
    same, complete, unit_ok, owner = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert same and complete and unit_ok and owner == 1


def test_bits_checksum_detects_one_bit():
    from paper_2511_08083_b200.shard import bits_checksum
    t = torch.randn(64, 8).to(torch.bfloat16)
    u = t.clone()
    u.view(torch.int16)[17, 3] ^= 1
    assert bits_checksum(t) != bits_checksum(u)
    assert bits_checksum(t) == bits_checksum(t.clone())
    p = t.flatten()[torch.randperm(t.numel())].reshape(t.shape)  # same multiset, permuted
    assert bits_checksum(p) != bits_checksum(t) or torch.equal(p, t)
