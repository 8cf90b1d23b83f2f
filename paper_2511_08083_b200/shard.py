"""Host-side multi-GPU partitioning of attention work units.

A unit is one (batch b, KV head kvh) pair: it is independent in the forward
and the backward (the only reduction, dK/dV over the G query heads of a KV
head, stays inside one unit), so ranks need no data-path collective.

Weak scaling (bench default): every rank owns a full per-GPU batch of B
sequences, global batches [rank*B, (rank+1)*B).
Strong scaling: a fixed global problem is split into contiguous, batch-major
unit ranges; when B >= world this is a plain batch split, otherwise KV-head
ranges are split (local Hq = G * local Hkv).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    batches: tuple      # global batch indices owned by this rank
    kv_heads: tuple     # global KV-head indices owned by this rank (within each batch)
    q_heads: tuple      # global query-head indices (the G heads of each owned KV head)

    @property
    def units(self):
        return len(self.batches) * len(self.kv_heads)


def weak_shard(rank: int, world: int, B: int, Hq: int, Hkv: int) -> Shard:
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return Shard(tuple(range(rank * B, (rank + 1) * B)), tuple(range(Hkv)), tuple(range(Hq)))


def strong_shard(rank: int, world: int, B: int, Hq: int, Hkv: int) -> Shard:
    """Contiguous batch-major split of the B*Hkv units of one global problem.
    Requires the split to be whole batches (B % world == 0) or whole KV-head
    groups inside one batch each (world % B == 0 and Hkv % (world // B) == 0)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    G = Hq // Hkv
    if B % world == 0:
        nb = B // world
        return Shard(tuple(range(rank * nb, (rank + 1) * nb)), tuple(range(Hkv)), tuple(range(Hq)))
    if world % B == 0 and Hkv % (world // B) == 0:
        per_b = world // B
        b = rank // per_b
        nk = Hkv // per_b
        k0 = (rank % per_b) * nk
        kv = tuple(range(k0, k0 + nk))
        return Shard((b,), kv, tuple(h for k in kv for h in range(k * G, (k + 1) * G)))
    raise ValueError(f"cannot split B={B}, Hkv={Hkv} units evenly over {world} ranks")


# ---------------------------------------------------------------- checking (not the hot path)
# NCCL carries only these checks (SURVEY §8(e) "Collectives"): per-unit checksums and one
# sampled unit's outputs gathered to rank 0. None of it is the method's arithmetic.

def _int_view(t):
    import torch
    t = t.contiguous()
    return t.view(torch.int16 if t.element_size() == 2 else torch.int32).to(torch.int64)


def bits_checksum(t):
    """Position-weighted sum of the raw bits (int64, wrapping): equal iff the values are
    bitwise equal (up to a 2^-64 collision), independent of the summation order."""
    import torch
    v = _int_view(t).reshape(-1)
    w = torch.arange(v.numel(), device=v.device, dtype=torch.int64) % 65521 + 1
    return (v * w).sum()


def unit_slices(outs, bi, ki, G):
    """The five outputs of local unit (batch index bi, KV-head index ki): O, LSE, dQ [.., G heads],
    dK, dV [.., one KV head] of the local [B', N, H', d] / [B', H', N] tensors."""
    hs = slice(ki * G, (ki + 1) * G)
    return (outs["O"][bi, :, hs], outs["LSE"][bi, hs], outs["dQ"][bi, :, hs], outs["dK"][bi, :, ki],
            outs["dV"][bi, :, ki])


def unit_checksums(outs, shard, G):
    """(ids [U, 2] int64 global (b, kvh), sums [U, 5] int64) for a rank's units."""
    import torch
    dev = outs["O"].device
    ids, sums = [], []
    for bi, b in enumerate(shard.batches):
        for ki, kvh in enumerate(shard.kv_heads):
            ids.append((b, kvh))
            sums.append(torch.stack([bits_checksum(t) for t in unit_slices(outs, bi, ki, G)]))
    return torch.tensor(ids, dtype=torch.int64, device=dev), torch.stack(sums)


def gather_checksums(ids, sums, world):
    """all_gather of every rank's (ids, sums) (equal unit counts per rank); returns a dict
    (b, kvh) -> tuple of 5 ints on every rank."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return {tuple(i): tuple(s) for i, s in zip(ids.tolist(), sums.tolist())}
    gi = [torch.empty_like(ids) for _ in range(world)]
    gs = [torch.empty_like(sums) for _ in range(world)]
    dist.all_gather(gi, ids)
    dist.all_gather(gs, sums)
    out = {}
    for a, s in zip(gi, gs):
        for i, v in zip(a.tolist(), s.tolist()):
            out[tuple(i)] = tuple(v)
    return out


def owner_of(unit, world, B, Hq, Hkv, scaling="strong"):
    """Rank owning global unit (b, kvh) and its local (bi, ki) indices."""
    split = strong_shard if scaling == "strong" else weak_shard
    for r in range(world):
        s = split(r, world, B, Hq, Hkv)
        if unit[0] in s.batches and unit[1] in s.kv_heads:
            return r, s.batches.index(unit[0]), s.kv_heads.index(unit[1])
    raise ValueError(f"unit {unit} has no owner")


def gather_unit_to_rank0(tensors, owner, rank, like):
    """Point-to-point copy of one unit's output tensors from `owner` to rank 0 (NCCL on an
    8-GPU box). `tensors`: the owner's tensors (ignored elsewhere); `like`: (shape, dtype,
    device) per tensor for rank 0's receive buffers. Returns rank 0's copies (None elsewhere)."""
    import torch
    import torch.distributed as dist
    if owner == 0:
        return [t.contiguous() for t in tensors] if rank == 0 else None
    if rank == owner:
        for t in tensors:
            dist.send(t.contiguous(), dst=0)
        return None
    if rank == 0:
        out = []
        for shape, dtype, device in like:
            buf = torch.empty(shape, dtype=dtype, device=device)
            dist.recv(buf, src=owner)
            out.append(buf)
        return out
    return None
