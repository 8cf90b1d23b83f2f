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
