"""Seeded synthetic inputs (shared by the oracle tests and the CUDA path).

Holds none of the method's arithmetic: only random-number generation.

Recipe (reading #15): Q, K, V and
dO are i.i.d. N(0, std^2) drawn in fp32 and rounded to bf16 (RNE), BNHD
contiguous, the paper's N(0,1) inputs. Every (tensor, b, kvh)
block is drawn from its own generator seeded with splitmix64(seed, t, b, kvh),
so a rank that owns only some batches produces exactly the values the 1-GPU
run would have for those batches.
"""
from __future__ import annotations

import torch

_M64 = (1 << 64) - 1
TENSOR_IDS = {"Q": 1, "K": 2, "V": 3, "dO": 4}


def splitmix64(*xs: int) -> int:
    """Fold integers through splitmix64; returns a 63-bit seed."""
    z = 0x9E3779B97F4A7C15
    for x in xs:
        z = (z + (int(x) & _M64) + 0x9E3779B97F4A7C15) & _M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        z = z ^ (z >> 31)
    return z & ((1 << 63) - 1)


def _block(shape, seed, device, std):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    return x.to(torch.bfloat16)


def make_inputs(B, N, Hq, Hkv, d, seed=0, device="cpu", std=1.0, batches=None,
                tensors=("Q", "K", "V", "dO"), std_qk=None, kv_heads=None):
    """Return dict name -> bf16 tensor. Q/dO [B', N, Hq', d], K/V [B', N, Hkv', d].

    `batches` (default all of range(B)) selects which global batch indices to
    generate, in order; `kv_heads` (default all of range(Hkv)) which KV heads
    (Hkv' = len(kv_heads), Hq' = G * Hkv': each KV head brings its G query
    heads). The values of a (b, kvh) unit do not depend on which other units
    are generated. `std` scales all four tensors; `std_qk` (if given)
    overrides it for Q and K only — the stress recipe Q, K ~ N(0, 4^2) with
    V, dO ~ N(0, 1) (SURVEY §8(c).4 "Stress distributions").
    """
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    G = Hq // Hkv
    batches = list(range(B)) if batches is None else list(batches)
    kv_heads = list(range(Hkv)) if kv_heads is None else list(kv_heads)
    out = {}
    for name in tensors:
        t = TENSOR_IDS[name]
        sd = std_qk if (std_qk is not None and name in ("Q", "K")) else std
        heads = G * len(kv_heads) if name in ("Q", "dO") else len(kv_heads)
        x = torch.empty((len(batches), N, heads, d), dtype=torch.bfloat16, device=device)
        for bi, b in enumerate(batches):
            for ki, kvh in enumerate(kv_heads):
                if name in ("Q", "dO"):
                    blk = _block((N, G, d), splitmix64(seed, t, b, kvh), device, sd)
                    x[bi, :, ki * G:(ki + 1) * G, :] = blk
                else:
                    blk = _block((N, d), splitmix64(seed, t, b, kvh), device, sd)
                    x[bi, :, ki, :] = blk
        out[name] = x
    return out


def sample_rows(N: int, count: int, seed: int, diag_tile: int = 128):
    """Row sample for ROW-mode checks: first 8, last 8, tile
    edges (multiples of 128 +- 1) and random rows; sorted, unique."""
    g = torch.Generator().manual_seed(splitmix64(seed, 99))
    rows = set(range(min(8, N))) | set(range(max(0, N - 8), N))
    for t in range(diag_tile, N, diag_tile):
        for r in (t - 1, t, t + 1):
            if 0 <= r < N and len(rows) < count // 2 + 16:
                rows.add(r)
    while len(rows) < min(count, N):
        rows.add(int(torch.randint(0, N, (1,), generator=g)))
    return sorted(rows)


def make_gemm_inputs(M: int, N: int, K: int, seed: int = 0, device="cpu", std: float = 1.0):
    """A [M, K] and B [N, K] bf16, i.i.d. N(0, std^2) rounded to bf16 -- the paper's
    GEMM inputs (N(0, 1)). Each operand has its own splitmix64 stream."""
    return {"A": _block((M, K), splitmix64(seed, 11), device, std),
            "B": _block((N, K), splitmix64(seed, 12), device, std)}


def make_ln_inputs(rows: int, D: int, seed: int = 0, device="cpu"):
    """x, residual [rows, D] bf16 N(0,1); weight ~ 1 + 0.1 N(0,1), bias ~ 0.1 N(0,1) bf16."""
    w = _block((D,), splitmix64(seed, 23), device, 0.1).float() + 1.0
    return {"x": _block((rows, D), splitmix64(seed, 21), device, 1.0),
            "residual": _block((rows, D), splitmix64(seed, 22), device, 1.0),
            "weight": w.to(torch.bfloat16),
            "bias": _block((D,), splitmix64(seed, 24), device, 0.1)}


def make_rope_inputs(B: int, N: int, H: int, d: int, seed: int = 0, device="cpu"):
    """x [B, N, H, d] bf16 N(0,1) (the Q or K tensor a rotary step transforms)."""
    return {"x": _block((B, N, H, d), splitmix64(seed, 31), device, 1.0)}


def make_qk_inputs(B: int, Nq: int, Nk: int, Hq: int, Hkv: int, d: int, seed: int = 0, device="cpu",
                   std: float = 1.0):
    """Nq != Nk (NEXT #4): Q, dO [B, Nq, Hq, d] and K, V [B, Nk, Hkv, d] bf16, N(0, std^2);
    each tensor has its own splitmix64 stream."""
    return {"Q": _block((B, Nq, Hq, d), splitmix64(seed, 41), device, std),
            "K": _block((B, Nk, Hkv, d), splitmix64(seed, 42), device, std),
            "V": _block((B, Nk, Hkv, d), splitmix64(seed, 43), device, std),
            "dO": _block((B, Nq, Hq, d), splitmix64(seed, 44), device, 1.0)}


def varlen_lengths(B: int, mean: int, seed: int = 0, lo: int = 1):
    """A length mix for packed batches: B lengths uniform in [lo, 2*mean - lo]
    (the document-length spread of a packed pre-training batch)."""
    g = torch.Generator().manual_seed(splitmix64(seed, 51))
    return [int(x) for x in torch.randint(lo, max(lo + 1, 2 * mean - lo + 1), (B,), generator=g)]


def make_varlen_inputs(lens_q, lens_k, Hq: int, Hkv: int, d: int, seed: int = 0, device="cpu", std: float = 1.0):
    """Packed variable-length batch: Q, dO [sum(lens_q), Hq, d], K, V [sum(lens_k), Hkv, d]
    bf16 N(0, std^2), and int32 offsets cu_q, cu_k [B+1] (cu[0] = 0, running sums)."""
    tq, tk = int(sum(lens_q)), int(sum(lens_k))
    cu_q = torch.tensor([0] + list(torch.tensor(list(lens_q)).cumsum(0).tolist()), dtype=torch.int32, device=device)
    cu_k = torch.tensor([0] + list(torch.tensor(list(lens_k)).cumsum(0).tolist()), dtype=torch.int32, device=device)
    return {"Q": _block((tq, Hq, d), splitmix64(seed, 61), device, std),
            "K": _block((tk, Hkv, d), splitmix64(seed, 62), device, std),
            "V": _block((tk, Hkv, d), splitmix64(seed, 63), device, std),
            "dO": _block((tq, Hq, d), splitmix64(seed, 64), device, 1.0),
            "cu_q": cu_q, "cu_k": cu_k}
