"""Plain fp64 oracles for the paper's memory-bound kernels.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Never imported by the
product package; the dropout hash below is implemented here independently of
the CUDA path (same counter-based generator, reading #20).

1. Fused dropout + residual + LayerNorm, following the listing's order
   (PAPER.md P:1214-1267 [App. Kernel listings > LayerNorm]):
       x~      = dropout(x, p) = x * keep / (1 - p)
       r       = residual + x~          -> stored as o_resid
       mean    = sum(r) / D
       var     = sum((r - mean)^2) / D
       o       = (r - mean) / sqrt(var + eps) * w + b
   eps = 1e-5. The listing keeps mean/var in bf16; the oracle is
   exact (fp64) and takes r after the bf16 rounding of the stored o_resid,
   as the product path does (reading #20).
   keep(i) for flat element index i = row * D + col (< 2^32):
   h(i) >= floor(p * 2^32), h = the "lowbias32" integer hash of
   (i * 0x9E3779B9 + seed) mod 2^32:
       x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16.

2. Rotary positional encoding (B=16, H=16, d=128), rotate-half
   form (reading #21): for x [B, N, H, d], cos/sin [N, d/2],
       out[..., i]       = x[..., i] cos[n, i] - x[..., i + d/2] sin[n, i]
       out[..., i + d/2] = x[..., i + d/2] cos[n, i] + x[..., i] sin[n, i]
   i.e. (x_i + j x_{i+d/2}) * exp(j theta_{n,i}).
"""
from __future__ import annotations

import numpy as np

def dropout_keep(n_elems: int, p: float, seed: int, offset: int = 0) -> np.ndarray:
    """Boolean keep mask for flat indices offset .. offset+n_elems-1 (uint32 arithmetic)."""
    if p <= 0.0:
        return np.ones(n_elems, dtype=bool)
    i = np.arange(offset, offset + n_elems, dtype=np.uint64)
    x = (i * np.uint64(0x9E3779B9) + np.uint64(seed & 0xFFFFFFFF)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(16)
    return x >= np.uint64(int(p * 4294967296.0))


def _bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp64 values to bf16 (round to nearest even) and back (for o_resid)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def layernorm_dropout_residual(x, residual, w, b, p: float = 0.0, seed: int = 0, eps: float = 1e-5,
                               round_resid: bool = True):
    """x, residual: [rows, D]; w, b: [D]. Returns (o [rows, D], o_resid [rows, D]) fp64."""
    x = np.asarray(x, dtype=np.float64)
    residual = np.asarray(residual, dtype=np.float64)
    rows, D = x.shape
    keep = dropout_keep(rows * D, p, seed).reshape(rows, D)
    xt = np.where(keep, x / (1.0 - p), 0.0) if p > 0 else x
    r = residual + xt
    if round_resid:
        r = _bf16_round(r)
    mean = r.sum(axis=1, keepdims=True) / D
    c = r - mean
    var = (c * c).sum(axis=1, keepdims=True) / D
    o = c / np.sqrt(var + eps) * np.asarray(w, dtype=np.float64) + np.asarray(b, dtype=np.float64)
    return o, r


def rope(x, cos, sin):
    """x [B, N, H, d]; cos, sin [N, d/2]. Rotate-half rotary embedding, fp64."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    h = d // 2
    c = np.asarray(cos, dtype=np.float64)[None, :, None, :]
    s = np.asarray(sin, dtype=np.float64)[None, :, None, :]
    x1, x2 = x[..., :h], x[..., h:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rope_tables(N: int, d: int, base: float = 10000.0):
    """cos/sin [N, d/2] for theta_{n,i} = n * base^(-2i/d) (the usual RoPE frequencies)."""
    i = np.arange(d // 2, dtype=np.float64)
    theta = np.arange(N, dtype=np.float64)[:, None] * base ** (-2.0 * i / d)[None, :]
    return np.cos(theta), np.sin(theta)
