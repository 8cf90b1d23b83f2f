"""Python binding of the C ABI (include/hk_attn.h): argument marshalling only.

Every step of the computation runs in libhkattn.so's sm_100a kernels; torch is
used for device memory and the current stream. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import HKError, check, check_diag, diag, lib  # noqa: F401


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_tensor(name, t, dtype=torch.bfloat16):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (BNHD)")
    if t.device != torch.device("cuda", torch.cuda.current_device()):
        raise ValueError(f"{name} must live on the current CUDA device")


def _expect_shape(name, t, shape):
    """Caller-supplied buffers reach the C ABI as raw pointers, so their sizes are checked here."""
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def _check_workspace(ws, nbytes):
    _check_tensor("workspace", ws, torch.float32)
    if ws.numel() * ws.element_size() < nbytes:
        raise ValueError(f"workspace must hold >= {nbytes} bytes, got {ws.numel() * ws.element_size()}")


def _shapes(q, k, v):
    """Returns B, Nq, Nk, Hq, Hkv, d (Nq != Nk allowed: bottom-right causal, hk_attn.h)."""
    if q.dim() != 4 or k.dim() != 4 or v.shape != k.shape:
        raise ValueError("q must be [B,Nq,Hq,d]; k, v [B,Nk,Hkv,d]")
    B, N, Hq, d = q.shape
    if k.shape[0] != B or k.shape[3] != d:
        raise ValueError("k/v shape mismatch with q")
    return B, N, k.shape[1], Hq, k.shape[2], d


def attn_fwd(q, k, v, causal: bool = False, out=None, lse=None):
    """O, LSE = attention(q, k, v). q [B,Nq,Hq,d], k/v [B,Nk,Hkv,d] bf16 CUDA.
    Returns (o [B,Nq,Hq,d] bf16, lse [B,Hq,Nq] fp32, natural log). Nq != Nk
    uses hk_attn_fwd_qk (causal mask bottom-right aligned)."""
    for n, t in (("q", q), ("k", k), ("v", v)):
        _check_tensor(n, t)
    B, N, Nk, Hq, Hkv, d = _shapes(q, k, v)
    o = torch.empty_like(q) if out is None else out
    L = torch.empty((B, Hq, N), dtype=torch.float32, device=q.device) if lse is None else lse
    _check_tensor("out", o)
    _check_tensor("lse", L, torch.float32)
    _expect_shape("out", o, q.shape)
    _expect_shape("lse", L, (B, Hq, N))
    if N == Nk:
        check(lib().hk_attn_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(L), B, Hq, Hkv, N, d, int(bool(causal)),
                                _stream()))
    else:
        check(lib().hk_attn_fwd_qk(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(L), B, Hq, Hkv, N, Nk, d,
                                   int(bool(causal)), _stream()))
    return o, L


def bwd_workspace_bytes(B, Hq, Hkv, N, d, Nk=None) -> int:
    if Nk is None or Nk == N:
        return int(lib().hk_attn_bwd_workspace_bytes(B, Hq, Hkv, N, d))
    return int(lib().hk_attn_bwd_qk_workspace_bytes(B, Hq, Hkv, N, Nk, d))


def bwd_ds_workspace_bytes(B, Hq, Hkv, N, d, Nk=None, causal=False) -> int:
    """Workspace size that selects the stored-dS backward (hk_attn_bwd_ds_workspace_bytes; equal to
    bwd_workspace_bytes where that path does not apply)."""
    return int(lib().hk_attn_bwd_ds_workspace_bytes(B, Hq, Hkv, N, N if Nk is None else Nk, d, int(bool(causal))))


# Largest stored-dS workspace attn_bwd allocates on its own (bytes; None = a quarter of the device's
# memory). Larger problems, or a caller-supplied workspace of the plain size, take the two-pass dQ.
DS_WORKSPACE_BUDGET = None


def _ds_budget(device) -> int:
    if DS_WORKSPACE_BUDGET is not None:
        return int(DS_WORKSPACE_BUDGET)
    return torch.cuda.get_device_properties(device).total_memory // 4


def default_bwd_workspace_bytes(B, Hq, Hkv, N, d, Nk=None, causal=False, device=None) -> int:
    """The workspace attn_bwd allocates when given none: the stored-dS size where that path applies
    and fits DS_WORKSPACE_BUDGET, else the plain size."""
    plain = bwd_workspace_bytes(B, Hq, Hkv, N, d, Nk)
    ds = bwd_ds_workspace_bytes(B, Hq, Hkv, N, d, Nk, causal)
    dev = torch.cuda.current_device() if device is None else device
    return ds if plain < ds <= _ds_budget(dev) else plain


HK_BWD_DETERMINISTIC = 1  # include/hk_attn.h
HK_BWD_ACCUMULATE_F32 = 2


def attn_bwd(q, k, v, o, lse, do, causal: bool = False, workspace=None, dq=None, dk=None, dv=None,
             deterministic: bool = False, accumulate: bool = False):
    """dQ, dK, dV of L = sum(O * dO) for O = attention(q, k, v).
    Returns (dq, dk, dv) bf16, plus the workspace holds D = rowsum(dO*O) then LSE*log2e.
    d = 64 runs the fused single-pass backward unless `deterministic` (hk_attn.h: dQ is then
    reproducible only up to fp32 reordering; dK, dV stay bitwise). accumulate: dq, dk, dv are
    caller-supplied fp32 tensors the results are ADDED into (HK_BWD_ACCUMULATE_F32)."""
    for n, t in (("q", q), ("k", k), ("v", v), ("o", o), ("do", do)):
        _check_tensor(n, t)
    _check_tensor("lse", lse, torch.float32)
    B, N, Nk, Hq, Hkv, d = _shapes(q, k, v)
    _expect_shape("o", o, q.shape)
    _expect_shape("do", do, q.shape)
    _expect_shape("lse", lse, (B, Hq, N))
    if accumulate and (dq is None or dk is None or dv is None):
        raise ValueError("accumulate=True needs the fp32 dq, dk, dv accumulators")
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    for n, t, ref in (("dq", dq, q), ("dk", dk, k), ("dv", dv, v)):
        _check_tensor(n, t, torch.float32 if accumulate else torch.bfloat16)
        _expect_shape(n, t, ref.shape)
    # no workspace given: the stored-dS backward (d = 128) when its workspace fits the budget
    nbytes = default_bwd_workspace_bytes(B, Hq, Hkv, N, d, Nk, causal, q.device) if workspace is None else 0
    ws = torch.empty((nbytes + 3) // 4, dtype=torch.float32, device=q.device) if workspace is None else workspace
    _check_workspace(ws, bwd_workspace_bytes(B, Hq, Hkv, N, d, Nk))
    check(lib().hk_attn_bwd_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(do), _ptr(dq), _ptr(dk),
                               _ptr(dv), _ptr(ws), ws.numel() * ws.element_size(), B, Hq, Hkv, N, Nk, d,
                               int(bool(causal)), (HK_BWD_DETERMINISTIC if deterministic else 0) |
                               (HK_BWD_ACCUMULATE_F32 if accumulate else 0), _stream()))
    return dq, dk, dv


def _varlen_args(q, k, v, cu_seqlens_q, cu_seqlens_k):
    for n, t in (("q", q), ("k", k), ("v", v)):
        _check_tensor(n, t)
    _check_tensor("cu_seqlens_q", cu_seqlens_q, torch.int32)
    _check_tensor("cu_seqlens_k", cu_seqlens_k, torch.int32)
    if q.dim() != 3 or k.dim() != 3 or v.shape != k.shape or k.shape[2] != q.shape[2]:
        raise ValueError("q must be [total_q,Hq,d]; k, v [total_k,Hkv,d]")
    if cu_seqlens_q.dim() != 1 or cu_seqlens_q.shape != cu_seqlens_k.shape or cu_seqlens_q.numel() < 2:
        raise ValueError("cu_seqlens_q / cu_seqlens_k must be int32 [B+1]")
    return cu_seqlens_q.numel() - 1, q.shape[0], k.shape[0], q.shape[1], k.shape[1], q.shape[2]


def check_cu_seqlens(cu_seqlens_q, cu_seqlens_k, total_q: int, total_k: int, max_seqlen_q: int,
                     max_seqlen_k: int):
    """Host-side check of the varlen offset contract of include/hk_attn.h (the library does not
    read device offsets on the host): cu[0] = 0, non-decreasing, cu[B] = total, every length
    <= max_seqlen. Copies the offsets to the host (a synchronisation): a debugging aid, not
    called on the fast path. Raises ValueError."""
    for name, cu, total, mx in (("q", cu_seqlens_q, total_q, max_seqlen_q), ("k", cu_seqlens_k, total_k,
                                                                              max_seqlen_k)):
        c = [int(x) for x in cu.detach().cpu().tolist()]
        lens = [b - a for a, b in zip(c, c[1:])]
        if c[0] != 0 or c[-1] != total or any(n < 0 for n in lens):
            raise ValueError(f"cu_seqlens_{name} must rise from 0 to total_{name}={total}: {c[:8]}...")
        if lens and max(lens) > mx:
            raise ValueError(f"a {name} sequence has length {max(lens)} > max_seqlen_{name}={mx}")


def attn_fwd_varlen(q, k, v, cu_seqlens_q, cu_seqlens_k, max_seqlen_q: int, max_seqlen_k: int,
                    causal: bool = False, out=None, lse=None, workspace=None, dynamic: bool = True):
    """Packed variable-length attention (hk_attn_fwd_varlen). q [total_q,Hq,d],
    k/v [total_k,Hkv,d] bf16; cu_seqlens_* int32 [B+1] on the device (not
    validated: see hk_attn.h). Returns (o [total_q,Hq,d], lse [Hq,total_q] fp32).
    dynamic: CTAs draw work items from a counter in `workspace` (>= 256 bytes;
    allocated here if None) — balanced when sequence lengths differ; False = static order."""
    B, tq, tk, Hq, Hkv, d = _varlen_args(q, k, v, cu_seqlens_q, cu_seqlens_k)
    o = torch.empty_like(q) if out is None else out
    L = torch.empty((Hq, tq), dtype=torch.float32, device=q.device) if lse is None else lse
    _check_tensor("out", o)
    _check_tensor("lse", L, torch.float32)
    _expect_shape("out", o, q.shape)
    _expect_shape("lse", L, (Hq, tq))
    ws = None
    if dynamic:
        ws = torch.empty(64, dtype=torch.int32, device=q.device) if workspace is None else workspace
        if not ws.is_cuda or not ws.is_contiguous() or ws.numel() * ws.element_size() < 256:
            raise ValueError("workspace must be a contiguous CUDA tensor of >= 256 bytes")
    check(lib().hk_attn_fwd_varlen(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(L), _ptr(cu_seqlens_q),
                                   _ptr(cu_seqlens_k), B, Hq, Hkv, tq, tk, int(max_seqlen_q), int(max_seqlen_k), d,
                                   int(bool(causal)), _ptr(ws) if ws is not None else None,
                                   ws.numel() * ws.element_size() if ws is not None else 0, _stream()))
    return o, L


def attn_bwd_varlen(q, k, v, o, lse, do, cu_seqlens_q, cu_seqlens_k, max_seqlen_q: int, max_seqlen_k: int,
                    causal: bool = False, workspace=None, dq=None, dk=None, dv=None, deterministic: bool = False):
    """Backward of attn_fwd_varlen (hk_attn_bwd_varlen_ex). Returns (dq, dk, dv) bf16. `deterministic`
    as in attn_bwd."""
    B, tq, tk, Hq, Hkv, d = _varlen_args(q, k, v, cu_seqlens_q, cu_seqlens_k)
    for n, t in (("o", o), ("do", do)):
        _check_tensor(n, t)
        _expect_shape(n, t, q.shape)
    _check_tensor("lse", lse, torch.float32)
    _expect_shape("lse", lse, (Hq, tq))
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    for n, t, ref in (("dq", dq, q), ("dk", dk, k), ("dv", dv, v)):
        _check_tensor(n, t)
        _expect_shape(n, t, ref.shape)
    nbytes = int(lib().hk_attn_bwd_varlen_workspace_bytes(B, Hq, Hkv, int(max_seqlen_q), int(max_seqlen_k), d))
    ws = torch.empty(nbytes // 4, dtype=torch.float32, device=q.device) if workspace is None else workspace
    _check_workspace(ws, nbytes)
    check(lib().hk_attn_bwd_varlen_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(do), _ptr(dq),
                                      _ptr(dk), _ptr(dv), _ptr(ws), ws.numel() * ws.element_size(),
                                      _ptr(cu_seqlens_q), _ptr(cu_seqlens_k), B, Hq, Hkv, tq, tk, int(max_seqlen_q),
                                      int(max_seqlen_k), d, int(bool(causal)),
                                      HK_BWD_DETERMINISTIC if deterministic else 0, _stream()))
    return dq, dk, dv


def set_max_ctas(n: int) -> None:
    """SM budget of the persistent kernels (hk_set_max_ctas): at most n CTAs per launch, n <= 0 =
    all SMs. Process-wide; results do not depend on it."""
    lib().hk_set_max_ctas(int(n))


def get_max_ctas() -> int:
    return int(lib().hk_get_max_ctas())


class sm_budget:
    """Context manager: persistent kernels leave `reserve` SMs free (for NCCL's copy kernels on
    another stream) inside the block; the previous budget is restored on exit."""

    def __init__(self, reserve: int):
        self.reserve = int(reserve)

    def __enter__(self):
        self.prev = get_max_ctas()
        if self.reserve > 0:
            sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            set_max_ctas(max(sms - self.reserve, 2))
        return self

    def __exit__(self, *exc):
        set_max_ctas(self.prev)
        return False


def accum_f32(acc, x):
    """acc += x for fp32 CUDA tensors of equal shape (hk_accum_f32, include/hk_ring.h)."""
    for name, t in (("acc", acc), ("x", x)):
        _check_tensor(name, t, torch.float32)
    _expect_shape("x", x, tuple(acc.shape))
    check(lib().hk_accum_f32(_ptr(acc), _ptr(x), ctypes.c_size_t(acc.numel()), _stream()))
    return acc


def gemm(a, b, out=None):
    """C = a @ b.T (bf16 in, fp32 accumulate, bf16 out) on the tcgen05 CTA-pair
    GEMM (include/hk_gemm.h). a [M, K], b [N, K] bf16 CUDA, contiguous;
    M, N multiples of 256 and K of 64."""
    _check_tensor("a", a)
    _check_tensor("b", b)
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[1]:
        raise ValueError(f"need a [M, K] and b [N, K]; got {tuple(a.shape)} and {tuple(b.shape)}")
    M, K = a.shape
    N = b.shape[0]
    c = torch.empty((M, N), dtype=torch.bfloat16, device=a.device) if out is None else out
    _check_tensor("out", c)
    _expect_shape("out", c, (M, N))
    check(lib().hk_gemm_bf16(_ptr(a), _ptr(b), _ptr(c), M, N, K, _stream()))
    return c


def ln_dropout_residual(x, residual, weight, bias, p: float = 0.0, seed: int = 0, eps: float = 1e-5,
                        out=None, out_resid=None):
    """Fused dropout + residual + LayerNorm (include/hk_membound.h). x, residual [..., D]
    bf16 CUDA contiguous; weight, bias [D] bf16. Returns (out, out_resid) bf16."""
    for n, t in (("x", x), ("residual", residual), ("weight", weight), ("bias", bias)):
        _check_tensor(n, t)
    if x.shape != residual.shape or weight.shape != (x.shape[-1],) or bias.shape != (x.shape[-1],):
        raise ValueError("x and residual must match, weight and bias must be [D]")
    D = x.shape[-1]
    rows = x.numel() // D
    o = torch.empty_like(x) if out is None else out
    r = torch.empty_like(x) if out_resid is None else out_resid
    for n, t in (("out", o), ("out_resid", r)):
        _check_tensor(n, t)
        _expect_shape(n, t, x.shape)
    check(lib().hk_ln_dropout_residual(_ptr(x), _ptr(residual), _ptr(weight), _ptr(bias), _ptr(o), _ptr(r), rows, D,
                                       float(p), int(seed) & 0xFFFFFFFF, float(eps), _stream()))
    return o, r


def rope(x, cos, sin, out=None, inverse: bool = False):
    """Rotary embedding (rotate-half) of x [B, N, H, d] bf16 with cos/sin [N, d/2] fp32
    (include/hk_membound.h). `out` may be `x` (in place). inverse: rotate by -theta (hk_rope_ex)."""
    _check_tensor("x", x)
    _check_tensor("cos", cos, torch.float32)
    _check_tensor("sin", sin, torch.float32)
    B, N, H, d = x.shape
    if cos.shape != (N, d // 2) or sin.shape != (N, d // 2):
        raise ValueError("cos and sin must be [N, d/2]")
    o = torch.empty_like(x) if out is None else out
    _check_tensor("out", o)
    _expect_shape("out", o, x.shape)
    check(lib().hk_rope_ex(_ptr(x), _ptr(cos), _ptr(sin), _ptr(o), B, N, H, d, int(bool(inverse)), _stream()))
    return o


def attn_fwd_rope(q, k, v, cos, sin, causal: bool = False, out=None, lse=None, k_rot=None):
    """O, LSE = attention(rope(q), rope(k), v) with the Q rotation fused into the forward kernel
    (hk_attn_fwd_rope). q [B,N,Hq,d], k/v [B,N,Hkv,d] bf16; cos/sin [N, d/2] fp32. Returns
    (o, lse, k_rot): k_rot = rope(k), which the backward (attn_bwd_rope) takes."""
    for n, t in (("q", q), ("k", k), ("v", v)):
        _check_tensor(n, t)
    B, N, Nk, Hq, Hkv, d = _shapes(q, k, v)
    if N != Nk:
        raise ValueError("attn_fwd_rope is self-attention: q and k need the same N")
    _check_tensor("cos", cos, torch.float32)
    _check_tensor("sin", sin, torch.float32)
    if cos.shape != (N, d // 2) or sin.shape != (N, d // 2):
        raise ValueError("cos and sin must be [N, d/2]")
    o = torch.empty_like(q) if out is None else out
    L = torch.empty((B, Hq, N), dtype=torch.float32, device=q.device) if lse is None else lse
    kr = torch.empty_like(k) if k_rot is None else k_rot
    for n, t, shp, dt in (("out", o, q.shape, torch.bfloat16), ("lse", L, (B, Hq, N), torch.float32),
                          ("k_rot", kr, k.shape, torch.bfloat16)):
        _check_tensor(n, t, dt)
        _expect_shape(n, t, shp)
    check(lib().hk_attn_fwd_rope(_ptr(q), _ptr(k), _ptr(v), _ptr(cos), _ptr(sin), _ptr(o), _ptr(L), _ptr(kr), B, Hq,
                                 Hkv, N, d, int(bool(causal)), _stream()))
    return o, L, kr


def attn_bwd_rope(q, k_rot, v, o, lse, do, cos, sin, causal: bool = False, deterministic: bool = False):
    """Gradients of attention(rope(q), rope(k), v) w.r.t. the UNrotated q, k and v: the backward
    runs on rope(q) and k_rot (from attn_fwd_rope) and maps dQ, dK back through the inverse
    rotation (R^T = R(-theta)). Every step is a libhkattn kernel. Returns (dq, dk, dv)."""
    qr = rope(q, cos, sin)
    dqr, dkr, dv = attn_bwd(qr, k_rot, v, o, lse, do, causal, deterministic=deterministic)
    return rope(dqr, cos, sin, out=dqr, inverse=True), rope(dkr, cos, sin, out=dkr, inverse=True), dv


class Attention(torch.autograd.Function):
    """autograd wrapper: Attention.apply(q, k, v, causal, deterministic=False) -> o."""

    @staticmethod
    def forward(ctx, q, k, v, causal=False, deterministic=False):
        o, lse = attn_fwd(q, k, v, causal)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.causal, ctx.deterministic = causal, deterministic
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        dq, dk, dv = attn_bwd(q, k, v, o, lse, do.contiguous(), ctx.causal, deterministic=ctx.deterministic)
        return dq, dk, dv, None, None


class AttentionRope(torch.autograd.Function):
    """autograd wrapper: AttentionRope.apply(q, k, v, cos, sin, causal) -> attention(rope(q), rope(k), v)."""

    @staticmethod
    def forward(ctx, q, k, v, cos, sin, causal=False):
        o, lse, kr = attn_fwd_rope(q, k, v, cos, sin, causal)
        ctx.save_for_backward(q, kr, v, o, lse, cos, sin)
        ctx.causal = causal
        return o

    @staticmethod
    def backward(ctx, do):
        q, kr, v, o, lse, cos, sin = ctx.saved_tensors
        dq, dk, dv = attn_bwd_rope(q, kr, v, o, lse, do.contiguous(), cos, sin, ctx.causal)
        return dq, dk, dv, None, None, None


class AttentionVarlen(torch.autograd.Function):
    """autograd wrapper: AttentionVarlen.apply(q, k, v, cu_q, cu_k, max_q, max_k, causal) -> o."""

    @staticmethod
    def forward(ctx, q, k, v, cu_q, cu_k, max_q, max_k, causal=False):
        o, lse = attn_fwd_varlen(q, k, v, cu_q, cu_k, max_q, max_k, causal)
        ctx.save_for_backward(q, k, v, o, lse, cu_q, cu_k)
        ctx.args = (max_q, max_k, causal)
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse, cu_q, cu_k = ctx.saved_tensors
        dq, dk, dv = attn_bwd_varlen(q, k, v, o, lse, do.contiguous(), cu_q, cu_k, *ctx.args)
        return dq, dk, dv, None, None, None, None, None


def diag_umma(a, b, n, k, a_tmem: bool, b_mn: bool):
    """Diagnostic single-tile tcgen05 GEMM (include/hk_attn_diag.h, libhkattn_diag.so)."""
    _check_tensor("a", a)
    _check_tensor("b", b)
    d = torch.empty((128, n), dtype=torch.float32, device=a.device)
    check_diag(diag().hk_diag_umma(_ptr(a), _ptr(b), _ptr(d), n, k, int(a_tmem), int(b_mn), _stream()))
    return d
