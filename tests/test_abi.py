"""CPU-side checks of the C ABI boundary: the library loads and exports every
symbol declared in include/*.h; the Python binding has a signature for each;
host-only validation paths return the documented statuses."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_08083_b200", "libhkattn.so")
LIB_DIAG = os.path.join(ROOT, "paper_2511_08083_b200", "libhkattn_diag.so")


def declared_symbols(which="all"):
    """hk_* functions declared in include/*.h: "diag" = hk_attn_diag.h (libhkattn_diag.so),
    "product" = every other header (libhkattn.so)."""
    names = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if which == "diag" and f != "hk_attn_diag.h" or which == "product" and f == "hk_attn_diag.h":
            continue
        if f.endswith(".h"):
            src = open(os.path.join(inc, f)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(hk_\w+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2511_08083_b200 import build
    build.build()
    return ctypes.CDLL(LIB)


def test_exports_every_declared_symbol(lib):
    names = declared_symbols("product")
    assert {"hk_attn_fwd", "hk_attn_bwd", "hk_attn_bwd_workspace_bytes", "hk_attn_last_error"} <= names
    for n in names:
        assert hasattr(lib, n), f"{n} not exported"
    diag = ctypes.CDLL(LIB_DIAG)
    for n in declared_symbols("diag"):
        assert hasattr(diag, n), f"{n} not exported by libhkattn_diag.so"
        assert not hasattr(lib, n), f"diagnostic {n} must not be in the product library"


def test_binding_covers_header():
    from paper_2511_08083_b200._lib import DIAG_SIGNATURES, SIGNATURES
    assert declared_symbols("product") == set(SIGNATURES)
    assert declared_symbols("diag") == set(DIAG_SIGNATURES)


def test_host_only_validation(lib):
    """Host-only paths (no GPU touched): version, status strings, workspace
    size, and argument validation that fails before any CUDA call."""
    from paper_2511_08083_b200 import _lib
    L = _lib.lib()
    assert L.hk_attn_abi_version() == 6
    assert L.hk_status_string(2) == b"HK_ERR_UNSUPPORTED"
    assert L.hk_attn_bwd_workspace_bytes(2, 4, 2, 256, 128) == 2 * 2 * 4 * 256 * 4 + 256
    # d = 64 adds the fused backward's fp32 dQ accumulator, B * Np * Hq * 64 floats
    assert L.hk_attn_bwd_workspace_bytes(2, 4, 2, 256, 64) == 2 * 2 * 4 * 256 * 4 + 256 + 2 * 256 * 4 * 256
    p = ctypes.c_void_p(16)
    assert L.hk_attn_fwd(p, p, p, p, p, 1, 2, 2, 128, 96, 0, None) == 2   # d = 96
    assert L.hk_attn_fwd(p, p, p, p, p, 1, 2, 2, 0, 64, 0, None) == 1     # N = 0
    assert L.hk_attn_bwd_workspace_bytes(1, 2, 2, 200, 128) == 2 * 2 * 256 * 4 + 256  # rows padded to 128
    assert L.hk_attn_fwd(p, p, p, p, p, 1, 3, 2, 128, 64, 0, None) == 1   # Hq % Hkv
    assert b"multiple" in L.hk_attn_last_error()
    assert L.hk_attn_fwd(p, p, p, p, p, 0, 2, 2, 128, 64, 0, None) == 1   # B = 0
    assert L.hk_attn_fwd(None, p, p, p, p, 1, 2, 2, 128, 64, 0, None) == 1
    assert L.hk_attn_fwd(ctypes.c_void_p(8), p, p, p, p, 1, 2, 2, 128, 64, 0, None) == 1
    # outputs aliasing inputs
    assert L.hk_attn_fwd(p, p, p, p, p, 1, 2, 2, 128, 64, 0, None) == 1
    assert b"alias" in L.hk_attn_last_error()
    # bwd: workspace too small
    a = [ctypes.c_void_p(16 * (i + 1) << 30) for i in range(10)]
    assert L.hk_attn_bwd(*a, 0, 1, 2, 2, 128, 64, 0, None) == 1
    assert b"workspace" in L.hk_attn_last_error()
    # bwd_ex: unknown flag bits are rejected before anything else
    assert L.hk_attn_bwd_ex(*a, 0, 1, 2, 2, 128, 128, 64, 0, 6, None) == 1
    assert b"flags" in L.hk_attn_last_error()


def test_host_only_validation_next4(lib):
    """Validation of the NEXT #4 entry points (Nq != Nk, varlen, ring merge / accumulate)
    fails before any CUDA call; workspace sizes follow the header formulas."""
    from paper_2511_08083_b200 import _lib
    L = _lib.lib()
    p = ctypes.c_void_p(16)
    Z = ctypes.c_size_t
    assert L.hk_attn_bwd_qk_workspace_bytes(2, 4, 2, 200, 1000, 64) == 2 * 2 * 4 * 256 * 4 + 256 + 2 * 256 * 4 * 256
    assert L.hk_attn_bwd_varlen_workspace_bytes(3, 4, 2, 129, 7, 128) == 2 * 3 * 4 * 256 * 4 + 256
    assert L.hk_attn_fwd_qk(p, p, p, p, p, 1, 2, 2, 128, 0, 64, 0, None) == 1     # Nk = 0
    assert L.hk_attn_fwd_qk(p, p, p, p, p, 1, 2, 2, 128, 256, 80, 0, None) == 2   # d = 80
    a = [ctypes.c_void_p(16 * (i + 1) << 30) for i in range(7)]
    # varlen: null offsets, zero totals, misaligned offsets, a too-small forward workspace
    assert L.hk_attn_fwd_varlen(*a[:5], None, a[6], 2, 2, 2, 100, 100, 64, 64, 64, 0, None, Z(0), None) == 1
    assert L.hk_attn_fwd_varlen(*a[:7], 2, 2, 2, 0, 100, 64, 64, 64, 0, None, Z(0), None) == 1
    assert L.hk_attn_fwd_varlen(*a[:5], ctypes.c_void_p(18), a[6], 2, 2, 2, 100, 100, 64, 64, 64, 0, None, Z(0),
                                None) == 1
    assert L.hk_attn_fwd_varlen(*a[:7], 2, 2, 2, 100, 100, 64, 64, 64, 0, ctypes.c_void_p(16 << 35), Z(64),
                                None) == 1
    assert b"workspace" in L.hk_attn_last_error()
    # ring building blocks
    assert L.hk_attn_merge(p, p, p, p, None, 1, 128, 2, 96, 0, None) == 2       # d not a power of two
    assert L.hk_attn_merge(p, p, p, p, None, 0, 128, 2, 64, 0, None) == 1       # B = 0
    assert L.hk_attn_merge(p, p, p, p, None, 1, 128, 2, 64, 0, None) == 1       # buffers overlap
    assert L.hk_accum_bf16(p, p, None, Z(12), 0, None) == 1                     # n % 8
    assert L.hk_accum_bf16(None, None, p, Z(16), 0, None) == 1                  # nothing to read


def test_stored_ds_workspace_size(lib):
    """hk_attn_bwd_ds_workspace_bytes (host only): the plain workspace rounded up to 1024 bytes plus
    one 32 KB bf16 dS tile per visited 128 x 128 block — the T(T+1)/2 triangle for causal Nq == Nk,
    the Tq x Tk rectangle otherwise — and exactly the plain size where the path does not apply (d = 64)."""
    from paper_2511_08083_b200 import _lib
    L = _lib.lib()
    for B, Hq, Hkv, Nq, Nk, causal in ((16, 32, 8, 8192, 8192, 1), (2, 4, 2, 300, 700, 1), (1, 6, 3, 777, 333, 0),
                                       (3, 2, 1, 128, 128, 1), (1, 1, 1, 1, 1, 0)):
        plain = L.hk_attn_bwd_qk_workspace_bytes(B, Hq, Hkv, Nq, Nk, 128)
        Tq, Tk = -(-Nq // 128), -(-Nk // 128)
        blocks = Tq * (Tq + 1) // 2 if (causal and Nq == Nk) else Tq * Tk
        want = -(-plain // 1024) * 1024 + B * Hq * blocks * 128 * 128 * 2
        assert L.hk_attn_bwd_ds_workspace_bytes(B, Hq, Hkv, Nq, Nk, 128, causal) == want
        assert L.hk_attn_bwd_ds_workspace_bytes(B, Hq, Hkv, Nq, Nk, 64, causal) == \
            L.hk_attn_bwd_qk_workspace_bytes(B, Hq, Hkv, Nq, Nk, 64)
    # C3: 34.9 GB of dS tiles (16 x 32 heads x 2080 blocks x 32 KB)
    assert L.hk_attn_bwd_ds_workspace_bytes(16, 32, 8, 8192, 8192, 128, 1) // 10**8 == 349
