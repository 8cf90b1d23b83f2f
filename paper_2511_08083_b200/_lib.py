"""ctypes loader for libhkattn.so (argument marshalling only).

There is no fallback: if the library is missing or fails to load, every call
raises. Build it with `python -m paper_2511_08083_b200.build` (or
`__graft_entry__.build()`)."""
from __future__ import annotations

import ctypes
import os

# HK_LIB=debug selects the -DHK_DEBUG_HANG build (barrier waits trap with a message).
# HK_LIB=trace selects the -DHK_TRACE build (in-kernel event trace, hk_diag_trace_read).
# Any other HK_LIB=<name> loads libhkattn_<name>.so (A/B timing of a saved build).
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                         f"libhkattn_{os.environ['HK_LIB']}.so" if os.environ.get("HK_LIB") else "libhkattn.so")
_lib = None

HK_STATUS = {0: "HK_OK", 1: "HK_ERR_INVALID_ARGUMENT", 2: "HK_ERR_UNSUPPORTED",
             3: "HK_ERR_DEVICE", 4: "HK_ERR_LAUNCH"}

# (name, restype, argtypes) for every symbol declared in include/hk_attn.h and hk_attn_diag.h
_P, _I, _Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
SIGNATURES = {
    "hk_attn_fwd": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hk_attn_bwd_workspace_bytes": (_Z, [_I, _I, _I, _I, _I]),
    "hk_attn_bwd": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _I, _I, _I, _I, _I, _I, _P]),
    "hk_attn_fwd_qk": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "hk_attn_bwd_qk_workspace_bytes": (_Z, [_I, _I, _I, _I, _I, _I]),
    "hk_attn_bwd_qk": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _I, _I, _I, _I, _I, _I, _I, _P]),
    "hk_attn_fwd_varlen": (_I, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _Z, _P]),
    "hk_attn_bwd_varlen_workspace_bytes": (_Z, [_I, _I, _I, _I, _I, _I]),
    "hk_attn_bwd_varlen": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P, _P, _I, _I, _I, _I, _I, _I, _I,
                                _I, _I, _P]),
    "hk_attn_merge": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P]),
    "hk_accum_bf16": (_I, [_P, _P, _P, _Z, _I, _P]),
    "hk_attn_last_error": (ctypes.c_char_p, []),
    "hk_status_string": (ctypes.c_char_p, [_I]),
    "hk_attn_abi_version": (_I, []),
    "hk_diag_umma": (_I, [_P, _P, _P, _I, _I, _I, _I, _P]),
    "hk_diag_rates": (_I, [_I, _I, _I, _P, _P]),
    "hk_diag_trace_read": (_I, [_P, _Z, _I]),
    "hk_gemm_bf16": (_I, [_P, _P, _P, _I, _I, _I, _P]),
    "hk_ln_dropout_residual": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, ctypes.c_float, ctypes.c_uint, ctypes.c_float, _P]),
    "hk_rope": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _P]),
    "hk_diag_bwd_phase": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _I, _I, _I, _I, _I, _I, _P]),
}


class HKError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{HK_STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} not built: run `python -m paper_2511_08083_b200.build`")
        L = ctypes.CDLL(_LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def check(status: int):
    if status != 0:
        raise HKError(status, lib().hk_attn_last_error().decode())
