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
# Those development builds hold the diagnostics too; the release build splits them into
# libhkattn_diag.so (include/hk_attn_diag.h), which the product path never loads.
_PKG = os.path.dirname(os.path.abspath(__file__))
_DEV = os.environ.get("HK_LIB")
_LIB_PATH = os.path.join(_PKG, f"libhkattn_{_DEV}.so" if _DEV else "libhkattn.so")
_DIAG_PATH = _LIB_PATH if _DEV else os.path.join(_PKG, "libhkattn_diag.so")
_lib = None
_diag = None

HK_STATUS = {0: "HK_OK", 1: "HK_ERR_INVALID_ARGUMENT", 2: "HK_ERR_UNSUPPORTED",
             3: "HK_ERR_DEVICE", 4: "HK_ERR_LAUNCH"}

_P, _I, _Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
# (restype, argtypes) for every symbol declared in include/hk_attn.h, hk_gemm.h, hk_membound.h, hk_ring.h
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
    "hk_attn_bwd_ex": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _I, _I, _I, _I, _I, _I, _I, ctypes.c_uint,
                            _P]),
    "hk_attn_bwd_varlen_ex": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P, _P, _I, _I, _I, _I, _I, _I, _I,
                                   _I, _I, ctypes.c_uint, _P]),
    "hk_attn_merge": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P]),
    "hk_accum_bf16": (_I, [_P, _P, _P, _Z, _I, _P]),
    "hk_accum_f32": (_I, [_P, _P, _Z, _P]),
    "hk_attn_bwd_ds_workspace_bytes": (_Z, [_I, _I, _I, _I, _I, _I, _I]),
    "hk_set_max_ctas": (None, [_I]),
    "hk_get_max_ctas": (_I, []),
    "hk_attn_last_error": (ctypes.c_char_p, []),
    "hk_status_string": (ctypes.c_char_p, [_I]),
    "hk_attn_abi_version": (_I, []),
    "hk_gemm_bf16": (_I, [_P, _P, _P, _I, _I, _I, _P]),
    "hk_ln_dropout_residual": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, ctypes.c_float, ctypes.c_uint, ctypes.c_float, _P]),
    "hk_rope": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _P]),
    "hk_rope_ex": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P]),
    "hk_attn_fwd_rope": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
}
# include/hk_attn_diag.h (libhkattn_diag.so)
DIAG_SIGNATURES = {
    "hk_diag_last_error": (ctypes.c_char_p, []),
    "hk_diag_umma": (_I, [_P, _P, _P, _I, _I, _I, _I, _P]),
    "hk_diag_rates": (_I, [_I, _I, _I, _P, _P]),
    "hk_diag_trace_read": (_I, [_P, _Z, _I]),
    "hk_diag_bwd_phase": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _I, _I, _I, _I, _I, _I, _P]),
}


class HKError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{HK_STATUS.get(status, status)}: {msg}")
        self.status = status


def _load(path, sigs):
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2511_08083_b200.build`")
    L = ctypes.CDLL(path)
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def lib():
    """libhkattn.so, the product C ABI."""
    global _lib
    if _lib is None:
        _lib = _load(_LIB_PATH, {**SIGNATURES, **(DIAG_SIGNATURES if _DEV else {})})
    return _lib


def diag():
    """libhkattn_diag.so (or the development build holding both): diagnostics only."""
    global _diag
    if _diag is None:
        _diag = lib() if _DEV else _load(_DIAG_PATH, DIAG_SIGNATURES)
    return _diag


def check(status: int):
    if status != 0:
        raise HKError(status, lib().hk_attn_last_error().decode())


def check_diag(status: int):
    if status != 0:
        raise HKError(status, diag().hk_diag_last_error().decode())
