"""Build libhkattn.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhkattn.so")
LIB_DEBUG = os.path.join(PKG, "libhkattn_debug.so")  # -DHK_DEBUG_HANG: barrier waits trap instead of hanging
LIB_TRACE = os.path.join(PKG, "libhkattn_trace.so")  # -DHK_TRACE: in-kernel clock64 event trace
SOURCES = [os.path.join(CSRC, "hk_attn.cu")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
         "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden", "-I", os.path.join(ROOT, "include")]


def _deps():
    files = list(SOURCES)
    for d in (CSRC, os.path.join(ROOT, "include")):
        files += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cuh", ".h", ".cu"))]
    return files


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def build(force: bool = False, verbose: bool = False, debug: bool = False, trace: bool = False,
          variant: str = "") -> str:
    """variant: build libhkattn_<variant>.so instead (A/B experiments with HK_EXTRA flags)."""
    lib = LIB_DEBUG if debug else LIB_TRACE if trace else LIB
    if variant:
        lib = os.path.join(PKG, f"libhkattn_{variant}.so")
    if not force and not (debug or trace or variant) and not needs_build():
        return LIB
    tmp = lib + ".tmp"
    extra = (["-DHK_DEBUG_HANG"] if debug else []) + (["-DHK_TRACE"] if trace else [])
    extra += os.environ.get("HK_EXTRA", "").split()  # e.g. tuning -D flags
    cmd = [NVCC, *FLAGS, *extra, "-o", tmp, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libhkattn.so")
    if verbose:
        sys.stderr.write(r.stderr)
    if not (debug or trace or variant):
        with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
            f.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv, trace="--trace" in sys.argv,
                variant=var))
