"""Build libhkattn.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhkattn.so")            # the product C ABI (include/hk_attn.h & co.)
LIB_DIAG = os.path.join(PKG, "libhkattn_diag.so")  # diagnostics (include/hk_attn_diag.h)
LIB_DEBUG = os.path.join(PKG, "libhkattn_debug.so")  # -DHK_DEBUG_HANG: barrier waits trap instead of hanging
LIB_TRACE = os.path.join(PKG, "libhkattn_trace.so")  # -DHK_TRACE: in-kernel clock64 event trace
SOURCES = [os.path.join(CSRC, "hk_attn.cu")]
SOURCES_DIAG = [os.path.join(CSRC, "hk_diag.cu")]
SOURCES_DEV = [os.path.join(CSRC, "hk_dev.cu")]  # debug / trace / variant builds: both in one library
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
         "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden", "-I", os.path.join(ROOT, "include")]


def _deps():
    files = list(SOURCES)
    for d in (CSRC, os.path.join(ROOT, "include")):
        files += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cuh", ".h", ".cu"))]
    return files


def needs_build() -> bool:
    for lib in (LIB, LIB_DIAG):
        if not os.path.exists(lib):
            return True
        t = os.path.getmtime(lib)
        if any(os.path.getmtime(f) > t for f in _deps()):
            return True
    return False


def _nvcc(sources, out, extra):
    tmp = out + ".tmp"
    return tmp, subprocess.Popen([NVCC, *FLAGS, *extra, "-o", tmp, *sources], stdout=subprocess.PIPE,
                                 stderr=subprocess.PIPE, text=True)


def build(force: bool = False, verbose: bool = False, debug: bool = False, trace: bool = False,
          variant: str = "") -> str:
    """Release: libhkattn.so + libhkattn_diag.so (compiled in parallel). debug / trace / variant
    (libhkattn_<variant>.so, A/B experiments with HK_EXTRA flags): one library holding both."""
    dev = debug or trace or bool(variant)
    lib = LIB_DEBUG if debug else LIB_TRACE if trace else LIB
    if variant:
        lib = os.path.join(PKG, f"libhkattn_{variant}.so")
    if not force and not dev and not needs_build():
        return LIB
    extra = (["-DHK_DEBUG_HANG"] if debug else []) + (["-DHK_TRACE"] if trace else [])
    extra += os.environ.get("HK_EXTRA", "").split()  # e.g. tuning -D flags
    jobs = [(lib, *_nvcc(SOURCES_DEV if dev else SOURCES, lib, extra))]
    if not dev:
        jobs.append((LIB_DIAG, *_nvcc(SOURCES_DIAG, LIB_DIAG, extra)))
    errs = []
    for out, tmp, proc in jobs:
        so, se = proc.communicate()
        if proc.returncode != 0:
            errs.append(so + se)
            continue
        if verbose:
            sys.stderr.write(se)
        if out == LIB and not dev:
            with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
                f.write(se)
        os.replace(tmp, out)
    if errs:
        sys.stderr.write("\n".join(errs))
        raise RuntimeError("nvcc failed building " + ", ".join(os.path.basename(j[0]) for j in jobs))
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv, trace="--trace" in sys.argv,
                variant=var))
