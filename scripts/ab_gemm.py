"""Interleaved A/B of two libhkattn builds' GEMM (hk_gemm_bf16) and cuBLAS (torch.matmul) on the same
inputs. Usage: python scripts/ab_gemm.py --a paper_2511_08083_b200/libhkattn_gbase.so
                                          --b paper_2511_08083_b200/libhkattn.so"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200.inputs import make_gemm_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", required=True)
    ap.add_argument("--b", required=True)
    ap.add_argument("--shapes", default="8192,8192,8192;4096,4096,4096;16384,16384,8192")
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    libs = {}
    for tag, path in (("A", a.a), ("B", a.b)):
        L = ctypes.CDLL(os.path.abspath(path))
        L.hk_gemm_bf16.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
        libs[tag] = L
    for sh in a.shapes.split(";"):
        M, N, K = (int(v) for v in sh.split(","))
        x = make_gemm_inputs(M, N, K, seed=0, device="cuda")
        A, Bm = x["A"], x["B"]
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        runs = {"A": lambda: libs["A"].hk_gemm_bf16(P(A), P(Bm), P(C), M, N, K, sp),
                "B": lambda: libs["B"].hk_gemm_bf16(P(A), P(Bm), P(C), M, N, K, sp),
                "cublas": lambda: torch.matmul(A, Bm.t())}
        t = {k: [] for k in runs}
        for rep in range(a.reps):
            order = list(runs) if rep % 2 == 0 else list(runs)[::-1]
            for k in order:
                for _ in range(3):
                    runs[k]()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record()
                for _ in range(a.iters):
                    runs[k]()
                e.record()
                torch.cuda.synchronize()
                t[k].append(s.elapsed_time(e) / a.iters)
        fl = 2.0 * M * N * K
        res = {k: round(fl / statistics.median(v) / 1e9, 1) for k, v in t.items()}
        print(json.dumps({"shape": [M, N, K], "tflops": res, "B_over_A": round(res["B"] / res["A"], 4),
                          "B_over_cublas": round(res["B"] / res["cublas"], 4)}), flush=True)


if __name__ == "__main__":
    main()
