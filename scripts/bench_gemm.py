"""BF16 GEMM C = A B^T (NEXT #2) on B200: our tcgen05 CTA-pair kernel vs cuBLAS
(torch.matmul, the library baseline on the same box), CUDA-event timed after
warm-up, inputs N(0,1) bf16. Prints one JSON line per shape.
  python scripts/bench_gemm.py [--shapes 8192,8192,8192;4096,4096,4096] [--iters 50]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import gemm  # noqa: E402
from paper_2511_08083_b200.inputs import make_gemm_inputs  # noqa: E402


def timed(fn, iters, warm):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="8192,8192,8192;4096,4096,4096;16384,16384,8192")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    a = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from bench import load_peaks  # MEASURED_PEAKS.json, else the profiling guide's fallback
    pk = load_peaks()
    for sh in a.shapes.split(";"):
        M, N, K = (int(v) for v in sh.split(","))
        x = make_gemm_inputs(M, N, K, seed=0, device="cuda")
        A, B = x["A"], x["B"]
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        flops = 2.0 * M * N * K
        # interleave ours / cuBLAS twice, keep the better of each (same thermal state)
        t_ours, t_cub = [], []
        for _ in range(2):
            t_ours.append(timed(lambda: gemm(A, B, out=C), a.iters, a.warmup))
            t_cub.append(timed(lambda: torch.matmul(A, B.t()), a.iters, a.warmup))
        mo, mc = min(t_ours), min(t_cub)
        rec = {"metric": "bf16 GEMM C = A B^T TFLOPS", "shape": [M, N, K], "ours_ms": round(mo, 4),
               "ours_tflops": round(flops / mo / 1e9, 1), "cublas_ms": round(mc, 4),
               "cublas_tflops": round(flops / mc / 1e9, 1), "ours_vs_cublas": round(mc / mo, 3),
               "roofline": {"bound": "tensor", "peak_burst": pk["burst"], "frac_of_burst":
                            round(flops / mo / 1e9 / pk["burst"], 3), "cublas_frac_of_burst":
                            round(flops / mc / 1e9 / pk["burst"], 3), "peaks_source": pk["source"]}}
        print(json.dumps(rec), flush=True)
        del x, A, B, C


if __name__ == "__main__":
    main()
