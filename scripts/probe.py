"""Quick kernel timing probe (not the bench): CUDA-event timing of
hk_attn_fwd / hk_attn_bwd on BASELINE-shaped configs."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import attn_bwd, attn_fwd  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

CONFIGS = {
    "C2-nc": (16, 4096, 16, 16, 128, False),
    "C2-c": (16, 4096, 16, 16, 128, True),
    "C3": (16, 8192, 32, 8, 128, True),
    "C4-8192": (16, 8192, 32, 32, 64, True),
    "C4-2048": (16, 2048, 32, 32, 64, True),
    "C5-4096-nc": (16, 4096, 64, 8, 128, False),
    "C5-4096-c": (16, 4096, 64, 8, 128, True),
    "C5-1024-nc": (16, 1024, 64, 8, 128, False),
    "C5-1024-c": (16, 1024, 64, 8, 128, True),
    "C5-8192-nc": (16, 8192, 64, 8, 128, False),
    "C5-16384-nc": (16, 16384, 64, 8, 128, False),
    "C5-16384-c": (16, 16384, 64, 8, 128, True),
    "C4-4096": (16, 4096, 32, 32, 64, True),
    "C4-16384": (16, 16384, 32, 32, 64, True),
}


def timeit(fn, iters, warm):
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
    ap.add_argument("--configs", default="C2-nc,C2-c,C3,C4-8192")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--bwd", action="store_true")
    ap.add_argument("--phases", action="store_true", help="time bwd pre / dkdv / dq separately")
    a = ap.parse_args()
    for name in a.configs.split(","):
        B, N, Hq, Hkv, d, causal = CONFIGS[name]
        x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
        flops = 4.0 * B * Hq * N * N * d * (0.5 if causal else 1.0)
        o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
        ms = timeit(lambda: attn_fwd(x["Q"], x["K"], x["V"], causal, out=o, lse=lse), a.iters, 3)
        rec = {"config": name, "fwd_ms": round(ms, 4), "fwd_tflops": round(flops / ms / 1e9, 1)}
        if a.bwd:
            dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
            ms_b = timeit(lambda: attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, dq=dq, dk=dk, dv=dv),
                          a.iters, 3)
            rec.update(bwd_ms=round(ms_b, 4), bwd_tflops=round(2.5 * flops / ms_b / 1e9, 1))
            if a.phases:
                import ctypes
                from paper_2511_08083_b200 import _lib
                from paper_2511_08083_b200.api import bwd_workspace_bytes
                L = _lib.diag()
                ws = torch.empty(bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4, device="cuda", dtype=torch.float32)
                P = lambda t: ctypes.c_void_p(t.data_ptr())
                sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
                for ph, name, fl in ((0, "pre", 0), (1, "dkdv", 2.0), (2, "dq", 1.5)):
                    f = lambda: _lib.check_diag(L.hk_diag_bwd_phase(ph, P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse),
                                                               P(x["dO"]), P(dq), P(dk), P(dv), P(ws), ws.numel() * 4,
                                                               B, Hq, Hkv, N, d, int(causal), sp))
                    t = timeit(f, a.iters, 2)
                    rec[name + "_ms"] = round(t, 4)
                    if fl:
                        rec[name + "_tflops"] = round(fl * flops / t / 1e9, 1)
        print(json.dumps(rec), flush=True)
        del x


if __name__ == "__main__":
    main()
