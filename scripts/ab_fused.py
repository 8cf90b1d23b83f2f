"""NEXT #1 A/B: the fused single-pass backward (default) vs the deterministic two-pass
backward (HK_BWD_DETERMINISTIC), interleaved in one process on the same inputs; public API calls,
CUDA events, medians of R repeats. Prints one JSON line per config."""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import attn_bwd, attn_fwd  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402

CONFIGS.update({"C4-4096": (16, 4096, 32, 32, 64, True), "C4-16384": (16, 16384, 32, 32, 64, True),
                "C5-8192-nc": (16, 8192, 64, 8, 128, False)})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C4-2048,C4-4096,C4-8192,C4-16384")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    for name in a.configs.split(","):
        B, N, Hq, Hkv, d, causal = CONFIGS[name]
        x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
        o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
        outs = {m: tuple(torch.empty_like(x[n]) for n in ("Q", "K", "V")) for m in ("fused", "det")}
        fl = 2.5 * 4.0 * B * Hq * N * N * d * (0.5 if causal else 1.0)
        t = {"fused": [], "det": []}
        for rep in range(a.reps):
            for m in (("fused", "det") if rep % 2 == 0 else ("det", "fused")):
                g = outs[m]
                f = lambda: attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, dq=g[0], dk=g[1], dv=g[2],
                                     deterministic=(m == "det"))
                f()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record()
                for _ in range(a.iters):
                    f()
                e.record()
                torch.cuda.synchronize()
                t[m].append(s.elapsed_time(e) / a.iters)
        torch.cuda.synchronize()
        dq_rel = float((outs["fused"][0].float() - outs["det"][0].float()).norm() / outs["det"][0].float().norm())
        same_dkdv = bool(torch.equal(outs["fused"][1], outs["det"][1]) and torch.equal(outs["fused"][2], outs["det"][2]))
        mf, md = statistics.median(t["fused"]), statistics.median(t["det"])
        print(json.dumps({"config": name, "fused_ms": round(mf, 4), "det_ms": round(md, 4),
                          "fused_bwd_tflops": round(fl / mf / 1e9, 1), "det_bwd_tflops": round(fl / md / 1e9, 1),
                          "speedup": round(md / mf, 4), "dq_rel_l2_vs_det": dq_rel, "dkdv_bitwise_equal": same_dkdv}),
              flush=True)
        del x, o, lse, outs


if __name__ == "__main__":
    main()
