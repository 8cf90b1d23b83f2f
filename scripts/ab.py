"""Interleaved A/B timing of two libhkattn builds in ONE process (same clocks,
same inputs): each kernel phase of lib A and lib B alternate, repeated R times,
medians reported. Usage:
  python scripts/ab.py --a paper_2511_08083_b200/libhkattn_base.so \
      --b paper_2511_08083_b200/libhkattn.so --configs C3,C5-1024-c
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402


def load(path):
    L = ctypes.CDLL(os.path.abspath(path))
    vp, i = ctypes.c_void_p, ctypes.c_int
    L.hk_attn_fwd.argtypes = [vp] * 5 + [i] * 6 + [vp]
    L.hk_diag_bwd_phase.argtypes = [i] + [vp] * 10 + [ctypes.c_size_t] + [i] * 6 + [vp]
    L.hk_attn_bwd_workspace_bytes.restype = ctypes.c_size_t
    L.hk_attn_bwd_workspace_bytes.argtypes = [i] * 5
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", required=True)
    ap.add_argument("--b", required=True)
    ap.add_argument("--configs", default="C3")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--phases", default="fwd,pre,dkdv,dq")
    a = ap.parse_args()
    libs = {"A": load(a.a), "B": load(a.b)}
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    for name in a.configs.split(","):
        B, N, Hq, Hkv, d, causal = CONFIGS[name]
        x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
        o = torch.empty_like(x["Q"])
        lse = torch.empty(B, Hq, N, device="cuda", dtype=torch.float32)
        dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
        # one workspace per build: their layouts may differ (e.g. r2's augmented K-step rows)
        wss = {t: torch.zeros(libs[t].hk_attn_bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4 + 64, device="cuda",
                              dtype=torch.float32) for t in libs}
        sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

        def run(L, ph):
            ws = wss["A"] if L is libs["A"] else wss["B"]
            if ph == "fwd":
                r = L.hk_attn_fwd(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), B, Hq, Hkv, N, d, int(causal), sp)
            else:
                k = {"pre": 0, "dkdv": 1, "dq": 2}[ph]
                r = L.hk_diag_bwd_phase(k, P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk),
                                        P(dv), P(ws), ws.numel() * 4, B, Hq, Hkv, N, d, int(causal), sp)
            assert r == 0, r

        run(libs["A"], "fwd")
        run(libs["A"], "pre")
        run(libs["B"], "pre")  # each build's own workspace
        res = {}
        for ph in a.phases.split(","):
            t = {"A": [], "B": []}
            for rep in range(a.reps):
                for tag in ("A", "B") if rep % 2 == 0 else ("B", "A"):
                    L = libs[tag]
                    run(L, ph)
                    if ph == "fwd" or ph == "pre":
                        pass
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    s.record()
                    for _ in range(a.iters):
                        run(L, ph)
                    e.record()
                    torch.cuda.synchronize()
                    t[tag].append(s.elapsed_time(e) / a.iters)
            ma, mb = statistics.median(t["A"]), statistics.median(t["B"])
            res[ph] = {"A_ms": round(ma, 4), "B_ms": round(mb, 4), "B_speedup": round(ma / mb, 4)}
        print(json.dumps({"config": name, **res}), flush=True)
        del x


if __name__ == "__main__":
    main()
