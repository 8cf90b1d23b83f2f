"""Stored-dS backward (workspace >= hk_attn_bwd_ds_workspace_bytes) against the two-pass backward of
the same library: dK, dV bitwise, dQ rel-L2, then interleaved public-API backward timing per config.
Usage: python scripts/ab_ds.py [--configs C3,C2-nc,...] [--check-only]"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import api  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs, make_qk_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402


def bwd(x, o, lse, causal, ws):
    return api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=ws)


def wss(B, Hq, Hkv, Nq, Nk, d, causal):
    plain = api.bwd_workspace_bytes(B, Hq, Hkv, Nq, d, Nk)
    big = api.bwd_ds_workspace_bytes(B, Hq, Hkv, Nq, d, Nk, causal)
    mk = lambda n: torch.zeros((n + 3) // 4, dtype=torch.float32, device="cuda")
    return mk(plain), mk(big), big > plain


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C2-nc,C2-c,C5-1024-c,C5-4096-c")
    ap.add_argument("--check-only", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    for (B, Nq, Nk, Hq, Hkv, causal) in [(1, 256, 256, 2, 1, True), (2, 1000, 1000, 8, 2, True),
                                         (1, 384, 384, 4, 4, False), (2, 200, 700, 4, 2, True),
                                         (1, 777, 333, 6, 3, False), (2, 2048, 2048, 16, 4, True)]:
        x = make_qk_inputs(B, Nq, Nk, Hq, Hkv, 128, seed=5, device="cuda")
        o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
        w0, w1, applies = wss(B, Hq, Hkv, Nq, Nk, 128, causal)
        g0 = bwd(x, o, lse, causal, w0)
        g1 = bwd(x, o, lse, causal, w1)
        g2 = bwd(x, o, lse, causal, w1)
        torch.cuda.synchronize()
        print(json.dumps({"shape": [B, Nq, Nk, Hq, Hkv, causal], "ds_path": applies,
                          "dk_dv_bitwise": bool(torch.equal(g0[1], g1[1]) and torch.equal(g0[2], g1[2])),
                          "dq_rel_l2_vs_two_pass": rel(g1[0], g0[0]),
                          "repeat_bitwise": all(bool(torch.equal(u, v)) for u, v in zip(g1, g2))}), flush=True)
    if a.check_only:
        return
    for name in a.configs.split(","):
        B, N, Hq, Hkv, d, causal = CONFIGS[name]
        x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
        o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
        w0, w1, applies = wss(B, Hq, Hkv, N, N, d, causal)
        t = {"A": [], "B": []}
        for rep in range(a.reps):
            for tag in ("A", "B") if rep % 2 == 0 else ("B", "A"):
                ws = w0 if tag == "A" else w1
                bwd(x, o, lse, causal, ws)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record()
                for _ in range(3):
                    bwd(x, o, lse, causal, ws)
                e.record()
                torch.cuda.synchronize()
                t[tag].append(s.elapsed_time(e) / 3)
        ma, mb = statistics.median(t["A"]), statistics.median(t["B"])
        fl = 2.5 * 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)
        print(json.dumps({"config": name, "ds_gb": round(w1.numel() * 4 / 1e9, 2), "two_pass_ms": round(ma, 3),
                          "stored_ds_ms": round(mb, 3), "speedup": round(ma / mb, 4),
                          "two_pass_bwd_tflops": round(fl / ma / 1e9, 1),
                          "stored_ds_bwd_tflops": round(fl / mb / 1e9, 1)}), flush=True)
        del x, o, lse, w0, w1
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
