"""Steady-state (power-capped) A/B of the two-pass and the stored-dS backward in the full training
step (public attn_fwd + attn_bwd, the workspace size selects the path): each mode runs --warm-s of
back-to-back steps, then --steps timed steps with the SM clock sampled; modes alternate --rounds
times. Usage: python scripts/ab_step_ds.py --config C3"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import api  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--warm-s", type=float, default=2.0)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        clk = lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pw = lambda: pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
    except Exception:
        clk = pw = lambda: -1
    B, N, Hq, Hkv, d, causal = CONFIGS[a.config]
    x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    o = torch.empty_like(x["Q"])
    lse = torch.empty(B, Hq, N, device="cuda", dtype=torch.float32)
    dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
    ws = {"two_pass": torch.zeros(api.bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4 + 64, device="cuda"),
          "stored_ds": torch.zeros(api.bwd_ds_workspace_bytes(B, Hq, Hkv, N, d, None, causal) // 4 + 64,
                                   device="cuda")}
    flops = 3.5 * 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)

    def step(w):
        api.attn_fwd(x["Q"], x["K"], x["V"], causal, out=o, lse=lse)
        api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=w, dq=dq, dk=dk, dv=dv)

    res = {m: {"ms": [], "mhz": [], "w": []} for m in ws}
    for rnd in range(a.rounds):
        for m in (list(ws) if rnd % 2 == 0 else list(ws)[::-1]):
            t0 = time.time()
            while time.time() - t0 < a.warm_s:
                step(ws[m])
                torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
            ev[0].record()
            for i in range(a.steps):
                step(ws[m])
                ev[i + 1].record()
                if i % 4 == 2:
                    res[m]["mhz"].append(clk())
                    res[m]["w"].append(pw())
            torch.cuda.synchronize()
            res[m]["ms"] += [ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)]
    out = {"config": a.config}
    for m, r in res.items():
        ms = statistics.median(r["ms"])
        out[m] = {"step_ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1),
                  "sm_mhz": statistics.median(r["mhz"]), "power_w": round(statistics.median(r["w"]), 1)}
    out["speedup"] = round(out["two_pass"]["step_ms"] / out["stored_ds"]["step_ms"], 4)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
