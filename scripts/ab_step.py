"""Steady-state (power-capped) A/B of several libhkattn builds on the full
training step (fwd + bwd), in one process: each build runs `--warm-s` seconds
of back-to-back steps, then `--steps` timed steps with the SM clock sampled;
builds rotate `--rounds` times. Usage:
  python scripts/ab_step.py --libs base,e00,e11 --config C3
(loads paper_2511_08083_b200/libhkattn_<name>.so; 'main' = libhkattn.so)
"""
import argparse
import ctypes
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402

PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2511_08083_b200")


def load(name):
    L = ctypes.CDLL(os.path.join(PKG, "libhkattn.so" if name == "main" else f"libhkattn_{name}.so"))
    vp, i = ctypes.c_void_p, ctypes.c_int
    L.hk_attn_fwd.argtypes = [vp] * 5 + [i] * 6 + [vp]
    L.hk_attn_bwd.argtypes = [vp] * 10 + [ctypes.c_size_t] + [i] * 6 + [vp]
    L.hk_attn_bwd_workspace_bytes.restype = ctypes.c_size_t
    L.hk_attn_bwd_workspace_bytes.argtypes = [i] * 5
    L.hk_attn_last_error.restype = ctypes.c_char_p
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--warm-s", type=float, default=1.5)
    ap.add_argument("--steps", type=int, default=15)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--ds", action="store_true", help="size the workspace for the stored-dS backward (d = 128)")
    a = ap.parse_args()
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        clk = lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        clk = lambda: -1
    B, N, Hq, Hkv, d, causal = CONFIGS[a.config]
    x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    o = torch.empty_like(x["Q"])
    lse = torch.empty(B, Hq, N, device="cuda", dtype=torch.float32)
    dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
    names = a.libs.split(",")
    libs = {n: load(n) for n in names}
    if a.ds:
        for L in libs.values():
            L.hk_attn_bwd_ds_workspace_bytes.restype = ctypes.c_size_t
            L.hk_attn_bwd_ds_workspace_bytes.argtypes = [ctypes.c_int] * 7
        wsb = max(L.hk_attn_bwd_ds_workspace_bytes(B, Hq, Hkv, N, N, d, int(causal)) for L in libs.values())
    else:
        wsb = max(L.hk_attn_bwd_workspace_bytes(B, Hq, Hkv, N, d) for L in libs.values())
    ws = torch.zeros(wsb // 4 + 64, device="cuda", dtype=torch.float32)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    flops = 3.5 * 4.0 * B * Hq * N * N * d * (0.5 if causal else 1.0)

    def step(L):
        r = L.hk_attn_fwd(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), B, Hq, Hkv, N, d, int(causal), sp)
        assert r == 0, (r, L.hk_attn_last_error())
        r = L.hk_attn_bwd(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk), P(dv), P(ws),
                          ws.numel() * 4, B, Hq, Hkv, N, d, int(causal), sp)
        assert r == 0, (r, L.hk_attn_last_error())

    res = {n: {"ms": [], "mhz": []} for n in names}
    for rnd in range(a.rounds):
        for n in (names if rnd % 2 == 0 else names[::-1]):
            L = libs[n]
            t0 = time.time()
            while time.time() - t0 < a.warm_s:
                step(L)
                torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            mhz = []
            for i in range(a.steps):
                step(L)
                if i % 3 == 0:
                    mhz.append(clk())
            e.record()
            torch.cuda.synchronize()
            res[n]["ms"].append(s.elapsed_time(e) / a.steps)
            res[n]["mhz"].extend(mhz)
    out = {n: {"ms_per_step": round(statistics.median(v["ms"]), 3),
               "tflops": round(flops / statistics.median(v["ms"]) / 1e9, 1),
               "sm_mhz_median": statistics.median(v["mhz"])} for n, v in res.items()}
    print(json.dumps({"config": a.config, **out}), flush=True)


if __name__ == "__main__":
    main()
