"""Sequence-length variants (NEXT #4) on B200: device-timed fwd and bwd TFLOPS of
  (a) a packed variable-length batch with the C3 head geometry (Llama-3 8B GQA,
      Hq=32, Hkv=8, d=128, causal): 131072 tokens as documents of uniform length
      in [1, 16383] (mean 8192), next to the dense C3 batch of the
      same token count;
  (b) Nq != Nk chunked prefill / ring-step shapes: B=16, Nq=1024 queries against
      Nk=16384 keys (bottom-right causal) with the same heads.
Algorithmic FLOPs count only visible (query, key) pairs: fwd = 4 d Hq x pairs,
bwd = 2.5 x fwd (reading #14). Prints one JSON line per workload."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import attn_bwd, attn_bwd_varlen, attn_fwd, attn_fwd_varlen  # noqa: E402
from paper_2511_08083_b200.inputs import (make_inputs, make_qk_inputs, make_varlen_inputs,  # noqa: E402
                                          varlen_lengths)


def pairs(lq, lk, causal):
    """Visible (query, key) pairs of one sequence under the bottom-right mask."""
    if not causal:
        return lq * lk
    off = lk - lq
    return sum(max(0, min(lk, i + off + 1)) for i in range(lq))


def timed(fn, iters, warm=3):
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


def report(name, cfg, npairs, Hq, d, t_f, t_b, peak):
    ff = 4.0 * d * Hq * npairs
    line = {"workload": name, **cfg, "fwd_ms": round(t_f, 4), "bwd_ms": round(t_b, 4),
            "fwd_tflops": round(ff / t_f / 1e9, 1), "bwd_tflops": round(2.5 * ff / t_b / 1e9, 1),
            "fwd_bwd_tflops": round(3.5 * ff / (t_f + t_b) / 1e9, 1)}
    line["frac_of_sustained"] = round(line["fwd_bwd_tflops"] / peak, 3)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pk = os.path.join(root, "MEASURED_PEAKS.json")
    peak = float(json.load(open(pk)).get("bf16_tflops_sustained", 1400.0)) if os.path.exists(pk) else 1400.0
    Hq, Hkv, d = 32, 8, 128
    causal = True

    # (a) packed documents vs dense C3 with the same token count
    total = 16 * 8192
    lens, s = [], 0
    for L in varlen_lengths(64, 8192, seed=7):
        if s + L > total:
            L = total - s
        lens.append(L)
        s += L
        if s == total:
            break
    x = make_varlen_inputs(lens, lens, Hq, Hkv, d, seed=1, device="cuda")
    mx = max(lens)
    o, lse = attn_fwd_varlen(x["Q"], x["K"], x["V"], x["cu_q"], x["cu_k"], mx, mx, causal)
    ws = torch.empty(int(2 * len(lens) * Hq * ((mx + 127) // 128 * 128) + 64), dtype=torch.float32, device="cuda")
    fws = torch.empty(64, dtype=torch.int32, device="cuda")
    t_fs = timed(lambda: attn_fwd_varlen(x["Q"], x["K"], x["V"], x["cu_q"], x["cu_k"], mx, mx, causal, out=o, lse=lse,
                                         dynamic=False), a.iters)
    t_f = timed(lambda: attn_fwd_varlen(x["Q"], x["K"], x["V"], x["cu_q"], x["cu_k"], mx, mx, causal, out=o, lse=lse,
                                        workspace=fws), a.iters)
    g = [torch.empty_like(x[n]) for n in ("Q", "K", "V")]
    t_b = timed(lambda: attn_bwd_varlen(x["Q"], x["K"], x["V"], o, lse, x["dO"], x["cu_q"], x["cu_k"], mx, mx, causal,
                                        workspace=ws, dq=g[0], dk=g[1], dv=g[2]), a.iters)
    npairs = sum(pairs(L, L, causal) for L in lens)
    report("varlen_C3_docs", {"docs": len(lens), "tokens": total, "max_len": mx, "Hq": Hq, "Hkv": Hkv, "d": d,
                              "causal": causal, "fwd_schedule": "dynamic",
                              "fwd_tflops_static_schedule": round(4.0 * d * Hq * npairs / t_fs / 1e9, 1)},
           npairs, Hq, d, t_f, t_b, peak)
    del x, o, lse, ws, g
    y = make_inputs(16, 8192, Hq, Hkv, d, seed=1, device="cuda")
    o, lse = attn_fwd(y["Q"], y["K"], y["V"], causal)
    t_f = timed(lambda: attn_fwd(y["Q"], y["K"], y["V"], causal, out=o, lse=lse), a.iters)
    g = [torch.empty_like(y[n]) for n in ("Q", "K", "V")]
    t_b = timed(lambda: attn_bwd(y["Q"], y["K"], y["V"], o, lse, y["dO"], causal, dq=g[0], dk=g[1], dv=g[2]),
                a.iters)
    report("dense_C3_same_tokens", {"B": 16, "N": 8192, "Hq": Hq, "Hkv": Hkv, "d": d, "causal": causal},
           16 * pairs(8192, 8192, causal), Hq, d, t_f, t_b, peak)
    del y, o, lse, g

    # (b) Nq != Nk
    for Nq, Nk in ((1024, 16384), (4096, 8192)):
        z = make_qk_inputs(16, Nq, Nk, Hq, Hkv, d, seed=2, device="cuda")
        for c in (False, True):
            o, lse = attn_fwd(z["Q"], z["K"], z["V"], c)
            t_f = timed(lambda: attn_fwd(z["Q"], z["K"], z["V"], c, out=o, lse=lse), a.iters)
            g = [torch.empty_like(z[n]) for n in ("Q", "K", "V")]
            t_b = timed(lambda: attn_bwd(z["Q"], z["K"], z["V"], o, lse, z["dO"], c, dq=g[0], dk=g[1], dv=g[2]),
                        a.iters)
            report("qk", {"B": 16, "Nq": Nq, "Nk": Nk, "Hq": Hq, "Hkv": Hkv, "d": d, "causal": c},
                   16 * pairs(Nq, Nk, c), Hq, d, t_f, t_b, peak)
            del o, lse, g
        del z


if __name__ == "__main__":
    main()
