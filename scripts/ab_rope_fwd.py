"""NEXT #3 cost check: hk_attn_fwd_rope (Q rotated in the forward kernel, K rotated once into Kr) vs
hk_attn_fwd on the same (unrotated) inputs, interleaved, CUDA events; also vs the unfused
hk_rope(Q) + hk_rope(K) + hk_attn_fwd. One JSON line per config."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (only for the cos/sin tables)
from paper_2511_08083_b200 import attn_fwd, attn_fwd_rope, rope  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

CONFIGS = {"C3": (16, 8192, 32, 8, 128, True), "C2-nc": (16, 4096, 16, 16, 128, False),
           "C4-8192": (16, 8192, 32, 32, 64, True), "C5-1024-c": (16, 1024, 64, 8, 128, True)}


def timed(f, iters=5):
    f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else CONFIGS):
    B, N, Hq, Hkv, d, causal = CONFIGS[name]
    x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    c, s = oracle.rope_tables(N, d)
    c = torch.from_numpy(c.astype(np.float32)).cuda()
    s = torch.from_numpy(s.astype(np.float32)).cuda()
    o, lse, kr = torch.empty_like(x["Q"]), torch.empty(B, Hq, N, device="cuda"), torch.empty_like(x["K"])
    qr = torch.empty_like(x["Q"])
    runs = {"plain": lambda: attn_fwd(x["Q"], x["K"], x["V"], causal, out=o, lse=lse),
            "fused_rope": lambda: attn_fwd_rope(x["Q"], x["K"], x["V"], c, s, causal, out=o, lse=lse, k_rot=kr),
            "unfused_rope": lambda: (rope(x["Q"], c, s, out=qr), rope(x["K"], c, s, out=kr),
                                     attn_fwd(qr, kr, x["V"], causal, out=o, lse=lse))}
    t = {k: [] for k in runs}
    for rep in range(5):
        for k in (list(runs) if rep % 2 == 0 else list(runs)[::-1]):
            t[k].append(timed(runs[k]))
    m = {k: statistics.median(v) for k, v in t.items()}
    print(json.dumps({"config": name, **{k + "_ms": round(v, 4) for k, v in m.items()},
                      "fused_vs_plain": round(m["plain"] / m["fused_rope"], 4),
                      "fused_vs_unfused": round(m["unfused_rope"] / m["fused_rope"], 4)}), flush=True)
    del x
