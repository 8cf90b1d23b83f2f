"""Interleaved A/B of hk_rope between two library builds (B=16, H=16, d=128, N in 1K/4K/16K)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200.inputs import make_rope_inputs  # noqa: E402


def load(path):
    L = ctypes.CDLL(os.path.abspath(path))
    vp, i = ctypes.c_void_p, ctypes.c_int
    L.hk_rope.argtypes = [vp, vp, vp, vp, i, i, i, i, vp]
    return L


libs = [load(a) for a in sys.argv[1:3]]
B, H, d = 16, 16, 128
for N in (1024, 4096, 16384):
    x = make_rope_inputs(B, N, H, d, seed=N, device="cuda")["x"]
    cos = torch.rand(N, d // 2, device="cuda")
    sin = torch.rand(N, d // 2, device="cuda")
    out = torch.empty_like(x)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = []
    for L in libs:
        for _ in range(5):
            assert L.hk_rope(P(x), P(cos), P(sin), P(out), B, N, H, d, sp) == 0
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            L.hk_rope(P(x), P(cos), P(sin), P(out), B, N, H, d, sp)
        e.record()
        torch.cuda.synchronize()
        res.append(s.elapsed_time(e) / 50)
    ref = out.clone()
    libs[0].hk_rope(P(x), P(cos), P(sin), P(out), B, N, H, d, sp)
    torch.cuda.synchronize()
    same = torch.equal(ref, out)
    nbytes = 4 * B * N * H * d
    print(json.dumps({"N": N, "A_ms": round(res[0], 4), "B_ms": round(res[1], 4), "A_GBs": round(nbytes / res[0] / 1e6),
                      "B_GBs": round(nbytes / res[1] / 1e6), "bitwise_equal": same}))
