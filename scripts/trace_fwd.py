"""Per-tile timeline of the forward kernel from the HK_TRACE build (one CTA in
the middle of the grid): softmax wait for S, softmax duration X, the
P-published -> next-S-ready chain, and MMA issue lag. HK_LIB=trace required."""
import ctypes
import json
import os
import statistics as st
import sys

import numpy as np
import torch

os.environ["HK_LIB"] = "trace"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import _lib, attn_fwd  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2-nc"
shapes = {"C2-nc": (16, 4096, 16, 16, 128, False), "C3": (16, 8192, 32, 8, 128, True),
          "C4-8192": (16, 8192, 32, 32, 64, True)}
B, N, Hq, Hkv, d, causal = shapes[cfg]
x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
L = _lib.lib()
attn_fwd(x["Q"], x["K"], x["V"], causal)
torch.cuda.synchronize()
buf = np.zeros(1 << 17, dtype=np.uint64)
L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1)
attn_fwd(x["Q"], x["K"], x["V"], causal)
torch.cuda.synchronize()
_lib.check(L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1))
n = int(buf[0])
w = buf[1:1 + n].reshape(-1, 2)
ev = {}
for hdr, clk in w:
    e, a, b = int(hdr) >> 48, (int(hdr) >> 32) & 0xFFFF, int(hdr) & 0xFFFFFFFF
    ev[(e, a, b)] = int(clk)
t0 = min(ev.values())
res = {}
for t in (0, 1):
    js = sorted(b for (e, a, b) in ev if e == 2 and a == t)
    if not js:
        continue
    wait = [ev[(2, t, j)] - ev[(1, t, j)] for j in js if (1, t, j) in ev]
    X = [ev[(3, t, j)] - ev[(2, t, j)] for j in js if (3, t, j) in ev]
    chain = [ev[(2, t, j + 1)] - ev[(3, t, j)] for j in js if (2, t, j + 1) in ev and (3, t, j) in ev]
    lag = [ev[(10 + t, j, 0)] - ev[(3, t, j)] for j in js if (10 + t, j, 0) in ev and (3, t, j) in ev]
    period = [ev[(2, t, j + 1)] - ev[(2, t, j)] for j in js if (2, t, j + 1) in ev]
    f = lambda v: round(st.median(v), 1) if v else None
    res[f"tile{t}"] = {"n": len(js), "wait_for_S": f(wait), "softmax_X": f(X), "P_to_nextS": f(chain),
                       "mma_lag_after_P": f(lag), "period": f(period)}
print(json.dumps(res, indent=1))
