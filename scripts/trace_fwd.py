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
          "C5-1024-c": (16, 1024, 64, 8, 128, True), "C5-1024-nc": (16, 1024, 64, 8, 128, False),
          "C4-8192": (16, 8192, 32, 32, 64, True)}
B, N, Hq, Hkv, d, causal = shapes[cfg]
x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
L = _lib.diag()
attn_fwd(x["Q"], x["K"], x["V"], causal)
torch.cuda.synchronize()
buf = np.zeros(64 * 1024, dtype=np.uint64)
L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1)
attn_fwd(x["Q"], x["K"], x["V"], causal)
torch.cuda.synchronize()
_lib.check_diag(L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1))
tab = buf.reshape(64, 1024)
ev = {(e, a): int(tab[e, a]) for e in range(64) for a in range(1024) if tab[e, a]}
res = {}
f = lambda v: round(st.median(v), 1) if v else None
for t in (0, 1):  # t = softmax warpgroup (column half)
    js = sorted(a for (e, a) in ev if e == 2 + 4 * t)
    if not js:
        continue
    E = lambda k, j: ev.get((k + 4 * t, j))
    d = lambda a, b: [b_ - a_ for a_, b_ in zip(a, b) if a_ and b_]
    wait = d([E(1, j) for j in js], [E(2, j) for j in js])
    X = d([E(2, j) for j in js], [E(3, j) for j in js])
    chain = d([E(3, j) for j in js], [E(2, j + 1) for j in js])
    lag = d([E(3, j) for j in js], [ev.get((10, j)) for j in js])
    period = d([E(2, j) for j in js], [E(2, j + 1) for j in js])
    sub = {}
    marks = [(2 + 4 * t, "S_ready"), (40 + 4 * t, "S_loaded"), (41 + 4 * t, "max_done"), (42 + 4 * t, "exps_done"),
             (43 + 4 * t, "st_done"), (3 + 4 * t, "P_pub")]
    for (e1, n1), (e2, n2) in zip(marks, marks[1:]):
        v = d([ev.get((e1, j)) for j in js], [ev.get((e2, j)) for j in js])
        if v:
            sub[f"{n1}->{n2}"] = f(v)
    res[f"tile{t}"] = {"n": len(js), "wait_for_S": f(wait), "softmax_X": f(X), "P_to_nextS": f(chain),
                       "mma_lag_after_P": f(lag), "period": f(period), "softmax_parts": sub}
t0c = ev.get((30, 0))
if t0c:
    firstS = min(v for (e, a), v in ev.items() if e in (2, 6) and a == 0)
    lastP = max(v for (e, a), v in ev.items() if e in (3, 7))
    end = max(ev.get((31, 0), 0), ev.get((32, 0), 0))
    res["cta"] = {"start_to_first_S": firstS - t0c, "first_S_to_last_P": lastP - firstS,
                  "last_P_to_epilogue_end": end - lastP, "total": end - t0c}
print(json.dumps(res, indent=1))
