"""Item-boundary cost in the persistent forward (HK_TRACE build, one CTA): the S-ready
-> S-ready period of consecutive steps of a Q tile, split into steps inside an item and
steps that cross into the next item (epilogue + next item's start). HK_LIB=trace."""
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

shapes = {"C5-1024-c": (16, 1024, 64, 8, 128, True), "C5-1024-nc": (16, 1024, 64, 8, 128, False),
          "qk-c": (16, 1024, 32, 8, 128, True, 16384), "qk-nc": (16, 1024, 32, 8, 128, False, 16384),
          "C3": (16, 8192, 32, 8, 128, True), "C4-2048": (16, 2048, 32, 32, 64, True)}
for cfg in sys.argv[1:]:
    B, N, Hq, Hkv, d, causal = shapes[cfg][:6]
    if len(shapes[cfg]) > 6:  # Nq != Nk
        from paper_2511_08083_b200.inputs import make_qk_inputs
        x = make_qk_inputs(B, N, shapes[cfg][6], Hq, Hkv, d, seed=0, device="cuda")
    else:
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
    out = {"config": cfg}
    for t in (0, 1):
        S = [int(tab[2 + 4 * t, a]) for a in range(1024) if tab[2 + 4 * t, a]]
        ep = sorted(int(tab[31 + t, a]) for a in range(1024) if tab[31 + t, a])
        inside, cross = [], []
        for a, b in zip(S, S[1:]):
            (cross if any(a < e < b for e in ep) else inside).append(b - a)
        X = [int(tab[3 + 4 * t, a]) - int(tab[2 + 4 * t, a]) for a in range(1024)
             if tab[2 + 4 * t, a] and tab[3 + 4 * t, a]]
        out[f"tile{t}"] = {"steps": len(S), "items": len(ep),
                           "period_inside_item": round(st.median(inside), 0) if inside else None,
                           "period_across_items": round(st.median(cross), 0) if cross else None,
                           "softmax_step": round(st.median(X), 0) if X else None}
    print(json.dumps(out), flush=True)
    del x
