"""Per-iteration timeline of the backward kernels from the HK_TRACE build (one
CTA in the middle of the grid). HK_LIB=trace is set here."""
import ctypes
import json
import os
import statistics as st
import sys

import numpy as np
import torch

os.environ["HK_LIB"] = "trace"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import _lib, attn_fwd, bwd_workspace_bytes  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2-nc"
shapes = {"C2-nc": (16, 4096, 16, 16, 128, False), "C3": (16, 8192, 32, 8, 128, True),
          "C4-8192": (16, 8192, 32, 32, 64, True), "C5-4096-nc": (16, 4096, 64, 8, 128, False)}
B, N, Hq, Hkv, d, causal = shapes[cfg]
x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
L = _lib.diag()
o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
ws = torch.empty(bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
buf = np.zeros(64 * 1024, dtype=np.uint64)


def run(phase):
    _lib.check_diag(L.hk_diag_bwd_phase(phase, P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk),
                                   P(dv), P(ws), ws.numel() * 4, B, Hq, Hkv, N, d, int(causal), None))
    torch.cuda.synchronize()


run(0)
out = {}
for phase, name in ((1, "dkdv"), (2, "dq")):
    run(phase)
    L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1)
    run(phase)
    _lib.check_diag(L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1))
    tab = buf.reshape(64, 1024)
    ev = {(e, a): int(tab[e, a]) for e in range(64) for a in range(1024) if tab[e, a]}
    its = sorted(a for (e, a) in ev if e == 2)
    f = lambda v: round(st.median(v), 1) if v else None
    g = lambda e1, e2, k=0: [ev[(e2, i + k)] - ev[(e1, i)] for i in its if (e1, i) in ev and (e2, i + k) in ev]
    out[name] = {"iters": len(its), "wait_S": f(g(1, 2)), "P_phase": f(g(2, 3)), "wait_dP": f(g(3, 4)),
                 "dS_phase": f(g(4, 5)), "dS_to_mma": f(g(5, 11)), "P_to_mma": f(g(3, 10)),
                 "period": f(g(2, 2, 1)), "total_cycles": max(ev.values()) - min(ev.values()),
                 "mma_wait_stage": f(g(12, 13)), "load_issue_to_landed": f(g(20, 13)),
                 "load_issue_lead_before_needed": f(g(20, 12)),
                 "mma_dV_to_S": f(g(10, 13, 1)), "mma_S_to_dK": f([ev[(11, i)] - ev[(13, i + 1)] for i in its
                                                                   if (11, i) in ev and (13, i + 1) in ev]),
                 "mma_dK_to_dP": f(g(11, 14, 1)), "mma_dP_to_nextdV": f(g(14, 10)),
                 "mma_dV_period": f(g(10, 10, 1)),
                 "mma_S_to_dQ(dq)": f(g(13, 11)) if name == "dq" else None,
                 "mma_dQ_to_dP(dq)": f(g(11, 14, 1)) if name == "dq" else None,
                 "mma_dQ_period(dq)": f(g(11, 11, 1)) if name == "dq" else None}
print(json.dumps(out, indent=1))
