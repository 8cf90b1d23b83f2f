"""Debug helper: run fwd + hk_attn_bwd (and each bwd phase) of a saved build
libhkattn_<name>.so at a given config, printing statuses."""
import ctypes
import sys

import torch

sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/scripts')
from ab_step import load  # noqa: E402
from probe import CONFIGS  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

cfg = sys.argv[1]
for name in sys.argv[2:]:
    L = load(name)
    L.hk_diag_bwd_phase.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 10 + [ctypes.c_size_t] + [ctypes.c_int] * 6 + \
        [ctypes.c_void_p]
    B, N, Hq, Hkv, d, causal = CONFIGS[cfg]
    x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    o = torch.empty_like(x["Q"])
    lse = torch.empty(B, Hq, N, device="cuda")
    dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
    ws = torch.zeros(L.hk_attn_bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4 + 64, device="cuda")
    a = (P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse))
    print(name, "fwd", L.hk_attn_fwd(*a, B, Hq, Hkv, N, d, int(causal), None), L.hk_attn_last_error())
    g = (P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk), P(dv), P(ws), ws.numel() * 4,
         B, Hq, Hkv, N, d, int(causal), None)
    print(name, "bwd", L.hk_attn_bwd(*g), L.hk_attn_last_error())
    torch.cuda.synchronize()
    for ph in (0, 1, 2):
        r = L.hk_diag_bwd_phase(ph, *g)
        torch.cuda.synchronize()
        print(name, "phase", ph, r, L.hk_attn_last_error())
    del x
