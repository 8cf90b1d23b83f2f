"""One forward + backward-phase launch sequence of a BASELINE config through the diagnostics ABI
(for ncu captures of a library variant): HK_LIB=<variant> python scripts/run_bwd_phase.py C2-nc 1"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import _lib, api  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402

B, N, Hq, Hkv, d, causal = CONFIGS[sys.argv[1]]
phase = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
ws = torch.zeros(api.bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4 + 64, device="cuda")
L = _lib.diag()
P = api._ptr
for ph in (0, phase, phase):
    _lib.check_diag(L.hk_diag_bwd_phase(ph, P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk),
                                        P(dv), P(ws), ws.numel() * 4, B, Hq, Hkv, N, d, int(causal), api._stream()))
torch.cuda.synchronize()
