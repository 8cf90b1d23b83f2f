import os, sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/scripts")
from paper_2511_08083_b200 import _lib, api
from paper_2511_08083_b200.inputs import make_inputs
from probe import CONFIGS
B, N, Hq, Hkv, d, causal = CONFIGS[sys.argv[1]]
x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
nb = api.bwd_ds_workspace_bytes(B, Hq, Hkv, N, d, None, causal) if sys.argv[2] == "ds" else api.bwd_workspace_bytes(B, Hq, Hkv, N, d)
ws = torch.zeros((nb + 3) // 4, device="cuda")
L = _lib.diag(); P = api._ptr
for k in (0, 1, 2, 1, 2):
    _lib.check_diag(L.hk_diag_bwd_phase(k, P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk), P(dv), P(ws), ws.numel() * 4, B, Hq, Hkv, N, d, int(causal), api._stream()))
torch.cuda.synchronize()
