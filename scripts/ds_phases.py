"""Per-phase times (hk_diag_bwd_phase: 0 preprocess, 1 dK/dV, 2 dQ) of the two-pass and the
stored-dS backward (the workspace size selects the path). Usage: python scripts/ds_phases.py C3"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import _lib, api  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402

for name in (sys.argv[1] if len(sys.argv) > 1 else "C3").split(","):
    B, N, Hq, Hkv, d, causal = CONFIGS[name]
    x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
    dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
    L = _lib.diag()
    P = api._ptr
    res = {"config": name}
    for tag, nb in (("two_pass", api.bwd_workspace_bytes(B, Hq, Hkv, N, d)),
                    ("stored_ds", api.bwd_ds_workspace_bytes(B, Hq, Hkv, N, d, None, causal))):
        ws = torch.zeros((nb + 3) // 4, device="cuda")

        def ph(k):
            _lib.check_diag(L.hk_diag_bwd_phase(k, P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq),
                                                P(dk), P(dv), P(ws), ws.numel() * 4, B, Hq, Hkv, N, d, int(causal),
                                                api._stream()))
        t = {0: [], 1: [], 2: []}
        for _ in range(5):
            for k in (0, 1, 2):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                ph(k)
                e.record()
                torch.cuda.synchronize()
                t[k].append(s.elapsed_time(e))
        res[tag] = {n: round(statistics.median(t[k][1:]), 3) for k, n in ((0, "pre"), (1, "dkdv"), (2, "dq"))}
        del ws
        torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)
