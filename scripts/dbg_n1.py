import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
from paper_2511_08083_b200 import attn_bwd, attn_fwd  # noqa: E402
from util import gen, np64  # noqa: E402

for (B, N, Hq, Hkv, d, causal) in [(1, 1, 2, 1, 64, 0), (1, 1, 2, 1, 128, 0), (1, 2, 2, 1, 64, 0), (1, 3, 1, 1, 64, 1)]:
    x = gen(B, N, Hq, Hkv, d, seed=7 * N + d)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], bool(causal))
    dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], bool(causal))
    torch.cuda.synchronize()
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), bool(causal))
    print((B, N, Hq, Hkv, d, causal), "lse", np64(lse).ravel()[:4], ref["LSE"].ravel()[:4])
    for n, t in (("dQ", dq), ("dK", dk), ("dV", dv)):
        g = np64(t)
        print("  ", n, "maxabs err", float(np.abs(g - ref[n]).max()), "ref norm", float(np.linalg.norm(ref[n])),
              "got[0,0,0,:4]", g.reshape(-1)[:4], "ref", ref[n].reshape(-1)[:4])
