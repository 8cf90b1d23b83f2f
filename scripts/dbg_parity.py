"""Print bwd/fwd parity errors for a list of small cases (debugging aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
from paper_2511_08083_b200 import attn_bwd, attn_fwd  # noqa: E402
from util import gen, np64, rel_l2  # noqa: E402

cases = [tuple(int(v) for v in c.split(",")) for c in sys.argv[1:]]
for B, N, Hq, Hkv, d, causal in cases:
    x = gen(B, N, Hq, Hkv, d, seed=7 * N + d)
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], bool(causal))
    dq, dk, dv = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], bool(causal))
    torch.cuda.synchronize()
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), bool(causal))
    e = {n: round(rel_l2(np64(t), ref[n]), 5) for n, t in (("dQ", dq), ("dK", dk), ("dV", dv))}
    bad = ""
    if e["dK"] > 0.01:
        err = np.linalg.norm((np64(dk) - ref["dK"]).reshape(B, N // 128, 128, Hkv, d), axis=(2, 4))
        bad = " dK err by (b, key tile, kvh): " + str(np.round(err, 2).tolist())
    print((B, N, Hq, Hkv, d, causal), e, bad, flush=True)
