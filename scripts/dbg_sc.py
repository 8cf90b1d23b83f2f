"""Tiny forward with a chosen library variant (HK_LIB) against the oracle; prints max errors."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2511_08083_b200 import attn_fwd
from paper_2511_08083_b200.inputs import make_inputs
for (B, N, Hq, Hkv, d, c) in ((1, 256, 2, 1, 128, False), (1, 512, 4, 2, 128, True), (1, 333, 2, 2, 64, True)):
    x = make_inputs(B, N, Hq, Hkv, d, seed=1, device="cuda")
    o, l = attn_fwd(x["Q"], x["K"], x["V"], c)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy().astype(np.float64)
    O, L = oracle.attn_fwd(f(x["Q"]), f(x["K"]), f(x["V"]), c)
    print((B, N, Hq, Hkv, d, c), "O", np.abs(f(o) - O).max(), "LSE", np.abs(f(l) - L).max(), flush=True)
