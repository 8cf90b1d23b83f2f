"""Forward error on the std-4 stress inputs (tests/test_gpu_fwd.py::test_fwd_stress_std4) against the
strict BASELINE bound (max-abs 2e-2), with the rows/columns where it peaks: evidence for DESIGN.md
reading #24."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2511_08083_b200 import attn_fwd  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

for causal in (False, True):
    for seed in (3, 4, 5):
        x = make_inputs(1, 512, 2, 1, 128, seed=seed, device="cuda", std_qk=4.0)
        o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
        torch.cuda.synchronize()
        f = lambda t: t.float().cpu().numpy().astype(np.float64)
        O, L = oracle.attn_fwd(f(x["Q"]), f(x["K"]), f(x["V"]), causal)
        e = np.abs(f(o) - O)
        i = np.unravel_index(e.argmax(), e.shape)
        print(json.dumps({"causal": causal, "seed": seed, "O_maxabs": float(e.max()), "at": [int(v) for v in i],
                          "O_ref_there": float(O[i]), "O_absmax": float(np.abs(O).max()),
                          "bf16_ulp_of_ref": float(2.0 ** (np.floor(np.log2(abs(O[i]))) - 7)) if O[i] else 0.0,
                          "LSE_maxabs": float(np.abs(f(lse) - L).max()),
                          "strict_pass": bool(e.max() <= 2e-2)}))
