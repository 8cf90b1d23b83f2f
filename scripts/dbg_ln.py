"""Debug: print the out_resid elements where the LN kernel and the oracle differ."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dropout_keep, layernorm_dropout_residual  # noqa: E402
from paper_2511_08083_b200 import ln_dropout_residual  # noqa: E402
from paper_2511_08083_b200.inputs import make_ln_inputs  # noqa: E402

rows, D, p, seed = 37, 2048, 0.1, 1234
x = make_ln_inputs(rows, D, seed=rows + D, device="cuda")
out, res = ln_dropout_residual(x["x"], x["residual"], x["weight"], x["bias"], p=p, seed=seed)
torch.cuda.synchronize()
f = lambda t: t.float().cpu().numpy().astype(np.float64)
p32 = float(np.float32(p))
_, r_ref = layernorm_dropout_residual(f(x["x"]), f(x["residual"]), f(x["weight"]), f(x["bias"]), p=p32, seed=seed)
g = f(res)
keep = dropout_keep(rows * D, p32, seed).reshape(rows, D)
bad = np.argwhere(np.abs(g - r_ref) > 2 ** -7 * np.abs(r_ref))
print("n bad", len(bad), "mask keep rate", keep.mean())
for r, c in bad[:10]:
    xv, rv = f(x["x"])[r, c], f(x["residual"])[r, c]
    print(r, c, "x", xv, "res", rv, "keep", keep[r, c], "gpu", g[r, c], "ref", r_ref[r, c],
          "exact", rv + (xv / (1 - p32) if keep[r, c] else 0.0))
