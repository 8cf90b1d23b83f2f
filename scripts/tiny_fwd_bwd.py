"""Tiny fwd+bwd for sanitizer runs (scripts/sanitize.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2511_08083_b200 import attn_bwd, attn_fwd  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

for d, causal in ((128, True), (64, False)):
    x = make_inputs(1, 256, 2, 1, d, seed=1, device="cuda")
    o, l = attn_fwd(x["Q"], x["K"], x["V"], causal)
    attn_bwd(x["Q"], x["K"], x["V"], o, l, x["dO"], causal)
torch.cuda.synchronize()
print("tiny fwd+bwd ran")
