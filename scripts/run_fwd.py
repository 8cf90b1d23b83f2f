"""One forward launch of a BASELINE config through the public API (for ncu captures of a
library variant: HK_LIB=<variant> python scripts/run_fwd.py C2-nc)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import attn_fwd  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402

B, N, Hq, Hkv, d, causal = CONFIGS[sys.argv[1]]
x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    attn_fwd(x["Q"], x["K"], x["V"], causal)
torch.cuda.synchronize()
