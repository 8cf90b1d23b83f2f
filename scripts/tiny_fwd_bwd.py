"""Small fwd+bwd+GEMM for sanitizer runs (scripts/sanitize.sh). Sizes are chosen so
the persistent kernels hand several items to each CTA (items > SMs) and the
dynamic scheduler, the cross-item barrier phases and the GEMM's CTA-pair
pipeline are all exercised."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2511_08083_b200 import attn_bwd, attn_fwd, gemm  # noqa: E402
from paper_2511_08083_b200.inputs import make_gemm_inputs, make_inputs  # noqa: E402

# (B, N, Hq, Hkv, d, causal): fwd 512 items, dQ 1024 items (> 148 SMs), dK/dV 256 items (MHA case)
for B, N, Hq, Hkv, d, causal in ((2, 1024, 64, 8, 128, True), (2, 1024, 16, 16, 64, False),
                                 (1, 200, 2, 1, 128, True)):
    x = make_inputs(B, N, Hq, Hkv, d, seed=1, device="cuda")
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
for M, N, K in ((4096, 4096, 128), (2048, 4096, 192)):  # 128 pair tiles (wide), 128 narrow-able
    g = make_gemm_inputs(M, N, K, seed=2, device="cuda")
    gemm(g["A"], g["B"])
torch.cuda.synchronize()
print("tiny fwd+bwd+gemm ran")
