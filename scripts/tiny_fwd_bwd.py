"""Small fwd+bwd+GEMM for sanitizer runs (scripts/sanitize.sh). Sizes are chosen so
the persistent kernels hand several items to each CTA (items > SMs) and the
dynamic scheduler, the cross-item barrier phases and the GEMM's CTA-pair
pipeline are all exercised."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2511_08083_b200 import (attn_bwd, attn_bwd_varlen, attn_fwd, attn_fwd_varlen, bwd_workspace_bytes,  # noqa: E402
                                   gemm, ring)
from paper_2511_08083_b200.inputs import make_gemm_inputs, make_inputs, make_qk_inputs, make_varlen_inputs  # noqa: E402

# (B, N, Hq, Hkv, d, causal): fwd 512 items, dQ 1024 items (> 148 SMs), dK/dV 256 items (MHA case)
for B, N, Hq, Hkv, d, causal in ((2, 1024, 64, 8, 128, True), (2, 1024, 16, 16, 64, False),
                                 (1, 200, 2, 1, 128, True)):
    x = make_inputs(B, N, Hq, Hkv, d, seed=1, device="cuda")
    o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
    attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)  # d = 128: the stored-dS backward
    ws = torch.empty(bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4, dtype=torch.float32, device="cuda")
    attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=ws)  # the two-pass backward
for M, N, K in ((4096, 4096, 128), (2048, 4096, 192)):  # 128 pair tiles (wide), 128 narrow-able
    g = make_gemm_inputs(M, N, K, seed=2, device="cuda")
    gemm(g["A"], g["B"])
# NEXT #4: Nq != Nk (incl. key-less rows), packed varlen with empty sequences, ring merge/accumulate
for Nq, Nk in ((384, 200), (100, 700)):
    z = make_qk_inputs(2, Nq, Nk, 8, 2, 128, seed=3, device="cuda")
    o, lse = attn_fwd(z["Q"], z["K"], z["V"], True)
    attn_bwd(z["Q"], z["K"], z["V"], o, lse, z["dO"], True)
v = make_varlen_inputs([300, 0, 129, 1000], [200, 50, 0, 1000], 8, 2, 64, seed=4, device="cuda")
for causal in (False, True):
    o, lse = attn_fwd_varlen(v["Q"], v["K"], v["V"], v["cu_q"], v["cu_k"], 1000, 1000, causal)
    attn_bwd_varlen(v["Q"], v["K"], v["V"], o, lse, v["dO"], v["cu_q"], v["cu_k"], 1000, 1000, causal)
x = make_inputs(1, 1024, 4, 2, 128, seed=5, device="cuda")
sh = {n: [ring.zigzag_shard(x[n], 2, r) for r in range(2)] for n in ("Q", "K", "V", "dO")}
fw = ring.ring_attn_fwd(sh["Q"], sh["K"], sh["V"], True, ring.LoopbackRing(2))
ring.ring_attn_bwd(sh["Q"], sh["K"], sh["V"], [f[0] for f in fw], [f[1] for f in fw], sh["dO"], True,
                   ring.LoopbackRing(2))
torch.cuda.synchronize()
print("tiny fwd+bwd+gemm+varlen+ring ran")
