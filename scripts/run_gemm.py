"""One 8192^3 GEMM each through our kernel and cuBLAS (torch.matmul), for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import gemm  # noqa: E402
from paper_2511_08083_b200.inputs import make_gemm_inputs  # noqa: E402

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x = make_gemm_inputs(M, N, K, seed=0, device="cuda")
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    gemm(x["A"], x["B"], out=C)
    torch.matmul(x["A"], x["B"].t())
torch.cuda.synchronize()
