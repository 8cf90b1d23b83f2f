import os, sys, json, statistics, torch
sys.path.insert(0, "/root/repo")
from paper_2511_08083_b200 import gemm
from paper_2511_08083_b200.inputs import make_gemm_inputs
for M, N, K in ((8192, 8192, 8192), (16384, 16384, 8192), (4096, 4096, 4096)):
    x = make_gemm_inputs(M, N, K, seed=0, device="cuda"); A, B = x["A"], x["B"]
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    def run(mode):
        if mode == "narrow": os.environ["HK_GEMM_NARROW"] = "1"
        else: os.environ.pop("HK_GEMM_NARROW", None)
        return (lambda: torch.matmul(A, B.t())) if mode == "cublas" else (lambda: gemm(A, B, out=C))
    t = {m: [] for m in ("wide", "narrow", "cublas")}
    for rep in range(6):
        for m in (("wide", "narrow", "cublas") if rep % 2 == 0 else ("cublas", "narrow", "wide")):
            f = run(m)
            for _ in range(3): f()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); s.record()
            for _ in range(20): f()
            e.record(); torch.cuda.synchronize(); t[m].append(s.elapsed_time(e) / 20)
    fl = 2.0 * M * N * K
    print(json.dumps({"shape": [M, N, K], **{m: round(fl / statistics.median(v) / 1e9, 1) for m, v in t.items()}}), flush=True)
