"""The d = 128 dK/dV pass on CTA pairs (-DHK_DKDV2=1 build) against the 1-CTA pass: bitwise dK, dV
(and dQ) on a set of shapes, then interleaved timing of the dK/dV phase on BASELINE configs.
Usage: python scripts/ab_dkdv2.py --a paper_2511_08083_b200/libhkattn_base.so \
           --b paper_2511_08083_b200/libhkattn_dkdv2.so [--configs C3,C2-nc] [--check-only]"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200.inputs import make_inputs, make_qk_inputs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import CONFIGS  # noqa: E402


def load(path):
    L = ctypes.CDLL(os.path.abspath(path))
    vp, i = ctypes.c_void_p, ctypes.c_int
    L.hk_attn_fwd_qk.argtypes = [vp] * 5 + [i] * 7 + [vp]
    L.hk_attn_bwd_qk.argtypes = [vp] * 10 + [ctypes.c_size_t] + [i] * 7 + [vp]
    L.hk_attn_bwd_qk_workspace_bytes.restype = ctypes.c_size_t
    L.hk_attn_bwd_qk_workspace_bytes.argtypes = [i] * 6
    L.hk_diag_bwd_phase.argtypes = [i] + [vp] * 10 + [ctypes.c_size_t] + [i] * 6 + [vp]
    L.hk_attn_last_error.restype = ctypes.c_char_p
    return L


P = lambda t: ctypes.c_void_p(t.data_ptr())


def run_bwd(L, x, B, Nq, Nk, Hq, Hkv, d, causal):
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    o = torch.empty_like(x["Q"])
    lse = torch.empty(B, Hq, Nq, device="cuda", dtype=torch.float32)
    r = L.hk_attn_fwd_qk(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), B, Hq, Hkv, Nq, Nk, d, int(causal), sp)
    assert r == 0, L.hk_attn_last_error()
    ws = torch.zeros(L.hk_attn_bwd_qk_workspace_bytes(B, Hq, Hkv, Nq, Nk, d) // 4 + 64, device="cuda")
    dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
    r = L.hk_attn_bwd_qk(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk), P(dv), P(ws),
                         ws.numel() * 4, B, Hq, Hkv, Nq, Nk, d, int(causal), sp)
    assert r == 0, L.hk_attn_last_error()
    torch.cuda.synchronize()
    return dq, dk, dv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", required=True)
    ap.add_argument("--b", required=True)
    ap.add_argument("--configs", default="C3,C2-nc,C2-c,C5-1024-c,C5-16384-c")
    ap.add_argument("--check-only", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    LA, LB = load(a.a), load(a.b)
    shapes = [(1, 256, 256, 2, 1, False), (1, 256, 256, 2, 1, True), (2, 1000, 1000, 8, 2, True),
              (1, 384, 384, 4, 4, False), (2, 200, 700, 4, 2, True), (1, 777, 333, 6, 3, False),
              (2, 2048, 2048, 16, 4, True), (1, 128, 128, 1, 1, True)]
    for (B, Nq, Nk, Hq, Hkv, causal) in shapes:
        x = make_qk_inputs(B, Nq, Nk, Hq, Hkv, 128, seed=5, device="cuda")
        ga = run_bwd(LA, x, B, Nq, Nk, Hq, Hkv, 128, causal)
        gb = run_bwd(LB, x, B, Nq, Nk, Hq, Hkv, 128, causal)
        same = [bool(torch.equal(u, v)) for u, v in zip(ga, gb)]
        diff = [float((u.float() - v.float()).abs().max()) for u, v in zip(ga, gb)]
        print(json.dumps({"shape": [B, Nq, Nk, Hq, Hkv, causal], "bitwise_dq_dk_dv": same, "maxdiff": diff}),
              flush=True)
    if a.check_only:
        return
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for name in a.configs.split(","):
        B, N, Hq, Hkv, d, causal = CONFIGS[name]
        if d != 128:
            continue
        x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
        o = torch.empty_like(x["Q"])
        lse = torch.empty(B, Hq, N, device="cuda", dtype=torch.float32)
        LA.hk_attn_fwd_qk(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), B, Hq, Hkv, N, N, d, int(causal), sp)
        dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
        ws = torch.zeros(LA.hk_attn_bwd_qk_workspace_bytes(B, Hq, Hkv, N, N, d) // 4 + 64, device="cuda")

        def ph(L, k):
            r = L.hk_diag_bwd_phase(k, P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk),
                                    P(dv), P(ws), ws.numel() * 4, B, Hq, Hkv, N, d, int(causal), sp)
            assert r == 0
        ph(LA, 0)
        t = {"A": [], "B": []}
        for rep in range(a.reps):
            for tag in ("A", "B") if rep % 2 == 0 else ("B", "A"):
                L = LA if tag == "A" else LB
                ph(L, 1)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record()
                for _ in range(3):
                    ph(L, 1)
                e.record()
                torch.cuda.synchronize()
                t[tag].append(s.elapsed_time(e) / 3)
        ma, mb = statistics.median(t["A"]), statistics.median(t["B"])
        fl = 4 * 2 * B * Hq * N * N * d * (0.5 if causal else 1.0)
        print(json.dumps({"config": name, "dkdv_A_ms": round(ma, 4), "dkdv_B_ms": round(mb, 4),
                          "B_speedup": round(ma / mb, 4), "A_tflops": round(fl / ma / 1e9, 1),
                          "B_tflops": round(fl / mb / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
