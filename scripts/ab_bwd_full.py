"""Interleaved A/B of the full public hk_attn_bwd (preprocess + dK/dV + dQ, including the
dQ fork) between two library builds: python scripts/ab_bwd_full.py libA.so libB.so C3,C5-1024-c"""
import sys, os, ctypes, torch, json, statistics
_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(_root, 'scripts')); sys.path.insert(0, _root)
from probe import CONFIGS
from paper_2511_08083_b200.inputs import make_inputs
def load(path):
    L = ctypes.CDLL(os.path.abspath(path)); vp, i = ctypes.c_void_p, ctypes.c_int
    L.hk_attn_fwd.argtypes = [vp]*5 + [i]*6 + [vp]
    L.hk_attn_bwd.argtypes = [vp]*10 + [ctypes.c_size_t] + [i]*6 + [vp]
    L.hk_attn_bwd_workspace_bytes.restype = ctypes.c_size_t; L.hk_attn_bwd_workspace_bytes.argtypes = [i]*5
    return L
A, Bl = load(sys.argv[1]), load(sys.argv[2])
for name in sys.argv[3].split(","):
    B, N, Hq, Hkv, d, c = CONFIGS[name]
    x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr()); sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    o = torch.empty_like(x["Q"]); lse = torch.empty((B, Hq, N), dtype=torch.float32, device="cuda")
    dq, dk, dv = (torch.empty_like(x[n]) for n in ("Q", "K", "V"))
    ws = torch.empty(A.hk_attn_bwd_workspace_bytes(B, Hq, Hkv, N, d)//4 + 64, dtype=torch.float32, device="cuda")
    A.hk_attn_fwd(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), B, Hq, Hkv, N, d, int(c), sp)
    def bwd(L):
        assert L.hk_attn_bwd(P(x["Q"]), P(x["K"]), P(x["V"]), P(o), P(lse), P(x["dO"]), P(dq), P(dk), P(dv), P(ws), ws.numel()*4, B, Hq, Hkv, N, d, int(c), sp) == 0
    def t(L, it=10):
        for _ in range(3): bwd(L)
        torch.cuda.synchronize(); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(it): bwd(L)
        e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/it
    ra, rb = [], []
    for _ in range(5): ra.append(t(A)); rb.append(t(Bl))
    ma, mb = statistics.median(ra), statistics.median(rb)
    print(json.dumps({"config": name, "A_bwd_ms": round(ma,4), "B_bwd_ms": round(mb,4), "B_speedup": round(ma/mb,4)}))
    del x
