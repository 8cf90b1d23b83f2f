"""Forward timing of Nq != Nk shapes, causal (bottom-right) vs non-causal (probe, not the bench)."""
import sys, torch, json
sys.path.insert(0, '/root/repo')
from paper_2511_08083_b200 import attn_fwd
from paper_2511_08083_b200.inputs import make_qk_inputs
def timed(fn, iters=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
for (B,Nq,Nk) in ((16,1024,16384),(16,1024,16256),(16,2048,16384),(4,4096,16384),(1,16384,16384)):
    x = make_qk_inputs(B, Nq, Nk, 32, 8, 128, seed=1, device="cuda")
    r = {}
    for c in (False, True):
        o, l = attn_fwd(x["Q"], x["K"], x["V"], c)
        r["causal" if c else "noncausal"] = round(timed(lambda: attn_fwd(x["Q"], x["K"], x["V"], c, out=o, lse=l)), 4)
    print(json.dumps({"B": B, "Nq": Nq, "Nk": Nk, **r}))
