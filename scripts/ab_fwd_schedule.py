"""A/B of the forward's work schedule on dense configs: dense static snake vs the same
batch through the varlen entry point (uniform lengths) with the static and the dynamic
scheduler. Prints min-of-3 ms per variant."""
import sys, torch, json
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2511_08083_b200 import attn_fwd, attn_fwd_varlen
from paper_2511_08083_b200.inputs import make_inputs
def timed(fn, iters=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
for (B,N,Hq,Hkv,d,c) in ((16,8192,32,8,128,True),(16,4096,16,16,128,False),(16,8192,32,32,64,True),(16,1024,64,8,128,True)):
    x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    cu = torch.arange(0, (B+1)*N, N, dtype=torch.int32, device="cuda")
    fl = lambda t: t.reshape(B*N, t.shape[2], d)
    q,k,v = fl(x["Q"]), fl(x["K"]), fl(x["V"])
    ws = torch.empty(64, dtype=torch.int32, device="cuda")
    o, l = attn_fwd(x["Q"], x["K"], x["V"], c)
    ov, lv = attn_fwd_varlen(q,k,v,cu,cu,N,N,c,workspace=ws)
    res = {}
    for rep in range(3):
        res.setdefault("dense_static",[]).append(timed(lambda: attn_fwd(x["Q"], x["K"], x["V"], c, out=o, lse=l)))
        res.setdefault("varlen_static",[]).append(timed(lambda: attn_fwd_varlen(q,k,v,cu,cu,N,N,c,out=ov,lse=lv,dynamic=False)))
        res.setdefault("varlen_dyn",[]).append(timed(lambda: attn_fwd_varlen(q,k,v,cu,cu,N,N,c,out=ov,lse=lv,workspace=ws)))
    print(json.dumps({"cfg": [B,N,Hq,Hkv,d,c], **{k_: round(min(v_),4) for k_,v_ in res.items()}}))
    del x
