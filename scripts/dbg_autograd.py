import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2511_08083_b200 import api  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

orig = api.attn_bwd


def spy(q, k, v, o, lse, do, causal=False, **kw):
    for n, t in (("q", q), ("k", k), ("v", v), ("o", o), ("lse", lse), ("do", do)):
        print(n, tuple(t.shape), t.stride(), t.dtype, hex(t.data_ptr()), t.is_contiguous(), flush=True)
    return orig(q, k, v, o, lse, do, causal, **kw)


api.attn_bwd = spy
x = make_inputs(1, 384, 4, 2, 128, seed=21, device="cuda")
q, k, v = (x[n].clone().requires_grad_() for n in ("Q", "K", "V"))
o = api.Attention.apply(q, k, v, False)
print("o", o.stride(), o.is_contiguous())
try:
    o.backward(x["dO"])
    torch.cuda.synchronize()
    print("ok")
except Exception as e:
    print("ERR", e)

import threading  # noqa: E402

res = {}


def worker():
    try:
        o2, l2 = api.attn_fwd(x["Q"], x["K"], x["V"], False)
        orig(x["Q"], x["K"], x["V"], o2, l2, x["dO"], False)
        torch.cuda.synchronize()
        res["ok"] = True
    except Exception as e:
        res["err"] = str(e)


th = threading.Thread(target=worker)
th.start()
th.join()
print("python thread:", res)
