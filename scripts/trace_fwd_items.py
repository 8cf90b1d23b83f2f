"""Item-boundary cost in the persistent forward (HK_TRACE build, one CTA): the S-ready
-> S-ready period of consecutive steps of a Q tile, split into steps inside an item and
steps that cross into the next item (epilogue + next item's start). HK_LIB=trace."""
import ctypes
import json
import os
import statistics as st
import sys

import numpy as np
import torch

os.environ["HK_LIB"] = "trace"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import _lib, attn_fwd  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402

shapes = {"C5-1024-c": (16, 1024, 64, 8, 128, True), "C5-1024-nc": (16, 1024, 64, 8, 128, False),
          "qk-c": (16, 1024, 32, 8, 128, True, 16384), "qk-nc": (16, 1024, 32, 8, 128, False, 16384),
          "C3": (16, 8192, 32, 8, 128, True), "C4-2048": (16, 2048, 32, 32, 64, True)}
for cfg in sys.argv[1:]:
    B, N, Hq, Hkv, d, causal = shapes[cfg][:6]
    if len(shapes[cfg]) > 6:  # Nq != Nk
        from paper_2511_08083_b200.inputs import make_qk_inputs
        x = make_qk_inputs(B, N, shapes[cfg][6], Hq, Hkv, d, seed=0, device="cuda")
    else:
        x = make_inputs(B, N, Hq, Hkv, d, seed=0, device="cuda")
    L = _lib.diag()
    attn_fwd(x["Q"], x["K"], x["V"], causal)
    torch.cuda.synchronize()
    buf = np.zeros(64 * 1024, dtype=np.uint64)
    L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1)
    attn_fwd(x["Q"], x["K"], x["V"], causal)
    torch.cuda.synchronize()
    _lib.check_diag(L.hk_diag_trace_read(ctypes.c_void_p(buf.ctypes.data), buf.nbytes, 1))
    tab = buf.reshape(64, 1024)
    out = {"config": cfg}
    for t in (0, 1):
        S = [int(tab[2 + 4 * t, a]) for a in range(1024) if tab[2 + 4 * t, a]]
        ep = sorted(int(tab[31 + t, a]) for a in range(1024) if tab[31 + t, a])
        inside, cross = [], []
        for a, b in zip(S, S[1:]):
            (cross if any(a < e < b for e in ep) else inside).append(b - a)
        X = [int(tab[3 + 4 * t, a]) - int(tab[2 + 4 * t, a]) for a in range(1024)
             if tab[2 + 4 * t, a] and tab[3 + 4 * t, a]]
        out[f"tile{t}"] = {"steps": len(S), "items": len(ep),
                           "period_inside_item": round(st.median(inside), 0) if inside else None,
                           "period_across_items": round(st.median(cross), 0) if cross else None,
                           "softmax_step": round(st.median(X), 0) if X else None}
    print(json.dumps(out), flush=True)
    del x
    # item-boundary breakdown (events: 12 MMA item start, 13 Q landed, 14 first S issued,
    # 15+t last PV of tile t issued, 18+t first PV of tile t may issue, 17 producer Q issued,
    # 33+t epilogue O complete, 35+t O read out, 31+t epilogue done; indices = busy item number)
    def ev(e, a):
        v = int(tab[e, a])
        return v if v else None
    nb = sum(1 for a in range(1024) if tab[12, a])
    rows = []
    for k in range(1, nb):
        r = {"q_issue": ev(17, k), "mma_start": ev(12, k), "q_landed": ev(13, k), "s_issued": ev(14, k),
             "k0_issue": ev(22, k), "k0_landed": ev(24, k), "loop_done": ev(20, k - 1),
             "s0_issued": ev(25, k), "s1_issued": ev(26, k)}
        for t in (0, 1):
            r[f"lastpv{t}"] = ev(15 + t, k - 1)
            r[f"ep_o{t}"] = ev(33 + t, k - 1)
            r[f"ep_read{t}"] = ev(35 + t, k - 1)
            r[f"ep_done{t}"] = ev(31 + t, k - 1)
            r[f"pv0_{t}"] = ev(18 + t, k)
        if all(v is not None for v in r.values()):
            rows.append(r)

    def med(f):
        return round(st.median([f(r) for r in rows]), 0) if rows else None
    out2 = {"config": cfg, "items": len(rows),
            "lastpv1->mma_next_start": med(lambda r: r["mma_start"] - r["lastpv1"]),
            "q_issue->q_landed": med(lambda r: r["q_landed"] - r["q_issue"]),
            "mma_start->q_landed": med(lambda r: r["q_landed"] - r["mma_start"]),
            "q_landed->s_issued": med(lambda r: r["s_issued"] - r["q_landed"]),
            "q_issue_before_lastpv1": med(lambda r: r["lastpv1"] - r["q_issue"]),
            "lastpv1->loop_done": med(lambda r: r["loop_done"] - r["lastpv1"]),
            "loop_done->mma_start": med(lambda r: r["mma_start"] - r["loop_done"]),
            "k0_issue->k0_landed": med(lambda r: r["k0_landed"] - r["k0_issue"]),
            "k0_issue_before_q_issue": med(lambda r: r["q_issue"] - r["k0_issue"]),
            "q_landed->k0_landed": med(lambda r: r["k0_landed"] - r["q_landed"]),
            "k0_landed->s0_issued": med(lambda r: r["s0_issued"] - r["k0_landed"]),
            "s0_issued->s1_issued": med(lambda r: r["s1_issued"] - r["s0_issued"]),
            "s1_issued->s_issued": med(lambda r: r["s_issued"] - r["s1_issued"])}
    for t in (0, 1):
        out2[f"t{t}"] = {"lastpv->O_complete": med(lambda r: r[f"ep_o{t}"] - r[f"lastpv{t}"]),
                         "O_complete->O_read": med(lambda r: r[f"ep_read{t}"] - r[f"ep_o{t}"]),
                         "O_read->ep_done": med(lambda r: r[f"ep_done{t}"] - r[f"ep_read{t}"]),
                         "lastpv->next_first_pv_ok": med(lambda r: r[f"pv0_{t}"] - r[f"lastpv{t}"]),
                         "s_issued->first_pv_ok": med(lambda r: r[f"pv0_{t}"] - r["s_issued"])}
    print(json.dumps(out2), flush=True)
