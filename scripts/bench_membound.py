"""Memory-bound kernels (NEXT #3) on B200 vs the HBM roofline and vs PyTorch eager:
fused dropout-residual-LayerNorm and rotary at the paper's B=16, H=16, d=128.
Bytes = algorithmic HBM bytes (each input read once, each output written once).
Prints one JSON line per kernel/shape."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import ln_dropout_residual, rope  # noqa: E402
from paper_2511_08083_b200.inputs import make_ln_inputs, make_rope_inputs  # noqa: E402


def timed(fn, iters=50, warm=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", default="1024,4096,16384")
    a = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from bench import load_peaks  # MEASURED_PEAKS.json, else the profiling guide's fallback (named in the output)
    pk = load_peaks()
    hbm, hbm_src = pk["hbm_gbs"], pk["source"]
    B, H, d = 16, 16, 128
    D = H * d
    for N in (int(v) for v in a.seqs.split(",")):
        rows = B * N
        x = make_ln_inputs(rows, D, seed=N, device="cuda")
        out, res = torch.empty_like(x["x"]), torch.empty_like(x["x"])
        for p in (0.0, 0.1):
            t = timed(lambda: ln_dropout_residual(x["x"], x["residual"], x["weight"], x["bias"], p=p, seed=1,
                                                  out=out, out_resid=res))

            def eager():
                xt = torch.nn.functional.dropout(x["x"], p=p, training=p > 0)
                r = x["residual"] + xt
                return torch.nn.functional.layer_norm(r, (D,), x["weight"], x["bias"], eps=1e-5), r
            te = timed(eager)
            nbytes = 4 * rows * D * 2
            print(json.dumps({"kernel": "ln_dropout_residual", "B": B, "N": N, "D": D, "p": p, "ms": round(t, 4),
                              "GB/s": round(nbytes / t / 1e6, 1), "hbm_peak_GB/s": hbm, "peak_source": hbm_src,
                              "frac": round(nbytes / t / 1e6 / hbm, 3) if hbm else None,
                              "torch_eager_ms": round(te, 4), "speedup_vs_eager": round(te / t, 2)}), flush=True)
        del x, out, res
        xr = make_rope_inputs(B, N, H, d, seed=N, device="cuda")["x"]
        pos = torch.arange(N, device="cuda", dtype=torch.float32)[:, None]
        inv = 10000.0 ** (-torch.arange(0, d // 2, device="cuda", dtype=torch.float32) * 2 / d)
        c, s = torch.cos(pos * inv).contiguous(), torch.sin(pos * inv).contiguous()
        o = torch.empty_like(xr)
        t = timed(lambda: rope(xr, c, s, out=o))

        def eager_rope():
            x1, x2 = xr[..., : d // 2].float(), xr[..., d // 2:].float()
            cc, ss = c[None, :, None, :], s[None, :, None, :]
            return torch.cat([x1 * cc - x2 * ss, x2 * cc + x1 * ss], -1).to(torch.bfloat16)
        te = timed(eager_rope)
        nbytes = 2 * B * N * H * d * 2
        print(json.dumps({"kernel": "rope", "B": B, "N": N, "H": H, "d": d, "ms": round(t, 4),
                          "GB/s": round(nbytes / t / 1e6, 1), "hbm_peak_GB/s": hbm, "peak_source": hbm_src,
                          "frac": round(nbytes / t / 1e6 / hbm, 3) if hbm else None,
                          "torch_eager_ms": round(te, 4), "speedup_vs_eager": round(te / t, 2)}), flush=True)
        del xr, o


if __name__ == "__main__":
    main()
