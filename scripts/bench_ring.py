"""Ring attention (NEXT #4) on one B200: P virtual ranks (LoopbackRing) run the whole
context-parallel schedule — chunk-pair attention calls, LSE merges, gradient
accumulation — back to back on one GPU, so the time is the sum of every rank's
compute. TFLOPS = the whole sequence's algorithmic fwd+bwd FLOPs (reading #14) /
that time, next to one dense call over the whole sequence: the ratio is the
decomposition overhead of the ring (smaller calls, merges, fp32 accumulators),
not its communication (which on 8 GPUs overlaps NVLink transfers with compute).
Workload: Llama-3 8B heads (Hq=32, Hkv=8, d=128), causal, B=1, N=32768 and 65536.
Prints one JSON line per (N, P)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import attn_bwd, attn_fwd, ring  # noqa: E402
from paper_2511_08083_b200.inputs import make_inputs  # noqa: E402


def timed(fn, iters=3, warm=2):
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
    Hq, Hkv, d, B, causal = 32, 8, 128, 1, True
    for N in (32768, 65536):
        x = make_inputs(B, N, Hq, Hkv, d, seed=1, device="cuda")
        flops = 3.5 * 4.0 * B * Hq * N * N * d * (0.5 if causal else 1.0)

        def dense():
            o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
            attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
        t_d = timed(dense)
        print(json.dumps({"workload": "ring_loopback", "N": N, "P": 1, "mode": "dense single call",
                          "ms": round(t_d, 3), "tflops": round(flops / t_d / 1e9, 1)}), flush=True)
        for P in (2, 4, 8):
            sh = {n: [ring.zigzag_shard(x[n], P, r) for r in range(P)] for n in ("Q", "K", "V", "dO")}
            comm = ring.LoopbackRing(P)

            def step(streams=1):
                fw = ring.ring_attn_fwd(sh["Q"], sh["K"], sh["V"], causal, comm, streams=streams)
                ring.ring_attn_bwd(sh["Q"], sh["K"], sh["V"], [f[0] for f in fw], [f[1] for f in fw], sh["dO"],
                                   causal, comm, streams=streams)
            t = timed(step)
            t_s = timed(lambda: step(4))
            # the same schedule captured once into a CUDA graph: no host launch overhead per kernel
            step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            t_g = timed(g.replay)
            print(json.dumps({"workload": "ring_loopback", "N": N, "P": P, "chunk": N // (2 * P), "Hq": Hq,
                              "Hkv": Hkv, "d": d, "causal": causal, "ms_all_ranks": round(t, 3),
                              "tflops": round(flops / t / 1e9, 1), "vs_dense": round(t_d / t, 3),
                              "graph_ms_all_ranks": round(t_g, 3), "graph_tflops": round(flops / t_g / 1e9, 1),
                              "graph_vs_dense": round(t_d / t_g, 3), "streams4_ms_all_ranks": round(t_s, 3),
                              "streams4_tflops": round(flops / t_s / 1e9, 1),
                              "streams4_vs_dense": round(t_d / t_s, 3)}), flush=True)
            del g
            del sh
        del x


if __name__ == "__main__":
    main()
