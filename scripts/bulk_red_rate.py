"""NEXT #1 decision data: throughput of the bulk-async (TMA) fp32 reduce-add that a
fused single-pass backward would use to accumulate dQ partials (one 128 x 128 fp32 tile = 64 KB per
(key tile, query tile, head) block), vs the red.global.add.v4 path measured in round 1. 148 CTAs,
one issuing thread each; wall time from CUDA events. Prints JSON lines."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import _lib  # noqa: E402

L = _lib.diag()
out = torch.zeros(148, device="cuda")
for mode, name in ((0, "cp.reduce.async.bulk.tensor.2d 128x128 fp32"), (1, "cp.reduce.async.bulk 128 x 512 B rows")):
    for row_tiles in (12, 64, 512):
        iters = 400
        for rep in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            _lib.check_diag(L.hk_diag_rates(6, mode * 100000 + row_tiles, iters, ctypes.c_void_p(out.data_ptr()), None))
            e.record()
            torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        byts = 148 * 65536 * iters
        region_mb = row_tiles * 128 * 32 * 512 / 1e6
        print(json.dumps({"op": name, "region_MB": round(region_mb, 1), "tiles_reduced": 148 * iters,
                          "ms": round(ms, 3), "TB_per_s": round(byts / ms / 1e9, 3),
                          "bytes_per_clk_chip": round(byts / (out.max().item()), 1)}), flush=True)
for tiles in (256, 4096):
    iters = 200
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.check_diag(L.hk_diag_rates(5, tiles, iters, ctypes.c_void_p(out.data_ptr()), None))
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(json.dumps({"op": "red.global.add.v4.f32 (256 threads)", "region_MB": tiles * 64 / 1024,
                      "ms": round(ms, 3), "TB_per_s": round(148 * 65536 * iters / ms / 1e9, 3)}), flush=True)
