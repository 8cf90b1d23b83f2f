"""Measure pipe issue rates and tcgen05.mma pacing on the GPU (diag entry point)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_08083_b200 import _lib  # noqa: E402

L = _lib.diag()
out = torch.zeros(148, device="cuda")
res = {}
names = ["ex2.f32", "cvt.bf16x2.f32", "fma.f32 (const operands)", "max.f32", "ex2.bf16x2", "add.f32",
         "fma.f32x2 (pairs, counted per element)", "add.f32x2 (pairs, counted per element)", "max3.f32",
         "int shift-add", "fma.f32 (3 register operands)"]
for op, nm in enumerate(names):
    iters = 4096
    for threads, tag in ((512, "16 warps/SM"), (128, "4 warps/SM (1 per SMSP)")):
        for _ in range(2):
            _lib.check_diag(L.hk_diag_rates(0, op + (100 if threads == 128 else 0), iters,
                                       ctypes.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        cyc = out.float().mean().item()
        res[f"{nm} per clk per SM, {tag}"] = round(threads * iters * 8 / cyc, 2)
for mode, mn in enumerate(["SS", "TS", "SS_Bmn"]):
    for n in (64, 128, 256):
        for _ in range(2):
            _lib.check_diag(L.hk_diag_rates(1, mode * 1000 + n, 2000, ctypes.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        cyc = out.float().mean().item()
        res[f"mma {mn} M=128 N={n} K=16 cycles"] = round(cyc, 2)
        res[f"mma {mn} M=128 N={n} flop/clk/SM"] = round(2 * 128 * n * 16 / cyc, 1)
for w in (4, 8, 16):
    iters = 1000
    for _ in range(2):
        _lib.check_diag(L.hk_diag_rates(2, w, iters, ctypes.c_void_p(out.data_ptr()), None))
    torch.cuda.synchronize()
    cyc = out.float().mean().item()
    res[f"tcgen05.ld 32x32b {w} warps bytes/clk/SM"] = round(w * 32 * 128 * 4 * iters / cyc, 1)
for emu in (0, 2, 3, 4, 5):
    for nwg in (1, 2):
        for _ in range(2):
            _lib.check_diag(L.hk_diag_rates(3, 10 * emu + nwg, 200, ctypes.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        res[f"softmax step emu {emu}/8, {nwg} WG: cycles/step"] = round(out.float().mean().item(), 1)
for rows in (64, 128):
    iters = 2000
    for _ in range(2):
        _lib.check_diag(L.hk_diag_rates(4, rows, iters, ctypes.c_void_p(out.data_ptr()), None))
    torch.cuda.synchronize()
    cyc = out.float().mean().item()
    res[f"TMA load {rows * 128 // 1024} KB boxes, 148 SMs, bytes/clk/SM"] = round(rows * 128 * iters / cyc, 1)
for tiles in (256, 4096):
    iters = 200
    for _ in range(2):
        _lib.check_diag(L.hk_diag_rates(5, tiles, iters, ctypes.c_void_p(out.data_ptr()), None))
    torch.cuda.synchronize()
    cyc = out.float().max().item()
    res[f"red.add.v4.f32 64KB tiles into {tiles * 64 // 1024} MB, bytes/clk chip"] = round(148 * 65536 * iters / cyc, 1)
print(json.dumps(res, indent=1))
