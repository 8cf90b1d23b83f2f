"""Forward softmax step in isolation (hk_diag_rates kind 3): cycles per 128-column step for
one or two warpgroups (two = both Q tiles' warpgroups running concurrently on the same SM
sub-partitions), per exp-emulation split."""
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
for emu in (0, 2, 3, 4, 5):
    for nwg in (1, 2):
        for _ in range(2):  # warm
            _lib.check_diag(L.hk_diag_rates(3, 10 * emu + nwg, 400, ctypes.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        res[f"emu{emu}_wg{nwg}"] = round(out.float().median().item(), 1)
print(json.dumps(res))
