"""PCIe bandwidth on the box (context for bench.py's e2e number): pinned H2D alone,
D2H alone, and both directions concurrently on two streams, 1 GiB each."""
import json

import torch

n = 1 << 30
h_a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_b = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, it=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_a, non_blocking=True)
    with torch.cuda.stream(s2):
        h_b.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timed(lambda: d_a.copy_(h_a, non_blocking=True))
t_d2h = timed(lambda: h_b.copy_(d_b, non_blocking=True))
t_both = timed(both)
print(json.dumps({"h2d_GBps": round(n / t_h2d / 1e6, 1), "d2h_GBps": round(n / t_d2h / 1e6, 1),
                  "concurrent_each_GBps": round(n / t_both / 1e6, 1)}))
