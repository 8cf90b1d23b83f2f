import json, torch
n = 1 << 29
K = 4
h_in = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(K)]
h_out = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(K)]
d_in = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(K)]
d_out = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(K)]
st = [torch.cuda.Stream() for _ in range(2 * K)]
def run(k_in, k_out):
    for i in range(k_in):
        with torch.cuda.stream(st[i]):
            d_in[i].copy_(h_in[i], non_blocking=True)
    for i in range(k_out):
        with torch.cuda.stream(st[K + i]):
            h_out[i].copy_(d_out[i], non_blocking=True)
    for s in st: torch.cuda.current_stream().wait_stream(s)
def timed(fn, it=4):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
for k in (1, 2, 4):
    t = timed(lambda: run(k, k))
    print(json.dumps({"streams_per_direction": k, "each_direction_GBps": round(k * n / t / 1e6, 1)}))
for k in (1, 2, 4):
    t = timed(lambda: run(k, 0))
    print(json.dumps({"h2d_only_streams": k, "GBps": round(k * n / t / 1e6, 1)}))
