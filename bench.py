"""bench.py — fused attention fwd+bwd throughput on B200 (driver contract).

A step = one pass of the whole hot path over one batch of synthetic input:
hk_attn_fwd (F0-F7) then hk_attn_bwd (B0 preprocess, B1 dK/dV, B2 dQ), both
through the public Python API (the C ABI calls a user makes; the backward forks
its dQ pass onto a side stream). Default workload (N=1): BASELINE.json
configs[2], Llama-3 8B GQA (Hq=32, Hkv=8, d=128) causal, B=16, N=8192 — the GQA
configuration the metric names that fits one GPU and is run at 1/2/4/8 GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
                    [--scaling strong|weak] [--impl reference]

Timed regions (CUDA events on the launching stream, W untimed warm-up steps,
barrier + synchronize around each, max over ranks):
  1. headline: K steps of the public attn_fwd + attn_bwd -> value, ms_per_step,
     step statistics (mean, median, min, first-10 vs last-10: P:880);
  2. breakdown: K steps of hk_attn_fwd + hk_attn_bwd's three kernels launched one
     per call (libhkattn_diag.so hk_diag_bwd_phase: same validation and kernels,
     no dQ fork) with events between kernels -> per-kernel ms and the roofline.
Sub-records (N=1): C4-8192 (d=64), C5-1024-c, C5-16384-c measured the same way
in the same run, so the driver's line carries the d=64 and 70B-GQA numbers.

Multi-GPU: one process per GPU (torchrun). Default strong
scaling: the fixed BASELINE problem (B=16) is split into contiguous batch-major
(b, kvh) unit ranges (shard.strong_shard) — no data-path collective. NCCL
carries only the checks: per-unit bit checksums all-gathered and compared with
a 1-GPU recomputation on rank 0, one sampled unit's outputs sent to rank 0 for
an oracle check on sampled rows, and the per-rank timings (max over ranks).

`--impl reference` times the fp64 CPU oracle (oracle/) on host cores on a
bounded sample of the same workload; it and the cpu_baseline leg are the only
places bench.py executes oracle/.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "attn fwd/bwd TFLOPS per GPU (GQA, d=64/128) and % of B200 BF16 dense peak"
UNIT = "TFLOPS"
SPEC_PEAK_TFLOPS = 2250.0
SUB_CONFIGS = ("C4-8192", "C5-1024-c", "C5-16384-c")

# name: (B, N, Hq, Hkv, d, causal, label) — B is the global batch of the BASELINE config
CONFIGS = {
    "C1": (1, 128, 2, 2, 64, False, "MHA B=1 H=2 N=128 d=64 non-causal"),
    "C2-nc": (16, 4096, 16, 16, 128, False, "MHA B=16 H=16 N=4096 d=128 non-causal"),
    "C2-c": (16, 4096, 16, 16, 128, True, "MHA B=16 H=16 N=4096 d=128 causal"),
    "C3": (16, 8192, 32, 8, 128, True, "Llama-3 8B GQA Hq=32 Hkv=8 d=128 causal B=16 N=8192"),
    "C4-2048": (16, 2048, 32, 32, 64, True, "d=64 MHA B=16 H=32 N=2048 causal"),
    "C4-4096": (16, 4096, 32, 32, 64, True, "d=64 MHA B=16 H=32 N=4096 causal"),
    "C4-8192": (16, 8192, 32, 32, 64, True, "d=64 MHA B=16 H=32 N=8192 causal"),
    "C4-16384": (16, 16384, 32, 32, 64, True, "d=64 MHA B=16 H=32 N=16384 causal"),
}
for _n in (1024, 2048, 4096, 8192, 16384, 32768):
    for _c in (False, True):
        CONFIGS[f"C5-{_n}-{'c' if _c else 'nc'}"] = (
            16, _n, 64, 8, 128, _c, f"Llama-3 70B GQA Hq=64 Hkv=8 d=128 {'causal' if _c else 'non-causal'} B=16 N={_n}")


def fwd_flops(B, N, Hq, d, causal):
    """FlashAttention convention (reading #14): 4 B Hq N^2 d, x1/2 causal."""
    return 4.0 * B * Hq * N * N * d * (0.5 if causal else 1.0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"burst": float(j["bf16_tflops"]), "sustained": float(j.get("bf16_tflops_sustained", j["bf16_tflops"])),
                "hbm_gbs": float(j["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)",
                "sustained_at_mhz": j.get("clocks_under_load", {}).get("sm_mhz_median")}
    return {"burst": 1590.0, "sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)",
            "sustained_at_mhz": None}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def step_stats(ms):
    """Mean (the paper's statistic), median, min, max and the first-10 vs last-10 means
    (NVIDIA throughput degrades with the iteration count)."""
    k = min(10, max(1, len(ms) // 2))
    return {"mean": round(statistics.fmean(ms), 4), "median": round(statistics.median(ms), 4),
            "min": round(min(ms), 4), "max": round(max(ms), 4), "first_mean": round(statistics.fmean(ms[:k]), 4),
            "last_mean": round(statistics.fmean(ms[-k:]), 4), "first_last_n": k}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index):
        self.samples, self.power, self.reasons, self.ok = [], [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = self._handle(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _handle(self, idx):
        import torch
        nv = self.nv
        try:
            pr = torch.cuda.get_device_properties(idx)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(idx)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w_median": round(statistics.median(self.power), 1) if self.power else None}


# ------------------------------------------------------------------ distributed
def dist_setup(backend="nccl"):
    """One process per GPU (torchrun env). backend="gloo" is a debugging aid that
    lets several ranks share one device (local rank modulo the device count) to
    exercise the multi-rank path on a single-GPU box; timings are then not
    per-GPU numbers."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dev = local % torch.cuda.device_count() if backend == "gloo" else local
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        local = dev
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _coll_device():
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_floats(xs, world):
    """all_gather of a small list of floats per rank -> list (rank-major) of lists."""
    if world == 1:
        return [list(xs)]
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(xs), dtype=torch.float64, device=_coll_device())
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


# ------------------------------------------------------------------ oracle legs (CPU)
def oracle_sample(cfg, seed, rows=None, x=None):
    """Time the fp64 oracle on one (b=0, kvh=0) unit of the workload, or on its
    first `rows` rows (a causal prefix is an exact sub-problem). `x` are the
    inputs the GPU used (D2H-copied here); if None they are generated on the
    CPU. Returns (tflops, seconds, description, flops, result)."""
    import numpy as np

    import oracle
    from paper_2511_08083_b200.inputs import make_inputs
    B, N, Hq, Hkv, d, causal, _ = cfg
    G = Hq // Hkv
    n = N if rows is None else rows
    if x is None:
        x = make_inputs(1, N, Hq, Hkv, d, seed=seed, device="cpu", batches=[0], kv_heads=[0])
    f = lambda t: t.float().cpu().numpy().astype(np.float64)
    Q = f(x["Q"][:1, :n, :G]); K = f(x["K"][:1, :n, :1]); V = f(x["V"][:1, :n, :1]); dO = f(x["dO"][:1, :n, :G])
    t0 = time.perf_counter()
    res = oracle.attn_fwd_bwd(Q, K, V, dO, causal)
    dt = time.perf_counter() - t0
    fl = 3.5 * fwd_flops(1, n, G, d, causal)
    desc = (f"one (b,kvh) unit of {B*Hkv}: G={G} heads x N={n}" if rows is None or rows == N else
            f"one (b,kvh) unit, G={G} heads, causal prefix of {n} of N={N} rows")
    return fl / dt / 1e12, dt, desc, fl, res


def oracle_cost(cfg, rows):
    """fp64 FLOPs the oracle executes on one unit (prefix of `rows` rows): 12 G n^2 d (x1/2 causal),
    SURVEY §8(d).9 — 6 n^2 d-sized GEMMs per head (S, PV, dP, dQ, dK, dV)."""
    B, N, Hq, Hkv, d, causal, _ = cfg
    return 12.0 * (Hq // Hkv) * rows * rows * d * (0.5 if causal else 1.0)


def oracle_full_cost(cfg):
    B, N, Hq, Hkv, d, causal, _ = cfg
    return 12.0 * B * Hq * N * N * d * (0.5 if causal else 1.0)


def run_reference(args, cfg):
    """--impl reference: the oracle as it stands, on host cores, bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    B, N, Hq, Hkv, d, causal, label = cfg
    nthreads = cores()
    # size one step to ~ (150 s / (K+W)) of CPU work: probe with a small prefix first
    rows = min(N, 1024)
    _, dt, _, fl, _ = oracle_sample(cfg, seed=0, rows=rows)
    rate = fl / dt
    target_s = max(1.0, min(20.0, 150.0 / (args.steps + args.warmup)))
    per_row2 = fl / (rows * rows)
    rows = int(min(N, max(128, math.sqrt(target_s * rate / per_row2))))
    if not causal:
        rows = N if fl / (rows * rows) * N * N / rate < 3 * target_s else rows
    for _ in range(args.warmup):
        oracle_sample(cfg, seed=0, rows=rows)
    times, flops, desc = [], 0.0, ""
    for _ in range(args.steps):
        _, dt, desc, fl, _ = oracle_sample(cfg, seed=0, rows=rows)
        times.append(dt)
        flops = fl
    v = flops * len(times) / sum(times) / 1e12
    gflops64 = oracle_cost(cfg, rows) / statistics.fmean(times) / 1e9
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": args.config, "label": label, "B": B, "N": N, "Hq": Hq, "Hkv": Hkv, "d": d,
                      "causal": causal},
           "impl": "reference",
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads, "kind": "oracle", "cpu_model": cpu_model(),
                            "sample": desc + " per step (fp64 numpy/OpenBLAS oracle)",
                            "fp64_gflops_achieved": round(gflops64, 2),
                            "extrapolated_full_problem_s": round(oracle_full_cost(cfg) / (gflops64 * 1e9), 1),
                            "extrapolated_note": "EXTRAPOLATION: full-problem oracle FLOPs / the achieved rate"},
           "step_ms_stats": step_stats([1e3 * t for t in times]),
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ GPU arm
class Problem:
    """The rank's local share of a config: inputs, outputs and workspace on the GPU."""

    def __init__(self, name, rank, world, scaling, seed):
        import torch

        from paper_2511_08083_b200.api import bwd_workspace_bytes, default_bwd_workspace_bytes
        from paper_2511_08083_b200.inputs import make_inputs
        from paper_2511_08083_b200.shard import strong_shard, weak_shard
        self.name = name
        self.cfg = CONFIGS[name]
        B, N, Hq, Hkv, d, causal, _ = self.cfg
        self.G = Hq // Hkv
        if scaling == "strong":
            self.shard = strong_shard(rank, world, B, Hq, Hkv)
            self.B_global = B
        else:
            self.shard = weak_shard(rank, world, B, Hq, Hkv)
            self.B_global = B * world
        self.B = len(self.shard.batches)
        self.Hkv = len(self.shard.kv_heads)
        self.Hq = self.G * self.Hkv
        self.N, self.d, self.causal = N, d, causal
        x = make_inputs(self.B_global, N, Hq, Hkv, d, seed=seed, device="cuda", batches=self.shard.batches,
                        kv_heads=self.shard.kv_heads)
        self.x = x
        self.q, self.k, self.v, self.do = x["Q"], x["K"], x["V"], x["dO"]
        self.o = torch.empty_like(self.q)
        self.lse = torch.empty((self.B, self.Hq, N), dtype=torch.float32, device="cuda")
        self.dq, self.dk, self.dv = torch.empty_like(self.q), torch.empty_like(self.k), torch.empty_like(self.v)
        # the workspace the public attn_bwd allocates itself: the stored-dS backward where it applies and
        # fits the budget (d = 128 dense), else the plain one
        nb = default_bwd_workspace_bytes(self.B, self.Hq, self.Hkv, N, d, None, causal)
        self.ds = nb > bwd_workspace_bytes(self.B, self.Hq, self.Hkv, N, d)
        self.ds_bytes = nb - bwd_workspace_bytes(self.B, self.Hq, self.Hkv, N, d) if self.ds else 0
        self.ws = torch.empty((nb + 3) // 4, dtype=torch.float32, device="cuda")
        self.fwd_flops = fwd_flops(self.B, N, self.Hq, d, causal)  # this rank's share
        in_bytes = sum(t.numel() * t.element_size() for t in (self.q, self.k, self.v, self.do))
        self.l2_note = "inputs larger than L2 (126 MB)" if in_bytes > 126e6 else "L2 flushed between steps"
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") if in_bytes <= 126e6 \
            else None

    def outputs(self):
        return {"O": self.o, "LSE": self.lse, "dQ": self.dq, "dK": self.dk, "dV": self.dv}

    def public_step(self):
        """The public API: hk_attn_fwd then hk_attn_bwd (which forks its dQ pass)."""
        from paper_2511_08083_b200 import attn_bwd, attn_fwd
        attn_fwd(self.q, self.k, self.v, self.causal, out=self.o, lse=self.lse)
        attn_bwd(self.q, self.k, self.v, self.o, self.lse, self.do, self.causal, workspace=self.ws, dq=self.dq,
                 dk=self.dk, dv=self.dv)


def time_headline(pb, steps, warmup, world, local, with_clocks=True):
    """Timed region 1: K public fwd+bwd steps, events around fwd and bwd of each step."""
    import torch
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        pb.public_step()
    torch.cuda.synchronize()
    barrier(world)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    clk = ClockSampler(local) if with_clocks else None
    ctx = clk if clk is not None else _Null()
    with ctx:
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        for i in range(steps):
            if pb.flush is not None:
                pb.flush.zero_()
            ev[i][0].record(st)
            attn_fwd(pb.q, pb.k, pb.v, pb.causal, out=pb.o, lse=pb.lse)
            ev[i][1].record(st)
            attn_bwd(pb.q, pb.k, pb.v, pb.o, pb.lse, pb.do, pb.causal, workspace=pb.ws, dq=pb.dq, dk=pb.dk, dv=pb.dv)
            ev[i][2].record(st)
        torch.cuda.synchronize()
        barrier(world)
        wall = time.perf_counter() - t0
    step_ms = [e[0].elapsed_time(e[2]) for e in ev]
    fwd_ms = [e[0].elapsed_time(e[1]) for e in ev]
    bwd_ms = [e[1].elapsed_time(e[2]) for e in ev]
    return step_ms, fwd_ms, bwd_ms, wall, (clk.summary() if clk is not None else None)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def time_breakdown(pb, steps, warmup, world):
    """Timed region 2: K steps of hk_attn_fwd + hk_attn_bwd's three kernels one per call
    (libhkattn_diag.so hk_diag_bwd_phase), events between kernels on the launching stream."""
    import ctypes

    import torch

    from paper_2511_08083_b200 import _lib, attn_fwd
    D = _lib.diag()
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)

    def phase(ph):
        _lib.check_diag(D.hk_diag_bwd_phase(ph, P(pb.q), P(pb.k), P(pb.v), P(pb.o), P(pb.lse), P(pb.do), P(pb.dq),
                                            P(pb.dk), P(pb.dv), P(pb.ws), pb.ws.numel() * 4, pb.B, pb.Hq, pb.Hkv,
                                            pb.N, pb.d, int(pb.causal), sp))

    def step(e=None):
        if e is not None:
            e[0].record(st)
        attn_fwd(pb.q, pb.k, pb.v, pb.causal, out=pb.o, lse=pb.lse)
        if e is not None:
            e[1].record(st)
        for ph in range(3):
            phase(ph)
            if e is not None:
                e[2 + ph].record(st)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    for i in range(steps):
        if pb.flush is not None:
            pb.flush.zero_()
        step(ev[i])
    torch.cuda.synchronize()
    barrier(world)
    # d = 64: hk_attn_bwd's default is the fused single pass (NEXT #1): phase 1 = dK/dV + dQ partials
    # (bulk reduce-add), phase 2 = the dQ convert pass
    names = ("fwd", "bwd_pre", "bwd_dkdv_dq", "dq_convert") if pb.d == 64 else \
        ("fwd", "bwd_pre", "bwd_dkdv_ds", "bwd_dq_ds") if pb.ds else ("fwd", "bwd_pre", "bwd_dkdv", "bwd_dq")
    per = {n: [e[i].elapsed_time(e[i + 1]) for e in ev] for i, n in enumerate(names)}
    return {n: statistics.fmean(t) for n, t in per.items()}


def bwd_path(pb):
    """Which backward the public attn_bwd runs for this problem (its default workspace decides)."""
    if pb.d == 64:
        return "fused single pass (dQ partials by bulk tensor reduce, NEXT #1)"
    if pb.ds:
        return f"stored dS ({pb.ds_bytes / 1e9:.1f} GB workspace): dK/dV pass + one-GEMM dQ pass"
    return "two-pass (dK/dV pass, dQ pass recomputing S and dP)"


def kernel_table(pb, kern_ms, peaks, world, sm_mhz=None):
    """Per-kernel algorithmic / executed rates and the roofline of the dominant kernel."""
    ff = pb.fwd_flops
    B, N, Hq, d = pb.B, pb.N, pb.Hq, pb.d
    # FLOPs per launch: executed = the tensor-core work the kernel issues; algorithmic = the share
    # of the method's 5 backward GEMMs (reading #14) it contributes.
    execd = {"fwd": ff, "bwd_dkdv": 2.0 * ff, "bwd_dq": 1.5 * ff,     # dkdv: S^T dP^T dV dK; dq: S dP dQ
             "bwd_dkdv_dq": 2.5 * ff,                                  # fused (d = 64): all 5 GEMMs once
             "bwd_dkdv_ds": 2.0 * ff, "bwd_dq_ds": 0.5 * ff}          # stored dS: dQ = dS K only
    alg = {"fwd": ff, "bwd_dkdv": 2.0 * ff, "bwd_dq": 0.5 * ff,       # dq: only dQ = dS K is not a recompute
           "bwd_dkdv_dq": 2.5 * ff, "bwd_dkdv_ds": 2.0 * ff, "bwd_dq_ds": 0.5 * ff}
    ds_bytes = getattr(pb, "ds_bytes", 0)  # stored dS: written by bwd_dkdv_ds, read by bwd_dq_ds
    pre_bytes = B * Hq * N * (4 * d + 4 + 4 + 4)  # read O, dO (bf16), LSE; write D, LSE2
    if d == 64:
        pre_bytes += B * Hq * N * d * 4          # + zero the fp32 dQ accumulator (fused backward)
    conv_bytes = B * Hq * N * d * (4 + 2)         # dq_convert: read fp32 dQ_acc, write bf16 dQ
    tot = sum(kern_ms.values())
    table = {}
    for n, ms in kern_ms.items():
        rec = {"ms": round(ms, 4), "share": round(ms / tot, 4)}
        if n in ("bwd_pre", "dq_convert"):
            nb = pre_bytes if n == "bwd_pre" else conv_bytes
            gbs = nb / (ms * 1e-3) / 1e9
            rec.update(gbs=round(gbs, 1), frac_of_hbm=round(gbs / peaks["hbm_gbs"], 4), algorithmic_bytes=nb)
        else:
            rec.update(tflops_executed=round(execd[n] / (ms * 1e-3) / 1e12, 1),
                       tflops_algorithmic=round(alg[n] / (ms * 1e-3) / 1e12, 1),
                       frac_of_burst_executed=round(execd[n] / (ms * 1e-3) / 1e12 / peaks["burst"], 4))
            if n in ("bwd_dkdv_ds", "bwd_dq_ds") and ds_bytes:
                # the dS round trip through HBM: written by the dK/dV pass, read (+ dQ written) by the dQ pass
                nb = ds_bytes + (B * Hq * N * d * 2 if n == "bwd_dq_ds" else 0)
                gbs = nb / (ms * 1e-3) / 1e9
                rec.update(hbm_gbs=round(gbs, 1), frac_of_hbm=round(gbs / peaks["hbm_gbs"], 4), hbm_bytes=nb)
        table[n] = rec
    dom = max((n for n in kern_ms if n not in ("bwd_pre", "dq_convert")), key=lambda n: kern_ms[n])
    ach = alg[dom] / (kern_ms[dom] * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{pb.name}:{dom}")
    roof = {"bound": "tensor", "kernel": dom, "achieved": round(ach, 1), "peak": peaks["burst"],
            "unit": "TFLOP/s", "frac": round(ach / peaks["burst"], 4), "traffic": traffic,
            "peak_kind": f"bf16 burst, {peaks['source']}",
            "frac_of_sustained": round(ach / peaks["sustained"], 4), "sustained_peak": peaks["sustained"],
            "sustained_measured_at_mhz": peaks["sustained_at_mhz"],
            "frac_of_spec_2250": round(ach / SPEC_PEAK_TFLOPS, 4),
            "algorithmic_flops_per_launch": alg[dom], "executed_flops_per_launch": execd[dom],
            "timing": "mean launch duration from CUDA events between kernels (timed region 2)"}
    # the backward as a whole: the method's 5 backward GEMMs (2.5 x the forward's FLOPs, reading #14)
    # over the summed kernel times, whichever path (two-pass / stored dS / fused) ran them
    bwd_ms = sum(ms for n, ms in kern_ms.items() if n != "fwd")
    if bwd_ms > 0:
        b_ach = 2.5 * ff / (bwd_ms * 1e-3) / 1e12
        roof["backward_path"] = {"kernels": [n for n in kern_ms if n != "fwd"], "ms": round(bwd_ms, 4),
                                 "algorithmic_tflops": round(b_ach, 1), "frac": round(b_ach / peaks["burst"], 4)}
    return table, roof, dom


def measure(pb, args, world, local, with_clocks=True):
    """Both timed regions for one problem; returns the record fields."""
    step_ms, fwd_ms, bwd_ms, wall, clk = time_headline(pb, args.steps, args.warmup, world, local, with_clocks)
    mean_ms = statistics.fmean(step_ms)
    ms = max_over_ranks(mean_ms, world)
    per_rank = gather_floats([mean_ms, statistics.fmean(fwd_ms), statistics.fmean(bwd_ms)], world)
    kern_ms = time_breakdown(pb, args.steps, max(3, args.warmup // 2), world)
    kern_ms = {n: max_over_ranks(v, world) for n, v in kern_ms.items()}
    return step_ms, fwd_ms, bwd_ms, wall, clk, ms, per_rank, kern_ms


def sub_record(name, args, peaks):
    """One extra config measured in the same run (N=1): public-API fwd / bwd TFLOPS and the
    per-kernel breakdown."""
    import torch
    pb = Problem(name, 0, 1, "strong", args.seed)
    steps = max(5, min(args.steps, int(4000 / max(1.0, _probe_ms(pb)))))
    a = argparse.Namespace(**{**vars(args), "steps": steps})
    step_ms, fwd_ms, bwd_ms, wall, clk, ms, _, kern_ms = measure(pb, a, 1, 0, with_clocks=True)
    ff = pb.fwd_flops
    table, roof, dom = kernel_table(pb, kern_ms, peaks, 1, (clk or {}).get("sm_mhz"))
    rec = {"workload": name, "label": pb.cfg[6], "steps": steps, "ms_per_step": round(ms, 4),
           "fwd_bwd_tflops": round(3.5 * ff / (ms * 1e-3) / 1e12, 1),
           "fwd_tflops": round(ff / (statistics.fmean(fwd_ms) * 1e-3) / 1e12, 1),
           "bwd_tflops": round(2.5 * ff / (statistics.fmean(bwd_ms) * 1e-3) / 1e12, 1),
           "pct_of_burst": round(100 * 3.5 * ff / (ms * 1e-3) / 1e12 / peaks["burst"], 2),
           "step_ms_stats": step_stats(step_ms), "kernels": table, "bwd_path": bwd_path(pb),
           "dominant": {"kernel": dom, "frac_of_burst": roof["frac"], "achieved": roof["achieved"]},
           "clocks": clk}
    del pb
    torch.cuda.empty_cache()
    return rec


def _probe_ms(pb):
    import torch
    pb.public_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pb.public_step()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)


def multi_gpu_checks(pb, args, rank, world):
    """SURVEY §8(e) checking over NCCL: (1) per-unit bit checksums all-gathered and compared with
    a 1-GPU recomputation of the whole problem on rank 0 (bitwise: no atomics, fixed order);
    (2) the sampled unit (B-1, Hkv-1) sent from its owner to rank 0 and checked against the
    oracle on 64 query rows of each of its heads (O, LSE max-abs; dQ relative L2)."""
    import numpy as np
    import torch

    from paper_2511_08083_b200.shard import (gather_checksums, gather_unit_to_rank0, owner_of, strong_shard,
                                             unit_checksums, unit_slices)
    B, N, Hq, Hkv, d, causal, _ = pb.cfg
    G = pb.G
    dev = _coll_device()
    ids, sums = unit_checksums(pb.outputs(), pb.shard, G)
    got = gather_checksums(ids.to(dev), sums.to(dev), world)
    unit = (pb.B_global - 1, Hkv - 1)
    owner, bi, ki = owner_of(unit, world, B, Hq, Hkv, args.scaling)
    mine = [t.to(dev) for t in unit_slices(pb.outputs(), bi, ki, G)] if rank == owner else None
    like = [(t.shape, t.dtype, dev) for t in unit_slices(pb.outputs(), 0, 0, G)]
    recv = gather_unit_to_rank0(mine, owner, rank, like)
    out = None
    if rank == 0:
        # (1) the same problem on this one GPU, all units
        full = Problem(pb.name, 0, 1, "strong", args.seed) if args.scaling == "strong" else None
        res = {"units_checked": len(got), "owner_of_sampled_unit": owner}
        if full is not None:
            full.public_step()
            torch.cuda.synchronize()
            want = gather_checksums(*unit_checksums(full.outputs(), strong_shard(0, 1, B, Hq, Hkv), G), 1)
            # O, LSE, dQ, dK, dV; the d = 64 fused backward adds fp32 dQ partials in arrival order, so
            # its dQ is compared by relative L2 on the sampled unit instead of bits
            idx = [0, 1, 2, 3, 4] if d == 128 else [0, 1, 3, 4]
            res["bitwise_outputs"] = [["O", "LSE", "dQ", "dK", "dV"][i] for i in idx]
            pick = lambda t: tuple(t[i] for i in idx)
            res["bitwise_equal_to_1gpu"] = bool(all(pick(got[u]) == pick(want[u]) for u in want))
            res["units_differing"] = [list(u) for u in want if pick(got.get(u, (0,) * 5)) != pick(want[u])][:8]
            if d == 64:
                fdq = unit_slices(full.outputs(), unit[0], unit[1], G)[2].float()
                res["sampled_unit_dq_rel_l2_vs_1gpu"] = float((recv[2].float().to(fdq.device) - fdq).norm() /
                                                              fdq.norm())
            del full
            torch.cuda.empty_cache()
        # (2) oracle on sampled rows of the gathered unit (inputs regenerated on the host)
        import oracle
        from paper_2511_08083_b200.inputs import make_inputs, sample_rows
        # regenerated on the GPU (the CUDA generator's stream, as every rank drew it), then copied
        xi = make_inputs(pb.B_global, N, Hq, Hkv, d, seed=args.seed, device="cuda", batches=[unit[0]],
                         kv_heads=[unit[1]])
        f = lambda t: t.float().cpu().numpy().astype(np.float64)
        Q, K, V, dO = f(xi["Q"]), f(xi["K"]), f(xi["V"]), f(xi["dO"])
        o_u, lse_u, dq_u = (f(t) for t in recv[:3])
        rows = sample_rows(N, 64, seed=args.seed + 7)
        eo = el = 0.0
        gdq, rdq = [], []
        for g in range(G):
            r = oracle.attn_rows(Q, K, V, dO, causal, 0, g, rows)
            eo = max(eo, float(np.abs(o_u[rows, g] - r["O"]).max()))
            el = max(el, float(np.abs(lse_u[g, rows] - r["LSE"]).max()))
            gdq.append(dq_u[rows, g])
            rdq.append(r["dQ"])
        gdq, rdq = np.stack(gdq), np.stack(rdq)
        res["sampled_unit_oracle"] = {"unit": list(unit), "rows": len(rows), "O_maxabs": eo, "LSE_maxabs": el,
                                      "dQ_rel_l2": float(np.linalg.norm(gdq - rdq) / np.linalg.norm(rdq)),
                                      "pass": bool(eo <= 2e-2 and el <= 2e-2 and
                                                   np.linalg.norm(gdq - rdq) / np.linalg.norm(rdq) <= 1e-2)}
        out = res
    barrier(world)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: split the fixed BASELINE problem over the GPUs (default); weak: B per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the same-run sub-records (C4-8192, C5-*)")
    ap.add_argument("--no-check", action="store_true", help="multi-GPU: skip the NCCL checks")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: debugging aid, ranks may share a GPU (not a per-GPU measurement)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch

    rank, world, local = dist_setup(args.dist_backend)
    peaks = load_peaks()
    pb = Problem(args.config, rank, world, args.scaling, args.seed)
    B, N, Hq, Hkv, d, causal, label = cfg
    step_ms, fwd_ms, bwd_ms, wall, clk, ms, per_rank, kern_ms = measure(pb, args, world, local)
    flops_rank = 3.5 * pb.fwd_flops
    flops_all = sum(gather_floats([flops_rank], world), [])
    total_flops = sum(flops_all)
    value = total_flops / (ms * 1e-3) / 1e12
    table, roofline, dom = kernel_table(pb, kern_ms, peaks, world, (clk or {}).get("sm_mhz"))
    fwd_all = max(r[1] for r in per_rank)
    bwd_all = max(r[2] for r in per_rank)

    checks = None
    if world > 1 and not args.no_check:
        checks = multi_gpu_checks(pb, args, rank, world)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pb, world)

    subs = None
    if world == 1 and not args.no_sub and rank == 0:
        subs = [sub_record(n, args, peaks) for n in SUB_CONFIGS if n != args.config]

    par = {"strong": f"(batch x KV-head) units of the fixed B={B} problem split over {world} GPU(s), no exchange",
           "weak": f"B={B} per GPU, (batch x KV-head) units sharded over {world} GPU(s), no exchange"}[args.scaling]
    if args.dist_backend != "nccl":
        par += " [gloo debug: ranks share a GPU]"
    out = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": args.scaling,
           "vs_baseline": None, "dtype": "bf16", "data": "synthetic (i.i.d. N(0,1) rounded to bf16, P:538)",
           "config": {"workload": args.config, "label": label, "global_batch": pb.B_global, "B_per_gpu": pb.B,
                      "N": N, "Hq": Hq, "Hkv": Hkv, "d": d, "causal": causal, "parallelism": par, "l2": pb.l2_note,
                      "bwd_path": bwd_path(pb)},
           "per_gpu_tflops": round(value / world, 2),
           "pct_of_peak": {"burst": round(100 * value / world / peaks["burst"], 2),
                           "sustained": round(100 * value / world / peaks["sustained"], 2),
                           "spec_2250": round(100 * value / world / SPEC_PEAK_TFLOPS, 2),
                           "peaks_source": peaks["source"]},
           "fwd_tflops_per_gpu": round(pb.fwd_flops / (fwd_all * 1e-3) / 1e12, 1),
           "bwd_tflops_per_gpu": round(2.5 * pb.fwd_flops / (bwd_all * 1e-3) / 1e12, 1),
           "step_ms_stats": step_stats(step_ms),
           "per_rank_ms": [round(r[0], 4) for r in per_rank],
           "per_rank_spread": round(max(r[0] for r in per_rank) / min(r[0] for r in per_rank) - 1, 4),
           "timing": "timed region 1 (value, ms_per_step, fwd/bwd): CUDA events around the public attn_fwd and "
                     "attn_bwd of each step on the launching stream (the dQ fork joins back before the last "
                     "event); timed region 2 (kernels, roofline): the same step with hk_attn_bwd's three kernels "
                     "launched one per call (libhkattn_diag.so), events between kernels",
           "kernels": table, "roofline": roofline, "gpu_launches": 4 * args.steps, "clocks": clk,
           "wall_s_timed_region": round(wall, 3), "e2e": e2e}
    if checks is not None:
        out["multi_gpu_checks"] = checks
    if subs is not None:
        out["sub_records"] = subs
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(pb, args)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_e2e(args, pb, world):
    """The same metric through the public API from pinned host buffers: per step H2D of Q, K, V,
    dO and D2H of O, LSE, dQ, dK, dV, pipelined on three streams over batch chunks."""
    import torch

    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    from paper_2511_08083_b200.api import default_bwd_workspace_bytes
    B, N, Hq, Hkv, d, causal = pb.B, pb.N, pb.Hq, pb.Hkv, pb.d, pb.causal
    x = pb.x
    chunk = 2 if B % 2 == 0 else 1
    nchunks = B // chunk
    h_in = {n: x[n].cpu().pin_memory() for n in ("Q", "K", "V", "dO")}
    dev_in = {n: torch.empty_like(x[n]) for n in h_in}
    o = torch.empty_like(x["Q"])
    lse = torch.empty((B, Hq, N), dtype=torch.float32, device="cuda")
    dq, dk, dv = torch.empty_like(x["Q"]), torch.empty_like(x["K"]), torch.empty_like(x["V"])
    h_out = {"O": torch.empty(o.shape, dtype=o.dtype, pin_memory=True),
             "LSE": torch.empty(lse.shape, dtype=lse.dtype, pin_memory=True),
             "dQ": torch.empty(dq.shape, dtype=dq.dtype, pin_memory=True),
             "dK": torch.empty(dk.shape, dtype=dk.dtype, pin_memory=True),
             "dV": torch.empty(dv.shape, dtype=dv.dtype, pin_memory=True)}
    dev_out = {"O": o, "LSE": lse, "dQ": dq, "dK": dk, "dV": dv}
    ws = torch.empty((default_bwd_workspace_bytes(chunk, Hq, Hkv, N, d, None, causal) + 3) // 4, dtype=torch.float32,
                     device="cuda")
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    done_cmp = [torch.cuda.Event() for _ in range(nchunks)]
    done_out = [torch.cuda.Event() for _ in range(nchunks)]
    started = [False] * nchunks

    def one_step():
        for c in range(nchunks):
            sl = slice(c * chunk, (c + 1) * chunk)
            with torch.cuda.stream(s_in):
                if started[c]:
                    s_in.wait_event(done_cmp[c])  # previous step's compute of chunk c read these inputs
                for n in h_in:
                    dev_in[n][sl].copy_(h_in[n][sl], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in)
                if started[c]:
                    s_cmp.wait_event(done_out[c])  # previous step's D2H of chunk c read these outputs
                qq, kk, vv, gg = (dev_in[n][sl] for n in ("Q", "K", "V", "dO"))
                attn_fwd(qq, kk, vv, causal, out=o[sl], lse=lse[sl])
                attn_bwd(qq, kk, vv, o[sl], lse[sl], gg, causal, workspace=ws, dq=dq[sl], dk=dk[sl], dv=dv[sl])
                done_cmp[c].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done_cmp[c])
                for n in h_out:
                    h_out[n][sl].copy_(dev_out[n][sl], non_blocking=True)
                done_out[c].record(s_out)
            started[c] = True

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    for _ in range(args.steps):
        one_step()
    s_in.wait_stream(s_out)
    s_in.wait_stream(s_cmp)
    e1.record(s_in)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    # the result really came back: spot-check the host copy against the device tensor
    assert torch.equal(h_out["dV"][-1], dv[-1].cpu())
    flops = sum(sum(gather_floats([3.5 * pb.fwd_flops], world), []))
    h2d = sum(t.numel() * t.element_size() for t in h_in.values())
    d2h = sum(t.numel() * t.element_size() for t in h_out.values())
    return {"value": round(flops / (ms * 1e-3) / 1e12, 2), "unit": UNIT, "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "pipeline": f"pinned host -> H2D / fwd+bwd / D2H on 3 streams over {nchunks} batch chunks of {chunk}"}


def cpu_baseline(pb, args):
    """The fp64 oracle, as it stands, on this host's cores, on one (b=0, kvh=0)
    unit (causal prefix if needed to stay ~10-30 s); also reports the GPU-vs-
    oracle errors on that sample (rows of the prefix are exact sub-problems), the
    achieved fp64 rate and the (labelled) extrapolated full-problem CPU time."""
    import numpy as np
    cfg = pb.cfg
    B, N, Hq, Hkv, d, causal, _ = cfg
    G = Hq // Hkv
    rows = N
    if oracle_cost(cfg, N) > 6e11:  # keep the sample ~10-30 s
        rows = int(math.sqrt(6e11 / (12.0 * G * d * (0.5 if causal else 1.0))))
        rows = max(128, (rows // 128) * 128)
    if not causal and rows != N:
        rows = N  # a non-causal prefix is not a sub-problem; take the full unit
    x = {n: pb.x[n][:1, :, :(G if n in ("Q", "dO") else 1)] for n in ("Q", "K", "V", "dO")}
    tf, dt, desc, fl, res = oracle_sample(cfg, seed=args.seed, rows=rows, x=x)
    f = lambda t: t.float().cpu().numpy().astype(np.float64)
    par = {"O_maxabs": float(np.abs(f(pb.o[:1, :rows, :G]) - res["O"]).max()),
           "LSE_maxabs": float(np.abs(f(pb.lse[:1, :G, :rows]) - res["LSE"]).max()),
           "dQ_rel_l2": float(np.linalg.norm(f(pb.dq[:1, :rows, :G]) - res["dQ"]) / np.linalg.norm(res["dQ"]))}
    if rows == N:
        for n, t in (("dK", pb.dk), ("dV", pb.dv)):
            par[f"{n}_rel_l2"] = float(np.linalg.norm(f(t[:1, :, :1]) - res[n]) / np.linalg.norm(res[n]))
    gflops64 = oracle_cost(cfg, rows) / dt / 1e9
    return {"value": round(tf, 6), "unit": UNIT, "cores": cores(), "kind": "oracle", "cpu_model": cpu_model(),
            "sample": desc + f" ({dt:.1f} s, fp64 numpy/OpenBLAS)", "seconds": round(dt, 2),
            "fp64_gflops_achieved": round(gflops64, 2),
            "extrapolated_full_problem_s": round(oracle_full_cost(cfg) / (gflops64 * 1e9), 1),
            "extrapolated_note": "EXTRAPOLATION: full-problem oracle FLOPs (12 B Hq N^2 d, x1/2 causal) / the "
                                 "achieved fp64 rate on the sample",
            "parity_on_sample": par}


if __name__ == "__main__":
    main()
