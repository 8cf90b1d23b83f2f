"""GPU parity of context-parallel ring attention (NEXT #4) through the C ABI:
the LSE merge kernel (hk_attn_merge) and the gradient accumulator (hk_accum_bf16)
against the fp64 oracle, and the whole ring forward + backward — P virtual ranks
driven by one process on one GPU (LoopbackRing: the same schedule and kernels as
DistRing, the exchange is a list rotation) — against the oracle's attention over
the whole sequence, at the BASELINE tolerances."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from util import TOL_MAXABS, TOL_RELL2, np64, rel_l2

pytestmark = pytest.mark.gpu


def test_merge_kernel_matches_oracle():
    from paper_2511_08083_b200 import _lib, api
    from paper_2511_08083_b200.inputs import make_qk_inputs
    B, Nq, Nk, Hq, Hkv, d = 2, 300, 700, 4, 2, 128
    x = make_qk_inputs(B, Nq, Nk, Hq, Hkv, d, seed=1, device="cuda")
    split = 333
    o1, l1 = api.attn_fwd(x["Q"], x["K"][:, :split].contiguous(), x["V"][:, :split].contiguous(), False)
    o2, l2 = api.attn_fwd(x["Q"], x["K"][:, split:].contiguous(), x["V"][:, split:].contiguous(), False)
    # a third partial that saw no key at all (LSE = -inf) must leave the result unchanged
    o3 = torch.zeros_like(o1)
    l3 = torch.full_like(l1, float("-inf"))
    acc = torch.empty(o1.shape, dtype=torch.float32, device="cuda")
    lacc = torch.empty_like(l1)
    out = torch.empty_like(o1)
    L = _lib.lib()
    for i, (o, lse) in enumerate(((o1, l1), (o3, l3), (o2, l2))):
        _lib.check(L.hk_attn_merge(api._ptr(acc), api._ptr(lacc), api._ptr(o), api._ptr(lse),
                                   api._ptr(out) if i == 2 else None, B, Nq, Hq, d, int(i == 0), api._stream()))
    torch.cuda.synchronize()
    ref_o, ref_l = oracle.attn_merge(*oracle.attn_merge(np64(o1), np64(l1), np64(o3), np64(l3)), np64(o2), np64(l2))
    assert np.abs(np64(acc) - ref_o).max() < 1e-5
    assert np.abs(np64(lacc) - ref_l).max() < 1e-5
    assert torch.equal(out, acc.to(torch.bfloat16))
    # and the merged result is the attention over all keys
    full = oracle.attn_fwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), False)
    assert np.abs(np64(out) - full[0]).max() <= TOL_MAXABS
    assert np.abs(np64(lacc) - full[1]).max() <= TOL_MAXABS


def test_accum_kernel():
    from paper_2511_08083_b200 import _lib, api
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn(4096, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3)]
    acc = torch.empty(4096, dtype=torch.float32, device="cuda")
    out = torch.empty(4096, dtype=torch.bfloat16, device="cuda")
    for i, x in enumerate(xs[:2]):
        _lib.check(L.hk_accum_bf16(api._ptr(acc), api._ptr(x), None, ctypes.c_size_t(4096), int(i == 0),
                                   api._stream()))
    _lib.check(L.hk_accum_bf16(api._ptr(acc), api._ptr(xs[2]), api._ptr(out), ctypes.c_size_t(4096), 0,
                               api._stream()))
    torch.cuda.synchronize()
    want = xs[0].double() + xs[1].double()
    assert torch.equal(acc, (xs[0].float() + xs[1].float()))
    assert torch.allclose(out.double(), want + xs[2].double(), rtol=2 ** -8, atol=1e-6)
    _lib.check(L.hk_accum_bf16(api._ptr(acc), None, api._ptr(out), ctypes.c_size_t(4096), 0, api._stream()))
    torch.cuda.synchronize()
    assert torch.equal(out, acc.to(torch.bfloat16))


def test_accum_f32_kernel():
    from paper_2511_08083_b200 import api
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(3, 1000, generator=g, device="cuda")
    b = torch.randn(3, 1000, generator=g, device="cuda")
    want = a + b
    api.accum_f32(a, b)
    torch.cuda.synchronize()
    assert torch.equal(a, want)  # one fp32 addition per element: the same rounding
    with pytest.raises(ValueError):
        api.accum_f32(a, b[:, :8])


def test_sm_budget_results_unchanged():
    """hk_set_max_ctas: the persistent kernels on 16 or 37 SMs (several items per CTA, another
    snake / counter order) give bitwise the results of the full-SM launch (reading #19)."""
    from paper_2511_08083_b200 import api
    from paper_2511_08083_b200.inputs import make_inputs
    for d, causal in ((128, True), (64, False)):
        x = make_inputs(2, 1000, 8, 2, d, seed=3, device="cuda")
        runs = []
        for reserve in (0, 148 - 37, 148 - 16):
            with api.sm_budget(reserve):
                assert api.get_max_ctas() == (0 if reserve == 0 else max(torch.cuda.get_device_properties(0)
                                                                         .multi_processor_count - reserve, 2))
                o, lse = api.attn_fwd(x["Q"], x["K"], x["V"], causal)
                g = api.attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, deterministic=True)
                c = api.gemm(x["Q"].reshape(-1, d)[:512].contiguous(), x["K"].reshape(-1, d)[:256].contiguous())
            assert api.get_max_ctas() == 0
            torch.cuda.synchronize()
            runs.append((o, lse) + tuple(g) + (c,))
        for other in runs[1:]:
            assert all(torch.equal(a, b) for a, b in zip(runs[0], other))


CASES = [
    # P, B, N, Hq, Hkv, d
    (2, 1, 1024, 4, 2, 128),
    (4, 2, 2048, 4, 1, 64),
    (3, 1, 1536, 8, 2, 128),   # c = 256
    (2, 2, 640, 2, 2, 64),     # c = 160: ragged 128-row tiles inside every chunk
    (8, 1, 2048, 4, 2, 128),   # P = 8: 16 chunks of 128 rows, 8 steps of fp32 accumulation
]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("case", CASES)
def test_ring_loopback_matches_whole_sequence(case, causal):
    from paper_2511_08083_b200 import ring
    from paper_2511_08083_b200.inputs import make_inputs
    P, B, N, Hq, Hkv, d = case
    x = make_inputs(B, N, Hq, Hkv, d, seed=7, device="cuda")
    sh = {n: [ring.zigzag_shard(x[n], P, r) for r in range(P)] for n in ("Q", "K", "V", "dO")}
    comm = ring.LoopbackRing(P)
    fw = ring.ring_attn_fwd(sh["Q"], sh["K"], sh["V"], causal, comm)
    o = [f[0] for f in fw]
    lse = [f[1] for f in fw]
    bw = ring.ring_attn_bwd(sh["Q"], sh["K"], sh["V"], o, lse, sh["dO"], causal, comm)
    # the same schedule with each step's calls on 3 side streams: the forward bitwise the same; the
    # backward there sums bf16-rounded per-call partials (calls sharing an fp32 accumulator would
    # race), so it agrees with the one-stream fp32-accumulating backward to bf16 rounding
    fw3 = ring.ring_attn_fwd(sh["Q"], sh["K"], sh["V"], causal, comm, streams=3)
    bw3 = ring.ring_attn_bwd(sh["Q"], sh["K"], sh["V"], o, lse, sh["dO"], causal, comm, streams=3)
    # SMs left free for the transfers (the NCCL setting): bitwise the same results
    fwr = ring.ring_attn_fwd(sh["Q"], sh["K"], sh["V"], causal, comm, reserve_sms=20)
    bwr = ring.ring_attn_bwd(sh["Q"], sh["K"], sh["V"], o, lse, sh["dO"], causal, comm, reserve_sms=20)
    torch.cuda.synchronize()
    for r in range(P):
        assert all(torch.equal(a, b) for a, b in zip(fw[r][0] + fw[r][1], fwr[r][0] + fwr[r][1]))
        assert all(torch.equal(a, b) for g1, g2 in zip(bw[r], bwr[r]) for a, b in zip(g1, g2))
    for r in range(P):
        assert all(torch.equal(a, b) for a, b in zip(fw[r][0] + fw[r][1], fw3[r][0] + fw3[r][1]))
        for g1, g3 in zip(bw[r], bw3[r]):
            for a, b in zip(g1, g3):
                assert rel_l2(np64(b), np64(a)) <= 4e-3
    O = ring.zigzag_unshard(o)
    LSE = ring.zigzag_unshard([(a.transpose(1, 2), b.transpose(1, 2)) for a, b in lse]).transpose(1, 2)
    dQ, dK, dV = (ring.zigzag_unshard([b[i] for b in bw]) for i in range(3))
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), causal)
    assert np.abs(np64(O) - ref["O"]).max() <= TOL_MAXABS
    assert np.abs(np64(LSE) - ref["LSE"]).max() <= TOL_MAXABS
    for n, t in (("dQ", dQ), ("dK", dK), ("dV", dV)):
        assert rel_l2(np64(t), ref[n]) <= TOL_RELL2, n


def _dist_worker(rank, world, port, causal, out):
    import os
    import torch.distributed as dist
    from paper_2511_08083_b200 import ring
    from paper_2511_08083_b200.inputs import make_inputs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    B, N, Hq, Hkv, d = 1, 1024, 4, 2, 128
    x = make_inputs(B, N, Hq, Hkv, d, seed=11, device="cuda")
    sh = {n: ring.zigzag_shard(x[n], world, rank) for n in ("Q", "K", "V", "dO")}
    comm = ring.DistRing()
    (o, lse), = ring.ring_attn_fwd([sh["Q"]], [sh["K"]], [sh["V"]], causal, comm)
    (dq, dk, dv), = ring.ring_attn_bwd([sh["Q"]], [sh["K"]], [sh["V"]], [o], [lse], [sh["dO"]], causal, comm)
    torch.cuda.synchronize()
    loop = ring.LoopbackRing(world)
    shl = {n: [ring.zigzag_shard(x[n], world, r) for r in range(world)] for n in ("Q", "K", "V", "dO")}
    fw = ring.ring_attn_fwd(shl["Q"], shl["K"], shl["V"], causal, loop)
    bw = ring.ring_attn_bwd(shl["Q"], shl["K"], shl["V"], [f[0] for f in fw], [f[1] for f in fw], shl["dO"],
                            causal, loop)
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(o + dq + dk + dv, fw[rank][0] + bw[rank][0] + bw[rank][1] +
                                                 bw[rank][2]))
    out.put((rank, bool(same)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("causal", [False, True])
def test_ring_two_processes_equal_loopback(causal):
    """Two processes (ranks) sharing the GPU, exchanging over gloo through DistRing,
    produce bitwise the loopback results (same kernels, same order of merges)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, causal, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert res[0] and res[1], res
