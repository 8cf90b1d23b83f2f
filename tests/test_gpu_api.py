"""Public API on the GPU: the autograd Function against the oracle, and the
shard property the multi-GPU split relies on (a batch slice computed alone is
bitwise identical to the same slice of the full run)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_08083_b200.inputs import make_inputs
from util import TOL_MAXABS, TOL_RELL2, gen, np64, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("causal", [False, True])
def test_autograd_function(causal):
    from paper_2511_08083_b200 import Attention
    x = gen(1, 384, 4, 2, 128, seed=21)
    q, k, v = (x[n].clone().requires_grad_() for n in ("Q", "K", "V"))
    o = Attention.apply(q, k, v, causal)
    o.backward(x["dO"])
    torch.cuda.synchronize()
    ref = oracle.attn_fwd_bwd(np64(x["Q"]), np64(x["K"]), np64(x["V"]), np64(x["dO"]), causal)
    assert np.abs(np64(o) - ref["O"]).max() <= TOL_MAXABS
    for name, t in (("dQ", q.grad), ("dK", k.grad), ("dV", v.grad)):
        assert rel_l2(np64(t), ref[name]) <= TOL_RELL2, name


@pytest.mark.parametrize("d,causal", [(128, True), (64, False)])
def test_batch_shard_bitwise(d, causal):
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    B, N, Hq, Hkv = 4, 512, 8, 2
    full = make_inputs(B, N, Hq, Hkv, d, seed=9, device="cuda")
    part = make_inputs(B, N, Hq, Hkv, d, seed=9, device="cuda", batches=[2, 3])
    outs = []
    for x in (full, part):  # the deterministic backward (d = 64 defaults to the fused, reordering one)
        o, lse = attn_fwd(x["Q"], x["K"], x["V"], causal)
        outs.append((o, lse) + attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, deterministic=True))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a[2:4], b)


def test_cuda_graph_capture_fwd_bwd():
    """fwd + bwd (whose dQ pass forks onto the library's side stream and joins back)
    captured into a CUDA graph and replayed: bitwise the eager results."""
    from paper_2511_08083_b200 import attn_bwd, attn_fwd, bwd_workspace_bytes
    B, N, Hq, Hkv, d, causal = 2, 640, 8, 2, 128, True
    x = make_inputs(B, N, Hq, Hkv, d, seed=31, device="cuda")
    o = torch.empty_like(x["Q"])
    lse = torch.empty((B, Hq, N), dtype=torch.float32, device="cuda")
    g3 = [torch.empty_like(x[n]) for n in ("Q", "K", "V")]
    ws = torch.empty(bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4, dtype=torch.float32, device="cuda")

    def step():
        attn_fwd(x["Q"], x["K"], x["V"], causal, out=o, lse=lse)
        attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal, workspace=ws, dq=g3[0], dk=g3[1], dv=g3[2])

    step()
    torch.cuda.synchronize()
    eager = [t.clone() for t in (o, lse, *g3)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for t in (o, lse, *g3):
        t.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, (o, lse, *g3)):
        assert torch.equal(a, b)


def test_wrong_buffer_shapes_raise():
    """caller buffers of the wrong shape or size are rejected before any launch."""
    from paper_2511_08083_b200 import attn_bwd, attn_fwd, bwd_workspace_bytes
    B, N, Hq, Hkv, d = 1, 256, 4, 2, 64
    x = make_inputs(B, N, Hq, Hkv, d, seed=1, device="cuda")
    q, k, v, do = x["Q"], x["K"], x["V"], x["dO"]
    with pytest.raises(ValueError, match="shape"):
        attn_fwd(q, k, v, out=torch.empty((B, N - 128, Hq, d), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError, match="shape"):
        attn_fwd(q, k, v, lse=torch.empty((B, Hq, N - 1), dtype=torch.float32, device="cuda"))
    o, lse = attn_fwd(q, k, v)
    with pytest.raises(ValueError, match="shape"):
        attn_bwd(q, k, v, o, lse, do, dk=torch.empty_like(q))
    with pytest.raises(ValueError, match="shape"):
        attn_bwd(q, k, v, o[:, :128], lse, do)
    small = torch.empty(bwd_workspace_bytes(B, Hq, Hkv, N, d) // 4 - 1, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError, match="workspace"):
        attn_bwd(q, k, v, o, lse, do, workspace=small)


def test_concurrent_backward_streams_independent():
    """the forked dQ pass has one side stream per caller stream, so two backward
    calls on two streams neither serialise on a shared side stream nor mix their results:
    each equals the same call made alone (bitwise)."""
    from paper_2511_08083_b200 import attn_bwd, attn_fwd
    B, N, Hq, Hkv, d, causal = 2, 512, 8, 2, 128, True
    xs = [make_inputs(B, N, Hq, Hkv, d, seed=s, device="cuda") for s in (5, 6)]
    fw = [attn_fwd(x["Q"], x["K"], x["V"], causal) for x in xs]
    alone = [attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal) for x, (o, lse) in zip(xs, fw)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [None, None]
    for rep in range(3):
        for i, (x, (o, lse)) in enumerate(zip(xs, fw)):
            streams[i].wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(streams[i]):
                outs[i] = attn_bwd(x["Q"], x["K"], x["V"], o, lse, x["dO"], causal)
        torch.cuda.synchronize()
        for a, b in zip(alone, outs):
            for u, w in zip(a, b):
                assert torch.equal(u, w)
