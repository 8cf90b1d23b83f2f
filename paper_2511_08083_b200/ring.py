"""Context-parallel (ring) attention over torch.distributed.

The sequence (length N) of a [B, N, H, d] batch is cut into 2P chunks of c = N / (2P)
rows; rank r holds chunks r and 2P-1-r of Q, K, V, dO ("zigzag": with a causal mask
every rank then does the same work). K and V travel around the ring (rank r sends
to r+1, receives from r-1) for P steps; at step s rank r holds the K/V chunks of
rank src = (r - s) mod P and computes, for each of its two query chunks qc and
each key chunk kc it holds:
    kc < qc  -> full (non-causal) attention         kc == qc -> causal
    kc > qc  -> nothing (causal only)
with the CUDA kernels of include/hk_attn.h, folding each partial (O, LSE) into an
fp32 accumulator with hk_attn_merge (include/hk_ring.h). The backward rotates K,
V and fp32 dK/dV accumulators; with the final O and LSE every hk_attn_bwd call
returns its key set's exact share of dQ, dK, dV, added straight into the fp32
accumulators (HK_BWD_ACCUMULATE_F32; with streams > 1, bf16 partials summed by
hk_accum_bf16), and one more rotation brings dK/dV home.

Every arithmetic step runs in libhkattn.so; this module only schedules calls and
moves tensors. The exchange is behind `RingComm`: `DistRing` (one rank per
process, torch.distributed P2P — NCCL over NVLink on a GPU box, CPU staging under
gloo) or `LoopbackRing` (all P ranks driven by one process on one device: the
same schedule and kernels, the exchange is a list rotation; used by the 1-GPU
tests and the measurement script).
"""
from __future__ import annotations

import ctypes

import torch

from . import api
from ._lib import check, lib


# ---------------------------------------------------------------- zigzag layout
def zigzag_chunks(P: int, r: int):
    """Global chunk indices (of 2P) held by rank r: (r, 2P-1-r)."""
    return (r, 2 * P - 1 - r)


def zigzag_shard(x: torch.Tensor, P: int, r: int):
    """Rank r's two chunks of a [B, N, ...] tensor, each contiguous [B, N/(2P), ...]."""
    N = x.shape[1]
    if N % (2 * P):
        raise ValueError(f"N={N} must be a multiple of 2P={2 * P}")
    c = N // (2 * P)
    return tuple(x[:, i * c:(i + 1) * c].contiguous() for i in zigzag_chunks(P, r))


def zigzag_unshard(parts):
    """Inverse of zigzag_shard over all ranks: parts[r] = (chunk r, chunk 2P-1-r)."""
    P = len(parts)
    chunks = [None] * (2 * P)
    for r, (a, b) in enumerate(parts):
        i, j = zigzag_chunks(P, r)
        chunks[i], chunks[j] = a, b
    return torch.cat(chunks, dim=1)


def visibility(qc: int, kc: int, causal: bool):
    """None (nothing visible), 'full' or 'causal' for query chunk qc vs key chunk kc."""
    if not causal or kc < qc:
        return "full"
    return "causal" if kc == qc else None


def plan(P: int, r: int, causal: bool):
    """The (step, q_half, k_half, mode) list rank r executes (deterministic)."""
    out = []
    for s in range(P):
        src = (r - s) % P
        qc, kc = zigzag_chunks(P, r), zigzag_chunks(P, src)
        for qh in (0, 1):
            for kh in (0, 1):
                m = visibility(qc[qh], kc[kh], causal)
                if m is not None:
                    out.append((s, qh, kh, m))
    return out


# ---------------------------------------------------------------- exchange
class RingComm:
    """ranks: the global ranks this process drives; world: P."""
    world: int
    ranks: list

    def start(self, per_rank):  # per_rank[i]: list of tensors of local rank i, sent to rank + 1
        raise NotImplementedError

    def finish(self, handle):  # -> per_rank list of received tensor lists (from rank - 1)
        raise NotImplementedError


class LoopbackRing(RingComm):
    """All P ranks in this process: the exchange is a rotation of the list."""

    def __init__(self, world: int):
        self.world, self.ranks = world, list(range(world))

    def start(self, per_rank):
        return [per_rank[(i - 1) % self.world] for i in range(self.world)]

    def finish(self, handle):
        return handle


class DistRing(RingComm):
    """One rank per process over torch.distributed point-to-point (batch_isend_irecv).
    Under NCCL the CUDA tensors go straight over NVLink; other backends (gloo) stage
    through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]
        self.staged = dist.get_backend(group) != "nccl"

    def _peer(self, d):
        r = (self.ranks[0] + d) % self.world
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def start(self, per_rank):
        send = per_rank[0]
        if self.staged:
            send = [t.cpu() for t in send]
        recv = [torch.empty_like(t) for t in send]
        ops = [self.dist.P2POp(self.dist.isend, t, self._peer(1), self.group) for t in send]
        ops += [self.dist.P2POp(self.dist.irecv, t, self._peer(-1), self.group) for t in recv]
        reqs = self.dist.batch_isend_irecv(ops)
        return reqs, recv, per_rank[0][0].device

    def finish(self, handle):
        reqs, recv, dev = handle
        for q in reqs:
            q.wait()
        if self.staged:
            recv = [t.to(dev) for t in recv]
        return [recv]


# ---------------------------------------------------------------- kernels
def _merge(o_acc, lse_acc, o_part, lse_part, o_out, init):
    B, c, H, d = o_part.shape
    check(lib().hk_attn_merge(api._ptr(o_acc), api._ptr(lse_acc), api._ptr(o_part), api._ptr(lse_part),
                              api._ptr(o_out) if o_out is not None else None, B, c, H, d, int(init),
                              api._stream()))


def _accum(acc, x, out=None, init=False):
    n = (x if x is not None else out).numel()
    check(lib().hk_accum_bf16(api._ptr(acc) if acc is not None else None,
                              api._ptr(x) if x is not None else None,
                              api._ptr(out) if out is not None else None, ctypes.c_size_t(n), int(init),
                              api._stream()))


class _Fanout:
    """Runs a step's independent attention calls on a pool of side streams (so the small
    chunk-pair kernels of one step fill the SMs together); the dependent merges and
    accumulations stay on the calling stream, in plan order, each after its call's event.
    n <= 1: everything on the calling stream, in order."""

    def __init__(self, n: int):
        self.main = torch.cuda.current_stream() if n > 1 else None  # n <= 1 touches no CUDA state
        self.side = [torch.cuda.Stream() for _ in range(n)] if n > 1 else []
        self.i = 0

    def begin(self):  # side streams see everything enqueued so far on the calling stream
        if self.side:
            e = torch.cuda.Event()
            e.record(self.main)
            for st in self.side:
                st.wait_event(e)

    def run(self, fn):
        if not self.side:
            fn()
            return None
        st = self.side[self.i % len(self.side)]
        self.i += 1
        with torch.cuda.stream(st):
            fn()
        e = torch.cuda.Event()
        e.record(st)
        return e

    def join(self, e):
        if e is not None:
            self.main.wait_event(e)


# ---------------------------------------------------------------- forward / backward
# SMs the persistent kernels leave free during a ring step when the exchange runs NCCL copy kernels
# on the same GPU (api.sm_budget): with every SM held by a one-CTA-per-SM kernel the transfer of the
# next step's K/V (and the dK/dV accumulators) cannot start until the step's kernels drain
RESERVE_SMS_NCCL = 8


def _reserve(comm: RingComm) -> int:
    return RESERVE_SMS_NCCL if isinstance(comm, DistRing) and not comm.staged else 0


def ring_attn_fwd(q, k, v, causal: bool, comm: RingComm, streams: int = 1, reserve_sms: int | None = None):
    """q, k, v: per local rank, (A, B) chunk pairs of [B, c, H, d] bf16 CUDA tensors
    (zigzag_shard). Returns per local rank ((oA, oB), (lseA, lseB)): O bf16
    [B, c, Hq, d], LSE fp32 [B, Hq, c] of the attention over the whole sequence.
    streams > 1: a step's attention calls run concurrently on that many side streams.
    reserve_sms: SMs the persistent kernels leave free for the K/V transfer (default: _reserve)."""
    with api.sm_budget(_reserve(comm) if reserve_sms is None else reserve_sms):
        return _ring_attn_fwd(q, k, v, causal, comm, streams)


def _ring_attn_fwd(q, k, v, causal, comm, streams):
    P = comm.world
    fan = _Fanout(streams)
    plans = [plan(P, r, causal) for r in comm.ranks]
    out = []
    for li, _ in enumerate(comm.ranks):
        qa = q[li][0]
        B, c, Hq, d = qa.shape
        out.append({"acc": [torch.empty(qa.shape, dtype=torch.float32, device=qa.device) for _ in range(2)],
                    "lse": [torch.empty((B, Hq, c), dtype=torch.float32, device=qa.device) for _ in range(2)],
                    "o": [torch.empty_like(qa) for _ in range(2)],
                    "seen": [0, 0],
                    "last": {qh: max(i for i, p in enumerate(plans[li]) if p[1] == qh) for qh in (0, 1)}})
    kv = [[k[li][0], k[li][1], v[li][0], v[li][1]] for li in range(len(comm.ranks))]
    for s in range(P):
        handle = comm.start(kv) if s + 1 < P else None
        fan.begin()
        parts = []
        for li in range(len(comm.ranks)):
            for i, (ps, qh, kh, mode) in enumerate(plans[li]):
                if ps != s:
                    continue
                qq, kk, vv = q[li][qh], kv[li][kh], kv[li][2 + kh]
                o_p = torch.empty_like(qq)
                l_p = torch.empty((qq.shape[0], qq.shape[2], qq.shape[1]), dtype=torch.float32, device=qq.device)
                e = fan.run(lambda qq=qq, kk=kk, vv=vv, o_p=o_p, l_p=l_p, m=mode:
                            api.attn_fwd(qq, kk, vv, m == "causal", out=o_p, lse=l_p))
                parts.append((li, i, qh, o_p, l_p, e))
        for li, i, qh, o_p, l_p, e in parts:
            st = out[li]
            fan.join(e)
            _merge(st["acc"][qh], st["lse"][qh], o_p, l_p, st["o"][qh] if i == st["last"][qh] else None,
                   st["seen"][qh] == 0)
            st["seen"][qh] += 1
        if handle is not None:
            kv = comm.finish(handle)
    return [((st["o"][0], st["o"][1]), (st["lse"][0], st["lse"][1])) for st in out]


def ring_attn_bwd(q, k, v, o, lse, do, causal: bool, comm: RingComm, streams: int = 1,
                  reserve_sms: int | None = None):
    """Backward of ring_attn_fwd. All arguments per local rank as (A, B) chunk pairs
    (o, lse from ring_attn_fwd). Returns per local rank ((dqA, dqB), (dkA, dkB), (dvA, dvB)).
    streams > 1: a step's backward calls run concurrently on that many side streams.
    reserve_sms: SMs the persistent kernels leave free for the transfers (default: _reserve)."""
    P = comm.world
    fan = _Fanout(streams)
    plans = [plan(P, r, causal) for r in comm.ranks]
    n_local = len(comm.ranks)
    dq_acc = [[torch.empty(q[li][h].shape, dtype=torch.float32, device=q[li][h].device) for h in (0, 1)]
              for li in range(n_local)]
    dq = [[torch.empty_like(q[li][h]) for h in (0, 1)] for li in range(n_local)]
    dq_seen = [[0, 0] for _ in range(n_local)]
    dq_last = [{qh: max(i for i, p in enumerate(plans[li]) if p[1] == qh) for qh in (0, 1)} for li in range(n_local)]
    # K, V travel one step ahead of the compute; the fp32 dK, dV accumulators travel one step
    # behind it: at step s each rank forms its contributions to the chunks it now holds in fresh
    # zeroed buffers while the accumulators of the same chunks (sent by the previous rank at the end
    # of step s - 1) are in flight, then adds the arrivals in (hk_accum_f32) and sends the sums on.
    # After the last step that send brings every chunk's dK, dV home (src = r + 1 at step P - 1).
    kv = [[k[li][0], k[li][1], v[li][0], v[li][1]] for li in range(n_local)]
    h_acc = None
    with api.sm_budget(_reserve(comm) if reserve_sms is None else reserve_sms):
        for s in range(P):
            h_kv = comm.start(kv) if s + 1 < P else None
            own = [[torch.zeros(kv[li][i].shape, dtype=torch.float32, device=kv[li][i].device) for i in range(4)]
                   for li in range(n_local)]
            fan.begin()
            parts = []
            for li in range(n_local):
                t = kv[li]
                for i, (ps, qh, kh, mode) in enumerate(plans[li]):
                    if ps != s:
                        continue
                    args = (q[li][qh], t[kh], t[2 + kh], o[li][qh], lse[li][qh], do[li][qh])
                    ws = torch.empty(api.bwd_workspace_bytes(args[0].shape[0], args[0].shape[2], args[1].shape[2],
                                                             args[0].shape[1], args[0].shape[3]) // 4,
                                     dtype=torch.float32, device=args[0].device)
                    if streams == 1:
                        # one stream: the call adds its share straight into the fp32 accumulators
                        # (HK_BWD_ACCUMULATE_F32) — no bf16 rounding of the per-step partials
                        if dq_seen[li][qh] == 0:
                            dq_acc[li][qh].zero_()
                        dq_seen[li][qh] += 1
                        api.attn_bwd(*args, mode == "causal", workspace=ws, dq=dq_acc[li][qh], dk=own[li][kh],
                                     dv=own[li][2 + kh], deterministic=True, accumulate=True)
                        if i == dq_last[li][qh]:
                            _accum(dq_acc[li][qh], None, dq[li][qh])
                        continue
                    g = [torch.empty_like(args[0]), torch.empty_like(args[1]), torch.empty_like(args[2])]
                    e = fan.run(lambda args=args, g=g, ws=ws, m=mode:
                                api.attn_bwd(*args, m == "causal", workspace=ws, dq=g[0], dk=g[1], dv=g[2],
                                             deterministic=True))
                    # the workspace (and the partials) stay referenced until the join: freed earlier, the
                    # caching allocator would hand the block to the next call while this one still runs
                    parts.append((li, i, qh, kh, g, e, ws))
            # streams > 1: calls sharing an accumulator would race, so each writes bf16 partials that are
            # summed here in fp32 (hk_accum_bf16)
            for li, i, qh, kh, (dq_p, dk_p, dv_p), e, _ws in parts:
                fan.join(e)
                last = i == dq_last[li][qh]
                _accum(dq_acc[li][qh], dq_p, dq[li][qh] if last else None, dq_seen[li][qh] == 0)
                dq_seen[li][qh] += 1
                _accum(own[li][kh], dk_p)
                _accum(own[li][2 + kh], dv_p)
            if h_acc is not None:  # the previous ranks' sums for the chunks this rank holds now
                inc = comm.finish(h_acc)
                for li in range(n_local):
                    for i in range(4):
                        api.accum_f32(own[li][i], inc[li][i])
            h_acc = comm.start(own)
            if h_kv is not None:
                kv = comm.finish(h_kv)
        home = comm.finish(h_acc)
    res = []
    for li in range(n_local):
        t = home[li]
        dk = [torch.empty_like(k[li][h]) for h in (0, 1)]
        dv = [torch.empty_like(v[li][h]) for h in (0, 1)]
        for h in (0, 1):
            _accum(t[h], None, dk[h])
            _accum(t[2 + h], None, dv[h])
        res.append(((dq[li][0], dq[li][1]), (dk[0], dk[1]), (dv[0], dv[1])))
    return res
