"""Multi-GPU partitioning of one evaluation: frames for spatial groups, pixels
for temporal groups, and a frame<->pixel all-to-all at every domain change.

Legality is the reference's own slicing rule (``slicer.py:263-280``,
``kernels.py:72-86``): spatial operators have receptive field 1 along b*t, so a
rank may own a range of whole frames (GroupNorm statistics stay local);
temporal operators have receptive field 1 along h and w, so a rank may own a
band of pixels with all frames.  SURVEY.md §8(e).

Storage model: a rank stores only its shard of every value, in the layout(s)
the value is read or written in (``Plan._layout_needs``), so its arena is
about 1/world of the single-GPU arena:

* ``S`` (spatial):  rows  F_r x all pixels   (F_r = the rank's frame range),
  row (f, p) at (f - F_r.start) * h*w + p
* ``T`` (temporal): rows  all frames x P_r   (P_r = the rank's pixel band),
  row (f, p) at f * |P_r| + (p - P_r.start)

An exchange S->T sends rank s the block F_r x P_s and receives F_s x P_r from
every peer; its own block F_r x P_r is a local copy between its two buffers.
T->S is the transpose.  A value exchanged once is valid in both layouts.

:func:`plan_exchanges` is the layout pass: it walks the compiled units of one
evaluation and inserts an exchange before every group whose input (or fused
residual operand) is not valid in the group's domain.  Transports:
:class:`NcclExchanger` (one process per GPU; torch.distributed
``all_to_all_single`` over NCCL/NVLink, or gloo on CPU for tests) and
:class:`LocalExchanger` (all ranks' plans on one device; direct block copies --
used to validate the partitioning with the real kernels on a single GPU).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N
from .errors import InvalidParam
from .kinds import Domain, OpKind

S, T = "S", "T"


def stream_of(handle: int):
    """torch stream object of a raw cudaStream_t handle (the current stream when it matches: a
    handle of 0 is the default stream, which ExternalStream does not map back to)."""
    cur = torch.cuda.current_stream()
    return cur if cur.cuda_stream == handle else torch.cuda.ExternalStream(handle)


def shard_range(extent: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous chunk of ``extent`` owned by ``rank``."""
    base, rem = divmod(extent, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


@dataclass(frozen=True)
class Block:
    """Rows {f in [f0,f1)} x {p in [p0,p1)} of a (frames*HW, C) value."""

    f0: int
    f1: int
    p0: int
    p1: int

    @property
    def n_outer(self) -> int:
        return self.f1 - self.f0

    @property
    def n_inner(self) -> int:
        return self.p1 - self.p0

    @property
    def rows(self) -> int:
        return self.n_outer * self.n_inner

    def empty(self) -> bool:
        return self.rows == 0


def send_block(src: str, dst: str, frames: int, hw: int, world: int, me: int, peer: int) -> Block:
    """Rows rank ``me`` sends to ``peer`` when converting src -> dst layout."""
    if (src, dst) == (S, T):
        f, p = shard_range(frames, world, me), shard_range(hw, world, peer)
    elif (src, dst) == (T, S):
        f, p = shard_range(frames, world, peer), shard_range(hw, world, me)
    else:
        raise InvalidParam(f"no exchange {src}->{dst}")
    return Block(f[0], f[1], p[0], p[1])


def recv_block(src: str, dst: str, frames: int, hw: int, world: int, me: int, peer: int) -> Block:
    return send_block(src, dst, frames, hw, world, peer, me)


def copy_block(stream, src_rows, dst_rows, blk: Block, C: int, copy_fn=None):
    """Strided copy of one block between two row views (view row (o,i) = frame o, pixel i)."""
    if blk.empty():
        return
    if copy_fn is not None:
        return copy_fn(src_rows, dst_rows, blk, C)
    N.call("sf_copy_rows", src_rows.view(), dst_rows.view(), blk.n_outer, blk.n_inner, C, stream)


# ---------------------------------------------------------------------------
# layout pass
# ---------------------------------------------------------------------------

@dataclass
class ExchangeOp:
    value: str        # graph value id whose rows move
    src: str
    dst: str
    at: int = -1      # schedule index it may start at (right after the value's producer)
    need: int = -1    # schedule index of the first unit that reads it in ``dst``
    done: object = None   # CUDA event recorded when the exchange completes (comm-stream mode)


def value_parts(plan, vid) -> list[str]:
    """Values whose storage makes up ``vid`` (a zero-copy concat is its operands)."""
    return plan._parts(plan._root_fn, vid)


def exchange_schedule(plan, root=None) -> list[ExchangeOp]:
    """Every frame<->pixel exchange of one evaluation, in schedule order.

    Walks ``GroupedGraph.schedule``: a group of domain d reads its input (and fused
    residual operand) in layout d; a value valid only in the other layout is exchanged.
    Each exchange may start right after the unit that last wrote the value (``at``) and
    must finish before its first reader (``need``); in between, on a comm stream, it
    overlaps with the compute of the units that do not depend on it.
    """
    root = root or plan._root_fn
    g = plan.graph
    layout: dict[str, set] = {}
    written: dict[str, int] = {}
    ops = []
    for si, (kind, ref) in enumerate(plan.grouped.schedule):
        if kind == "node":
            n = g.nodes[ref]
            if n.id in plan.fused_adds:
                continue
            if n.kind is OpKind.CONCAT and all(root(plan._storage_id(v)) == root(plan._storage_id(n.id))
                                                for v in n.inputs):
                continue              # zero-copy concat: its operands wrote straight into its buffer
            raise InvalidParam(f"sharded execution needs every boundary op fused; {n.kind.value} {n.id} is not")
        grp = plan.grouped.groups[ref]
        if grp.ops[0].id in plan.emb_nodes:
            continue
        d = S if grp.domain is Domain.SPATIAL else T
        needed = [grp.head_input]
        tail = grp.tail
        out_vals = [tail]
        if tail in plan.epilogue_of:
            add_id, other, is_emb = plan.epilogue_of[tail]
            if not is_emb:
                needed.append(other)
            out_vals.append(add_id)
        for v in needed:
            if v == "x":              # the latent: fp32, consumed by in_conv on local frames only
                continue
            for part in plan._parts(root, v):
                have = layout.get(part, set())
                if d not in have:
                    if not have:
                        raise InvalidParam(f"value {part} consumed before it is produced")
                    src = S if S in have else T
                    ops.append(ExchangeOp(part, src, d, at=written[part] + 1, need=si))
                    have.add(d)
                    layout[part] = have
        for v in out_vals:
            layout[v] = {d}
            written[v] = si
    return ops


def plan_exchanges(plan) -> list[tuple[int, ExchangeOp]]:
    """(schedule index of the first reader, op) for one evaluation, in order."""
    return [(op.need, op) for op in exchange_schedule(plan)]


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class NcclExchanger:
    """One rank per process: pack -> all_to_all_single -> unpack.

    ``group``: a torch.distributed process group (NCCL on GPUs, gloo on CPU).
    ``copy_fn``: optional host-side block copy (CPU tests); default = sf_copy_rows.
    """

    def __init__(self, rank: int, world: int, group=None, copy_fn=None, comm_stream: bool = False):
        self.rank, self.world, self.group, self.copy_fn = rank, world, group, copy_fn
        self.send = None
        self.recv = None
        self.bytes_moved = 0
        # comm-stream mode: pack / all_to_all / unpack run on their own stream, ordered after the
        # value's producer and before its reader by CUDA events (Plan._insert_exchanges)
        self.comm = torch.cuda.Stream() if comm_stream and torch.cuda.is_available() else None

    def _buffers(self, numel, dtype, device):
        if self.send is None or self.send.numel() < numel or self.send.dtype != dtype:
            self.send = torch.empty(numel, dtype=dtype, device=device)
            self.recv = torch.empty(numel, dtype=dtype, device=device)
        return self.send, self.recv

    def exchange_views(self, stream, src_view, dst_view, frames: int, hw: int, C: int, src: str, dst: str,
                       dtype, device):
        """Move one value between layouts; ``src_view(blk)`` / ``dst_view(blk)`` give the row view of
        a block's first row (frame blk.f0, pixel blk.p0) in the source / destination layout."""
        import torch.distributed as dist
        from .device import Rows
        me, W = self.rank, self.world
        sblk = [send_block(src, dst, frames, hw, W, me, s) for s in range(W)]
        rblk = [recv_block(src, dst, frames, hw, W, me, s) for s in range(W)]
        own = sblk[me]
        sblk[me] = rblk[me] = Block(0, 0, 0, 0)
        s_rows = [b.rows * C for b in sblk]
        r_rows = [b.rows * C for b in rblk]
        send, recv = self._buffers(max(sum(s_rows), sum(r_rows), 1), dtype, device)
        off = 0
        for s, b in enumerate(sblk):
            if not b.empty():
                copy_block(stream, src_view(b), Rows(send[off:off + s_rows[s]].view(b.rows, C), 0, b.n_inner), b, C,
                           self.copy_fn)
            off += s_rows[s]
        # this rank's own block moves between its two layouts without leaving the GPU
        copy_block(stream, src_view(own), dst_view(own), own, C, self.copy_fn)
        dist.all_to_all_single(recv[:sum(r_rows)], send[:sum(s_rows)], r_rows, s_rows, group=self.group)
        off = 0
        for s, b in enumerate(rblk):
            if not b.empty():
                copy_block(stream, Rows(recv[off:off + r_rows[s]].view(b.rows, C), 0, b.n_inner), dst_view(b), b, C,
                           self.copy_fn)
            off += r_rows[s]
        self.bytes_moved += sum(s_rows) * send.element_size()

    def exchange(self, plan, op: ExchangeOp, stream):
        s = plan.shapes[op.value]
        t = plan.values[op.value].store[op.src][0]

        def go(st):
            self.exchange_views(st, lambda b: plan.block_rows(op.value, op.src, b.f0, b.p0),
                                lambda b: plan.block_rows(op.value, op.dst, b.f0, b.p0),
                                s.b * s.t, s.h * s.w, s.c, op.src, op.dst, t.dtype, t.device)
        if self.comm is None:
            go(stream)
            return
        start = torch.cuda.Event()
        start.record(stream_of(stream))
        self.comm.wait_event(start)
        with torch.cuda.stream(self.comm):
            go(self.comm.cuda_stream)
        op.done.record(self.comm)


class LocalExchanger:
    """All ranks' plans on one device: block copies straight between their arenas.

    ``comm_stream``: run the copies on a side stream ordered by the plans' exchange events,
    exercising on one GPU the same producer -> exchange -> reader ordering as NcclExchanger."""

    def __init__(self, plans, comm_stream: bool = False):
        self.plans = plans
        self.world = len(plans)
        self.comm = torch.cuda.Stream() if comm_stream else None

    def exchange_all(self, op: ExchangeOp, stream, index: int | None = None):
        if self.comm is not None:
            start = torch.cuda.Event()
            start.record(stream_of(stream))
            self.comm.wait_event(start)
            self._copies(op, self.comm.cuda_stream)
            for p in self.plans:          # every rank's copy of this exchange is now complete
                p.units[index].exchange.done.record(self.comm)
            return
        self._copies(op, stream)

    def _copies(self, op: ExchangeOp, stream):
        W = self.world
        for me in range(W):
            src_plan = self.plans[me]
            s = src_plan.shapes[op.value]
            frames, hw = s.b * s.t, s.h * s.w
            for peer in range(W):
                b = send_block(op.src, op.dst, frames, hw, W, me, peer)
                copy_block(stream, src_plan.block_rows(op.value, op.src, b.f0, b.p0),
                           self.plans[peer].block_rows(op.value, op.dst, b.f0, b.p0), b, s.c)


# ---------------------------------------------------------------------------
# all ranks on one device (partitioning check with the real kernels)
# ---------------------------------------------------------------------------

class VirtualShards:
    """``world`` sharded plans of one network on a single GPU, run in lockstep.

    Every unit runs on every virtual rank over that rank's frames / pixels;
    exchange units move blocks directly between the ranks' arenas.  The
    result is assembled from each rank's own frames.  This exercises exactly
    the per-rank launch sequences the NCCL path runs, with a device-local copy
    in place of the all-to-all ("bitwise agreement with the
    sharded run's per-shard math").
    """

    def __init__(self, cfg, world: int, exec_cfg=None, K: int | None = None, comm_stream: bool = False):
        from dataclasses import replace

        from .executor import ExecConfig
        from .harness import Denoiser
        base = exec_cfg or ExecConfig()
        self.world = world
        self.dens = []
        dw = None
        for r in range(world):
            d = Denoiser(cfg, replace(base, rank=r, world=world), K=K, device_weights=dw)
            dw = d.model.dw
            self.dens.append(d)
        self.K = self.dens[0].K
        self.local = LocalExchanger([d.plan for d in self.dens], comm_stream)
        for d in self.dens:
            d.plan.exchanger = self.local

    def run(self, x0, schedule=None):
        import numpy as np

        from .harness import alpha
        st = torch.cuda.current_stream().cuda_stream
        for d in self.dens:
            d.set_latent(x0)
        keys = set(range(self.K)) if schedule is None else set(schedule.key_steps)
        plans = [d.plan for d in self.dens]
        for s in range(self.K):
            if s in keys:
                for d in self.dens:
                    d.plan.emb_launch(st, d.emb_table[s].data_ptr())
                units = [p.units for p in plans]
            else:
                units = [p.tail_units for p in plans]
            for i, u in enumerate(units[0]):
                if u.exchange is not None:
                    self.local.exchange_all(u.exchange, st, plans[0].units.index(u))
                else:
                    for r in range(self.world):
                        units[r][i].run(st)
            for p in plans:
                N.call("sf_axpy_f32", p.latent_local.data_ptr(), p.eps.data_ptr(), alpha(s, self.K),
                       p.latent_local.numel(), st)
        xs = self.dens[0].model.x_shape
        hw = xs.h * xs.w
        full = torch.empty_like(plans[0].latent)
        for r, p in enumerate(plans):
            f0, f1 = shard_range(xs.b * xs.t, self.world, r)
            full[f0 * hw:f1 * hw] = p.latent[f0 * hw:f1 * hw]
        d0 = self.dens[0]
        return d0.model.download(d0.model.latent_to_bcthw(st, full))
