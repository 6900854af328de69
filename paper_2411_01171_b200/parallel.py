"""Multi-GPU partitioning of one evaluation: frames for spatial groups, pixels
for temporal groups, and a frame<->pixel all-to-all at every domain change.

Legality is the reference's own slicing rule (``slicer.py:263-280``,
``kernels.py:72-86``): spatial operators have receptive field 1 along b*t, so a
rank may own a range of whole frames (GroupNorm statistics stay local);
temporal operators have receptive field 1 along h and w, so a rank may own a
band of pixels with all frames.  SURVEY.md §8(e).

Storage model: every rank allocates the full-size arena (rows of all frames
and pixels); a value is *valid* on a rank only on the rows of its layout:

* ``S`` (spatial):  rows  F_r x all pixels   (F_r = the rank's frame range)
* ``T`` (temporal): rows  all frames x P_r   (P_r = the rank's pixel band)

An exchange S->T sends rank s the block F_r x P_s and receives F_s x P_r from
every peer; T->S is the transpose.  Because blocks land at their global row
positions, no unpack permutation is needed beyond the strided copy, and a
value exchanged once is valid in both layouts (``S|T``).

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


def value_parts(plan, vid) -> list[str]:
    """Values whose storage makes up ``vid`` (a zero-copy concat is its operands)."""
    n = plan.graph.nodes.get(vid)
    if n is not None and n.kind is OpKind.CONCAT and all(
            plan.values[v].buf == plan.values[vid].buf for v in n.inputs):
        out = []
        for v in n.inputs:
            out.extend(value_parts(plan, v))
        return out
    return [vid]


def plan_exchanges(plan) -> list[tuple[int, ExchangeOp]]:
    """(index of the unit it must precede, op) for one evaluation, in order."""
    g = plan.graph
    layout: dict[str, set] = {}
    inserts = []
    for ui, u in enumerate(plan.units):
        kind, ref = u.ref
        if kind == "node":
            n = g.nodes[ref]
            raise InvalidParam(f"sharded execution needs every boundary op fused; {n.kind.value} {n.id} is not")
        grp = plan.grouped.groups[ref]
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
            for part in value_parts(plan, v):
                have = layout.get(part, set())
                if d not in have:
                    if not have:
                        raise InvalidParam(f"value {part} consumed before it is produced")
                    src = S if S in have else T
                    inserts.append((ui, ExchangeOp(part, src, d)))
                    have.add(d)
                    layout[part] = have
        for v in out_vals:
            layout[v] = {d}
    return inserts


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

def _value_rows(plan, vid):
    from .device import Rows
    v = plan.values[vid]
    s = plan.shapes[vid]
    return Rows(v.tensor, 0, s.h * s.w, v.col0), s


class NcclExchanger:
    """One rank per process: pack -> all_to_all_single -> unpack.

    ``group``: a torch.distributed process group (NCCL on GPUs, gloo on CPU).
    ``copy_fn``: optional host-side block copy (CPU tests); default = sf_copy_rows.
    """

    def __init__(self, rank: int, world: int, group=None, copy_fn=None):
        self.rank, self.world, self.group, self.copy_fn = rank, world, group, copy_fn
        self.send = None
        self.recv = None
        self.bytes_moved = 0

    def _buffers(self, numel, dtype, device):
        if self.send is None or self.send.numel() < numel or self.send.dtype != dtype:
            self.send = torch.empty(numel, dtype=dtype, device=device)
            self.recv = torch.empty(numel, dtype=dtype, device=device)
        return self.send, self.recv

    def exchange_rows(self, stream, rows, frames: int, hw: int, C: int, src: str, dst: str):
        """Move the blocks of one (frames*hw, C) row view between layouts."""
        import torch.distributed as dist
        from .device import Rows
        me, W = self.rank, self.world
        sblk = [send_block(src, dst, frames, hw, W, me, s) for s in range(W)]
        rblk = [recv_block(src, dst, frames, hw, W, me, s) for s in range(W)]
        for s in (me,):
            sblk[s] = Block(0, 0, 0, 0)
            rblk[s] = Block(0, 0, 0, 0)
        s_rows = [b.rows * C for b in sblk]
        r_rows = [b.rows * C for b in rblk]
        send, recv = self._buffers(max(sum(s_rows), sum(r_rows), 1), rows.t.dtype, rows.t.device)
        off = 0
        for s, b in enumerate(sblk):
            if not b.empty():
                src_v = rows.shifted(rows=b.f0 * hw + b.p0)
                dst_v = Rows(send[off:off + s_rows[s]].view(b.rows, C), 0, b.n_inner)
                copy_block(stream, src_v, dst_v, b, C, self.copy_fn)
            off += s_rows[s]
        dist.all_to_all_single(recv[:sum(r_rows)], send[:sum(s_rows)], r_rows, s_rows, group=self.group)
        off = 0
        for s, b in enumerate(rblk):
            if not b.empty():
                src_v = Rows(recv[off:off + r_rows[s]].view(b.rows, C), 0, b.n_inner)
                dst_v = rows.shifted(rows=b.f0 * hw + b.p0)
                copy_block(stream, src_v, dst_v, b, C, self.copy_fn)
            off += r_rows[s]
        self.bytes_moved += sum(s_rows) * rows.t.element_size()

    def exchange(self, plan, op: ExchangeOp, stream):
        rows, s = _value_rows(plan, op.value)
        self.exchange_rows(stream, rows, s.b * s.t, s.h * s.w, s.c, op.src, op.dst)


class LocalExchanger:
    """All ranks' plans on one device: block copies straight between arenas."""

    def __init__(self, plans):
        self.plans = plans
        self.world = len(plans)

    def exchange_all(self, op: ExchangeOp, stream):
        W = self.world
        for me in range(W):
            src_rows, s = _value_rows(self.plans[me], op.value)
            frames, hw = s.b * s.t, s.h * s.w
            for peer in range(W):
                if peer == me:
                    continue
                b = send_block(op.src, op.dst, frames, hw, W, me, peer)
                dst_rows, _ = _value_rows(self.plans[peer], op.value)
                off = b.f0 * hw + b.p0
                copy_block(stream, src_rows.shifted(rows=off), dst_rows.shifted(rows=off), b, s.c)


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

    def __init__(self, cfg, world: int, exec_cfg=None, K: int | None = None):
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
        self.local = LocalExchanger([d.plan for d in self.dens])

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
                    self.local.exchange_all(u.exchange, st)
                else:
                    for r in range(self.world):
                        units[r][i].run(st)
            for p in plans:
                N.call("sf_axpy_f32", p.latent.data_ptr(), p.eps.data_ptr(), alpha(s, self.K), p.latent.numel(), st)
        xs = self.dens[0].model.x_shape
        hw = xs.h * xs.w
        full = torch.empty_like(plans[0].latent)
        for r, p in enumerate(plans):
            f0, f1 = shard_range(xs.b * xs.t, self.world, r)
            full[f0 * hw:f1 * hw] = p.latent[f0 * hw:f1 * hw]
        d0 = self.dens[0]
        return d0.model.download(d0.model.latent_to_bcthw(st, full))
