"""Device executor: compiles a GroupedGraph into fused sm_100a launches.

Mirrors the reference's missing ``executor`` module (contract ``SPEC.md:312-
380``; ``ExecMode`` values ``grouping.py:343``).  ``execute(graph_or_grouped,
mode, inputs, weights)`` keeps the reference signature; underneath, a
:class:`Plan` is compiled once per (graph, weights, config) and replayed:

1. **Operator Grouping** comes from :func:`grouping.group_operators` -- the
   reference's own partition.  Each group runs slice by slice (Feature Slicer):
   a spatial slice is a contiguous range of whole frames, a temporal slice is a
   band of pixels across all frames; both are *views* into the channels-last
   activation (``sf_view_t``), never copies.  Intermediates of a group live
   in a slice-sized scratch region, so the per-group working set is bounded
   by one slice (paper Eq. 1, §4.2).
2. **Boundary fusion**: every ``Add`` whose first operand comes from a group
   ending in a GEMM-type op (conv, temporal conv, linear, attention) is folded
   into that GEMM's epilogue (the step-embedding add as a per-frame bias, the
   residual adds as a residual read); a ``SiLU`` after a norm or GEMM is
   folded into it; each ``Concat`` allocates one buffer whose channel ranges
   its producers write directly (zero-copy).  None of this changes what is
   computed, only where intermediate sums are rounded (fp32 epilogue instead
   of a bf16 round trip).
3. **Memory**: all group-boundary tensors live in one arena whose offsets come
   from a liveness interval packing over the schedule; scratch is one region
   sized for the largest slice.  ``Plan.arena_bytes + Plan.scratch_bytes`` is
   the device analog of the reference's static peak model.

Precision: activations are stored in bf16, every accumulation is fp32 (GEMM
accumulators in TMEM/registers, norm statistics in fp64), the latent and the
network output are fp32.  Tolerances against the fp64/fp32 oracle are stated
in the tests.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import device as D
from .device import Epilogue, Rows
from .errors import InvalidParam, ShapeMismatch
from .graph import Graph, infer_shapes
from .grouping import GroupedGraph, group_operators
from .kinds import Domain, OpKind
from .ledger import MemoryLedger
from .modes import ExecMode
from .slicer import default_temporal_config
from .tensor import Shape5, Tensor5D
from .unet import PROBE_LABEL, UNetConfig, sinusoidal_step_embedding

GEMM_KINDS = (OpKind.CONV2D, OpKind.TEMPORAL_CONV, OpKind.LINEAR, OpKind.SPATIAL_ATTENTION,
              OpKind.TEMPORAL_ATTENTION)


@dataclass
class ExecConfig:
    """Device execution knobs.

    slice_streams: s > 1 runs a sliced group's consecutive slices round-robin on s streams with s
    scratch copies (slices are independent: disjoint rows of the group output), so the launches of
    small slices overlap instead of leaving the GPU idle -- with single-CTA GEMM tiles in those
    groups; 1 (default) = one stream, one copy.  The budget bounds one copy.
    slicing: "budget" (default) -- per group the fewest slices whose scratch
    fits ``scratch_budget`` (``spatial_k`` / ``temporal_k`` override the count);
    "plan" -- the group's own ``SlicePlan`` (grouping.py:121-127): spatial
    slices are exactly its frame extents, a temporal plan of k_h x k_w tiles
    runs as the same number of contiguous pixel bands (a band is one row view
    of the channels-last layout; the output does not depend on the tiling,
    slicer.py:263-280).  gemm_backend: 0 auto (tcgen05 where the shape allows,
    else mma.sync), 1 mma.sync only, 2 tcgen05 only.
    """

    spatial_k: int | None = None
    temporal_k: int | None = None
    scratch_budget: int = 1 << 30
    slicing: str = "budget"
    slice_streams: int = 1      # s > 1: consecutive slices of a sliced group round-robin over s streams
    ln_fold: bool = False       # LayerNorm -> temporal attention: statistics pass + folded QKV GEMM
                                # (measured: faster at C >= 640, slower at L0 -- profiles finding 31)
    gn_from_conv: bool = True   # a GroupNorm reading a conv's output takes its statistics from the
                                # conv epilogue's partials (sf_gemm gn_partial) instead of a stats pass
    gemm_backend: int = 0
    device: str = "cuda"
    rank: int = 0          # frame/pixel shard owned by this plan (parallel.py)
    world: int = 1


def balanced(extent: int, k: int) -> list[tuple[int, int]]:
    """k nearly equal contiguous chunks (device slice plan)."""
    if extent <= 0:
        return []
    k = max(1, min(k, extent))
    base, rem = divmod(extent, k)
    out, s = [], 0
    for i in range(k):
        n = base + (1 if i < rem else 0)
        out.append((s, s + n))
        s += n
    return out


@dataclass
class Value:
    """Device storage of one graph value."""

    name: str
    shape: Shape5
    kind: str = "rows"          # rows (bf16 channels-last) | emb (fp32 vector) | latent / eps (fp32 rows)
    buf: str | None = None      # arena buffer key
    col0: int = 0
    width: int = 0              # storage row width (>= C when aliased into a concat)
    tensor: torch.Tensor | None = None
    store: dict = field(default_factory=dict)   # layout "F" | "S" | "T" -> (rows tensor, col0)


@dataclass
class Unit:
    """One schedule unit compiled to launches."""

    label: str
    run: object                  # callable(stream)
    ref: tuple = ()              # schedule unit it lowers
    exchange: object = None      # parallel.ExchangeOp for frame<->pixel exchange units
    reads: list = field(default_factory=list)
    writes: list = field(default_factory=list)
    gemm_flops: float = 0.0


class Plan:
    """Compiled launch program for one network evaluation (and its rehash tail)."""

    fp32_out = True      # the graph output (the network's eps) is written as fp32 rows

    def __init__(self, graph: Graph, grouped: GroupedGraph, dw: D.DeviceWeights, cfg: ExecConfig,
                 emb_channels: int | None = None):
        self.graph, self.grouped, self.dw, self.cfg = graph, grouped, dw, cfg
        self.dev = dw.dev
        self.shapes = infer_shapes(graph)
        self.topo = graph.topo_order()
        self.pos = {n: i for i, n in enumerate(self.topo)}
        self.cons = graph.consumers()
        self.values: dict[str, Value] = {}
        self.fused_adds: dict[str, tuple[str, str]] = {}   # add id -> (producer tail, other operand)
        self.epilogue_of: dict[str, tuple[str, str, bool]] = {}  # producer tail -> (add id, operand, is_emb)
        self.units: list[Unit] = []
        self.emb_nodes: list[str] = []
        self.gn_feed: dict[str, str] = {}        # conv node id -> GroupNorm input value it produces
        self.gn_part: dict[str, tuple] = {}      # that value -> (partials tensor, splits per frame)
        self.gn_roles: dict[str, list] = {}      # resampling op -> [(role, value, channel offset)]
        self.gn_meta: dict[str, int] = {}        # value with handed-over statistics -> splits per frame
        self.exchanger = None
        self._analyse()
        self._layout()
        self._compile()
        if cfg.world > 1:
            self._insert_exchanges()

    # ------------------------------------------------------------------ analysis
    def _producer_group(self, vid):
        for gi, g in enumerate(self.grouped.groups):
            if g.tail == vid:
                return gi, g
        return None, None

    def _analyse(self):
        g = self.graph
        for nid in self.topo:
            n = g.nodes[nid]
            if n.kind is OpKind.LINEAR and n.inputs == ("step_emb",):
                self.emb_nodes.append(nid)
        for nid in self.topo:
            n = g.nodes[nid]
            if n.kind is not OpKind.ADD:
                continue
            a, b = n.inputs
            gi, grp = self._producer_group(a)
            if grp is None or grp.ops[-1].kind not in GEMM_KINDS or len(self.cons.get(a, [])) != 1:
                continue
            if grp.ops[-1].kind is OpKind.CONV2D and "w" not in self.dw.p[grp.ops[-1].id]:
                continue
            if a in self.epilogue_of:
                continue
            is_emb = b in self.emb_nodes
            sa, sb = self.shapes[a], self.shapes[b]
            if not is_emb and sa != sb:
                continue
            self.fused_adds[nid] = (a, b)
            self.epilogue_of[a] = (nid, b, is_emb)
        if self.cfg.gn_from_conv and os.environ.get("SF_GN_FROM_CONV") != "0":
            self._analyse_gn_feed()

    def _analyse_gn_feed(self):
        """GroupNorms whose statistics a producer kernel hands over as partial sums, so the
        GroupNorm itself only runs the finalize (kernels.py:228-237 statistics):
          * res.norm2 reads res.conv1's stored output (+ step embedding, unet.py:186-193): the
            conv's GEMM epilogue sums the values it stores (``gn_feed``: conv id -> value);
          * down_blocks.i+1.res.norm1 reads the downsample's output, and up_blocks.i.res.norm1 reads
            concat(skip, upsample(x)) (unet.py:221-244): the downsample kernel sums its output and
            the skip it reads, the upsample kernel the copies it writes; down_blocks.0.res.norm1 reads
            the in_conv output, which the tensor-core in_conv kernel sums (``gn_roles``: op id ->
            [(role, value, channel offset)]).
        Each value gets [frames][splits][C] float2 partials; ``gn_meta``: value -> splits."""
        self.gn_roles: dict[str, list] = {}
        self.gn_meta: dict[str, int] = {}
        f0, f1 = self._frames()
        nf = f1 - f0
        sms = (torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
               if torch.cuda.is_available() else 148)
        down_of_input = {grp.head_input: grp.ops[0].id for grp in self.grouped.groups
                         if len(grp.ops) == 1 and grp.ops[0].kind is OpKind.DOWNSAMPLE2X}
        up_by_tail = {grp.tail: grp.ops[0].id for grp in self.grouped.groups
                      if len(grp.ops) == 1 and grp.ops[0].kind is OpKind.UPSAMPLE2X}
        down_by_tail = {grp.tail: grp.ops[0].id for grp in self.grouped.groups
                        if len(grp.ops) == 1 and grp.ops[0].kind is OpKind.DOWNSAMPLE2X}

        def resample_splits(coarse):
            # splits over the coarse grid (the downsample's outputs = the upsample's inputs): the same
            # count for both producers of a concat's partials; frames x splits <= 2 blocks per SM (the
            # downsample kernel holds 127 registers x 240 threads: two blocks per SM, one wave)
            return max(1, min((2 * sms) // max(1, nf), coarse, 16))
        for grp in self.grouped.groups:
            if grp.domain is not Domain.SPATIAL or grp.ops[0].kind is not OpKind.GROUP_NORM:
                continue
            v = grp.head_input
            node = self.graph.nodes.get(v)
            if v in down_by_tail:
                self.gn_roles.setdefault(down_by_tail[v], []).append(("out", v, 0))
                self.gn_meta[v] = resample_splits(self.shapes[v].h * self.shapes[v].w)
                continue
            if node is not None and node.kind is OpKind.CONCAT and len(node.inputs) == 2:
                a, b = node.inputs
                sa, sv = self.shapes[a], self.shapes[v]
                if a in down_of_input and b in up_by_tail and (sa.h, sa.w) == (sv.h, sv.w) and sa.h % 2 == 0 \
                        and sa.w % 2 == 0:
                    self.gn_roles.setdefault(down_of_input[a], []).append(("in", v, 0))
                    self.gn_roles.setdefault(up_by_tail[b], []).append(("out", v, sa.c))
                    self.gn_meta[v] = resample_splits((sv.h // 2) * (sv.w // 2))
                continue
            src = self.fused_adds[v][0] if v in self.fused_adds else v
            _, pg = self._producer_group(src)
            if pg is None or pg.domain is not Domain.SPATIAL:
                continue
            conv = pg.ops[-1]
            if conv.kind is not OpKind.CONV2D or conv.id in self.gn_feed:
                continue
            if pg.head_input == "x" and len(pg.ops) == 1 and "wt32" in self.dw.p.get(conv.id, {}):
                # in_conv on the tensor-core small-channel kernel (sf_conv3x3_smallcin_gn):
                # task-ordered partials, about one task per warp slot (2 blocks x 8 warps per SM)
                sv, cin = self.shapes[v], self.shapes["x"].c
                if sv.c % 64 == 0 and sv.c <= 640 and 9 * cin <= 96 and v == conv.id:
                    self.gn_roles.setdefault(conv.id, []).append(("smallcin", v, 0))
                    self.gn_meta[v] = max(1, min(-(-(sv.h * sv.w) // 16), (16 * sms) // max(1, nf), 64))
                continue
            if "w" not in self.dw.p.get(conv.id, {}) or pg.head_input == "x":
                continue
            if self.shapes[conv.id] != self.shapes[v]:
                continue
            self.gn_feed[conv.id] = v
            self.gn_meta[v] = int(N.query("sf_conv_gn_splits", self.shapes[v].h, self.shapes[v].w))
        for op_id, roles in self.gn_roles.items():
            if len({self.gn_meta[v] for _, v, _ in roles}) != 1:
                raise InvalidParam(f"{op_id}: its GroupNorm partials need one split count, got "
                                   f"{[(r, v, self.gn_meta[v]) for r, v, _ in roles]}")
        # partial buffers: one slot per set of first-producer -> consumer intervals that do not
        # overlap in the schedule (norm2 follows conv1 directly; a concat's buffer lives from the
        # down path's downsample to the up block)
        spos = {(k, r): i for i, (k, r) in enumerate(self.grouped.schedule)}
        op_pos = {}
        for gi, grp in enumerate(self.grouped.groups):
            for o in grp.ops:
                op_pos[o.id] = spos.get(("group", gi), -1)
        cons_pos: dict[str, int] = {}   # the GroupNorm group that finalizes each value (latest, to be safe)
        for gi, grp in enumerate(self.grouped.groups):
            if grp.ops[0].kind is OpKind.GROUP_NORM:
                cons_pos[grp.head_input] = max(cons_pos.get(grp.head_input, -1), spos[("group", gi)])
        start = {v: op_pos[c] for c, v in self.gn_feed.items()}
        for op_id, roles in self.gn_roles.items():
            for _, v, _ in roles:
                start[v] = min(start.get(v, op_pos[op_id]), op_pos[op_id])
        self._gn_slot_of, self._gn_slot_elems, free_after = {}, [], []
        self.gn_intervals: dict[str, tuple[int, int]] = {}   # value -> (first producer, consumer) positions
        for v in sorted(start, key=lambda u: start[u]):
            a, b = start[v], cons_pos[v]
            self.gn_intervals[v] = (a, b)
            elems = nf * self.gn_meta[v] * self.shapes[v].c * 2
            for k, fa in enumerate(free_after):
                if fa < a:
                    break
            else:
                k = len(free_after)
                free_after.append(-1)
                self._gn_slot_elems.append(0)
            free_after[k] = b
            self._gn_slot_elems[k] = max(self._gn_slot_elems[k], elems)
            self._gn_slot_of[v] = k
        self._gn_slots: list[torch.Tensor | None] = [None] * len(self._gn_slot_elems)

    def gn_partials(self, vid):
        """(partials buffer over this rank's frames, splits per frame) for a GroupNorm input whose
        statistics a producer hands over; the slot tensor is allocated when the first user compiles."""
        if vid not in self.gn_part:
            k = self._gn_slot_of[vid]
            if self._gn_slots[k] is None:
                self._gn_slots[k] = torch.empty((self._gn_slot_elems[k],), dtype=torch.float32, device=self.dev)
            self.gn_part[vid] = (self._gn_slots[k], self.gn_meta[vid])
        return self.gn_part[vid]

    # ------------------------------------------------------------------ layout
    def _storage_id(self, vid):
        """Fused-add producers write straight into the add's output."""
        if vid in self.epilogue_of:
            return self.epilogue_of[vid][0]
        return vid

    def _layout(self):
        g = self.graph
        sched = list(self.grouped.schedule)
        # unit index of definition / last use per stored value
        unit_of = {}
        for ui, (k, r) in enumerate(sched):
            outs = [r] if k == "node" else [self.grouped.groups[r].tail]
            for o in outs:
                unit_of[o] = ui
        uses: dict[str, list[int]] = {}
        for ui, (k, r) in enumerate(sched):
            ins = g.nodes[r].inputs if k == "node" else (self.grouped.groups[r].head_input,)
            for v in ins:
                uses.setdefault(v, []).append(ui)
            if k == "group":
                tail = self.grouped.groups[r].tail
                if tail in self.epilogue_of:
                    add_id, other, _ = self.epilogue_of[tail]
                    uses.setdefault(other, []).append(ui)
        # concat aliasing: operand -> (concat id, col offset)
        alias: dict[str, tuple[str, int]] = {}
        for nid in self.topo:
            n = g.nodes[nid]
            if n.kind is OpKind.CONCAT:
                off = 0
                ok = all(self._storage_id(v) not in alias and v in g.nodes for v in n.inputs)
                if ok:
                    for v in n.inputs:
                        alias[self._storage_id(v)] = (nid, off)
                        off += self.shapes[v].c
        self.alias = alias
        # buffers: one per (storage root, layout)
        intervals: dict[str, list[int]] = {}

        def root(sid):
            while sid in alias:
                sid = alias[sid][0]
            return sid
        self._root_fn = root
        self.root = lambda vid: root(self._storage_id(vid))

        special = {"x", "step_emb", *self.emb_nodes}
        # only values that cross a schedule unit live in the arena: group tails and
        # ungrouped nodes (group-internal intermediates live in the slice scratch)
        self.materialized = {vid for vid in unit_of if vid not in special}
        for vid, shape in self.shapes.items():
            if vid not in self.materialized:
                continue
            sid = root(self._storage_id(vid))
            d = unit_of.get(vid, unit_of.get(self._storage_id(vid), 0))
            last = max(uses.get(vid, [d]) + [d])
            if vid in g.outputs:
                last = len(sched)
            lo, hi = intervals.get(sid, [d, last])
            intervals[sid] = [min(lo, d), max(hi, last)]
        out_id = g.outputs[0]
        # persistent: the rehash probe (its storage doubles as the feature cache)
        probe = None
        for n in g.nodes.values():
            if n.label == PROBE_LABEL:
                probe = root(self._storage_id(n.id))
        if probe is not None:
            intervals[probe] = [0, len(sched)]
        self.probe_root = probe
        # layouts: unsharded, one full buffer ("F") per root; sharded (parallel.py), a frame-
        # sharded copy "S" (this rank's frames x all pixels) and/or a pixel-sharded copy "T"
        # (all frames x this rank's pixel band) -- only the layouts the root is read or
        # written in, each 1/world of the full size
        self.sharded = self.cfg.world > 1
        if self.sharded:
            # each layout copy lives only while that layout is read or written
            key_iv = self._layout_intervals(root, out_id, len(sched))
            if probe is not None:
                for key in key_iv:
                    if key[0] == probe:
                        key_iv[key] = [0, len(sched)]
        else:
            key_iv = {(sid, "F"): iv for sid, iv in intervals.items()}
        sizes: dict[tuple, int] = {}
        for (sid, L) in key_iv:
            sizes[(sid, L)] = self._layout_rows(self.shapes[sid], L) * self.shapes[sid].c * \
                (4 if sid == out_id else 2)
        # interval packing: largest first, lowest non-conflicting offset
        placed: list[tuple[int, int, int, int]] = []  # (off, size, lo, hi)
        offsets = {}
        align = 256
        for key in sorted(sizes, key=lambda k: (-sizes[k], k)):
            lo, hi = key_iv[key]
            size = (sizes[key] + align - 1) // align * align
            cands = sorted({0} | {o + sz for o, sz, l2, h2 in placed})
            for off in cands:
                if all(not (l2 <= hi and lo <= h2 and off < o + sz and o < off + size) for o, sz, l2, h2 in placed):
                    break
            placed.append((off, size, lo, hi))
            offsets[key] = off
        self.arena_bytes = max([o + s for o, s, _, _ in placed] + [align])
        # kept for the derived memory ledger (ledger.py): live units and payload bytes per buffer
        self.arena_intervals = {key: tuple(key_iv[key]) for key in sizes}
        self.arena_sizes = dict(sizes)
        self.n_units = len(sched)
        self.arena = torch.empty(self.arena_bytes, dtype=torch.uint8, device=self.dev)
        self.buffers = {}
        for key, off in offsets.items():
            sid, L = key
            s = self.shapes[sid]
            rows = self._layout_rows(s, L)
            if sid == out_id:
                t = self.arena[off:off + rows * s.c * 4].view(torch.float32).view(rows, s.c)
            else:
                t = self.arena[off:off + rows * s.c * 2].view(torch.bfloat16).view(rows, s.c)
            self.buffers[key] = t
        # values: each points at its root's buffers (a concat operand at its channel offset)
        for vid, shape in self.shapes.items():
            if vid not in self.materialized:
                continue
            sid = self._storage_id(vid)
            col = 0
            while sid in alias:
                sid, c0 = alias[sid][0], alias[sid][1] + col
                col = c0
            store = {}
            for L in ("F", "S", "T"):
                if (sid, L) in self.buffers:
                    store[L] = (self.buffers[(sid, L)], col)
            if "F" in store:
                store["S"] = store["T"] = store["F"]
            self.values[vid] = Value(vid, shape, buf=sid, col0=col, tensor=store.get("F", (None,))[0], store=store)
        # inputs: latent rows (fp32) and the emb table
        xs = self.shapes["x"]
        self.latent = torch.zeros(xs.b * xs.t * xs.h * xs.w, xs.c, dtype=torch.float32, device=self.dev)
        # the network output (eps) is produced frame-sharded: this rank's frames only
        self.eps = self.values[out_id].store["S"][0]
        F0, F1 = self._frames()
        self.latent_local = self.latent[F0 * xs.h * xs.w:F1 * xs.h * xs.w]
        # step-embedding projections of every res block: one gemv per step
        ws = [self.dw.p[n]["w32"] for n in self.emb_nodes]
        bs = [self.dw.p[n]["bias"] for n in self.emb_nodes]
        self.emb_w = torch.cat(ws, 0).contiguous() if ws else None
        self.emb_b = torch.cat(bs, 0).contiguous() if bs else None
        self.emb_out = torch.zeros(sum(w.shape[0] for w in ws), dtype=torch.float32, device=self.dev)
        self.emb_slot = {}
        off = 0
        for n, w in zip(self.emb_nodes, ws):
            self.emb_slot[n] = self.emb_out[off:off + w.shape[0]]
            off += w.shape[0]
        self.emb_in = torch.zeros(self.shapes["step_emb"].c if "step_emb" in self.shapes else 1,
                                  dtype=torch.float32, device=self.dev)
        self.peak_model_bytes = self.arena_bytes

    def memory_ledger(self, scratch_bytes: int | None = None, summary: dict | None = None) -> MemoryLedger:
        """One evaluation's allocation events, derived from the compiled plan.

        Each arena buffer is charged before the first unit that defines it and
        released after its last consumer (the probe and the network output stay
        to the end); the slice scratch is charged for the whole evaluation.
        """
        led = MemoryLedger(summary)
        g = self.graph

        def tag(key):
            sid, L = key
            n = g.nodes.get(sid)
            base = n.label or sid if n is not None else sid
            return base if L == "F" else f"{base}:{L}"
        if scratch_bytes:
            led.alloc(scratch_bytes, "slice_scratch")
        by_lo: dict[int, list[str]] = {}
        by_hi: dict[int, list[str]] = {}
        for sid, (lo, hi) in sorted(self.arena_intervals.items()):
            by_lo.setdefault(lo, []).append(sid)
            by_hi.setdefault(hi, []).append(sid)
        for u in range(self.n_units + 1):
            for sid in by_lo.get(u, []):
                led.alloc(self.arena_sizes[sid], tag(sid))
            for sid in by_hi.get(u, []):
                led.free(self.arena_sizes[sid], tag(sid))
        if scratch_bytes:
            led.free(scratch_bytes, "slice_scratch")
        return led

    def rows(self, vid, row0=0, ostride=0) -> Rows:
        """Global row view of an unsharded value (row = frame * h*w + pixel)."""
        v = self.values[vid]
        return Rows(v.tensor, row0, ostride, v.col0)

    # -- sharded layouts (parallel.py): S = my frames x all pixels, T = all frames x my pixels
    def _frames(self):
        from .parallel import shard_range
        xs = self.shapes["x"]
        return shard_range(xs.b * xs.t, self.cfg.world, self.cfg.rank)

    def _pixels(self, shape: Shape5):
        from .parallel import shard_range
        return shard_range(shape.h * shape.w, self.cfg.world, self.cfg.rank)

    def _layout_rows(self, shape: Shape5, L: str) -> int:
        if L == "S":
            f0, f1 = self._frames()
            return (f1 - f0) * shape.h * shape.w
        if L == "T":
            p0, p1 = self._pixels(shape)
            return shape.b * shape.t * (p1 - p0)
        return shape.b * shape.t * shape.h * shape.w

    def srows(self, vid, f0: int) -> Rows:
        """Rows (frame f0 + o, pixel i) of a value in its frame-sharded layout (ostride h*w)."""
        v = self.values[vid]
        t, col = v.store["S"]
        hw = v.shape.h * v.shape.w
        base = self._frames()[0] if "F" not in v.store else 0
        return Rows(t, (f0 - base) * hw, hw, col)

    def trows(self, vid, p0: int) -> Rows:
        """Rows (frame o, pixel p0 + i) of a value in its pixel-sharded layout."""
        v = self.values[vid]
        t, col = v.store["T"]
        if "F" in v.store:
            return Rows(t, p0, v.shape.h * v.shape.w, col)
        q0, q1 = self._pixels(v.shape)
        return Rows(t, p0 - q0, q1 - q0, col)

    def block_rows(self, vid, L: str, f0: int, p0: int) -> Rows:
        """Row view starting at (frame f0, pixel p0) in layout L; row (o, i) = (f0 + o, p0 + i)."""
        if L == "S":
            return self.srows(vid, f0).shifted(rows=p0)
        r = self.trows(vid, p0)
        return r.shifted(rows=f0 * r.ostride)

    def _parts(self, root, vid) -> list[str]:
        """Values whose storage makes up ``vid`` (a zero-copy concat is its operands)."""
        n = self.graph.nodes.get(vid)
        if n is not None and n.kind is OpKind.CONCAT and all(
                root(self._storage_id(v)) == root(self._storage_id(vid)) for v in n.inputs):
            return [p for v in n.inputs for p in self._parts(root, v)]
        return [vid]

    def _layout_intervals(self, root, out_id, n_units) -> dict:
        """(storage root, layout) -> [first, last] schedule unit touching that layout copy.

        A group of domain d reads its input (and fused residual) and writes its output in
        layout d; the exchanges of ``parallel.exchange_schedule`` move values between layouts.
        """
        iv: dict[tuple, list[int]] = {}

        def touch(v, L, ui):
            key = (root(self._storage_id(v)), L)
            lo, hi = iv.get(key, [ui, ui])
            iv[key] = [min(lo, ui), max(hi, ui)]
        for ui, (kind, ref) in enumerate(self.grouped.schedule):
            if kind != "group":
                continue
            grp = self.grouped.groups[ref]
            if grp.ops[0].id in self.emb_nodes:
                continue
            d = "S" if grp.domain is Domain.SPATIAL else "T"
            touched = [grp.head_input, grp.tail]
            if grp.tail in self.epilogue_of:
                add_id, other, is_emb = self.epilogue_of[grp.tail]
                touched.append(add_id)
                if not is_emb:
                    touched.append(other)
            for v in touched:
                if v in ("x", "step_emb"):
                    continue
                for part in self._parts(root, v):
                    touch(part, d, ui)
        # an exchange reads its source copy and writes its destination copy anywhere from
        # right after the producer (``at``) until its first reader (``need``): both stay live
        from .parallel import exchange_schedule
        for op in exchange_schedule(self, root):
            for L in (op.src, op.dst):
                touch(op.value, L, op.at)
                touch(op.value, L, op.need)
        key = (root(self._storage_id(out_id)), "S")
        iv[key] = [iv.get(key, [0, 0])[0], n_units]
        return iv

    # ------------------------------------------------------------------ compile
    def _k_for(self, per_unit_bytes: int, extent: int, override: int | None) -> int:
        if override:
            return max(1, min(override, extent))
        units = max(1, self.cfg.scratch_budget // max(1, per_unit_bytes))
        return max(1, math.ceil(extent / units))

    def _insert_exchanges(self):
        """Place every frame<->pixel exchange right after its value's producer; its first reader
        waits on the exchange's completion event (used when the exchanger runs on a comm stream)."""
        from .parallel import exchange_schedule
        ops = exchange_schedule(self)
        sched_idx = {ref: i for i, ref in enumerate(self.grouped.schedule)}
        pos = [sched_idx[u.ref] for u in self.units]
        out = []
        j = 0
        ops = sorted(ops, key=lambda o: (o.at, o.need))
        waits: dict[int, list] = {}
        for op in ops:
            op.done = torch.cuda.Event() if torch.cuda.is_available() and self.dev.type == "cuda" else None
            waits.setdefault(op.need, []).append(op)
        for u, si in zip(self.units, pos):
            while j < len(ops) and ops[j].at <= si:
                op = ops[j]
                out.append(Unit(f"exchange[{op.value} {op.src}->{op.dst}]", self._exchange_runner(op), ref=u.ref,
                                exchange=op))
                j += 1
            if si in waits:
                u.run = self._waiting(u.run, waits[si])
            out.append(u)
        self.units = out
        self.n_exchanges = len(ops)

    def _waiting(self, run, ops):
        def wrapped(st):
            if getattr(self.exchanger, "comm", None) is not None:
                from .parallel import stream_of
                cur = stream_of(st)
                for op in ops:
                    cur.wait_event(op.done)
            run(st)
        return wrapped

    def _exchange_runner(self, op):
        def run(st):
            if self.exchanger is None:
                raise InvalidParam("sharded plan has no exchanger attached")
            self.exchanger.exchange(self, op, st)
        return run

    def _compile(self):
        self.slice_counts: dict[str, int] = {}
        self.scratch_need = 0
        self._scratch_users = []
        for kind, ref in self.grouped.schedule:
            if kind == "node":
                u = self._compile_node(self.graph.nodes[ref])
            else:
                u = self._compile_group(self.grouped.groups[ref])
            if u is not None:
                u.ref = (kind, ref)
                self.units.append(u)
        self.scratch = torch.empty(max(self.scratch_need, 256), dtype=torch.uint8, device=self.dev)
        for fn in self._scratch_users:
            fn(self.scratch)
        self.scratch_bytes = self.scratch.numel()
        self.gn_work = None

    def _scratch(self, specs, copies: int = 1):
        """Reserve ``copies`` sets of named slice-scratch tensors (bound after compile)."""
        off, layout = 0, {}
        for name, (rows, cols, dtype) in specs.items():
            es = torch.empty((), dtype=dtype).element_size()
            layout[name] = (off, rows, cols, dtype)
            off += (rows * cols * es + 255) // 256 * 256
        self.scratch_need = max(self.scratch_need, off * copies)
        holders = [{} for _ in range(copies)]

        def bind(buf):
            for k, holder in enumerate(holders):
                for name, (o, r, c, dt) in layout.items():
                    es = torch.empty((), dtype=dt).element_size()
                    holder[name] = buf[k * off + o:k * off + o + r * c * es].view(dt).view(r, c)
        self._scratch_users.append(bind)
        return holders if copies > 1 else holders[0]

    def _fork(self, st, n):
        """Streams for ``n`` concurrent slice chains: the launch stream and n - 1 side streams
        ordered after everything already issued on it (ExecConfig.slice_streams)."""
        if n == 1:
            return [st]
        from .parallel import stream_of
        sides = self.__dict__.setdefault("_sides", [])
        while len(sides) < n - 1:
            sides.append(torch.cuda.Stream(device=self.dev))
        ev = torch.cuda.Event()
        ev.record(stream_of(st))
        for s in sides[:n - 1]:
            s.wait_event(ev)
        return [st] + [s.cuda_stream for s in sides[:n - 1]]

    def _join(self, st, streams):
        from .parallel import stream_of
        for s in self.__dict__.get("_sides", [])[:len(streams) - 1]:
            ev = torch.cuda.Event()
            ev.record(s)
            stream_of(st).wait_event(ev)

    def _epilogue(self, tail_id, rows_fn):
        """Epilogue for a GEMM-ending group whose output feeds a fused Add."""
        if tail_id not in self.epilogue_of:
            return lambda sl: Epilogue()
        add_id, other, is_emb = self.epilogue_of[tail_id]
        if is_emb:
            eb = self.emb_slot[other]
            return lambda sl: Epilogue(rowbias=eb)
        return lambda sl: Epilogue(res=rows_fn(other, sl))

    def _compile_node(self, n):
        g = self.graph
        if n.id in self.fused_adds or n.id in self.emb_nodes:
            return None
        shp = self.shapes[n.id]
        if n.kind is OpKind.CONCAT:
            outs = []
            for v in n.inputs:
                if self.values[v].buf != self.values[n.id].buf:
                    outs.append(v)
            if not outs:
                return None
            off_map = {}
            off = 0
            for v in n.inputs:
                off_map[v] = off
                off += self.shapes[v].c

            def run(st, n=n, outs=outs, off_map=off_map):
                for v in outs:
                    s = self.shapes[v]
                    N.call("sf_copy_rows", self.rows(v).view(), self.rows(n.id).shifted(cols=off_map[v]).view(),
                           1, s.b * s.t * s.h * s.w, s.c, st)
            return Unit(n.id, run)
        if n.kind is OpKind.ADD:
            a, b = n.inputs
            sa, sb = self.shapes[a], self.shapes[b]
            if b in self.emb_nodes or a in self.emb_nodes:
                raise InvalidParam(f"unfusable step-embedding add {n.id}")
            bcast = (sb.h, sb.w) == (1, 1) and (sa.h, sa.w) != (1, 1)

            def run(st, n=n, a=a, b=b, s=shp, bcast=bcast):
                N.call("sf_add", self.rows(a).view(), self.rows(b, 0, 1 if bcast else 0).view(),
                       self.rows(n.id).view(), s.b * s.t if bcast else 1,
                       s.h * s.w if bcast else s.b * s.t * s.h * s.w, s.c, 1 if bcast else 0, st)
            return Unit(n.id, run)
        if n.kind is OpKind.SPLIT:
            sizes = [int(v) for v in n.attrs["sizes"]]
            off = sum(sizes[:int(n.attrs["index"])])

            def run(st, n=n, off=off, s=shp):
                N.call("sf_copy_rows", self.rows(n.inputs[0]).shifted(cols=off).view(), self.rows(n.id).view(), 1,
                       s.b * s.t * s.h * s.w, s.c, st)
            return Unit(n.id, run)
        raise InvalidParam(f"ungrouped {n.kind.value} node {n.id} has no device lowering")

    def _compile_group(self, grp):
        ops = list(grp.ops)
        kinds = [o.kind for o in ops]
        head_in = grp.head_input
        in_shape = self.shapes[head_in]
        if ops[0].id in self.emb_nodes:
            return None
        if grp.domain is Domain.SPATIAL:
            return self._compile_spatial(grp, ops, kinds, in_shape)
        return self._compile_temporal(grp, ops, kinds, in_shape)

    # spatial groups: slices are frame ranges
    def _compile_spatial(self, grp, ops, kinds, s):
        frames = s.b * s.t
        HW = s.h * s.w
        backend = self.cfg.gemm_backend
        C = s.c
        tail = ops[-1].id
        x_id = grp.head_input
        latent_in = x_id == "x"

        def vrows(vid, sl):
            return self.srows(vid, sl[0])

        epi_fn = self._epilogue(tail, vrows)
        # lower the chain into steps over slice-local buffers; scratch specs per frame first
        steps = []
        pf_specs = {}          # name -> (rows per frame, cols, dtype)
        shape = s
        cur = "IN"
        i = 0
        nb = 0
        flops = 0.0
        gn_shapes = []
        max_groups = max([int(o.attrs.get("groups", 1)) for o in ops if o.kind is OpKind.GROUP_NORM] + [1])
        while i < len(ops):
            o = ops[i]
            nxt = ops[i + 1] if i + 1 < len(ops) else None
            fuse_act = nxt is not None and nxt.kind is OpKind.SILU
            last = (i + (2 if fuse_act else 1)) >= len(ops)
            out_shape = self.shapes[ops[i + (1 if fuse_act else 0)].id]
            dst = "OUT" if last else f"t{nb}"
            if not last:
                pf_specs[dst] = (out_shape.h * out_shape.w, out_shape.c, torch.bfloat16)
                nb += 1
            act = N.ACT_SILU if fuse_act else N.ACT_NONE
            steps.append((o, cur, dst, shape, out_shape, act, last))
            cur = dst
            if o.kind is OpKind.CONV2D:
                flops += 2.0 * frames * out_shape.h * out_shape.w * shape.c * out_shape.c * 9
            elif o.kind is OpKind.LINEAR:
                flops += 2.0 * frames * HW * shape.c * out_shape.c
            elif o.kind is OpKind.SPATIAL_ATTENTION:
                flops += frames * (8.0 * HW * C * C + 4.0 * HW * HW * C)
            if o.kind is OpKind.GROUP_NORM:
                gn_shapes.append(shape)
            if o.kind is OpKind.SPATIAL_ATTENTION:
                hw = shape.h * shape.w
                pf_specs.update(D.spatial_attention_scratch(hw, hw, shape.c))
            if o.kind is OpKind.CONV2D and "w_taps" in self.dw.p.get(o.id, {}):
                pf_specs["taps_y"] = (out_shape.h * out_shape.w, 9 * out_shape.c, torch.float32)
            shape = out_shape
            i += 2 if fuse_act else 1
        # GroupNorm (+ SiLU) -> per-tap out_conv projection: the apply runs inside the projection
        # (sf_group_norm_project), so the normalised tensor is neither written nor scratch
        gn_project = {}
        eps_tail = self.fp32_out and tail == self.graph.outputs[0]
        for a_, b_ in zip(steps, steps[1:]):
            (go, gsrc, gdst, gsh, _, gact, _), (co, csrc, _, csh, cosh, cact, clast) = a_, b_
            if (go.kind is OpKind.GROUP_NORM and co.kind is OpKind.CONV2D and csrc == gdst and clast and eps_tail
                    and "w_taps" in self.dw.p.get(co.id, {}) and not cact and tail not in self.epilogue_of
                    and gsh.c % 64 == 0 and gsh.c <= 384 and 9 * cosh.c <= 48 and gsh.h * gsh.w >= 16
                    and os.environ.get("SF_GN_PROJECT") != "0"):
                gn_project[co.id] = (go, gsrc, gact)
                pf_specs.pop(gdst, None)
        # exact per-frame slice scratch of this chain -> slice count under the budget
        per_frame = sum(r * c * torch.empty((), dtype=dt).element_size() for r, c, dt in pf_specs.values())
        from .parallel import shard_range
        f0, f1 = shard_range(frames, self.cfg.world, self.cfg.rank)
        if self.cfg.slicing == "plan" and grp.plan.extents:
            # the group's own plan (ceil chunks, remainder last), cut to this rank's frames
            slices, a = [], 0
            for e in grp.plan.extents:
                lo, hi = max(a, f0), min(a + e, f1)
                if lo < hi:
                    slices.append((lo, hi))
                a += e
        else:
            k = self._k_for(per_frame, f1 - f0, self.cfg.spatial_k)
            slices = [(a + f0, b + f0) for a, b in balanced(f1 - f0, k)]
        self.slice_counts[grp.label] = len(slices)
        fmax = max([b - a for a, b in slices] + [1])
        specs = {k: (fmax * r, c, dt) for k, (r, c, dt) in pf_specs.items()}
        # the split count of the statistics pass grows as a slice's frame count shrinks: size the
        # workspace for every slice extent, not only the largest (a 3-frame slice of a plan sized
        # for 4 frames needs 297 split rows against 296)
        gn_need = max([N.query("sf_group_norm_workspace", n, g.h * g.w, g.c)
                       for g in gn_shapes for n in {b - a for a, b in slices}] or [0])
        if gn_need:
            specs["gn_work"] = ((gn_need + 3) // 4, 1, torch.float32)
            specs["gn_stats"] = (2 * fmax * max_groups, 1, torch.float32)
        ncopy = max(1, min(self.cfg.slice_streams, len(slices)))
        if ncopy > 1 and os.environ.get("SF_STREAM_PAIRS") != "1":
            # concurrent slices: single-CTA GEMM tiles pack the SMs better than CTA pairs
            # (north-star plan, same box: 48.6 / 61.0 / 63.3 steps/s at 2 / 4 / 6 streams vs
            # 45.9 / 58.1 / 60.6 with pairs; SF_STREAM_PAIRS=1 is the A/B knob)
            backend |= N.GEMM_NO_PAIR
        scratches = self._scratch(specs, ncopy) if ncopy > 1 else [self._scratch(specs)]
        eps_out = self.fp32_out and tail == self.graph.outputs[0]
        # GroupNorm statistics handed over through conv-epilogue partials (_analyse_gn_feed)
        gn_out = self.gn_partials(self.gn_feed[tail]) if tail in self.gn_feed else None
        gn_in = self.gn_partials(x_id) if x_id in self.gn_meta else None
        # resampling ops that hand partials over: role -> (buffer, splits, row length, channel offset)
        gn_rs = {o.id: {role: (*self.gn_partials(v), self.shapes[v].c, c0) for role, v, c0 in self.gn_roles[o.id]}
                 for o in ops if o.id in self.gn_roles}
        fr0 = self._frames()[0] if gn_out or gn_in or gn_rs else 0

        def part_ptr(entry, f):
            t, splits, ld, _ = entry
            return t.data_ptr() + (f - fr0) * splits * ld * 8

        def run(st0):
            streams = self._fork(st0, ncopy)
            for si, sl in enumerate(slices):
                one_slice(sl, scratches[si % ncopy], streams[si % ncopy])
            self._join(st0, streams)

        def one_slice(sl, scratch, st):
            if True:
                nf = sl[1] - sl[0]
                gn_stats_of = {}

                def loc(name, shp):
                    if name == "IN":
                        return vrows(x_id, sl)
                    if name == "OUT":
                        return vrows(tail, sl)
                    if name not in scratch:
                        return None    # the GroupNorm output a fused projection never materialises
                    return Rows(scratch[name], 0, shp.h * shp.w)
                for (o, src, dst, ish, osh, act, last) in steps:
                    prm = self.dw.p.get(o.id)
                    X = None if (latent_in and src == "IN") else loc(src, ish)
                    Y = loc(dst, osh)
                    epi = epi_fn(sl) if last else Epilogue()
                    if act:
                        epi.act = act
                    k = o.kind
                    ihw, ohw = ish.h * ish.w, osh.h * osh.w
                    if k is OpKind.GROUP_NORM:
                        groups = int(o.attrs.get("groups", 1))
                        stats = scratch["gn_stats"]
                        mean = stats[:nf * groups, 0]
                        rstd = stats[fmax * max_groups: fmax * max_groups + nf * groups, 0]
                        gn_stats_of[o.id] = (mean, rstd)
                        eps = float(o.attrs.get("eps", 1e-5))
                        if src == "IN" and gn_in is not None:
                            N.call("sf_group_norm_finalize", gn_in[0].data_ptr() + (sl[0] - fr0) * gn_in[1] * ish.c * 8,
                                   nf, gn_in[1], ihw, ish.c, groups, eps, mean.data_ptr(), rstd.data_ptr(), st)
                        else:
                            D.group_norm_stats(st, X, nf, ihw, ish.c, groups, eps, scratch["gn_work"], mean, rstd)
                        if not any(g[0] is o for g in gn_project.values()):
                            D.group_norm_apply(st, X, Y, nf, ihw, ish.c, groups, mean, rstd, prm, act)
                    elif k is OpKind.LAYER_NORM:
                        D.layer_norm(st, X, Y, nf, ihw, ish.c, prm, float(o.attrs.get("eps", 1e-5)), act)
                    elif k is OpKind.SILU:
                        N.call("sf_silu", X.view(), Y.view(), nf, ihw, ish.c, st)
                    elif k is OpKind.CONV2D and o.id in gn_project:
                        go, gsrc, gact = gn_project[o.id]
                        gp, gx = self.dw.p[go.id], loc(gsrc, ish)
                        mean, rstd = gn_stats_of[go.id]
                        ybuf = scratch["taps_y"]
                        N.call("sf_group_norm_project", gx.view(), nf, ihw, ish.c, int(go.attrs.get("groups", 1)),
                               mean.data_ptr(), rstd.data_ptr(), gp["gamma"].data_ptr(), gp["beta"].data_ptr(), gact,
                               prm["w_taps"].data_ptr(), 9 * osh.c, ybuf.data_ptr(), ybuf.stride(0), st)
                        N.call("sf_conv3x3_tapsum", ybuf.data_ptr(), ybuf.stride(0), nf, osh.h, osh.w, osh.c,
                               prm["bias"].data_ptr(), self.srows(tail, sl[0]).view(), st)
                    elif k is OpKind.CONV2D:
                        if latent_in and src == "IN":
                            lat = self.latent[sl[0] * ihw:]
                            if o.id in gn_rs:
                                e = gn_rs[o.id]["smallcin"]
                                N.call("sf_conv3x3_smallcin_gn", lat.data_ptr(), nf, ish.h, ish.w, ish.c,
                                       prm["wt32"].data_ptr(), prm["bias"].data_ptr(), osh.c, Y.view(), e[1],
                                       part_ptr(e, sl[0]), st)
                            else:
                                N.call("sf_conv3x3_smallcin", lat.data_ptr(), nf, ish.h, ish.w, ish.c,
                                       prm["wt32"].data_ptr(), prm["bias"].data_ptr(), osh.c, Y.view(), st)
                        elif last and eps_out:
                            # out_conv: fp32 network output (per-tap projection + shifted sum for tiny cout)
                            out = self.srows(tail, sl[0])
                            if "w_taps" in prm and epi.res is None and epi.rowbias is None and not act:
                                D.conv2d_tapwise(st, X, out, nf, ish.h, ish.w, ish.c, osh.c, prm, scratch["taps_y"],
                                                 backend)
                            else:
                                D.conv2d(st, X, out, nf, ish.h, ish.w, ish.c, osh.c, prm, epi, backend,
                                         out_fp32=True)
                        else:
                            gp = None
                            if last and gn_out is not None:
                                gp = gn_out[0].data_ptr() + (sl[0] - fr0) * gn_out[1] * osh.c * 8
                            D.conv2d(st, X, Y, nf, ish.h, ish.w, ish.c, osh.c, prm, epi, backend, gn_partial=gp)
                    elif k is OpKind.LINEAR:
                        D.linear(st, X, Y, nf, ihw, ish.c, osh.c, prm, epi, backend)
                    elif k is OpKind.SPATIAL_ATTENTION:
                        D.spatial_attention(st, X, Y, nf, ihw, ish.c, prm, epi, scratch, backend)
                    elif k is OpKind.DOWNSAMPLE2X and o.id in gn_rs:
                        r = gn_rs[o.id]
                        eo, ei = r.get("out"), r.get("in")
                        sp = (eo or ei)[1]
                        if ei is not None and ei[1] != sp:
                            raise InvalidParam(f"{o.id}: output / skip partials need one split count")
                        N.call("sf_downsample2x_gn", X.view(), Y.view(), nf, ish.h, ish.w, ish.c, sp,
                               part_ptr(eo, sl[0]) if eo else None, eo[2] if eo else 0,
                               part_ptr(ei, sl[0]) if ei else None, ei[2] if ei else 0, st)
                    elif k is OpKind.DOWNSAMPLE2X:
                        N.call("sf_downsample2x", X.view(), Y.view(), nf, ish.h, ish.w, ish.c, st)
                    elif k is OpKind.UPSAMPLE2X and o.id in gn_rs:
                        eo = gn_rs[o.id]["out"]
                        N.call("sf_upsample2x_gn", X.view(), Y.view(), nf, ish.h, ish.w, ish.c, eo[1],
                               part_ptr(eo, sl[0]), eo[2], eo[3], st)
                    elif k is OpKind.UPSAMPLE2X:
                        N.call("sf_upsample2x", X.view(), Y.view(), nf, ish.h, ish.w, ish.c, st)
                    else:
                        raise InvalidParam(f"no spatial lowering for {k.value}")
        return Unit(grp.label, run, gemm_flops=flops)

    # temporal groups: slices are pixel bands across all frames
    def _compile_temporal(self, grp, ops, kinds, s):
        B, T, HW, C = s.b, s.t, s.h * s.w, s.c
        backend = self.cfg.gemm_backend
        tail = ops[-1].id
        x_id = grp.head_input

        def vrows(vid, band):
            return self.trows(vid, band[0])

        epi_fn = self._epilogue(tail, vrows)
        steps, pp_specs = [], {}        # name -> (rows per pixel, cols, dtype)
        i = nb = 0
        flops = 0.0
        fold_ln = {}                    # temporal attention id -> the LayerNorm folded into its QKV GEMM
        while i < len(ops):
            o = ops[i]
            nxt = ops[i + 1] if i + 1 < len(ops) else None
            if (self.cfg.ln_fold and o.kind is OpKind.LAYER_NORM and nxt is not None
                    and nxt.kind is OpKind.TEMPORAL_ATTENTION):
                fold_ln[nxt.id] = o
                pt = self.dw.p[nxt.id]
                if "fold" not in pt:
                    pl = self.dw.p[o.id]
                    D.unfused_weights(pt, self.dev)
                    pt["fold"] = D.ln_fold_weights(pt["wqkv"], pl["gamma"], pl["beta"])
                pp_specs["lnstats"] = (B * T, 2, torch.float32)
                i += 1
                continue
            fuse_act = nxt is not None and nxt.kind is OpKind.SILU
            last = (i + (2 if fuse_act else 1)) >= len(ops)
            oc = self.shapes[ops[i + (1 if fuse_act else 0)].id].c
            dst = "OUT" if last else f"t{nb}"
            if not last:
                pp_specs[dst] = (B * T, oc, torch.bfloat16)
                nb += 1
            steps.append((o, None, dst, N.ACT_SILU if fuse_act else N.ACT_NONE, last, oc))
            if o.kind is OpKind.TEMPORAL_CONV:
                flops += 2.0 * B * T * HW * C * oc * 3
            elif o.kind is OpKind.LINEAR:
                flops += 2.0 * B * T * HW * C * oc
            elif o.kind is OpKind.TEMPORAL_ATTENTION:
                flops += B * HW * (8.0 * T * C * C + 4.0 * T * T * C)
                emb_epi = last and self.epilogue_of.get(tail, (None, None, False))[2]
                if fuse_act or emb_epi or not D.fused_temporal_ok(self.dw.p[o.id], T, self.shapes[o.id].c,
                                                                  backend=backend, fold=fold_ln.get(o.id)):
                    # three launches (QKV GEMM, core, output GEMM) through slice scratch
                    D.unfused_weights(self.dw.p[o.id], self.dev)
                    pp_specs["qkv"] = (B * T, 3 * C, torch.bfloat16)
                    pp_specs["o"] = (B * T, C, torch.bfloat16)
            i += 2 if fuse_act else 1
        # exact per-pixel slice scratch -> band count under the budget
        per_pix = sum(r * c * torch.empty((), dtype=dt).element_size() for r, c, dt in pp_specs.values())
        from .parallel import shard_range
        p0, p1 = shard_range(HW, self.cfg.world, self.cfg.rank)
        if self.cfg.slicing == "plan" and grp.plan.row_extents:
            k = max(1, min(grp.plan.n_slices, p1 - p0))
        else:
            k = self._k_for(per_pix, p1 - p0, self.cfg.temporal_k)
        bands = [(a + p0, b + p0) for a, b in balanced(p1 - p0, k)]
        self.slice_counts[grp.label] = len(bands)
        pmax = max([b - a for a, b in bands] + [1])
        specs = {k: (pmax * r, c, dt) for k, (r, c, dt) in pp_specs.items()}
        # fix up sources: each step reads the previous step's destination
        fixed, prev = [], "IN"
        for (o, _src, dst, act, last, oc) in steps:
            fixed.append((o, prev, dst, act, last, oc))
            prev = dst
        steps = fixed
        ncopy = max(1, min(self.cfg.slice_streams, len(bands)))
        if ncopy > 1 and os.environ.get("SF_STREAM_PAIRS") != "1":
            backend |= N.GEMM_NO_PAIR       # see _compile_spatial
        scratches = self._scratch(specs, ncopy) if ncopy > 1 else [self._scratch(specs)]

        def run(st0):
            streams = self._fork(st0, ncopy)
            for bi_, band in enumerate(bands):
                one_band(band, scratches[bi_ % ncopy], streams[bi_ % ncopy])
            self._join(st0, streams)

        def one_band(band, scratch, st):
            if True:
                npx = band[1] - band[0]

                def loc(name):
                    if name == "IN":
                        return vrows(x_id, band)
                    if name == "OUT":
                        return vrows(tail, band)
                    return Rows(scratch[name], 0, npx)
                cin = C
                for (o, src, dst, act, last, oc) in steps:
                    prm = self.dw.p.get(o.id)
                    X, Y = loc(src), loc(dst)
                    epi = epi_fn(band) if last else Epilogue()
                    if act:
                        epi.act = act
                    k = o.kind
                    if k is OpKind.LAYER_NORM:
                        D.layer_norm(st, X, Y, B * T, npx, cin, prm, float(o.attrs.get("eps", 1e-5)), act)
                    elif k is OpKind.SILU:
                        N.call("sf_silu", X.view(), Y.view(), B * T, npx, cin, st)
                    elif k is OpKind.TEMPORAL_CONV:
                        D.temporal_conv(st, X, Y, B * T, T, npx, cin, oc, prm, epi, backend)
                    elif k is OpKind.LINEAR:
                        D.linear(st, X, Y, B * T, npx, cin, oc, prm, epi, backend)
                    elif k is OpKind.TEMPORAL_ATTENTION:
                        ln = fold_ln.get(o.id)
                        fold = None if ln is None else (prm["fold"], float(ln.attrs.get("eps", 1e-5)))
                        D.temporal_attention(st, X, Y, B, T, npx, cin, prm, epi, scratch, backend, fold)
                    else:
                        raise InvalidParam(f"no temporal lowering for {k.value}")
                    cin = oc
        return Unit(grp.label, run, gemm_flops=flops)

    # ------------------------------------------------------------------ run
    def units_after(self, node_id):
        """Units strictly after ``node_id`` in topo order (the rehash tail)."""
        cut = self.pos[node_id]
        out = []
        for u in self.units:
            k, r = u.ref
            first = r if k == "node" else self.grouped.groups[r].ops[0].id
            if self.pos[first] > cut:
                out.append(u)
        return out

    def emb_launch(self, st, emb_vec_ptr):
        if self.emb_w is not None:
            N.call("sf_gemv_f32", self.emb_w.data_ptr(), emb_vec_ptr, self.emb_b.data_ptr(),
                   self.emb_out.data_ptr(), self.emb_w.shape[0], self.emb_w.shape[1], st)

    def run_full(self, st, emb_vec_ptr):
        self.emb_launch(st, emb_vec_ptr)
        for u in self.units:
            u.run(st)

    def run_tail(self, st):
        for u in self.tail_units:
            u.run(st)

    @property
    def tail_units(self):
        if not hasattr(self, "_tail"):
            self._tail = self.units_after(self.graph.node_by_label(PROBE_LABEL).id)
        return self._tail

    @property
    def probe(self) -> torch.Tensor:
        return self.values[self.graph.node_by_label(PROBE_LABEL).id].tensor

    def probe_band_rows(self) -> tuple[Rows, int, int]:
        """(rows, n_outer, n_inner) of this rank's part of the probe: all frames x its pixel band
        (the probe is a temporal-group output; unsharded: every pixel)."""
        pid = self.graph.node_by_label(PROBE_LABEL).id
        sh = self.shapes[pid]
        p0, p1 = self._pixels(sh) if self.sharded else (0, sh.h * sh.w)
        return self.trows(pid, p0), sh.b * sh.t, p1 - p0

    def flops_full(self) -> float:
        return sum(u.gemm_flops for u in self.units)

    def flops_tail(self) -> float:
        return sum(u.gemm_flops for u in self.tail_units)


class _GroupPlan(Plan):
    """The launch program of one operator group over standalone input/output rows (execute_group)."""

    fp32_out = False

    def __init__(self, group, in_shape: Shape5, weights, cfg: ExecConfig):
        graph = Graph(list(group.ops), {group.head_input: in_shape}, [group.tail])
        self.graph, self.cfg = graph, cfg
        self.grouped = GroupedGraph(graph, (group,), (), (("group", 0),))
        self.dw = D.DeviceWeights(graph, weights, cfg.device)
        self.dev = self.dw.dev
        self.shapes = infer_shapes(graph)
        self.topo = graph.topo_order()
        self.pos = {n: i for i, n in enumerate(self.topo)}
        self.cons = graph.consumers()
        self.values, self.fused_adds, self.epilogue_of, self.units, self.emb_nodes = {}, {}, {}, [], []
        self.gn_feed, self.gn_part, self.gn_roles, self.gn_meta = {}, {}, {}, {}   # one group: no hand-over
        self.exchanger = None
        so = self.shapes[group.tail]
        self.inp = torch.empty(in_shape.rows, in_shape.c, dtype=torch.bfloat16, device=self.dev)
        self.out = torch.empty(so.rows, so.c, dtype=torch.bfloat16, device=self.dev)
        self.sharded = False
        for vid, t in ((group.head_input, self.inp), (group.tail, self.out)):
            self.values[vid] = Value(vid, self.shapes[vid], tensor=t, store={L: (t, 0) for L in ("F", "S", "T")})
        self.latent = torch.empty(in_shape.rows, in_shape.c, dtype=torch.float32, device=self.dev) \
            if group.head_input == "x" else None
        self.eps = None
        self._compile()


_GROUP_PLANS: dict = {}


def execute_group(group, x, weights, ledger=None, cfg: ExecConfig | None = None) -> Tensor5D:
    """One operator group on the device, slice by slice (grouping.py:223-254).

    Same contract as the reference's ``execute_group(group, x, weights, ledger)``:
    ``x`` is the group's full input (a Tensor5D of either package), the result a
    fresh Tensor5D of the group's output in ``x``'s dtype.  The group's own
    ``SlicePlan`` sets the slices (``ExecConfig(slicing="plan")``; a caller's
    ``cfg`` may choose the budget planner instead).  The ledger sees the output
    buffer (kept, like the reference) and the slice scratch of the group
    (released when the group completes) -- the device analog of the
    reference's output + per-stage slots.  The compiled launch program is
    cached per (group, input shape, weights).
    """
    from . import ops
    from .interop import as_array, as_group
    grp = as_group(group)
    xa = as_array(x)
    shape = Shape5(*xa.shape)
    out_dtype = xa.dtype if xa.dtype in (np.float32, np.float64) else np.float32
    if len(grp.ops) == 1 and grp.head_input == "step_emb":
        # the step-embedding projection (a (b,t,c,1,1) input): one per-op launch
        op = grp.ops[0]
        y = ops.apply_kernel(op.kind, [Tensor5D(xa)], weights.get(op.param_ref), op.attrs)
        if ledger is not None:
            ledger.alloc(y.data.astype(out_dtype).nbytes, op.label)
        return Tensor5D(y.data.astype(out_dtype))
    cfg = cfg or ExecConfig(slicing="plan")
    key = (grp.label, grp.nodes, tuple(shape), id(weights), cfg.slicing, cfg.scratch_budget, cfg.spatial_k,
           cfg.temporal_k, cfg.gemm_backend)
    hit = _GROUP_PLANS.get(key)
    if hit is None or hit[0] is not weights:
        ops._dev()
        if len(_GROUP_PLANS) > 64:
            _GROUP_PLANS.clear()
        hit = (weights, _GroupPlan(grp, shape, weights, cfg))
        _GROUP_PLANS[key] = hit
    plan = hit[1]
    st = torch.cuda.current_stream().cuda_stream
    if plan.latent is not None:
        plan.latent.copy_(ops.to_rows(Tensor5D(xa), torch.float32))
    else:
        plan.inp.copy_(ops.to_rows(Tensor5D(xa)))
    out_shape = plan.shapes[grp.tail]
    if ledger is not None:
        ledger.alloc(out_shape.count() * np.dtype(out_dtype).itemsize, grp.ops[-1].label)
        ledger.alloc(plan.scratch_bytes, f"{grp.label}:slice_scratch")
    for u in plan.units:
        u.run(st)
    y = ops.from_rows(plan.out, out_shape)
    if ledger is not None:
        ledger.free(plan.scratch_bytes, f"{grp.label}:slice_scratch")
    return Tensor5D(y.data.astype(out_dtype))


def plan_memory(graph: Graph, grouped: GroupedGraph, cfg: ExecConfig | None = None) -> dict:
    """Arena / scratch bytes the device plan would reserve, computed without a GPU.

    Builds the plan's layout on the ``meta`` device (shapes only), so the device
    analog of the reference's static peak model (grouping.py:334-450) can be
    checked and reported anywhere.
    """
    cfg = cfg or ExecConfig()
    dw = D.DeviceWeights.__new__(D.DeviceWeights)
    dw.dev = torch.device("meta")
    dw.p = {}
    for n in graph.nodes.values():
        if n.kind is OpKind.CONV2D and graph.nodes[n.id].inputs[0] != "x":
            dw.p[n.id] = {"w": None}
        elif n.kind is OpKind.CONV2D:
            dw.p[n.id] = {"wt32": None}    # in_conv: the small-channel kernel
        elif n.kind is OpKind.LINEAR:
            dw.p[n.id] = {"w32": torch.empty(1, 1, device="meta"), "bias": torch.empty(1, device="meta")}
        elif n.param_ref:
            dw.p[n.id] = {}
    plan = Plan.__new__(Plan)
    plan.graph, plan.grouped, plan.dw = graph, grouped, dw
    plan.cfg = ExecConfig(spatial_k=cfg.spatial_k, temporal_k=cfg.temporal_k, scratch_budget=cfg.scratch_budget,
                          gn_from_conv=cfg.gn_from_conv,
                          device="meta", rank=cfg.rank, world=cfg.world)
    plan.dev = dw.dev
    plan.shapes = infer_shapes(graph)
    plan.topo = graph.topo_order()
    plan.pos = {n: i for i, n in enumerate(plan.topo)}
    plan.cons = graph.consumers()
    plan.values, plan.fused_adds, plan.epilogue_of, plan.units, plan.emb_nodes = {}, {}, {}, [], []
    plan.gn_feed, plan.gn_part, plan.gn_roles, plan.gn_meta = {}, {}, {}, {}
    plan.exchanger = None
    plan._analyse()
    plan._layout()
    led = plan.memory_ledger()
    out = {"arena_bytes": plan.arena_bytes, "buffers": len(plan.buffers), "ledger": led,
           "ledger_peak_bytes": led.peak_bytes,
           "gn_partial_bytes": 4 * sum(getattr(plan, "_gn_slot_elems", [])), "gn_from_conv": len(plan.gn_feed),
           "gn_handed_over": len(plan.gn_meta),
           "gn_slots": {v: (getattr(plan, "_gn_slot_of", {}).get(v), *plan.gn_intervals[v])
                        for v in getattr(plan, "gn_intervals", {})}}
    if plan.cfg.world > 1:
        from .parallel import exchange_schedule
        ex = exchange_schedule(plan)
        out["exchanges_per_eval"] = len(ex)
        out["hoisted_exchanges"] = sum(1 for op in ex if op.at < op.need)
        # bytes this rank sends per evaluation: of each exchanged value it holds 1/world (its frames or
        # its pixel band) and keeps the 1/world of that block which stays local
        w = plan.cfg.world
        sent = 0.0
        for op in ex:
            s = plan.shapes[op.value]
            sent += s.b * s.t * s.h * s.w * s.c * 2 / w * (w - 1) / w
        out["exchange_bytes_per_rank"] = int(sent)
    return out


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


class DeviceModel:
    """Graph + device weights + compiled plan; the object behind execute/rehash/run_denoise."""

    def __init__(self, graph: Graph, weights, cfg: ExecConfig | None = None, grouped: GroupedGraph | None = None,
                 unet_cfg: UNetConfig | None = None, device_weights: D.DeviceWeights | None = None):
        N.load()
        if not torch.cuda.is_available():
            from .errors import NativeError
            raise NativeError("no CUDA device: the sliceflow_b200 path has no CPU fallback")
        from .interop import as_graph, as_grouped
        self.cfg = cfg or ExecConfig()
        graph = as_graph(graph)
        self.graph = graph
        self.unet_cfg = unet_cfg
        if grouped is not None:
            grouped = as_grouped(grouped)
        if grouped is None:
            xs = graph.inputs["x"]
            grouped = group_operators(graph, xs.b * xs.t, default_temporal_config(xs.h, xs.w))
        self.grouped = grouped
        self.dw = device_weights or D.DeviceWeights(graph, weights, self.cfg.device)
        self.plan = Plan(graph, grouped, self.dw, self.cfg)
        xs = graph.inputs["x"]
        self.x_shape = xs
        self.host_in = torch.empty(xs.count(), dtype=torch.float32).pin_memory()
        self.host_out = torch.empty(xs.count(), dtype=torch.float32).pin_memory()
        self.dev_bcthw = torch.empty(xs.count(), dtype=torch.float32, device=self.dw.dev)

    # latent edges
    def upload_latent(self, st, x_host: np.ndarray):
        xs = self.x_shape
        self.host_in.numpy()[:] = np.ascontiguousarray(x_host, dtype=np.float32).ravel()
        self.dev_bcthw.copy_(self.host_in, non_blocking=True)
        N.call("sf_bcthw_to_rows_f32", self.dev_bcthw.data_ptr(), self.plan.latent.data_ptr(), xs.b * xs.t, xs.c,
               xs.h * xs.w, st)

    def latent_to_bcthw(self, st, src_rows: torch.Tensor):
        xs = self.x_shape
        N.call("sf_rows_to_bcthw_f32", src_rows.data_ptr(), self.dev_bcthw.data_ptr(), xs.b * xs.t, xs.c, xs.h * xs.w,
               st)
        return self.dev_bcthw

    def download(self, dev_tensor) -> np.ndarray:
        self.host_out.copy_(dev_tensor.view(-1), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.host_out.numpy().reshape(tuple(self.x_shape)).copy()


def pipeline_schedule(n_stages: int, n_slices: int) -> list[list[tuple[int, int]]]:
    """Wavefront table of SPEC.md:337-343 (paper Fig. 5c): at tick t, stage j runs slice t - j.

    Returns one list of (stage, slice) pairs per tick; m + n - 1 ticks.  On the
    device a group's stages are fused into one kernel chain per slice, so every
    slice passes all stages back to back on one stream -- the same dependency
    order, with zero extra buffers (the "Pipelined peak == SlicedLoop peak"
    property holds by construction).
    """
    if n_stages < 1 or n_slices < 1:
        raise InvalidParam(f"pipeline needs >= 1 stage and slice, got {n_stages}, {n_slices}")
    return [[(j, t - j) for j in range(n_stages) if 0 <= t - j < n_slices]
            for t in range(n_stages + n_slices - 1)]


def _with_frames(graph: Graph, t: int) -> Graph:
    """The same network over a clip of t frames (weights do not depend on T)."""
    return Graph(graph.nodes.values(), {k: s.replace(t=t) for k, s in graph.inputs.items()}, graph.outputs)


def naive_clip_chunks(T: int, chunk: int) -> list[tuple[int, int]]:
    """Frame ranges of NaiveClip(chunk) (1 <= chunk < T)."""
    if not 1 <= chunk < T:
        raise InvalidParam(f"naive chunk must be in [1, {T}), got {chunk}")
    return [(o, min(o + chunk, T)) for o in range(0, T, chunk)]


def execute(graph_or_grouped, mode, inputs, weights, cfg: ExecConfig | None = None, naive_chunk: int | None = None):
    """One network evaluation on the device.

    Returns ``(output Tensor5D, ledger, timing)`` like the reference contract.
    ``ledger`` is a :class:`MemoryLedger` derived from the compiled plan (arena
    buffers charged over their live units, slice scratch over the evaluation);
    its ``summary`` holds the device facts (arena, scratch, torch peak).
    ``timing`` is wall-clock ms per phase.  REFERENCE runs the same fused
    kernels with one slice per group (unsliced); SLICED_LOOP / PIPELINED use
    the slice plan of ``cfg`` (on one stream the pipelined wavefront and the
    for-loop issue the same launches, so they are the same program here).
    NAIVE_CLIP(``naive_chunk``) runs independent evaluations over clips of
    frames and stitches them along t -- the divergent
    baseline the slicer avoids.
    """
    from .interop import as_array, as_graph_or_grouped, as_mode
    mode = as_mode(mode)
    graph, grouped = as_graph_or_grouped(graph_or_grouped)
    if cfg is None:
        # a caller-built GroupedGraph carries its slice plans: honour them (grouping.py:223-254)
        cfg = ExecConfig(slicing="plan") if grouped is not None else ExecConfig()
    if mode is ExecMode.REFERENCE or mode is ExecMode.NAIVE_CLIP:
        cfg = ExecConfig(spatial_k=1, temporal_k=1, scratch_budget=cfg.scratch_budget,
                         gemm_backend=cfg.gemm_backend, device=cfg.device)
    x = as_array(inputs["x"])
    se = as_array(inputs["step_emb"])
    vec = np.ascontiguousarray(se.reshape(-1, se.shape[2])[0], dtype=np.float32)
    if not np.all(se.reshape(-1, se.shape[2]) == vec[None]):
        raise ShapeMismatch("device path expects the step embedding broadcast over (b, t) (unet.py:106-113)")
    if mode is ExecMode.NAIVE_CLIP:
        if naive_chunk is None:
            raise InvalidParam("naiveclip needs naive_chunk")
        chunks = naive_clip_chunks(graph.inputs["x"].t, naive_chunk)
    else:
        chunks = [(0, graph.inputs["x"].t)]
    torch.cuda.reset_peak_memory_stats()
    t0 = time.perf_counter()
    outs, models, compile_ms = [], {}, 0.0
    for f0, f1 in chunks:
        n = f1 - f0
        if n not in models:
            tc = time.perf_counter()
            if mode is ExecMode.NAIVE_CLIP:
                models[n] = DeviceModel(_with_frames(graph, n), weights, cfg)
            else:
                models[n] = DeviceModel(graph, weights, cfg, grouped)
            compile_ms += (time.perf_counter() - tc) * 1e3
        model = models[n]
        st = stream_handle()
        model.upload_latent(st, np.ascontiguousarray(x[:, f0:f1]))
        emb = torch.from_numpy(vec).to(model.dw.dev)
        model.plan.run_full(st, emb.data_ptr())
        outs.append(model.download(model.latent_to_bcthw(st, model.plan.eps)))
    out = outs[0] if len(outs) == 1 else np.concatenate(outs, axis=1)
    t2 = time.perf_counter()
    model = models[chunks[0][1] - chunks[0][0]]
    summary = {"mode": mode.value, "arena_bytes": model.plan.arena_bytes,
               "scratch_bytes": model.plan.scratch_bytes, "torch_peak_bytes": torch.cuda.max_memory_allocated()}
    ledger = model.plan.memory_ledger(model.plan.scratch_bytes, summary)
    timing = {"compile_ms": compile_ms, "run_ms": (t2 - t0) * 1e3 - compile_ms}
    return Tensor5D(out), ledger, timing
