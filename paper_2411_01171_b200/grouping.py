"""Operator Grouping pass (paper §4.2) and the static peak-memory model.

Reference: ``sliceflow/grouping.py``.  ``group_operators`` reproduces the
greedy maximal-chain pass exactly (``grouping.py:130-200``) -- same groups,
same plans, same schedule -- because the device executor launches one fused
kernel sequence per group of exactly this partition.  The liveness model
(``grouping.py:300-450``) is kept so the measured device peak can be reported
next to the reference's own estimate.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping

import numpy as np

from .errors import InvalidParam, ShapeInferenceFailure
from .graph import Graph, OpNode, infer_shapes
from .kinds import Domain, output_shape, scratch_bytes
from .modes import ExecMode
from .slicer import SliceMode, SlicePlan, plan_spatial, plan_temporal, validate_lossless
from .tensor import Shape5, resolve_dtype


@dataclass(frozen=True)
class OperatorGroup:
    ops: tuple[OpNode, ...]
    domain: Domain
    plan: SlicePlan
    label: str

    @property
    def nodes(self) -> tuple[str, ...]:
        return tuple(o.id for o in self.ops)

    @property
    def head_input(self) -> str:
        return self.ops[0].inputs[0]

    @property
    def tail(self) -> str:
        return self.ops[-1].id


@dataclass(frozen=True)
class GroupedGraph:
    graph: Graph
    groups: tuple[OperatorGroup, ...]
    ungrouped: tuple[str, ...]
    schedule: tuple[tuple[str, object], ...]

    def unit_outputs(self) -> dict[str, tuple[str, object]]:
        return {(self.groups[r].tail if k == "group" else r): (k, r) for k, r in self.schedule}


def make_plan(domain: Domain, in_shape: Shape5, spatial_k: int, temporal_cfg: tuple[int, int]) -> SlicePlan:
    """Clamp k to the extents and plan (grouping.py:121-127)."""
    if domain is Domain.SPATIAL:
        bt = in_shape.b * in_shape.t
        return plan_spatial(bt, min(spatial_k, bt))
    kh, kw = temporal_cfg
    return plan_temporal(in_shape.h, in_shape.w, min(kh, in_shape.h), min(kw, in_shape.w))


def group_operators(graph: Graph, spatial_k: int, temporal_cfg: tuple[int, int]) -> GroupedGraph:
    """Greedy maximal chains of same-domain, losslessly sliceable ops (grouping.py:130-200)."""
    from .interop import as_graph
    graph = as_graph(graph)
    if spatial_k < 1:
        raise InvalidParam(f"spatial_k must be >= 1, got {spatial_k}")
    if min(temporal_cfg) < 1:
        raise InvalidParam(f"temporal slice counts must be >= 1, got {temporal_cfg}")
    shapes = infer_shapes(graph)
    cons = graph.consumers()
    topo = graph.topo_order()
    pos = {nid: i for i, nid in enumerate(topo)}
    taken: set[str] = set()
    groups: list[OperatorGroup] = []
    loose: list[str] = []
    units: list[tuple[int, tuple[str, object]]] = []

    def leave_ungrouped(nid):
        taken.add(nid)
        loose.append(nid)
        units.append((pos[nid], ("node", nid)))

    for nid in topo:
        if nid in taken:
            continue
        head = graph.nodes[nid]
        if head.domain is Domain.BOUNDARY or len(head.inputs) != 1:
            leave_ungrouped(nid)
            continue
        plan = make_plan(head.domain, shapes[head.inputs[0]], spatial_k, temporal_cfg)
        chain = [nid]
        if not validate_lossless(graph, chain, plan):
            leave_ungrouped(nid)
            continue
        while True:
            nxt_ids = cons.get(chain[-1], [])
            if len(nxt_ids) != 1:
                break
            nxt = graph.nodes[nxt_ids[0]]
            if (nxt.id in taken or len(nxt.inputs) != 1 or nxt.domain is not head.domain
                    or not validate_lossless(graph, chain + [nxt.id], plan)):
                break
            chain.append(nxt.id)
        taken.update(chain)
        ops = tuple(graph.nodes[c] for c in chain)
        label = (f"group[{ops[0].label}->{ops[-1].label}]" if len(ops) > 1 else f"group[{ops[0].label}]")
        groups.append(OperatorGroup(ops, head.domain, plan, label))
        units.append((pos[chain[0]], ("group", len(groups) - 1)))

    for g in groups:
        assert validate_lossless(graph, list(g.nodes), g.plan), g.label
    grouped = {n for g in groups for n in g.nodes}
    assert not grouped & set(loose) and grouped | set(loose) == set(graph.nodes)
    units.sort(key=lambda u: u[0])
    return GroupedGraph(graph, tuple(groups), tuple(loose), tuple(u for _, u in units))


# ---------------------------------------------------------------------------
# static peak-memory model (grouping.py:265-450)
# ---------------------------------------------------------------------------

def sliced_shape(full: Shape5, plan: SlicePlan, index: int = 0) -> Shape5:
    if plan.mode is SliceMode.SPATIAL_BT:
        return Shape5(1, plan.extents[index], full.c, full.h, full.w)
    ri, ci = divmod(index, len(plan.col_extents))
    return Shape5(full.b, full.t, full.c, plan.row_extents[ri], plan.col_extents[ci])


def group_output_shape(group: OperatorGroup, in_shape: Shape5) -> Shape5:
    s = in_shape
    for o in group.ops:
        s = output_shape(o.kind, [s], o.attrs)
    return s


def group_slot_sizes(group: OperatorGroup, in_shape: Shape5, itemsize: int) -> dict[str, int]:
    """One slice-sized slot per stage boundary + attention scratch (grouping.py:274-287)."""
    plan = group.plan
    full = in_shape
    sizes = {"slot0": sliced_shape(full, plan).nbytes(itemsize)}
    for j, o in enumerate(group.ops):
        sb = scratch_bytes(o.kind, sliced_shape(full, plan), itemsize)
        if sb:
            sizes[f"scratch{j}"] = sb
        full = output_shape(o.kind, [full], o.attrs)
        sizes[f"slot{j + 1}"] = sliced_shape(full, plan).nbytes(itemsize)
    return sizes


def group_working_set_bytes(group: OperatorGroup, in_shape: Shape5, itemsize: int) -> int:
    return sum(group_slot_sizes(group, in_shape, itemsize).values()) + \
        group_output_shape(group, in_shape).nbytes(itemsize)


class _Live:
    def __init__(self):
        self.cur = 0
        self.peak = 0
        self.live: dict[str, int] = {}

    def alloc(self, key, n):
        self.live[key] = n
        self.bump(n)

    def bump(self, n):
        self.cur += n
        self.peak = max(self.peak, self.cur)

    def free(self, key):
        self.cur -= self.live.pop(key)


def _reference_peak(graph: Graph, itemsize: int, input_shapes: Mapping[str, Shape5]) -> int:
    shapes = infer_shapes(graph, input_shapes)
    sim = _Live()
    refs: dict[str, int] = {}
    for n in graph.nodes.values():
        for r in dict.fromkeys(n.inputs):
            refs[r] = refs.get(r, 0) + 1
    for o in graph.outputs:
        refs[o] = refs.get(o, 0) + 1
    for name, s in input_shapes.items():
        sim.alloc(name, Shape5(*s).nbytes(itemsize))
    for nid in graph.topo_order():
        n = graph.nodes[nid]
        sb = scratch_bytes(n.kind, shapes[n.inputs[0]], itemsize)
        sim.bump(sb)
        sim.alloc(nid, shapes[nid].nbytes(itemsize))
        sim.cur -= sb
        for r in dict.fromkeys(n.inputs):
            refs[r] -= 1
            if refs[r] == 0 and r in sim.live:
                sim.free(r)
    return sim.peak


def _grouped_peak(gg: GroupedGraph, itemsize: int) -> int:
    graph = gg.graph
    shapes = infer_shapes(graph)
    sim = _Live()

    def consumed(unit):
        k, r = unit
        return list(dict.fromkeys(graph.nodes[r].inputs)) if k == "node" else [gg.groups[r].head_input]

    refs: dict[str, int] = {}
    for u in gg.schedule:
        for r in consumed(u):
            refs[r] = refs.get(r, 0) + 1
    for o in graph.outputs:
        refs[o] = refs.get(o, 0) + 1
    for name, s in graph.inputs.items():
        sim.alloc(name, s.nbytes(itemsize))
    for u in gg.schedule:
        k, r = u
        if k == "node":
            n = graph.nodes[r]
            sb = scratch_bytes(n.kind, shapes[n.inputs[0]], itemsize)
            sim.bump(sb)
            sim.alloc(r, shapes[r].nbytes(itemsize))
            sim.cur -= sb
        else:
            g = gg.groups[r]
            sim.alloc(g.tail, shapes[g.tail].nbytes(itemsize))
            slots = sum(group_slot_sizes(g, shapes[g.head_input], itemsize).values())
            sim.bump(slots)
            sim.cur -= slots
        for ref in consumed(u):
            refs[ref] -= 1
            if refs[ref] == 0 and ref in sim.live:
                sim.free(ref)
    return sim.peak


def estimate_peak_memory(g, mode, dtype="float32", naive_chunk: int | None = None) -> int:
    """Static liveness peak of one evaluation (grouping.py:334-364)."""
    from .interop import as_graph_or_grouped, as_mode
    mode = as_mode(mode)
    itemsize = np.dtype(resolve_dtype(dtype)).itemsize if dtype not in ("bfloat16", "bf16") else 2
    graph, grouped = as_graph_or_grouped(g)
    if mode in (ExecMode.SLICED_LOOP, ExecMode.PIPELINED):
        if grouped is None:
            raise ShapeInferenceFailure(f"{mode.value} requires a GroupedGraph")
        return _grouped_peak(grouped, itemsize)
    if mode is ExecMode.REFERENCE:
        return _reference_peak(graph, itemsize, graph.inputs)
    if mode is ExecMode.NAIVE_CLIP:
        if naive_chunk is None:
            raise InvalidParam("naive_chunk required for naiveclip estimates")
        t = graph.inputs["x"].t
        if not 1 <= naive_chunk < t:
            raise InvalidParam(f"naive chunk must be in [1, {t}), got {naive_chunk}")
        held = sum(s.nbytes(itemsize) for s in graph.inputs.values())
        held += infer_shapes(graph)[graph.outputs[0]].nbytes(itemsize)
        peak, off = held, 0
        while off < t:
            ct = min(naive_chunk, t - off)
            inner = _reference_peak(graph, itemsize, {k: s.replace(t=ct) for k, s in graph.inputs.items()})
            peak = max(peak, held + inner)
            off += ct
        return peak
    raise InvalidParam(f"unknown mode {mode}")


def grouped_graph_report(gg: GroupedGraph, dtype="float32") -> dict:
    """JSON summary per group (grouping.py:457-476)."""
    from .interop import as_grouped
    gg = as_grouped(gg)
    itemsize = np.dtype(resolve_dtype(dtype)).itemsize
    shapes = infer_shapes(gg.graph)
    rows = [{"label": g.label, "nodes": list(g.nodes), "node_count": len(g.nodes), "domain": g.domain.value,
             "plan": g.plan.to_json_dict(),
             "working_set_bytes": group_working_set_bytes(g, shapes[g.head_input], itemsize)}
            for g in gg.groups]
    return {"groups": rows, "ungrouped": list(gg.ungrouped), "group_count": len(rows),
            "ungrouped_count": len(gg.ungrouped)}
