"""Accept the reference's own objects at the boundary (drop-in by value, not identity).

The reference (``/root/reference/pkg/src/sliceflow``) defines its own
``OpKind``/``Domain`` enums (``kernels.py:35-54``), ``OpNode``/``Graph``
(``graph.py:20-45``), ``SlicePlan`` (``slicer.py:58-80``), ``OperatorGroup``/
``GroupedGraph`` (``grouping.py:84-118``), ``Tensor5D`` (``tensor.py:64-113``)
and ``WeightBundle`` (``kernels.py:400-465``).  Those are different Python
classes from this package's, so an enum comparison by identity
(``n.kind is OpKind.LINEAR``) fails on a reference-built graph.  Every public
entry point of this package therefore normalises its arguments here first:
enums by ``.value``, containers by their attributes.  Objects that already
are this package's pass through untouched.
"""

from __future__ import annotations

import numpy as np

from .graph import Graph, OpNode
from .grouping import GroupedGraph, OperatorGroup
from .kinds import Domain, OpKind
from .modes import ExecMode
from .slicer import SliceMode, SlicePlan
from .tensor import Shape5, Tensor5D


def _enum(cls, v):
    return v if isinstance(v, cls) else cls(getattr(v, "value", v))


def as_node(n) -> OpNode:
    if isinstance(n, OpNode):
        return n
    return OpNode(id=n.id, kind=_enum(OpKind, n.kind), domain=_enum(Domain, n.domain), inputs=tuple(n.inputs),
                  param_ref=n.param_ref, label=getattr(n, "label", ""), attrs=dict(getattr(n, "attrs", {}) or {}))


def as_graph(g) -> Graph:
    """This package's Graph for ``g`` (identity if it already is one)."""
    if isinstance(g, Graph):
        return g
    return Graph([as_node(n) for n in g.nodes.values()], {k: Shape5(*v) for k, v in g.inputs.items()},
                 list(g.outputs))


def as_plan(p) -> SlicePlan:
    if isinstance(p, SlicePlan):
        return p
    return SlicePlan(mode=_enum(SliceMode, p.mode), k=getattr(p, "k", None), k_h=getattr(p, "k_h", None),
                     k_w=getattr(p, "k_w", None), extents=tuple(getattr(p, "extents", ()) or ()),
                     row_extents=tuple(getattr(p, "row_extents", ()) or ()),
                     col_extents=tuple(getattr(p, "col_extents", ()) or ()))


def as_group(grp, graph: Graph | None = None) -> OperatorGroup:
    if isinstance(grp, OperatorGroup):
        return grp
    ops = tuple(graph.nodes[o.id] if graph is not None else as_node(o) for o in grp.ops)
    return OperatorGroup(ops, _enum(Domain, grp.domain), as_plan(grp.plan), grp.label)


def as_grouped(gg) -> GroupedGraph:
    """This package's GroupedGraph for ``gg``: same groups, plans and schedule."""
    if isinstance(gg, GroupedGraph):
        return gg
    graph = as_graph(gg.graph)
    groups = tuple(as_group(grp, graph) for grp in gg.groups)
    return GroupedGraph(graph, groups, tuple(gg.ungrouped), tuple((str(k), r) for k, r in gg.schedule))


def is_grouped(obj) -> bool:
    return isinstance(obj, GroupedGraph) or (hasattr(obj, "groups") and hasattr(obj, "schedule")
                                             and hasattr(obj, "graph"))


def as_graph_or_grouped(obj):
    """(graph, grouped-or-None) for ``execute``'s first argument."""
    if is_grouped(obj):
        gg = as_grouped(obj)
        return gg.graph, gg
    return as_graph(obj), None


def as_array(x) -> np.ndarray:
    """Tensor5D (either package's) or array-like -> ndarray."""
    if isinstance(x, Tensor5D):
        return x.data
    if hasattr(x, "data") and hasattr(x, "shape") and not isinstance(x, np.ndarray):
        return np.asarray(x.data)
    return np.asarray(x)


def as_mode(m) -> ExecMode:
    return _enum(ExecMode, m)
