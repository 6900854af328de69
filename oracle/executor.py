"""Oracle executor: Reference and SlicedLoop walks (test oracle only).

The reference specifies ``execute(graph_or_grouped, mode, inputs, weights)``
(``SPEC.md:333-341``) but ships no ``executor.py`` (``grouping.py:343`` imports
it).  This restates the two modes the parity tests need:

* REFERENCE: every node of ``graph.topo_order()`` through ``apply_kernel``
  (``kernels.py:323``), unsliced.
* SLICED_LOOP: walk ``GroupedGraph.schedule`` (``grouping.py:104-118``); a
  group runs slice by slice exactly like ``execute_group``
  (``grouping.py:223-254``): copy the slice, run the chain, write the slice
  result into the full output.

``start_after`` restricts the walk to units strictly after a node in topo
order -- the Step Rehash tail (``SPEC.md:425``, survey Appendix A).
"""

from __future__ import annotations

import time

import numpy as np

from paper_2411_01171_b200.grouping import GroupedGraph, group_output_shape
from paper_2411_01171_b200.modes import ExecMode
from paper_2411_01171_b200.slicer import SliceMode, plan_regions
from paper_2411_01171_b200.tensor import Shape5

from . import kernels as K


def _params(weights, node):
    return weights.get(node.param_ref) if node.param_ref else None


def run_chain(ops, x, weights):
    for op in ops:
        x = K.apply_kernel(op.kind, [x], _params(weights, op), op.attrs)
    return x


def run_group_sliced(group, x, weights, max_slices=None, slice_times=None):
    """Slice, run the chain per slice, reassemble (grouping.py:223-254).

    ``slice_times`` (a list) receives the wall time of every slice that ran."""
    shape = Shape5(*x.shape)
    out_shape = group_output_shape(group, shape)
    # zeros, not empty: a sampled run (max_slices) leaves the other slices unwritten
    out = np.zeros(tuple(out_shape), dtype=x.dtype)
    regions = plan_regions(shape, group.plan)
    if max_slices is not None:
        regions = regions[:max_slices]
    for reg in regions:
        t0 = time.perf_counter()
        if reg.mode is SliceMode.SPATIAL_BT:
            a, b = reg.bt
            part = x.reshape(shape.b * shape.t, *x.shape[2:])[a:b].copy()[None]
            res = run_chain(group.ops, part, weights)
            out.reshape(out_shape.b * out_shape.t, *out.shape[2:])[a:b] = res[0]
        else:
            (r0, r1), (c0, c1) = reg.rows, reg.cols
            part = np.ascontiguousarray(x[:, :, :, r0:r1, c0:c1])
            out[:, :, :, r0:r1, c0:c1] = run_chain(group.ops, part, weights)
        if slice_times is not None:
            slice_times.append(time.perf_counter() - t0)
    return out


def units_for(graph, grouped: GroupedGraph | None, mode: ExecMode):
    if mode is ExecMode.REFERENCE or grouped is None:
        return [("node", nid) for nid in graph.topo_order()]
    return list(grouped.schedule)


def evaluate(graph, weights, feeds, mode=ExecMode.REFERENCE, grouped=None, start_after=None,
             capture=(), max_slices=None, timing=None):
    """One network evaluation; returns (output, {label: captured array}).

    ``max_slices`` runs only the first slices of every group (a bounded CPU
    timing sample); ``timing`` (a list) receives (unit, sample_s, extrapolated_s).
    """
    mode = ExecMode(mode)
    topo = graph.topo_order()
    pos = {n: i for i, n in enumerate(topo)}
    vals = dict(feeds)
    units = units_for(graph, grouped, mode)
    if start_after is not None:
        cut = pos[start_after]
        units = [u for u in units
                 if pos[u[1] if u[0] == "node" else grouped.groups[u[1]].ops[0].id] > cut]
    captured = {}
    timings = [] if timing is not None else None
    for kind, ref in units:
        t0 = time.perf_counter()
        if kind == "node":
            n = graph.nodes[ref]
            vals[ref] = K.apply_kernel(n.kind, [vals[r] for r in n.inputs], _params(weights, n), n.attrs)
            done = [ref]
        else:
            g = grouped.groups[ref]
            st = []
            vals[g.tail] = run_group_sliced(g, vals[g.head_input], weights, max_slices, st)
            done = [g.tail]
        if timings is not None:
            dt = time.perf_counter() - t0
            est = dt
            if kind == "group" and max_slices is not None:
                # unsampled slices at the median of the sampled ones after the first (the first
                # slice of a group pays cold caches: extrapolating it alone overstated a full C3
                # evaluation by 55 %, profiles/r02_cpu_full_eval_c3.json)
                n = grouped.groups[ref].plan.n_slices
                warm = sorted(st[1:] or st)
                est = dt + (n - len(st)) * warm[len(warm) // 2]
            timings.append((ref if kind == "node" else grouped.groups[ref].label, dt, est))
        for d in done:
            lbl = graph.nodes[d].label
            if lbl in capture:
                captured[lbl] = vals[d]
    if timing is not None:
        timing.extend(timings)
    return vals[graph.outputs[0]], captured
