"""Generate golden fixtures by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified reference package ``sliceflow`` from
``/root/reference/pkg/src`` (it cannot travel to the GPU box, so its outputs are
frozen here as small ``.npz``/``.json`` fixtures).  The reference ships no
executor/rehash/harness modules; the ~30 lines of glue
below (walk the schedule, alpha_s update rule, Algorithm A1) drive only the
reference's own public functions: ``build_toy_unet``, ``group_operators``,
``execute_group``, ``apply_kernel``, ``step_embedding_tensor``,
``cosine_similarity``, ``estimate_peak_memory`` and ``WeightBundle.save``.
"""

from __future__ import annotations

import enum
import hashlib
import json
import os
import sys
import tempfile
import types

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

# grouping.estimate_peak_memory imports the missing sliceflow.executor for its
# ExecMode enum only (grouping.py:343); provide exactly that enum.
_stub = types.ModuleType("sliceflow.executor")


class ExecMode(str, enum.Enum):
    REFERENCE = "reference"
    SLICED_LOOP = "slicedloop"
    PIPELINED = "pipelined"
    NAIVE_CLIP = "naiveclip"


_stub.ExecMode = ExecMode
sys.modules["sliceflow.executor"] = _stub

from sliceflow import kernels as RK  # noqa: E402
from sliceflow.graph import infer_shapes, receptive_field  # noqa: E402
from sliceflow.grouping import (estimate_peak_memory, execute_group, group_operators,  # noqa: E402
                                grouped_graph_report)
from sliceflow.slicer import default_temporal_config, plan_spatial, plan_temporal  # noqa: E402
from sliceflow.tensor import Tensor5D  # noqa: E402
from sliceflow.unet import PROBE_LABEL, UNetConfig, build_toy_unet, step_embedding_tensor  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def walk(grouped, W, feeds, start_after=None, capture=()):
    g = grouped.graph
    topo = g.topo_order()
    pos = {n: i for i, n in enumerate(topo)}
    vals = {k: Tensor5D(v) if isinstance(v, np.ndarray) else v for k, v in feeds.items()}
    cap = {}
    for kind, ref in grouped.schedule:
        first = ref if kind == "node" else grouped.groups[ref].ops[0].id
        if start_after is not None and pos[first] <= pos[start_after]:
            continue
        if kind == "node":
            n = g.nodes[ref]
            vals[ref] = RK.apply_kernel(n.kind, [vals[r] for r in n.inputs],
                                        W.get(n.param_ref) if n.param_ref else None, n.attrs)
            out = ref
        else:
            grp = grouped.groups[ref]
            vals[grp.tail] = execute_group(grp, vals[grp.head_input], W)
            out = grp.tail
        if g.nodes[out].label in capture:
            cap[g.nodes[out].label] = vals[out].data.copy()
    return vals[g.outputs[0]].data, cap


def a1(S, gamma):
    K = len(S)
    i = j = 0
    G = [0]
    while i < K:
        if S[i][j] >= gamma:
            i += 1
        else:
            G.append(i)
            j = i
    G.append(K - 1)
    return sorted(set(G))


def denoise(cfg, dtype, K, spatial_k=None, G=None):
    graph, w64 = build_toy_unet(cfg)
    W = w64.astype(dtype)
    sk = spatial_k or cfg.effective_batch * cfg.frames
    grouped = group_operators(graph, sk, default_temporal_config(cfg.height, cfg.width))
    probe_id = graph.node_by_label(PROBE_LABEL).id
    x = np.random.default_rng(cfg.seed + 1).standard_normal(tuple(cfg.input_shape())).astype(dtype)
    keys = set(range(K)) if G is None else set(G)
    probes, eps_list, cache = [], [], None
    for s in range(K):
        if s in keys:
            feeds = {"x": x, "step_emb": step_embedding_tensor(cfg, s, dtype)}
            eps, cap = walk(grouped, W, feeds, capture=(PROBE_LABEL,))
            cache = cap[PROBE_LABEL]
            probes.append(cache)
        else:
            eps, _ = walk(grouped, W, {probe_id: cache}, start_after=probe_id)
        eps_list.append(eps)
        x = x - np.dtype(dtype).type(0.08 * (1.0 - s / K)) * eps
    return x, probes, eps_list


def structure(cfg, spatial_k):
    graph, w64 = build_toy_unet(cfg)
    grouped = group_operators(graph, spatial_k, default_temporal_config(cfg.height, cfg.width))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "w.slfw")
        w64.save(p)
        sha = hashlib.sha256(open(p, "rb").read()).hexdigest()
    shapes = infer_shapes(graph)
    return {
        "topo": graph.topo_order(),
        "graph_json": graph.to_json_dict(),
        "schedule": [[k, r] for k, r in grouped.schedule],
        "report": grouped_graph_report(grouped),
        "shapes": {k: list(v) for k, v in shapes.items()},
        "weights": {f"{k}/{n}": [float(a.sum()), float(np.abs(a).sum()), list(a.shape)]
                    for k, grp in w64.entries.items() for n, a in grp.items()},
        "slfw_sha256": sha,
        "peak": {m: estimate_peak_memory(grouped if m != "reference" else graph, m)
                 for m in ("reference", "slicedloop", "pipelined")},
        "peak_naive2": estimate_peak_memory(graph, "naiveclip", naive_chunk=2),
    }


def kernel_vectors():
    """Seeded per-kernel input/output vectors through the reference apply_kernel."""
    rng = np.random.default_rng(1234)
    out = {}
    cases = []
    for dt in ("float64", "float32"):
        x = rng.standard_normal((1, 3, 16, 6, 8))
        cases += [
            (dt, "conv2d", (1, 3, 16, 6, 8), {"out_channels": 24},
             {"weight": rng.standard_normal((24, 16, 3, 3)) * 0.1, "bias": rng.standard_normal(24)}),
            (dt, "temporal_conv", (1, 5, 16, 3, 4), {"out_channels": 16},
             {"weight": rng.standard_normal((16, 16, 3)) * 0.1, "bias": rng.standard_normal(16)}),
            (dt, "group_norm", (1, 3, 16, 6, 8), {"groups": 4, "eps": 1e-5},
             {"gamma": rng.standard_normal(16), "beta": rng.standard_normal(16)}),
            (dt, "layer_norm", (1, 3, 16, 6, 8), {"eps": 1e-5},
             {"gamma": rng.standard_normal(16), "beta": rng.standard_normal(16)}),
            (dt, "silu", (1, 3, 16, 6, 8), {}, None),
            (dt, "linear", (1, 3, 16, 6, 8), {"out_features": 40},
             {"weight": rng.standard_normal((40, 16)) * 0.2, "bias": rng.standard_normal(40)}),
            (dt, "spatial_attention", (1, 2, 32, 6, 8), {},
             {k: rng.standard_normal((32, 32)) * 0.2 for k in ("wq", "wk", "wv", "wo")}),
            (dt, "temporal_attention", (1, 7, 32, 3, 4), {},
             {k: rng.standard_normal((32, 32)) * 0.2 for k in ("wq", "wk", "wv", "wo")}),
            (dt, "downsample2x", (1, 3, 16, 6, 8), {}, None),
            (dt, "upsample2x", (1, 3, 16, 3, 4), {}, None),
        ]
    for i, (dt, kind, shape, attrs, params) in enumerate(cases):
        x = rng.standard_normal(shape).astype(dt)
        # the pipeline always casts weights to the run dtype (unet.py:214-215)
        params = None if params is None else {n: np.asarray(a).astype(dt) for n, a in params.items()}
        y = RK.apply_kernel(RK.OpKind(kind), [Tensor5D(x)], params, attrs).data
        key = f"{i:02d}_{kind}_{dt}"
        out[f"{key}/x"] = x
        out[f"{key}/y"] = y
        for n, a in (params or {}).items():
            out[f"{key}/p_{n}"] = np.asarray(a)
        out[f"{key}/attrs"] = np.frombuffer(json.dumps(attrs).encode(), dtype=np.uint8)
    # boundary ops
    a = rng.standard_normal((1, 3, 8, 4, 4))
    bias = rng.standard_normal((1, 3, 8, 1, 1))
    out["add_bias/a"], out["add_bias/b"] = a, bias
    out["add_bias/y"] = RK.apply_kernel(RK.OpKind.ADD, [Tensor5D(a), Tensor5D(bias)]).data
    c2 = rng.standard_normal((1, 3, 5, 4, 4))
    out["concat/a"], out["concat/b"] = a, c2
    out["concat/y"] = RK.apply_kernel(RK.OpKind.CONCAT, [Tensor5D(a), Tensor5D(c2)]).data
    # cosine
    p = rng.standard_normal((1, 4, 8, 8, 8))
    q = p + 0.3 * rng.standard_normal(p.shape)
    out["cos/a"], out["cos/b"] = p, q
    out["cos/y"] = np.array([RK.cosine_similarity(Tensor5D(p), Tensor5D(q))])
    return out


def main():
    meta = {}
    # --- C1 (BASELINE config 1): 8f x 4x32x32, base 8, 10 steps -------------
    c1 = UNetConfig(channels=4, frames=8, height=32, width=32, base_channels=8, norm_groups=4, steps=10)
    arrays = {}
    for dt in ("float64", "float32"):
        x, probes, eps = denoise(c1, dt, 10)
        arrays[f"c1_{dt}_final"] = x
        arrays[f"c1_{dt}_eps0"] = eps[0]
        arrays[f"c1_{dt}_probe0"] = probes[0]
        S = np.ones((10, 10))
        for i in range(10):
            for j in range(i + 1, 10):
                S[i, j] = S[j, i] = RK.cosine_similarity(Tensor5D(probes[i]), Tensor5D(probes[j]))
        arrays[f"c1_{dt}_S"] = S
    S = arrays["c1_float64_S"]
    gammas = [0.85, 0.9, 0.93, 0.95, 0.97]
    meta["c1_G"] = {str(g): a1(S, g) for g in gammas}
    G = a1(S, 0.93)
    for dt in ("float64", "float32"):
        xr, _, _ = denoise(c1, dt, 10, G=G)
        arrays[f"c1_{dt}_rehash_g093_final"] = xr
    # unsliced (spatial_k=1, one temporal tile) single eval for losslessness pins
    x0 = np.random.default_rng(c1.seed + 1).standard_normal(tuple(c1.input_shape()))
    graph, w64 = build_toy_unet(c1)
    g1 = group_operators(graph, 1, (1, 1))
    arrays["c1_float64_eps0_unsliced"], _ = walk(g1, w64, {"x": x0, "step_emb": step_embedding_tensor(c1, 0, "float64")})
    meta["c1_structure"] = structure(c1, 8)
    # --- SPEC default toy: c=8, K=25 ----------------------------------------
    d = UNetConfig()
    meta["default_structure"] = structure(d, 8)
    x, probes, _ = denoise(d, "float32", 25, spatial_k=8)
    S = np.ones((25, 25))
    for i in range(25):
        for j in range(i + 1, 25):
            S[i, j] = S[j, i] = RK.cosine_similarity(Tensor5D(probes[i]), Tensor5D(probes[j]))
    arrays["default_float32_final"] = x
    arrays["default_float32_S"] = S
    # --- wide config (every width a multiple of 64: exercises the tcgen05 path)
    cw = UNetConfig(channels=4, frames=4, height=16, width=16, base_channels=64, norm_groups=32, steps=3)
    for dt in ("float64",):
        x, probes, eps = denoise(cw, dt, 3)
        arrays[f"wide_{dt}_final"] = x
        arrays[f"wide_{dt}_eps0"] = eps[0]
    meta["wide_structure"] = {k: v for k, v in structure(cw, 4).items() if k in ("slfw_sha256", "peak", "schedule")}
    # --- slicer / rf examples --------------------
    meta["plans"] = {
        "spatial": {f"{bt},{k}": list(plan_spatial(bt, k).extents)
                    for bt, k in [(14, 7), (14, 4), (5, 1), (25, 8), (25, 4), (25, 2), (64, 8), (16, 16)]},
        "temporal": {f"{h},{w},{kh},{kw}": [list(p.row_extents), list(p.col_extents)]
                     for h, w, kh, kw in [(8, 8, 4, 4), (7, 7, 4, 4), (6, 6, 1, 1), (72, 128, 16, 16),
                                          (9, 16, 9, 16)]
                     for p in [plan_temporal(h, w, kh, kw)]},
    }
    np.savez_compressed(os.path.join(OUT, "reference_runs.npz"), **arrays)
    np.savez_compressed(os.path.join(OUT, "reference_kernels.npz"), **kernel_vectors())
    with open(os.path.join(OUT, "reference_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
