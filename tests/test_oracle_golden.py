"""Pin the CPU oracle and the shared host logic against the real reference's outputs.

Fixtures come from tests/golden/make_golden.py (the unmodified reference run in
the build container).  CPU only.
"""

import hashlib
import json

import numpy as np
import pytest

from oracle import kernels as K
from oracle.harness import Model, run_full, run_rehash
from oracle.rehash import key_step_search, similarity_map
from paper_2411_01171_b200.grouping import estimate_peak_memory, group_operators, grouped_graph_report
from paper_2411_01171_b200.graph import infer_shapes
from paper_2411_01171_b200.kinds import OpKind
from paper_2411_01171_b200.slicer import default_temporal_config, plan_spatial, plan_temporal
from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet

C1 = UNetConfig(channels=4, frames=8, height=32, width=32, base_channels=8, norm_groups=4, steps=10)


def _rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("name,cfg,sk", [("c1_structure", C1, 8), ("default_structure", UNetConfig(), 8)])
def test_builder_and_grouping_match_reference(golden, name, cfg, sk):
    ref = golden["meta"][name]
    graph, w = build_toy_unet(cfg)
    assert graph.topo_order() == ref["topo"]
    assert json.loads(json.dumps(graph.to_json_dict())) == ref["graph_json"]
    # the reference-written JSON loads here (cli --graph) and describes the same graph
    from paper_2411_01171_b200.graph import Graph
    assert Graph.from_json_dict(ref["graph_json"]).to_json_dict() == graph.to_json_dict()
    gg = group_operators(graph, sk, default_temporal_config(cfg.height, cfg.width))
    assert [[k, r] for k, r in gg.schedule] == ref["schedule"]
    assert json.loads(json.dumps(grouped_graph_report(gg))) == ref["report"]
    assert {k: list(v) for k, v in infer_shapes(graph).items()} == ref["shapes"]
    for key, (s, a, shape) in ref["weights"].items():
        op, n = key.split("/")
        arr = w.get(op)[n]
        assert list(arr.shape) == shape
        assert float(arr.sum()) == s and float(np.abs(arr).sum()) == a, key
    assert hashlib.sha256(w.to_bytes()).hexdigest() == ref["slfw_sha256"]
    for mode, peak in ref["peak"].items():
        assert estimate_peak_memory(gg if mode != "reference" else graph, mode) == peak
    assert estimate_peak_memory(graph, "naiveclip", naive_chunk=2) == ref["peak_naive2"]


def test_plans_match_reference(golden):
    p = golden["meta"]["plans"]
    for key, ext in p["spatial"].items():
        bt, k = map(int, key.split(","))
        assert list(plan_spatial(bt, k).extents) == ext
    for key, (rows, cols) in p["temporal"].items():
        h, w, kh, kw = map(int, key.split(","))
        pl = plan_temporal(h, w, kh, kw)
        assert list(pl.row_extents) == rows and list(pl.col_extents) == cols


def _kernel_cases(golden):
    kv = golden["kernels"]
    keys = sorted({k.split("/")[0] for k in kv.files if k[:2].isdigit()})
    return kv, keys


def test_oracle_kernels_match_reference_vectors(golden):
    kv, keys = _kernel_cases(golden)
    assert len(keys) == 20
    for key in keys:
        kind = OpKind("_".join(key.split("_")[1:-1]))
        dt = key.split("_")[-1]
        attrs = json.loads(bytes(kv[f"{key}/attrs"]).decode())
        params = {f[len(key) + 3:]: kv[f] for f in kv.files if f.startswith(f"{key}/p_")} or None
        y = K.apply_kernel(kind, [kv[f"{key}/x"]], params, attrs)
        ref = kv[f"{key}/y"]
        assert y.dtype == ref.dtype and y.shape == ref.shape
        tol = 1e-13 if dt == "float64" else 2e-6
        assert _rel(y, ref) <= tol, (key, _rel(y, ref))
    y = K.apply_kernel(OpKind.ADD, [kv["add_bias/a"], kv["add_bias/b"]])
    assert np.array_equal(y, kv["add_bias/y"])
    y = K.apply_kernel(OpKind.CONCAT, [kv["concat/a"], kv["concat/b"]])
    assert np.array_equal(y, kv["concat/y"])
    assert abs(K.cosine_similarity(kv["cos/a"], kv["cos/b"]) - kv["cos/y"][0]) < 1e-14


def test_spec_kernel_examples():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((1, 2, 8, 4, 4))
    assert np.all(K.silu(np.zeros(5)) == 0)
    assert np.all(K.apply_kernel(OpKind.ADD, [x, -x]) == 0)
    w = np.zeros((8, 8, 3, 3))
    w[np.arange(8), np.arange(8), 1, 1] = 1
    assert np.array_equal(K.conv2d(x, w, np.zeros(8)), x)
    y = K.group_norm(x, np.ones(8), np.zeros(8), 4, 1e-5).reshape(1, 2, 4, 2, 4, 4)
    assert np.abs(y.mean(axis=(3, 4, 5))).max() < 1e-5
    assert np.abs(y.var(axis=(3, 4, 5)) - 1).max() < 1e-4
    assert K.cosine_similarity(x, x) == pytest.approx(1.0)
    assert K.cosine_similarity(x, -x) == pytest.approx(-1.0)
    e1, e2 = np.zeros(16), np.zeros(16)
    e1[0], e2[1] = 1, 1
    assert K.cosine_similarity(e1, e2) == 0.0


def test_a1_spec_examples():
    K5 = np.full((5, 5), 0.5) + 0.5 * np.eye(5)
    assert key_step_search(K5, 0.9) == [0, 1, 2, 3, 4]
    assert key_step_search(np.ones((6, 6)), 0.95) == [0, 5]
    S = np.full((6, 6), 0.5)
    np.fill_diagonal(S, 1.0)
    for i in range(3):
        S[i, 0] = 0.99
    S[4, 3] = S[5, 3] = 0.99
    assert key_step_search(S, 0.95) == [0, 3, 5]


def test_a1_matches_bruteforce_on_random_maps():
    rng = np.random.default_rng(3)
    for _ in range(1000):
        k = int(rng.integers(1, 33))
        S = rng.uniform(0.5, 1.0, (k, k))
        S = (S + S.T) / 2
        np.fill_diagonal(S, 1.0)
        g = float(rng.uniform(0.01, 1.0))
        # independent literal trace
        i = j = 0
        G = [0]
        while i < k:
            if S[i][j] >= g:
                i += 1
            else:
                G.append(i)
                j = i
        G.append(k - 1)
        out = key_step_search(S, g)
        assert out == sorted(set(G)) and out[0] == 0 and out[-1] == k - 1


@pytest.mark.parametrize("dt,tol", [("float64", 1e-12), ("float32", 2e-5)])
def test_oracle_c1_denoise_matches_reference(golden, dt, tol):
    runs = golden["runs"]
    m = Model(C1, np.dtype(dt))
    x, probes, eps = run_full(m)
    assert _rel(eps[0], runs[f"c1_{dt}_eps0"]) <= tol
    assert _rel(probes[0], runs[f"c1_{dt}_probe0"]) <= tol
    assert _rel(x, runs[f"c1_{dt}_final"]) <= tol
    S = similarity_map(probes)
    assert np.abs(S - runs[f"c1_{dt}_S"]).max() <= tol
    for g, G in golden["meta"]["c1_G"].items():
        assert key_step_search(runs["c1_float64_S"], float(g)) == G
    G = golden["meta"]["c1_G"]["0.93"]
    xr, ev = run_rehash(m, G)
    assert ev.count("full") == len(G)
    assert _rel(xr, runs[f"c1_{dt}_rehash_g093_final"]) <= tol


def test_slicing_is_lossless_fp64(golden):
    runs = golden["runs"]
    assert _rel(runs["c1_float64_eps0"], runs["c1_float64_eps0_unsliced"]) < 1e-12


def test_torch_ref_pinned_to_goldens(golden):
    """oracle/torch_ref.py (the fp64 checker used at C2/C3 on the GPU) against the reference's own
    fp64 runs: C1 10-step all-key run, its similarity map, eps at s=0, the gamma=0.93 rehash run,
    and the base-64 WIDE run.  Bar: <= 1e-12 (measured ~1e-15)."""
    from oracle import torch_ref as TR
    runs = golden["runs"]
    ref = TR.TorchRef(C1)
    x, S, eps = TR.run_full(ref, eps_steps=(0,))
    assert _rel(x.numpy(), runs["c1_float64_final"]) <= 1e-12
    assert float(np.abs(S - runs["c1_float64_S"]).max()) <= 1e-12
    assert _rel(eps[0].numpy(), runs["c1_float64_eps0"]) <= 1e-12
    xr = TR.run_rehash(ref, golden["meta"]["c1_G"]["0.93"])
    assert _rel(xr.numpy(), runs["c1_float64_rehash_g093_final"]) <= 1e-12
    for g, G in golden["meta"]["c1_G"].items():
        assert key_step_search(S, float(g)) == G, g
    wide = UNetConfig(channels=4, frames=4, height=16, width=16, base_channels=64, norm_groups=32, steps=3)
    xw, _, ew = TR.run_full(TR.TorchRef(wide), eps_steps=(0,))
    assert _rel(xw.numpy(), runs["wide_float64_final"]) <= 1e-12
    assert _rel(ew[0].numpy(), runs["wide_float64_eps0"]) <= 1e-12
