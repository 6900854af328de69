"""CLI subcommands that drive the device (-m gpu): run / compare / similarity."""

import json

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_01171_b200.build import build  # noqa: E402
from paper_2411_01171_b200.cli import main  # noqa: E402
from paper_2411_01171_b200.rehash import SimilarityMap  # noqa: E402

build()

SMALL = ["--frames", "4", "--height", "16", "--width", "16", "--base-channels", "8", "--norm-groups", "4",
         "--channels", "4", "--steps", "5"]


def test_run_modes(tmp_path):
    sums = {}
    for mode in ("reference", "slicedloop", "pipelined"):
        d = tmp_path / mode
        assert main(["run", "--mode", mode, *SMALL, "--spatial-k", "4", "--out", str(d)]) == 0
        rep = json.loads((d / "run_report.json").read_text())
        assert rep["mode"] == mode and rep["peak_bytes"] > 0 and rep["static_model_bytes"] > 0
        sums[mode] = rep["output_checksum"]
    assert sums["pipelined"] == sums["slicedloop"]          # same launches, bit-identical output


def test_compare_flags_naive_divergence(tmp_path):
    assert main(["compare", "--modes", "reference,slicedloop,naiveclip", "--naive-chunk", "2", *SMALL,
                 "--out", str(tmp_path)]) == 0
    rows = {r["mode"]: r for r in json.loads((tmp_path / "compare.json").read_text())["rows"]}
    assert rows["reference"]["max_rel_error"] == 0.0
    assert rows["slicedloop"]["max_rel_error"] <= 1e-2
    assert rows["naiveclip"]["diverged"]


def test_similarity_then_search(tmp_path):
    assert main(["similarity", *SMALL, "--out", str(tmp_path)]) == 0
    S = SimilarityMap.parse_csv((tmp_path / "similarity.csv").read_text())
    assert S.K == 5 and abs(S.values[0, 0] - 1.0) < 1e-6
    assert main(["search-steps", "--similarity", str(tmp_path / "similarity.csv"), "--target-count", "3",
                 "--out", str(tmp_path)]) == 0
    assert len(json.loads((tmp_path / "schedule.json").read_text())["key_steps"]) == 3


def test_run_from_exported_model(tmp_path):
    """run --graph/--weights (exported files) == run_denoise on the same graph with the fp32 bundle in
    memory (bit-exact), and matches the fp64-built network within the bf16 storage tolerance."""
    import numpy as np
    from paper_2411_01171_b200.harness import DenoiseRunConfig, run_denoise
    from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet
    assert main(["export", *SMALL, "--out", str(tmp_path / "m")]) == 0
    assert main(["run", *SMALL, "--graph", str(tmp_path / "m" / "graph.json"), "--weights",
                 str(tmp_path / "m" / "weights.slfw"), "--save-output", "--out", str(tmp_path / "f")]) == 0
    y_file = np.load(tmp_path / "f" / "output.npy")
    ucfg = UNetConfig(frames=4, height=16, width=16, base_channels=8, norm_groups=4, channels=4, steps=5)
    g, w = build_toy_unet(ucfg)
    y32, _ = run_denoise(DenoiseRunConfig(unet=ucfg, graph=g, weights=w.astype(np.float32)))
    assert np.array_equal(y_file, y32.data)
    y64, _ = run_denoise(DenoiseRunConfig(unet=ucfg))
    assert float(np.abs(y_file - y64.data).max() / np.abs(y64.data).max()) <= 5e-3
