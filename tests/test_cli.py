"""CLI validation, exit codes and the host-only search-steps subcommand."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2411_01171_b200.cli import main
from paper_2411_01171_b200.rehash import SimilarityMap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_validation_exit_codes(tmp_path, capsys):
    assert main(["run", "--mode", "slicedloop", "--spatial-k", "0", "--out", str(tmp_path)]) == 2
    assert "spatial-k must be >= 1" in capsys.readouterr().err
    assert main(["run", "--mode", "bogus", "--out", str(tmp_path)]) == 2
    assert main(["run", "--mode", "naiveclip", "--out", str(tmp_path)]) == 2
    assert main(["run", "--gamma", "1.01", "--out", str(tmp_path)]) == 2
    assert main(["run", "--unknown-flag", "--out", str(tmp_path)]) == 2
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"frames": 4, "nonsense": 1}))
    assert main(["run", "--config", str(cfg), "--out", str(tmp_path)]) == 2
    assert "nonsense" in capsys.readouterr().err


def _write_map(path, vals):
    path.write_text(SimilarityMap(len(vals), np.asarray(vals, dtype=float)).export_csv())


def test_search_steps_all_ones(tmp_path):
    m = tmp_path / "s.csv"
    _write_map(m, np.ones((6, 6)))
    assert main(["search-steps", "--similarity", str(m), "--gamma", "0.95", "--out", str(tmp_path)]) == 0
    doc = json.loads((tmp_path / "schedule.json").read_text())
    assert doc["key_steps"] == [0, 5] and doc["K"] == 6


def test_search_steps_target_count(tmp_path):
    K = 25
    i = np.arange(K)
    vals = np.exp(-0.02 * np.abs(i[:, None] - i[None, :]))      # similarity decaying with step distance
    m = tmp_path / "s.csv"
    _write_map(m, vals)
    assert main(["search-steps", "--similarity", str(m), "--target-count", "13", "--out", str(tmp_path)]) == 0
    assert len(json.loads((tmp_path / "schedule.json").read_text())["key_steps"]) == 13
    assert main(["search-steps", "--similarity", str(m), "--gamma", "1.01", "--out", str(tmp_path)]) == 2
    assert main(["search-steps", "--similarity", str(m), "--out", str(tmp_path)]) == 2
    assert main(["search-steps", "--similarity", str(m), "--target-count", "99", "--out", str(tmp_path)]) == 2


def test_module_entry_point(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_2411_01171_b200", "run", "--spatial-k", "0",
                        "--out", str(tmp_path)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 2 and "spatial-k" in r.stderr


SMALL = ["--frames", "4", "--height", "16", "--width", "16", "--base-channels", "8", "--norm-groups", "4",
         "--channels", "4", "--steps", "5"]


def test_export_round_trip(tmp_path):
    """export writes the config's network as graph.json + weights.slfw (graph.py:127-169,
    kernels.py:397-465); both load back to the built graph and the fp32 weights."""
    from paper_2411_01171_b200.graph import Graph
    from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet
    from paper_2411_01171_b200.weights import WeightBundle
    assert main(["export", *SMALL, "--out", str(tmp_path)]) == 0
    g, w = build_toy_unet(UNetConfig(frames=4, height=16, width=16, base_channels=8, norm_groups=4, channels=4,
                                     steps=5))
    g2 = Graph.load(tmp_path / "graph.json")
    assert g2.to_json_dict() == g.to_json_dict()
    w2 = WeightBundle.load(tmp_path / "weights.slfw")
    assert sorted(w2.entries) == sorted(w.entries)
    for k, arrs in w.entries.items():
        for n, a in arrs.items():
            assert np.array_equal(w2.get(k)[n], a.astype(np.float32))


def test_model_file_flags_validated(tmp_path, capsys):
    assert main(["export", *SMALL, "--out", str(tmp_path)]) == 0
    g, wf = str(tmp_path / "graph.json"), str(tmp_path / "weights.slfw")
    assert main(["run", *SMALL, "--graph", g, "--out", str(tmp_path / "r")]) == 2         # weights missing
    assert "together" in capsys.readouterr().err
    assert main(["run", *SMALL, "--graph", str(tmp_path / "nope.json"), "--weights", wf,
                 "--out", str(tmp_path / "r")]) == 2
    assert main(["run", *SMALL, "--graph", g, "--weights", g, "--out", str(tmp_path / "r")]) == 2  # bad magic
    # a graph for another latent shape is rejected before any device work
    assert main(["run", "--frames", "8", *SMALL[2:], "--graph", g, "--weights", wf,
                 "--out", str(tmp_path / "r")]) == 2
    assert "does not match" in capsys.readouterr().err
