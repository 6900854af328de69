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
