"""CPU baseline timing of the reference algorithm (oracle port) on the host cores.

Used only by ``bench.py`` (the ``cpu_baseline`` object of our line and the
``--impl reference`` arm).  Follows BASELINE.md §2: fp32, SlicedLoop,
spatial_k = B*T, temporal preset capped16, OpenBLAS on all host cores.

Bounded sample: every group runs only its first ``max_slices`` slices (one frame
for spatial groups, one capped16 tile for temporal groups); the unsampled slices
are charged at the median time of the sampled ones after the first (the first
slice pays cold caches) -- the for-loop executor's slices are independent and
identically shaped up to the remainder (grouping.py:241-254).  Checked once
against a complete C3 evaluation on the GPU box's 16 host cores
(tests/cpu_full_eval.py, profiles/r02_cpu_full_eval_c3.json).
Ungrouped Add/Concat nodes run in full.  One full (key) step and one tail
(skipped) step are sampled; a K-step rehash run is extrapolated as
|G| * full + (K - |G|) * tail.
"""

from __future__ import annotations

import os
import time

import numpy as np

from paper_2411_01171_b200.modes import ExecMode
from paper_2411_01171_b200.unet import PROBE_LABEL, step_embedding_tensor

from .executor import evaluate
from .harness import Model, initial_latent


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class CpuBaseline:
    def __init__(self, cfg, max_slices: int | None = 4):
        self.cfg = cfg
        self.max_slices = max_slices
        self.model = Model(cfg, np.float32)
        self.x = initial_latent(cfg)
        self.probe_id = self.model.graph.node_by_label(PROBE_LABEL).id

    def sample(self, step: int = 0) -> dict:
        m = self.model
        feeds = {"x": self.x, "step_emb": step_embedding_tensor(self.cfg, step, "float32").data}
        t_full = []
        t0 = time.perf_counter()
        _, cap = evaluate(m.graph, m.weights, feeds, ExecMode.SLICED_LOOP, m.grouped, capture=(PROBE_LABEL,),
                          max_slices=self.max_slices, timing=t_full)
        t1 = time.perf_counter()
        t_tail = []
        evaluate(m.graph, m.weights, {self.probe_id: cap[PROBE_LABEL]}, ExecMode.SLICED_LOOP, m.grouped,
                 start_after=self.probe_id, max_slices=self.max_slices, timing=t_tail)
        t2 = time.perf_counter()
        run = sum(t[1] for t in t_full + t_tail)
        extrap = sum(t[2] for t in t_full + t_tail)
        return {"full_s": sum(t[2] for t in t_full), "tail_s": sum(t[2] for t in t_tail),
                "sample_s": t2 - t0, "sample_full_s": t1 - t0,
                "fraction": run / extrap if extrap else 1.0}   # share of the extrapolated time actually run

    def steps_per_s(self, n_keys: int, K: int, sample: dict) -> float:
        run_s = n_keys * sample["full_s"] + (K - n_keys) * sample["tail_s"]
        return K / run_s
