"""Oracle denoise loop + rehash run (restates SPEC.md:422-430, 479-487).

x <- x - alpha_s * f(x, s), alpha_s = float32(0.08 * (1 - s/K)); x0 =
default_rng(seed+1).standard_normal(input_shape) (survey §8d: the builder's
documented choice for the unpinned "seeded initial x").  Test oracle only.
"""

from __future__ import annotations

import numpy as np

from paper_2411_01171_b200.grouping import group_operators
from paper_2411_01171_b200.modes import ExecMode
from paper_2411_01171_b200.slicer import default_temporal_config
from paper_2411_01171_b200.unet import PROBE_LABEL, build_toy_unet, step_embedding_tensor

from .executor import evaluate
from .rehash import donors


def initial_latent(cfg, dtype=np.float32):
    return np.random.default_rng(cfg.seed + 1).standard_normal(tuple(cfg.input_shape())).astype(dtype)


def alpha(s, K, dtype=np.float32):
    return dtype(0.08 * (1.0 - s / K))


class Model:
    """Graph + cast weights + grouping, built once."""

    def __init__(self, cfg, dtype=np.float32, spatial_k=None, temporal_cfg=None):
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        self.graph, w64 = build_toy_unet(cfg)
        self.weights = w64.astype(self.dtype)
        sk = spatial_k or cfg.effective_batch * cfg.frames
        tc = temporal_cfg or default_temporal_config(cfg.height, cfg.width)
        self.grouped = group_operators(self.graph, sk, tc)

    def eps(self, x, s, mode=ExecMode.SLICED_LOOP, capture=()):
        feeds = {"x": x, "step_emb": step_embedding_tensor(self.cfg, s, self.dtype.name).data}
        return evaluate(self.graph, self.weights, feeds, mode, self.grouped, capture=capture)

    def tail(self, cache, mode=ExecMode.SLICED_LOOP):
        return evaluate(self.graph, self.weights, {PROBE_LABEL: cache}, mode, self.grouped,
                        start_after=self.graph.node_by_label(PROBE_LABEL).id)[0]


def run_full(model, K=None, mode=ExecMode.SLICED_LOOP, capture_probe=True):
    """Plain K-step loop; returns (final x, [probe per step], [eps per step])."""
    cfg = model.cfg
    K = K or cfg.steps
    x = initial_latent(cfg, model.dtype.type)
    probes, epss = [], []
    for s in range(K):
        e, cap = model.eps(x, s, mode, capture=(PROBE_LABEL,) if capture_probe else ())
        if capture_probe:
            probes.append(cap[PROBE_LABEL])
        epss.append(e)
        x = x - alpha(s, K, model.dtype.type) * e
        assert np.isfinite(x).all(), f"non-finite latent at step {s}"
    return x, probes, epss


def run_rehash(model, G, K=None, mode=ExecMode.SLICED_LOOP):
    """Key steps full + cache the probe; skipped steps run the tail on the donor's cache."""
    cfg = model.cfg
    K = K or cfg.steps
    keys = set(G)
    x = initial_latent(cfg, model.dtype.type)
    cache = None
    evals = []
    for s in range(K):
        if s in keys:
            e, cap = model.eps(x, s, mode, capture=(PROBE_LABEL,))
            cache = cap[PROBE_LABEL]
            evals.append("full")
        else:
            e = model.tail(cache, mode)
            evals.append("tail")
        x = x - alpha(s, K, model.dtype.type) * e
    return x, evals


__all__ = ["Model", "run_full", "run_rehash", "initial_latent", "alpha", "donors"]
