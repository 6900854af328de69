"""Step Rehash (paper §4.3, Appendix B) on the device.

The reference specifies this module (``SPEC.md:382-462``) but does not ship
it; ``unet.py:28-36`` fixes the probe.  Here:

* the similarity map is a Gram matrix of the K cached probe tensors computed
  by one fixed-order fp64 reduction kernel (``sf_gram_bf16``) -- the probes
  stay in HBM, only K*K doubles come back;
* the key-step search (Algorithm A1) and the target-count gamma search are
  host logic over that K x K map;
* :func:`rehash_execute` runs the denoising loop where key steps evaluate the
  full network (their probe output *is* the feature cache: the probe's arena
  slot is persistent) and skipped steps evaluate only the tail strictly after
  the probe (``SPEC.md:425``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import BadThreshold, InvalidParam, ScheduleMismatch, TargetUnreachable, ZeroNorm


@dataclass
class SimilarityMap:
    """K x K cosine similarities at a probe layer."""

    K: int
    values: np.ndarray
    probe_label: str = ""

    def export_csv(self) -> str:
        """K x K CSV with step-index header row/column."""
        lines = ["step," + ",".join(str(j) for j in range(self.K))]
        for i in range(self.K):
            lines.append(str(i) + "," + ",".join(repr(float(v)) for v in self.values[i]))
        return "\n".join(lines) + "\n"

    @classmethod
    def parse_csv(cls, text: str, probe_label: str = "") -> "SimilarityMap":
        rows = [r.split(",") for r in text.strip().splitlines()[1:]]
        vals = np.array([[float(v) for v in r[1:]] for r in rows])
        return cls(len(rows), vals, probe_label)


@dataclass
class StepSchedule:
    """Key steps G, K and gamma."""

    key_steps: list
    K: int
    gamma: float | None = None
    margin: float | None = None
    donors: list = field(default_factory=list)

    def __post_init__(self):
        if not self.donors:
            d, keys = 0, set(self.key_steps)
            for s in range(self.K):
                if s in keys:
                    d = s
                self.donors.append(d)

    def is_key(self, s: int) -> bool:
        return s in set(self.key_steps)

    def to_json_dict(self) -> dict:
        return {"K": self.K, "gamma": self.gamma, "key_steps": list(self.key_steps)}


def gram_partial(probes: list[torch.Tensor]) -> np.ndarray:
    """K x K fp64 Gram matrix <p_i, p_j> of device probes (one fixed-order reduction)."""
    K = len(probes)
    n = probes[0].numel()
    dev = probes[0].device
    if any(p.data_ptr() % 16 for p in probes):
        raise InvalidParam("sf_gram_bf16 needs 16-byte aligned probes")
    ptrs = torch.tensor([p.data_ptr() for p in probes], dtype=torch.int64, device=dev)
    work = torch.empty(N.query("sf_gram_workspace", K, n), dtype=torch.uint8, device=dev)
    out = torch.empty(K * K, dtype=torch.float64, device=dev)
    N.call("sf_gram_bf16", ptrs.data_ptr(), K, n, work.data_ptr(), out.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    return out.cpu().numpy().reshape(K, K)


def gram_similarity(probes: list[torch.Tensor], probe_label: str = "") -> SimilarityMap:
    """S[i][j] = <p_i, p_j> / (|p_i| |p_j|) from one device Gram reduction."""
    return similarity_from_gram(gram_partial(probes), probe_label)


def similarity_from_gram(G: np.ndarray, probe_label: str = "") -> SimilarityMap:
    """Normalise a (possibly rank-summed) Gram matrix into the cosine map (kernels.py:386-390)."""
    K = G.shape[0]
    d = np.diag(G).copy()
    if np.any(d == 0.0):
        raise ZeroNorm("cosine similarity undefined for an identically-zero tensor")
    S = G / np.sqrt(np.outer(d, d))
    S = np.clip(S, -1.0, 1.0)
    np.fill_diagonal(S, 1.0)
    return SimilarityMap(K, S, probe_label)


def key_step_search(S, gamma: float, K: int | None = None) -> StepSchedule:
    """Algorithm A1, duplicates removed."""
    if not (0.0 < gamma <= 1.0):
        raise BadThreshold(f"gamma must be in (0,1], got {gamma}")
    vals = S.values if isinstance(S, SimilarityMap) else np.asarray(S)
    K = vals.shape[0] if K is None else K
    if vals.shape[0] != K:
        raise ScheduleMismatch(f"similarity map is {vals.shape[0]}x{vals.shape[0]}, run has K={K}")
    i = j = 0
    G = [0]
    margin = math.inf
    while i < K:
        v = vals[i][j]
        if i != j:
            margin = min(margin, abs(v - gamma))
        if v >= gamma:
            i += 1
        else:
            G.append(i)
            j = i
    G.append(K - 1)
    return StepSchedule(sorted(set(G)), K, gamma, margin if margin != math.inf else None)


def gamma_for_target(S, target: int, tol: float = 1e-6) -> float:
    """Bisection over (0, 1] to 1e-6 for |G| == target, ties to larger gamma.

    Returns the midpoint of the final bracket's gamma interval that yields
    ``target`` keys when it can be found, which maximises the decision margin
    (survey §7 hard part 3: a gamma sitting on a similarity entry flips G under
    bf16 rounding).
    """
    vals = S.values if isinstance(S, SimilarityMap) else np.asarray(S)
    K = vals.shape[0]
    if not 1 <= target <= K or len(key_step_search(vals, 1.0).key_steps) < target:
        raise TargetUnreachable(f"no gamma yields {target} key steps")
    lo, hi = 0.0, 1.0
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if len(key_step_search(vals, max(mid, 1e-12)).key_steps) >= target:
            hi = mid
        else:
            lo = mid
    if len(key_step_search(vals, hi).key_steps) != target:
        raise TargetUnreachable(f"no gamma yields exactly {target} key steps")
    # widen to the interval of similarity values around hi that keeps |G|
    cands = np.unique(vals[np.triu_indices(K, 1)])
    above = cands[cands >= hi]
    below = cands[cands < hi]
    if len(above) and len(below):
        mid = 0.5 * (below.max() + above.min())
        if len(key_step_search(vals, mid).key_steps) == target and (
                key_step_search(vals, mid).key_steps == key_step_search(vals, hi).key_steps):
            return float(mid)
    return hi


def op_count_report(graph, schedule: StepSchedule, tail_nodes: int) -> dict:
    """Executed vs skipped node evaluations per step."""
    full = len(graph.nodes)
    per = [full if schedule.is_key(s) else tail_nodes for s in range(schedule.K)]
    return {"per_step": per, "executed": sum(per), "full_run": full * schedule.K,
            "fraction": sum(per) / (full * schedule.K), "tail_nodes": tail_nodes}
