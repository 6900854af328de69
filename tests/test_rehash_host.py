"""Step Rehash host logic on CPU: Algorithm A1 edge cases, the target-count gamma
search and the error semantics SPEC.md specifies (
errors.py:72-80 of the reference).  No GPU needed: the device side (the Gram
reduction) is covered by tests/test_gpu_parity.py.
"""

import math

import numpy as np
import pytest

from paper_2411_01171_b200.errors import BadThreshold, ScheduleMismatch, TargetUnreachable, ZeroNorm
from paper_2411_01171_b200.rehash import (SimilarityMap, StepSchedule, gamma_for_target, key_step_search,
                                          similarity_from_gram)


def walk_map(K, seed, n=4096, drift=0.35):
    """Cosine map of a random walk of feature tensors (adjacent steps similar, like a denoising trace)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    probes = []
    for _ in range(K):
        x = x + drift * rng.standard_normal(n) * rng.uniform(0.2, 1.5)
        probes.append(x.copy())
    P = np.stack(probes)
    return similarity_from_gram(P @ P.T).values


@pytest.mark.parametrize("gamma", [0.0, -0.5, 1.0000001, 2.0, math.nan])
def test_bad_threshold(gamma):
    with pytest.raises(BadThreshold):
        key_step_search(np.eye(4), gamma)


def test_schedule_mismatch():
    with pytest.raises(ScheduleMismatch):
        key_step_search(np.ones((5, 5)), 0.9, K=6)


@pytest.mark.parametrize("target", [0, -1, 11])
def test_target_unreachable(target):
    with pytest.raises(TargetUnreachable):
        gamma_for_target(walk_map(10, 0), target)


def test_degenerate_maps():
    # every step identical to step 0: only the mandatory first and last steps are keys
    assert key_step_search(np.ones((7, 7)), 0.99).key_steps == [0, 6]
    # K = 1: a single key step
    assert key_step_search(np.ones((1, 1)), 0.5).key_steps == [0]
    # gamma = 1 on a map with every off-diagonal entry < 1: every step is a key
    S = walk_map(9, 1)
    assert key_step_search(S, 1.0).key_steps == list(range(9))


@pytest.mark.parametrize("seed", range(6))
def test_schedule_invariants(seed):
    K = 25
    S = walk_map(K, seed)
    for gamma in np.linspace(0.05, 1.0, 40):
        sch = key_step_search(S, float(gamma))
        G = sch.key_steps
        assert G[0] == 0 and G[-1] == K - 1
        assert G == sorted(set(G)) and all(0 <= g < K for g in G)
        # donor of a skipped step = the latest key step at or before it
        for s in range(K):
            assert sch.donors[s] == max(g for g in G if g <= s)
            assert sch.is_key(s) == (s in G)
        if sch.margin is not None:
            assert sch.margin >= 0


@pytest.mark.parametrize("seed", range(4))
def test_gamma_for_target_hits_every_reachable_count(seed):
    K = 25
    S = walk_map(K, 100 + seed)
    n_max = len(key_step_search(S, 1.0).key_steps)
    hit = 0
    for target in range(2, n_max + 1):
        try:
            g = gamma_for_target(S, target)
        except TargetUnreachable:
            # |G| is not monotone in gamma on arbitrary maps: a count can be skipped
            continue
        assert 0.0 < g <= 1.0
        assert len(key_step_search(S, g).key_steps) == target
        hit += 1
    assert hit >= (n_max - 1) // 2


def test_similarity_from_gram_properties():
    rng = np.random.default_rng(7)
    P = rng.standard_normal((6, 300))
    S = similarity_from_gram(P @ P.T, "probe").values
    want = (P @ P.T) / np.outer(np.linalg.norm(P, axis=1), np.linalg.norm(P, axis=1))
    assert np.allclose(S, want, atol=1e-14)
    assert np.array_equal(S, S.T) and np.all(np.diag(S) == 1.0)
    P[3] = 0.0
    with pytest.raises(ZeroNorm):
        similarity_from_gram(P @ P.T)


def test_similarity_csv_and_schedule_json_round_trip():
    S = SimilarityMap(8, walk_map(8, 3), "up_blocks.3.temporal.0")
    back = SimilarityMap.parse_csv(S.export_csv())
    assert back.K == 8 and np.array_equal(back.values, S.values)
    sch = key_step_search(S, 0.9)
    d = sch.to_json_dict()
    assert d == {"K": 8, "gamma": 0.9, "key_steps": sch.key_steps}
    assert StepSchedule(d["key_steps"], d["K"]).donors == sch.donors
