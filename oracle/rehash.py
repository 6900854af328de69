"""Oracle Step Rehash: similarity map, Algorithm A1, target-gamma search.

Restates ``SPEC.md:382-462`` (the reference ships no ``rehash.py``;
``unet.py:28-36`` names its probe).  Test oracle only.
"""

from __future__ import annotations

import numpy as np

from paper_2411_01171_b200.errors import BadThreshold, TargetUnreachable

from .kernels import cosine_similarity


def similarity_map(trace):
    """S[i][j] = cos(trace_i, trace_j)."""
    k = len(trace)
    s = np.ones((k, k))
    for i in range(k):
        for j in range(i + 1, k):
            s[i, j] = s[j, i] = cosine_similarity(trace[i], trace[j])
    return s


def key_step_search(S, gamma, K=None):
    """Algorithm A1 as printed; dedupe + sort."""
    if not (0.0 < gamma <= 1.0):
        raise BadThreshold(f"gamma must be in (0,1], got {gamma}")
    S = np.asarray(S)
    K = S.shape[0] if K is None else K
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


def donors(G, K):
    """Donor of every step = latest key step <= it."""
    out, d = [], 0
    keys = set(G)
    for s in range(K):
        if s in keys:
            d = s
        out.append(d)
    return out


def gamma_for_target(S, target, tol=1e-6):
    """Binary search over (0,1] for |G| = target, ties toward larger gamma."""
    K = np.asarray(S).shape[0]
    if not 1 <= target <= K:
        raise TargetUnreachable(f"target {target} outside [1, {K}]")
    lo, hi = 0.0, 1.0
    # smallest gamma with |G| >= target, searched on the literal algorithm
    if len(key_step_search(S, 1.0)) < target:
        raise TargetUnreachable(f"no gamma yields {target} key steps")
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if len(key_step_search(S, max(mid, 1e-12))) >= target:
            hi = mid
        else:
            lo = mid
    if len(key_step_search(S, hi)) != target:
        raise TargetUnreachable(f"no gamma yields exactly {target} key steps")
    return hi
