"""Feature Slicer host API: extract_slice / slice_tensor / unslice (slicer.py:193-256).

The device path never copies slices (they are row views); these are the reference's
public host utilities.  Checked against the SPEC examples, the round-trip property on
random shapes and plans (hypothesis), the error classes, and -- where the reference is
importable (build container) -- element-for-element against the reference's own output.
"""

import os
import sys

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2411_01171_b200.errors import IncompleteCover, OverlappingRegions, PlanShapeMismatch
from paper_2411_01171_b200.slicer import (SubFeature, extract_slice, plan_spatial, plan_temporal, slice_tensor,
                                          unslice)
from paper_2411_01171_b200.tensor import Tensor5D


def _x(shape, seed=0):
    return Tensor5D(np.random.default_rng(seed).standard_normal(shape))


def test_spec_examples():
    x = _x((1, 4, 3, 4, 4))
    # identity plan -> one sub-feature equal to X
    (only,) = slice_tensor(x, plan_spatial(4, 1))
    assert np.array_equal(only.data.data, x.data)
    # bt = 4, k = 2 -> two parts, bit-identical reassembly
    parts = slice_tensor(x, plan_spatial(4, 2))
    assert len(parts) == 2 and parts[0].region.bt == (0, 2)
    assert np.array_equal(unslice(parts).data, x.data)
    # h = w = 4, k_h = k_w = 2 -> four tiles, bit-identical reassembly
    tiles = slice_tensor(x, plan_temporal(4, 4, 2, 2))
    assert len(tiles) == 4 and tiles[3].region.rows == (2, 4) and tiles[3].region.cols == (2, 4)
    assert np.array_equal(unslice(list(reversed(tiles))).data, x.data)


def test_slices_are_copies_and_validated():
    x = _x((2, 3, 2, 5, 6))
    s = extract_slice(x, plan_spatial(6, 4), 1)
    assert s.region.bt == (2, 4) and tuple(s.data.shape) == (1, 2, 2, 5, 6)
    assert not np.shares_memory(s.data.data, x.data)
    assert np.array_equal(s.data.data[0], x.data.reshape(6, 2, 5, 6)[2:4])
    with pytest.raises(PlanShapeMismatch):
        SubFeature(x.shape, s.region, Tensor5D(np.zeros((1, 3, 2, 5, 6))))
    with pytest.raises(PlanShapeMismatch):
        slice_tensor(x, plan_spatial(5, 2))


def test_unslice_errors():
    x = _x((1, 6, 2, 3, 3))
    parts = slice_tensor(x, plan_spatial(6, 3))
    with pytest.raises(IncompleteCover):
        unslice(parts[:2])
    with pytest.raises(OverlappingRegions):
        unslice(parts + parts[:1])
    with pytest.raises(IncompleteCover):
        unslice([])
    tiles = slice_tensor(x, plan_temporal(3, 3, 2, 2))
    with pytest.raises(IncompleteCover):
        unslice(tiles[1:])
    with pytest.raises(OverlappingRegions):
        unslice(tiles + tiles[-1:])
    with pytest.raises(PlanShapeMismatch):
        unslice(parts[:1] + tiles)


@settings(max_examples=60, deadline=None)
@given(b=st.integers(1, 2), t=st.integers(1, 6), c=st.integers(1, 3), h=st.integers(1, 7), w=st.integers(1, 7),
       data=st.data())
def test_round_trip_property(b, t, c, h, w, data):
    x = _x((b, t, c, h, w), seed=b * 1000 + t * 100 + h * 10 + w)
    if data.draw(st.booleans()):
        plan = plan_spatial(b * t, data.draw(st.integers(1, b * t)))
    else:
        plan = plan_temporal(h, w, data.draw(st.integers(1, h)), data.draw(st.integers(1, w)))
    parts = slice_tensor(x, plan)
    assert len(parts) == plan.n_slices
    perm = data.draw(st.permutations(parts))
    assert np.array_equal(unslice(perm).data, x.data)


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")
def test_matches_reference_slices():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from sliceflow import slicer as RS
    from sliceflow.tensor import Tensor5D as RT
    x = _x((1, 5, 3, 7, 9), seed=3)
    for mine, theirs in ((plan_spatial(5, 2), RS.plan_spatial(5, 2)),
                         (plan_temporal(7, 9, 3, 4), RS.plan_temporal(7, 9, 3, 4))):
        a = slice_tensor(x, mine)
        r = RS.slice_tensor(RT(x.data), theirs)
        assert len(a) == len(r)
        for p, q in zip(a, r):
            assert (p.region.bt, p.region.rows, p.region.cols) == (q.region.bt, q.region.rows, q.region.cols)
            assert np.array_equal(p.data.data, q.data.data)
