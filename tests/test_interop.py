"""Drop-in with the reference's own objects (build container: /root/reference importable).

The reference's ``Graph`` / ``GroupedGraph`` / ``OpKind`` / ``SlicePlan`` /
``Tensor5D`` are different classes from this package's; every entry point
normalises them by value (``paper_2411_01171_b200/interop.py``).  These tests
hand objects built by the UNMODIFIED reference to this package's host entry
points and check the results equal the ones computed from this package's own
objects.  Skipped where the reference is absent (the GPU box).
"""

import enum
import os
import sys
import types

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")


@pytest.fixture(scope="module")
def ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    if "sliceflow.executor" not in sys.modules:
        # grouping.estimate_peak_memory imports the (unshipped) executor for ExecMode only
        stub = types.ModuleType("sliceflow.executor")

        class ExecMode(str, enum.Enum):
            REFERENCE = "reference"
            SLICED_LOOP = "slicedloop"
            PIPELINED = "pipelined"
            NAIVE_CLIP = "naiveclip"
        stub.ExecMode = ExecMode
        sys.modules["sliceflow.executor"] = stub
    from sliceflow import grouping as G
    from sliceflow import slicer as SL
    from sliceflow import tensor as T
    from sliceflow import unet as U
    return types.SimpleNamespace(U=U, G=G, SL=SL, T=T, ExecMode=sys.modules["sliceflow.executor"].ExecMode)


def _cfgs(ref):
    return [ref.U.UNetConfig(channels=4, frames=8, height=32, width=32, base_channels=8, norm_groups=4, steps=10),
            ref.U.UNetConfig()]


def test_reference_graph_through_host_entry_points(ref):
    from paper_2411_01171_b200.graph import infer_shapes, receptive_field
    from paper_2411_01171_b200.grouping import estimate_peak_memory, group_operators, grouped_graph_report
    from paper_2411_01171_b200.slicer import default_temporal_config
    from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet
    for rc in _cfgs(ref):
        rgraph, _ = ref.U.build_toy_unet(rc)
        mine, _ = build_toy_unet(UNetConfig(**{f: getattr(rc, f) for f in rc.__dataclass_fields__}))
        # shape inference on the reference's Graph (was: ShapeInferenceFailure 'unknown kind OpKind.LINEAR')
        assert {k: tuple(v) for k, v in infer_shapes(rgraph).items()} == \
            {k: tuple(v) for k, v in infer_shapes(mine).items()}
        tc = default_temporal_config(rc.height, rc.width)
        gg_from_ref = group_operators(rgraph, 8, tc)
        gg_mine = group_operators(mine, 8, tc)
        assert gg_from_ref.schedule == gg_mine.schedule
        assert grouped_graph_report(gg_from_ref) == grouped_graph_report(gg_mine)
        # the reference's own GroupedGraph (built by its grouping pass) is accepted as is
        rgg = ref.G.group_operators(rgraph, 8, tc)
        assert grouped_graph_report(rgg) == grouped_graph_report(gg_mine)
        for mode in ("reference", ref.ExecMode.SLICED_LOOP, ref.ExecMode.PIPELINED):
            g = rgraph if mode == "reference" else rgg
            gm = mine if mode == "reference" else gg_mine
            assert estimate_peak_memory(g, mode) == estimate_peak_memory(gm, getattr(mode, "value", mode))
            # and equals the reference's own static model
            assert estimate_peak_memory(g, mode) == ref.G.estimate_peak_memory(g, ref.ExecMode(getattr(mode, "value", mode)))
        seg = list(rgg.groups[0].nodes)
        assert receptive_field(rgraph, seg, "bt") == receptive_field(mine, seg, "bt")


def test_reference_grouped_graph_converts_by_value(ref):
    from paper_2411_01171_b200.interop import as_grouped, as_plan
    from paper_2411_01171_b200.kinds import Domain, OpKind
    from paper_2411_01171_b200.slicer import SliceMode, plan_spatial, plan_temporal
    rc = _cfgs(ref)[0]
    rgraph, _ = ref.U.build_toy_unet(rc)
    rgg = ref.G.group_operators(rgraph, 3, (4, 4))
    gg = as_grouped(rgg)
    assert len(gg.groups) == len(rgg.groups)
    for a, b in zip(gg.groups, rgg.groups):
        assert a.label == b.label and a.nodes == b.nodes
        assert isinstance(a.domain, Domain) and a.domain.value == b.domain.value
        assert all(isinstance(o.kind, OpKind) for o in a.ops)
        assert a.plan.n_slices == b.plan.n_slices
        assert a.plan.to_json_dict() == b.plan.to_json_dict()
    p = as_plan(ref.SL.plan_spatial(25, 8))
    assert p.mode is SliceMode.SPATIAL_BT and p.extents == plan_spatial(25, 8).extents
    p = as_plan(ref.SL.plan_temporal(9, 16, 4, 4))
    assert p.row_extents == plan_temporal(9, 16, 4, 4).row_extents


def test_reference_tensor_and_modes_accepted(ref):
    from paper_2411_01171_b200.interop import as_array, as_mode
    from paper_2411_01171_b200.modes import ExecMode
    x = np.arange(2 * 3 * 4 * 2 * 2, dtype=np.float32).reshape(1, 2, 12, 2, 2)
    t = ref.T.Tensor5D(x)
    assert np.array_equal(as_array(t), x)
    assert as_mode(ref.ExecMode.PIPELINED) is ExecMode.PIPELINED
    assert as_mode("slicedloop") is ExecMode.SLICED_LOOP
