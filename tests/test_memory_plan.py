"""Device arena vs the reference's static peak model (grouping.py:334-450), CPU only.

The arena holds only values that cross schedule units (group inputs/outputs,
skip tensors, zero-copy concat buffers, the persistent rehash probe and the
fp32 network output); group intermediates live in slice scratch.  Its size
must stay close to the reference's own grouped liveness floor in bf16.
"""

import pytest

from paper_2411_01171_b200.executor import plan_memory
from paper_2411_01171_b200.grouping import estimate_peak_memory, group_operators
from paper_2411_01171_b200.slicer import default_temporal_config
from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet


@pytest.mark.parametrize("cfg", [
    UNetConfig(channels=4, frames=8, height=32, width=32, base_channels=8, norm_groups=4),
    UNetConfig(channels=4, frames=25, height=72, width=128, base_channels=320, norm_groups=32),
])
def test_arena_close_to_reference_static_floor(cfg):
    g, _ = build_toy_unet(cfg)
    gg = group_operators(g, cfg.frames, default_temporal_config(cfg.height, cfg.width))
    # reference liveness walk in fp32 bytes -> bf16 activations are half
    floor_bf16 = estimate_peak_memory(gg, "slicedloop") / 2
    mem = plan_memory(g, gg)
    print(cfg.base_channels, mem, floor_bf16)
    assert mem["arena_bytes"] <= 1.25 * floor_bf16 + (1 << 20)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_groupnorm_statistics_hand_over(name):
    """15-16 of the 19 GroupNorms per evaluation take their statistics from a producer kernel (9 conv1
    epilogues, 3 downsamples, 3 concats fed by a downsample + an upsample, the tensor-core in_conv); the analysis checks that
    every producer writes one split count for all the partials it emits."""
    import bench
    from paper_2411_01171_b200.executor import ExecConfig, plan_memory
    from paper_2411_01171_b200.grouping import group_operators
    from paper_2411_01171_b200.slicer import default_temporal_config
    from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet
    cfg = UNetConfig(**bench.CONFIGS[name])
    g, _ = build_toy_unet(cfg)
    gg = group_operators(g, cfg.frames, default_temporal_config(cfg.height, cfg.width))
    m = plan_memory(g, gg, ExecConfig())
    # + the in_conv's own partials where it runs on the tensor-core kernel (cout % 64 == 0)
    assert m["gn_from_conv"] == 9 and m["gn_handed_over"] == (16 if cfg.base_channels % 64 == 0 else 15)
    assert 0 < m["gn_partial_bytes"] < max(0.06 * m["arena_bytes"], 1 << 20)
    off = plan_memory(g, gg, ExecConfig(gn_from_conv=False))
    assert off["gn_handed_over"] == 0 and off["gn_partial_bytes"] == 0


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_groupnorm_partial_slots_do_not_overlap(name):
    """Partial buffers are shared only between hand-overs whose [first producer, consumer] schedule
    intervals are disjoint (a concat's lives from the down path's downsample to the up block)."""
    import bench
    from paper_2411_01171_b200.executor import ExecConfig, plan_memory
    from paper_2411_01171_b200.grouping import group_operators
    from paper_2411_01171_b200.slicer import default_temporal_config
    from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet
    cfg = UNetConfig(**bench.CONFIGS[name])
    g, _ = build_toy_unet(cfg)
    gg = group_operators(g, cfg.frames, default_temporal_config(cfg.height, cfg.width))
    slots = plan_memory(g, gg, ExecConfig())["gn_slots"]
    assert len(slots) >= 15
    by_slot = {}
    for v, (k, a, b) in slots.items():
        assert a < b, v
        by_slot.setdefault(k, []).append((a, b, v))
    for k, iv in by_slot.items():
        iv.sort()
        for (a0, b0, v0), (a1, b1, v1) in zip(iv, iv[1:]):
            assert b0 < a1, f"slot {k}: {v0} [{a0}, {b0}] overlaps {v1} [{a1}, {b1}]"
    assert len(by_slot) >= 2     # the concats' long-lived partials need slots of their own
