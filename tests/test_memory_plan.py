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
