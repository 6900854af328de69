"""Two-stream slice execution vs one stream, repeated (the concurrency check of profiles finding 30).

    python tools/race_check.py [runs]

A ragged C3 plan (7 frame slices; GroupNorm -> conv groups in flight on two streams) evaluated
``runs`` times eagerly; every result must equal the one-stream result bit for bit.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2411_01171_b200.build import build  # noqa: E402

build()
from paper_2411_01171_b200.executor import ExecConfig, execute  # noqa: E402
from paper_2411_01171_b200.harness import initial_latent  # noqa: E402
from paper_2411_01171_b200.modes import ExecMode  # noqa: E402
from paper_2411_01171_b200.tensor import Tensor5D  # noqa: E402
from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet, step_embedding_tensor  # noqa: E402

c3 = UNetConfig(channels=4, frames=25, height=72, width=128, base_channels=320, norm_groups=32, steps=25)
g, w = build_toy_unet(c3)
inp = {"x": Tensor5D(initial_latent(c3)), "step_emb": step_embedding_tensor(c3, 5)}
ref = execute(g, ExecMode.SLICED_LOOP, inp, w, cfg=ExecConfig(spatial_k=7, slice_streams=1))[0].data
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
bad = sum(not np.array_equal(execute(g, ExecMode.SLICED_LOOP, inp, w,
                                     cfg=ExecConfig(spatial_k=7, slice_streams=2))[0].data, ref) for _ in range(n))
print(f"two streams vs one: {bad} of {n} runs differ", flush=True)
