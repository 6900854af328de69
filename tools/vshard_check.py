"""Frame/pixel-sharded plans emulated on one GPU at C3 scale vs the single-GPU run.

    python tools/vshard_check.py [world] [runs]

Runs the sharded launch sequences (per-rank S/T storage, 34 exchanges per evaluation), two
denoising steps (one key + one tail): inline exchanges once, then ``runs`` times with the exchanges
on a side stream ordered by CUDA events (the NCCL comm-stream protocol), which must reproduce the
inline result bit for bit; and the max deviation from the unsharded run (the GroupNorm statistics
are summed in a per-shard order, so it is small but not zero at this size).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2411_01171_b200.build import build  # noqa: E402

build()
from paper_2411_01171_b200.harness import Denoiser, initial_latent  # noqa: E402
from paper_2411_01171_b200.parallel import VirtualShards  # noqa: E402
from paper_2411_01171_b200.rehash import StepSchedule  # noqa: E402
from paper_2411_01171_b200.unet import UNetConfig  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = UNetConfig(channels=4, frames=25, height=72, width=128, base_channels=320, norm_groups=32, steps=2)
x0 = initial_latent(cfg)
sched = StepSchedule([0], 2)
ref = Denoiser(cfg).run(x0, sched)
inline = VirtualShards(cfg, world).run(x0, sched)
dev = float(np.abs(inline - ref).max() / np.abs(ref).max())
vs = VirtualShards(cfg, world, comm_stream=True)
bad = sum(not np.array_equal(vs.run(x0, sched), inline) for _ in range(runs))
print(f"world {world}: sharded vs unsharded max_rel {dev:.2e}; comm-stream runs differing from inline: {bad} of "
      f"{runs}", flush=True)
