"""Run one eager key step and one tail step of a config (for ncu launch lists).

    python tools/step_once.py [--config c3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2411_01171_b200.executor import ExecConfig  # noqa: E402
from paper_2411_01171_b200.harness import Denoiser, initial_latent  # noqa: E402
from paper_2411_01171_b200.unet import UNetConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--backend", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
cfg = UNetConfig(**CONFIGS[a.config])
den = Denoiser(cfg, ExecConfig(gemm_backend=a.backend), K=2)
den.set_latent(initial_latent(cfg))
st = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    den.plan.run_full(st, den.emb_table[0].data_ptr())
    den.plan.run_tail(st)
torch.cuda.synchronize()
print("ok", len(den.plan.units), "units")
