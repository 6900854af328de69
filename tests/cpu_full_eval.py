"""Time ONE real, complete CPU evaluation of the reference algorithm (test infrastructure).

    python tests/cpu_full_eval.py c3 [--out FILE]

The bench's ``cpu_baseline`` extrapolates from the first slice of every group;
this runs every slice of every group (oracle port, fp32, SlicedLoop, capped16
temporal preset, spatial k = B*T -- BASELINE.md §2) for one full evaluation
and one tail evaluation, so the extrapolation can be checked against a real
run on the same host cores.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle.cpu_baseline import CpuBaseline, host_cores  # noqa: E402
from paper_2411_01171_b200.unet import UNetConfig  # noqa: E402
from parity_sd import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = UNetConfig(**CONFIGS[a.config])
    sampled = CpuBaseline(cfg).sample()
    full = CpuBaseline(cfg, max_slices=None)
    t0 = time.perf_counter()
    real = full.sample()
    wall = time.perf_counter() - t0
    rec = {"config": a.config, "cores": host_cores(), "full_eval_s": real["sample_full_s"],
           "tail_eval_s": real["sample_s"] - real["sample_full_s"], "wall_s": wall,
           "extrapolated_full_s": sampled["full_s"], "extrapolated_tail_s": sampled["tail_s"],
           "extrapolation_error": sampled["full_s"] / real["sample_full_s"] - 1.0,
           "sample_run_s": sampled["sample_s"]}
    print(json.dumps(rec), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rec, fh, indent=1)


if __name__ == "__main__":
    main()
