"""Step Rehash ablation (BASELINE config 5): slicing+grouping only vs rehash at
several similarity thresholds, on one GPU.

    python tools/rehash_ablation.py [--config c2] [--gammas 0.90 0.93 0.95 0.97] [--target 13]

For every gamma: the key-step schedule G from Algorithm A1 on the calibration
map (measured on the device), its decision margin, device time of the whole
K-step run (CUDA graph), and the final latent's deviation from the all-key
(no-skip) run.  "Skip schedule matched to the CPU oracle" (BASELINE config 5):
A1 is also run on the fp64 oracle's own similarity map (committed record
profiles/r02_parity_<config>.json, tests/parity_sd.py) at the same gamma, and
``G_oracle_match`` says whether the device's schedule is the oracle's.
Prints one JSON line per setting.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2411_01171_b200.harness import Denoiser, initial_latent  # noqa: E402
from paper_2411_01171_b200.rehash import StepSchedule, gamma_for_target, key_step_search  # noqa: E402
from paper_2411_01171_b200.unet import UNetConfig  # noqa: E402


def timed_run(den, x0, sched, reps=3):
    key = den.prepare(sched)
    den.set_latent(x0)
    x0_rows = den.plan.latent.clone()
    den.launch(key)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        den.plan.latent.copy_(x0_rows)
        den.launch(key)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, den.result()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--gammas", type=float, nargs="*", default=[0.85, 0.90, 0.93, 0.95, 0.97, 0.99])
    ap.add_argument("--target", type=int, default=13)
    a = ap.parse_args()
    cfg = UNetConfig(**CONFIGS[a.config])
    K = cfg.steps
    den = Denoiser(cfg)
    x0 = initial_latent(cfg)
    _, S = den.calibrate(x0)
    den.trace = None
    rec_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            f"r02_parity_{a.config}.json")
    S_ref = np.asarray(json.load(open(rec_path))["S_ref"]) if os.path.exists(rec_path) else None
    adj = [S.values[i, i + 1] for i in range(K - 1)]
    print(json.dumps({"config": a.config, "similarity": {"mean_adjacent": float(np.mean(adj)),
                                                          "min_adjacent": float(np.min(adj))}}))
    full_ms, x_full = timed_run(den, x0, StepSchedule(list(range(K)), K))
    scale = float(np.abs(x_full).max())
    print(json.dumps({"setting": "slicing+grouping only (all key)", "keys": K, "run_ms": round(full_ms, 3),
                      "steps_per_s": round(K / full_ms * 1e3, 3)}))
    settings = [(g, None) for g in a.gammas] + [(None, a.target)]
    for g, tgt in settings:
        gamma = g if g is not None else gamma_for_target(S, tgt)
        sched = key_step_search(S, gamma, K)
        ms, x = timed_run(den, x0, sched)
        oracle = {}
        if S_ref is not None:
            so = key_step_search(S_ref, gamma, K)
            oracle = {"G_oracle": so.key_steps, "G_oracle_match": so.key_steps == sched.key_steps,
                      "oracle_margin": so.margin, "s_err": float(np.abs(S.values - S_ref).max())}
        print(json.dumps({
            "setting": f"rehash gamma={gamma:.6f}" + (f" (target {tgt})" if tgt else ""),
            "keys": len(sched.key_steps), "key_steps": sched.key_steps,
            "decision_margin": sched.margin, "run_ms": round(ms, 3), "steps_per_s": round(K / ms * 1e3, 3),
            "speedup_vs_all_key": round(full_ms / ms, 3),
            "final_max_rel_vs_all_key": float(np.abs(x - x_full).max() / scale), **oracle}))


if __name__ == "__main__":
    main()
