"""Parity of the device path against the fp64 oracle at SD widths (BASELINE configs 2/3).

Test infrastructure: imported by ``tests/test_gpu_parity_sd.py`` and runnable as

    python tests/parity_sd.py c3 [--out profiles/r02_parity_c3.json]

to write the committed parity record that ``bench.py`` checks its own
schedule against.  The oracle is ``oracle/torch_ref.py`` (torch fp64 on the
same GPU, pinned to the reference's own fp64 goldens at <= 1e-12).

What is compared (tolerances for bf16 storage + fp32 accumulation):
  * eps0   -- one network evaluation at s = 0 from the seeded latent: max_rel
  * S      -- the full K x K calibration similarity map (all-key run): max |S_dev - S_ref|
  * G      -- the Step Rehash key steps at the bench's gamma (target 13 of 25) from both maps,
              and the decision margin |S_ij - gamma| along the oracle's A1 path
  * x_allkey / x_rehash -- final latents of the all-key run and of the 13/25 rehash run
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np
import torch

from oracle import torch_ref as TR
from paper_2411_01171_b200.executor import ExecConfig
from paper_2411_01171_b200.harness import Denoiser, initial_latent
from paper_2411_01171_b200.rehash import StepSchedule, gamma_for_target, key_step_search
from paper_2411_01171_b200.unet import UNetConfig

CONFIGS = {
    "c2": dict(channels=4, frames=16, height=64, width=64, base_channels=320, norm_groups=32, steps=25),
    "c3": dict(channels=4, frames=25, height=72, width=128, base_channels=320, norm_groups=32, steps=25),
    "wide": dict(channels=4, frames=4, height=16, width=16, base_channels=64, norm_groups=32, steps=10),
    # long clip (BASELINE C4's T = 64) on a small plane: the fused temporal attention with 2 pixels
    # per tile at L0 and the tcgen05 temporal core at C = 640 / 1280
    "long": dict(channels=4, frames=64, height=32, width=32, base_channels=320, norm_groups=32, steps=25),
}


def rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def a1_margin(S, gamma) -> float:
    """Smallest |S[i][j] - gamma| over the comparisons Algorithm A1 makes on S."""
    return key_step_search(S, gamma).margin


def target_keys(K: int) -> int:
    return max(2, math.ceil(K * 13 / 25))


def run(name: str, exec_cfg: ExecConfig | None = None, log=print) -> dict:
    cfg = UNetConfig(**CONFIGS[name])
    K = cfg.steps
    t0 = time.perf_counter()
    den = Denoiser(cfg, exec_cfg or ExecConfig())
    x0 = initial_latent(cfg)
    # one evaluation at s = 0
    st = torch.cuda.current_stream().cuda_stream
    den.set_latent(x0)
    den.plan.run_full(st, den.emb_table[0].data_ptr())
    eps0_dev = den.model.download(den.model.latent_to_bcthw(st, den.plan.eps))
    x_allkey_dev, S_dev = den.calibrate(x0)
    nk = target_keys(K)
    gamma = gamma_for_target(S_dev, nk)                  # the bench's gamma (bench.py)
    G_dev = key_step_search(S_dev, gamma).key_steps
    x_rehash_dev = den.run(x0, StepSchedule(G_dev, K))
    den.trace = None
    del den
    torch.cuda.empty_cache()
    t_dev = time.perf_counter() - t0
    log(f"[{name}] device done in {t_dev:.1f} s")

    t1 = time.perf_counter()
    ref = TR.TorchRef(cfg, "cuda")
    probes = []
    x_allkey_ref, S_ref, eps = TR.run_full(ref, eps_steps=(0,), probe_sink=probes)
    # how much of the S error bf16 storage of the probe alone would explain: the oracle's own
    # fp64 probes rounded to bf16, Gram in fp64
    S_ref_bf16probe = TR.similarity_from_gram(TR.gram([p.to(torch.bfloat16).double() for p in probes]))
    del probes
    eps0_ref = eps[0].cpu().numpy()
    x_allkey_ref = x_allkey_ref.cpu().numpy()
    G_ref = key_step_search(S_ref, gamma).key_steps
    gamma_ref = gamma_for_target(S_ref, nk)
    G_ref_target = key_step_search(S_ref, gamma_ref).key_steps
    x_rehash_ref = TR.run_rehash(ref, G_ref).cpu().numpy()
    t_ref = time.perf_counter() - t1
    log(f"[{name}] oracle done in {t_ref:.1f} s")

    s_err = float(np.abs(S_dev.values - S_ref).max())
    fixed = {}
    for g in (0.90, 0.93, 0.95, 0.97):
        sr, sd = key_step_search(S_ref, g), key_step_search(S_dev.values, g)
        fixed[f"{g:.2f}"] = {"G_ref": list(sr.key_steps), "G_dev": list(sd.key_steps),
                             "match": list(sr.key_steps) == list(sd.key_steps), "margin_ref": sr.margin}
    x0d = x0.astype(np.float64)
    rec = {
        "config": name, "unet": CONFIGS[name], "K": K, "target_keys": nk,
        "eps0_max_rel": rel(eps0_dev, eps0_ref), "eps0_max_abs": float(np.abs(eps0_dev - eps0_ref).max()),
        "eps0_rms_rel": float(np.sqrt(np.mean((eps0_dev - eps0_ref) ** 2) / np.mean(eps0_ref ** 2))),
        "update_allkey_max_rel": rel(x_allkey_dev - x0d, x_allkey_ref - x0d),
        "update_rehash_max_rel": rel(x_rehash_dev - x0d, x_rehash_ref - x0d),
        "x_allkey_max_rel": rel(x_allkey_dev, x_allkey_ref),
        "x_allkey_max_abs": float(np.abs(x_allkey_dev - x_allkey_ref).max()),
        "s_err": s_err,
        "s_err_bf16_probe_storage_only": float(np.abs(S_ref_bf16probe - S_ref).max()),
        "fixed_gamma": fixed,
        "gamma": gamma, "G_dev": list(G_dev), "G_ref": list(G_ref), "G_match": list(G_dev) == list(G_ref),
        "margin_ref": a1_margin(S_ref, gamma), "margin_dev": a1_margin(S_dev.values, gamma),
        "gamma_ref_target": gamma_ref, "G_ref_target": list(G_ref_target),
        "G_target_match": list(G_ref_target) == list(G_dev),
        "x_rehash_max_rel": rel(x_rehash_dev, x_rehash_ref),
        "x_rehash_max_abs": float(np.abs(x_rehash_dev - x_rehash_ref).max()),
        "S_dev": S_dev.values.tolist(), "S_ref": S_ref.tolist(),
        "oracle": "oracle/torch_ref.py (torch fp64 on the same GPU, reference-mode walk)",
        "device_s": round(t_dev, 1), "oracle_s": round(t_ref, 1),
    }
    return rec


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    from paper_2411_01171_b200.build import build
    build()
    rec = run(a.config, log=lambda m: print(m, file=sys.stderr, flush=True))
    short = {k: v for k, v in rec.items() if k not in ("S_dev", "S_ref")}
    print(json.dumps(short), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rec, fh, indent=1)


if __name__ == "__main__":
    main()
