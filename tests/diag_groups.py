"""Per-group local error of the device path against the fp64 oracle (diagnostic, test infrastructure).

    python tests/diag_groups.py c2 [--out FILE]

One oracle evaluation at s = 0 (torch fp64, every value kept); then every
operator group and every ungrouped node runs ALONE on the device from the
oracle's own input (``executor.execute_group`` / ``ops.apply_kernel``), and
its output is compared with the oracle's: the error that unit adds by
itself (max |dev - ref| / max |ref|), plus the attention logit range.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np
import torch

from oracle import torch_ref as TR
from paper_2411_01171_b200 import ops
from paper_2411_01171_b200.executor import execute_group
from paper_2411_01171_b200.grouping import group_operators
from paper_2411_01171_b200.slicer import default_temporal_config
from paper_2411_01171_b200.tensor import Tensor5D
from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from parity_sd import CONFIGS  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    from paper_2411_01171_b200.build import build
    build()
    cfg = UNetConfig(**CONFIGS[a.config])
    graph, w64 = build_toy_unet(cfg)
    ref = TR.TorchRef(cfg, "cuda", graph, w64)
    feeds = {"x": ref.initial_latent(), "step_emb": ref.step_emb(0)}
    vals = dict(feeds)
    for nid in ref.topo:
        n = graph.nodes[nid]
        vals[nid] = TR.apply(n.kind, [vals[r] for r in n.inputs], ref.W.get(nid), n.attrs)
    gg = group_operators(graph, cfg.frames, default_temporal_config(cfg.height, cfg.width))
    w32 = w64.astype(np.float32)
    rows = []
    for kind, r in gg.schedule:
        if kind == "group":
            grp = gg.groups[r]
            xin = vals[grp.head_input].float().cpu().numpy()
            y = execute_group(grp, Tensor5D(xin), w32).data
            out = grp.tail
            label = grp.label
        else:
            n = graph.nodes[r]
            xs = [Tensor5D(vals[i].float().cpu().numpy()) for i in n.inputs]
            y = ops.apply_kernel(n.kind, xs, w32.get(n.param_ref) if n.param_ref else None, n.attrs).data
            out, label = r, n.label
        yr = vals[out].cpu().numpy()
        err = float(np.abs(y - yr).max() / np.abs(yr).max())
        rows.append({"unit": label, "rel": err, "max_ref": float(np.abs(yr).max())})
        print(f"{err:9.2e}  {label}", flush=True)
    # attention logit ranges (spatial: first frame)
    logits = {}
    for nid in ref.topo:
        n = graph.nodes[nid]
        if n.kind.value.endswith("attention"):
            x = vals[n.inputs[0]]
            B, T, C, H, W = x.shape
            if n.kind.value == "spatial_attention":
                tok = x[0, :1].reshape(1, C, H * W).transpose(1, 2)
            else:
                tok = x.permute(0, 3, 4, 1, 2).reshape(-1, T, C)[:64]
            q, k = tok @ ref.W[nid]["wq"], tok @ ref.W[nid]["wk"]
            s = (q @ k.transpose(1, 2)) / C ** 0.5
            logits[n.label] = [float(s.min()), float(s.max())]
    print(json.dumps(logits, indent=1))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"config": a.config, "units": rows, "logits": logits}, fh, indent=1)


if __name__ == "__main__":
    main()
