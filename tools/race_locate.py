"""Locate a slice-stream race: run a one-stream plan and an s-stream plan of the same network in
lockstep, unit by unit, on identical inputs (the s-stream plan's arena is reset to the one-stream
plan's state before every repetition), and report every unit whose output ever differs.

    python tools/race_locate.py [--streams 4] [--reps 6] [--spatial-k 7] [--temporal-k 5]

Prints one line per differing (unit, repetition) with the value(s) and the frame / row / column
ranges that differ, then a summary JSON line.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01171_b200.build import build  # noqa: E402

build()
from paper_2411_01171_b200.executor import DeviceModel, ExecConfig  # noqa: E402
from paper_2411_01171_b200.harness import initial_latent  # noqa: E402
from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet, step_embedding_tensor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--spatial-k", type=int, default=7)
    ap.add_argument("--temporal-k", type=int, default=5)
    ap.add_argument("--backend", type=int, default=0)
    a = ap.parse_args()
    c3 = UNetConfig(channels=4, frames=25, height=72, width=128, base_channels=320, norm_groups=32, steps=25)
    g, w = build_toy_unet(c3)
    mk = lambda s, dw=None: DeviceModel(g, w, ExecConfig(spatial_k=a.spatial_k, temporal_k=a.temporal_k,
                                                         slice_streams=s, gemm_backend=a.backend),
                                        device_weights=dw)
    A = mk(1)
    B = mk(a.streams, A.dw)
    assert A.plan.arena_bytes == B.plan.arena_bytes
    st = torch.cuda.current_stream().cuda_stream
    x = initial_latent(c3)
    se = step_embedding_tensor(c3, 5).data
    emb = torch.from_numpy(se.reshape(-1, se.shape[2])[0].astype("float32").copy()).cuda()
    for m in (A, B):
        m.upload_latent(st, x)
        m.plan.emb_launch(st, emb.data_ptr())
    torch.cuda.synchronize()
    B.plan.emb_out.copy_(A.plan.emb_out)
    # value -> (byte offset in the arena, rows, cols, element size)
    base = A.plan.arena.data_ptr()
    spans = []
    for (sid, _), t in A.plan.buffers.items():
        spans.append((t.data_ptr() - base, t.numel() * t.element_size(), sid, t.shape, t.element_size()))
    bad = {}
    for i, (ua, ub) in enumerate(zip(A.plan.units, B.plan.units)):
        assert ua.label == ub.label
        for r in range(a.reps):
            B.plan.arena.copy_(A.plan.arena)
            B.plan.latent.copy_(A.plan.latent)
            torch.cuda.synchronize()
            ub.run(st)
            torch.cuda.synchronize()
            if r == 0:
                snap = A.plan.arena.clone()
                ua.run(st)
                torch.cuda.synchronize()
                ref = A.plan.arena.clone()
                A.plan.arena.copy_(snap)
            diff = (B.plan.arena != ref).nonzero().flatten()
            if diff.numel():
                lo, hi = int(diff.min()), int(diff.max())
                where = []
                for off, nb, vid, shape, es in spans:
                    if off <= hi and lo < off + nb:
                        d = diff[(diff >= off) & (diff < off + nb)] - off
                        if d.numel():
                            rows = (d // (shape[1] * es)).unique()
                            cols = ((d % (shape[1] * es)) // es).unique()
                            where.append({"value": vid, "rows": [int(rows.min()), int(rows.max())],
                                          "n_rows": int(rows.numel()), "cols": [int(cols.min()), int(cols.max())],
                                          "n_bytes": int(d.numel())})
                print(json.dumps({"unit": i, "label": ua.label, "rep": r, "diff_bytes": int(diff.numel()),
                                  "where": where}), flush=True)
                bad.setdefault(ua.label, 0)
                bad[ua.label] += 1
        A.plan.arena.copy_(ref)
    print(json.dumps({"streams": a.streams, "reps": a.reps, "units": len(A.plan.units), "bad_units": bad}))


if __name__ == "__main__":
    main()
