"""GroupNorm statistics + apply at the C3 level shapes, CUDA-event timed (median of 20, L2 flushed).

    python tools/gn_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200 import device as D  # noqa: E402
from paper_2411_01171_b200.build import build  # noqa: E402
from paper_2411_01171_b200.device import Rows  # noqa: E402

build()
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
out = {}
for (hw, C) in ((9216, 320), (9216, 960), (2304, 640), (2304, 1920), (576, 1280), (144, 1280), (576, 2560)):
    F = 25
    x = torch.randn(F * hw, C, device=dev).to(torch.bfloat16)
    y = torch.empty_like(x)
    work = torch.zeros(N.query("sf_group_norm_workspace", F, hw, C), dtype=torch.uint8, device=dev)
    mean = torch.empty(F * 32, device=dev)
    rstd = torch.empty(F * 32, device=dev)
    g = torch.ones(C, device=dev)
    b = torch.zeros(C, device=dev)
    res = {}
    for name in ("stats", "apply"):
        ts = []
        for r in range(23):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            if name == "stats":
                D.group_norm_stats(st, Rows(x, 0, hw), F, hw, C, 32, 1e-5, work, mean, rstd)
            else:
                D.group_norm_apply(st, Rows(x, 0, hw), Rows(y, 0, hw), F, hw, C, 32, mean, rstd,
                                   {"gamma": g, "beta": b}, N.ACT_SILU)
            e.record()
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        us = ts[len(ts) // 2]
        nbytes = F * hw * C * 2 * (1 if name == "stats" else 2)
        res[name] = {"us": round(us, 1), "TBps": round(nbytes / us / 1e6, 2)}
    ref = torch.nn.functional.group_norm(x.float().view(F, hw, C).permute(0, 2, 1), 32, eps=1e-5)
    got_m = mean.view(F, 32)
    xm = x.float().view(F, hw, 32, C // 32).mean(dim=(1, 3))
    res["mean_err"] = float((got_m - xm).abs().max())
    out[f"{hw}x{C}"] = res
print(json.dumps(out))
