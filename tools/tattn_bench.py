"""Fused temporal attention (one sf_temporal_attention_fused launch) vs the three-launch path
(QKV GEMM, mma.sync core, output GEMM + residual) at a given shape, CUDA-event timed, L2 flushed
between repetitions.

    python tools/tattn_bench.py [--T 25] [--P 9216] [--C 320] [--reps 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01171_b200.build import build  # noqa: E402

build()
from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200 import device as D  # noqa: E402
from paper_2411_01171_b200.device import Epilogue, Rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=1)
    ap.add_argument("--T", type=int, default=25)
    ap.add_argument("--P", type=int, default=9216)
    ap.add_argument("--C", type=int, default=320)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    B, T, P, C = a.B, a.T, a.P, a.C
    dev = torch.device("cuda")
    rows = B * T * P
    x = (torch.randn(rows, C, device=dev)).to(torch.bfloat16)
    res = (torch.randn(rows, C, device=dev)).to(torch.bfloat16)
    y = torch.empty_like(x)
    ws = [torch.randn(C, C, dtype=torch.float64) / C ** 0.5 for _ in range(4)]
    prm = {"wqkv": torch.cat([w.t() for w in ws[:3]]).to(dev).to(torch.bfloat16).contiguous(),
           "wo": ws[3].t().contiguous().to(dev).to(torch.bfloat16),
           "wfused": D.temporal_fused_weights(*(w.numpy() for w in ws), dev)}
    scratch = {"qkv": torch.empty(rows, 3 * C, device=dev, dtype=torch.bfloat16),
               "o": torch.empty(rows, C, device=dev, dtype=torch.bfloat16)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    epi = Epilogue(res=Rows(res, 0, P))

    def run(fused):
        os.environ["SF_TATTN_FUSED"] = "1" if fused else "0"
        D.temporal_attention(st, Rows(x, 0, P), Rows(y, 0, P), B, T, P, C, prm, epi, scratch)

    out = {}
    for fused in (True, False):
        for _ in range(3):
            run(fused)
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run(fused)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        out["fused_us" if fused else "three_launch_us"] = round(ts[len(ts) // 2], 1)
        if fused:
            yf = y.clone()
    rel = float((yf.float() - y.float()).abs().max() / y.float().abs().max())
    hbm = 3 * rows * C * 2   # x, res in; y out
    out.update({"B": B, "T": T, "P": P, "C": C, "fused_vs_three_launch_max_rel": rel,
                "fused_algorithmic_GBps": round(hbm / out["fused_us"] / 1e3, 1),
                "fused_TFLOPs_issued": round(B * -(-P // (128 // T)) * (4 * 128 * C * C + 4 * 128 * 128 * C)
                                            / out["fused_us"] / 1e6, 1)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
