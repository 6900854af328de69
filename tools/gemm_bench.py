"""Time one sf_gemm shape in isolation (CUDA events), for tuning and ncu captures.

    python tools/gemm_bench.py plain 230400 320 320 [--res] [--reps 20]
    python tools/gemm_bench.py conv 25x72x128 320 320          # frames x H x W, cin, cout
    python tools/gemm_bench.py tconv 25x9216 320 320           # T x pixels, cin, cout
    python tools/gemm_bench.py vt 25x9216 320 320              # frames x pixels: v^T = wv^T x^T per frame

Prints time, TFLOP/s and the algorithmic HBM bytes/s (A read once, out (+res) once).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200 import device as D  # noqa: E402
from paper_2411_01171_b200.device import Rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["plain", "conv", "tconv", "vt"])
    ap.add_argument("m")
    ap.add_argument("cin", type=int)
    ap.add_argument("n", type=int)
    ap.add_argument("--res", action="store_true")
    ap.add_argument("--silu", action="store_true")
    ap.add_argument("--gn", action="store_true", help="conv: GroupNorm partials from the epilogue (gn_partial)")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda")
    st = torch.cuda.current_stream().cuda_stream
    dims = [int(v) for v in a.m.split("x")]
    rows = 1
    for d in dims:
        rows *= d
    taps = {"plain": 1, "conv": 9, "tconv": 3, "vt": 1}[a.mode]
    x = (torch.randn(rows, a.cin, device=dev)).to(torch.bfloat16)
    w = (torch.randn(a.n, taps * a.cin, device=dev) * (taps * a.cin) ** -0.5).to(torch.bfloat16)
    bias = torch.randn(a.n, device=dev)
    out = torch.empty(rows, a.n, device=dev, dtype=torch.bfloat16)
    res = torch.randn(rows, a.n, device=dev).to(torch.bfloat16) if a.res else None
    act = N.ACT_SILU if a.silu else N.ACT_NONE
    part = None
    if a.gn and a.mode == "conv":
        F_, H, W = dims
        part = torch.empty(F_ * N.query("sf_conv_gn_splits", H, W) * a.n * 2, device=dev)

    def run():
        if a.mode == "plain":
            D.gemm(st, mode=N.GEMM_PLAIN, n_outer=1, n_inner=rows, cin=a.cin, n=a.n, a=Rows(x), w=w, out=Rows(out),
                   bias=bias, act=act, res=Rows(res) if res is not None else None)
        elif a.mode == "conv":
            F_, H, W = dims
            D.gemm(st, mode=N.GEMM_CONV3X3, n_outer=F_, n_inner=H * W, H=H, W=W, cin=a.cin, n=a.n,
                   a=Rows(x, 0, H * W), w=w, out=Rows(out, 0, H * W), bias=bias, act=act,
                   res=Rows(res, 0, H * W) if res is not None else None,
                   gn_partial=part.data_ptr() if part is not None else None)
        elif a.mode == "vt":
            # the spatial-attention v^T projection (device.spatial_attention): A = wv (M = C),
            # B = the frame's tokens (K-major), batched over frames
            F_, P = dims
            D.gemm(st, mode=N.GEMM_PLAIN, n_outer=1, n_inner=a.n, cin=a.cin, n=P, a=Rows(w), w=out,
                   w_ptr=x.data_ptr(), w_ld=a.cin, out=Rows(out, 0, 0), batch=F_, a_bstride=0,
                   w_bstride=P * a.cin, out_bstride=a.n * P)
        else:
            T, P = dims
            D.gemm(st, mode=N.GEMM_TCONV3, n_outer=T, n_inner=P, T=T, cin=a.cin, n=a.n, a=Rows(x, 0, P), w=w,
                   out=Rows(out, 0, P), bias=bias, act=act, res=Rows(res, 0, P) if res is not None else None)
    run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        run()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.reps
    fl = 2.0 * rows * a.n * taps * a.cin
    by = rows * a.cin * 2 + rows * a.n * 2 * (2 if a.res else 1)
    print(f"gemm {a.mode} M={rows} K={taps * a.cin} N={a.n} res={a.res} gn={part is not None}: {ms * 1e3:.1f} us  "
          f"{fl / ms / 1e9:.1f} TF/s  {by / ms / 1e6:.0f} GB/s algorithmic")


if __name__ == "__main__":
    main()
