"""Isolate the out_conv slice-stream race (tools/race_locate.py): the tap-wise 3x3 convolution
(plain GEMM into fp32 per-tap rows + shifted tap sum, device.conv2d_tapwise) of consecutive frame
slices on s streams with s scratch copies, against the same slices on one stream.

    python tools/race_tapwise.py [--streams 4] [--reps 20] [--stage gemm|tapsum|both] [--backend 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01171_b200.build import build  # noqa: E402

build()
from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200 import device as D  # noqa: E402
from paper_2411_01171_b200.executor import balanced  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--backend", type=int, default=N.GEMM_NO_PAIR)
    ap.add_argument("--frames", type=int, default=25)
    ap.add_argument("--k", type=int, default=7)
    ap.add_argument("--hog-mb", type=int, default=0, help="HBM copy on a fifth stream during the slices")
    a = ap.parse_args()
    H, W, C, CO = 72, 128, 320, 4
    HW = H * W
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    src = torch.randn(a.frames * HW, C, device=dev, generator=g).to(torch.bfloat16)
    prm = {"w_taps": (torch.randn(9 * CO, C, device=dev, generator=g) * 0.05).to(torch.bfloat16),
           "bias": torch.randn(CO, device=dev, generator=g)}
    slices = balanced(a.frames, a.k)
    fmax = max(b - s for s, b in slices)
    S = a.streams
    xs = [torch.empty(fmax * HW, C, device=dev, dtype=torch.bfloat16) for _ in range(S)]
    ys = [torch.empty(fmax * HW, 9 * CO, device=dev, dtype=torch.float32) for _ in range(S)]
    out = torch.empty(a.frames * HW, CO, device=dev, dtype=torch.float32)
    streams = [torch.cuda.Stream() for _ in range(S)]
    hog_stream = torch.cuda.Stream()
    if a.hog_mb:
        hog_src = torch.empty(a.hog_mb << 20, dtype=torch.uint8, device=dev)
        hog_dst = torch.empty_like(hog_src)

    def run(nstreams):
        out.fill_(float("nan"))
        main = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(main)
        for s in streams:
            s.wait_event(ev)
        if a.hog_mb and nstreams > 1:
            hog_stream.wait_event(ev)
            with torch.cuda.stream(hog_stream):
                for _ in range(4):
                    hog_dst.copy_(hog_src)
        for si, (f0, f1) in enumerate(slices):
            k = si % nstreams
            st = streams[k].cuda_stream if nstreams > 1 else main.cuda_stream
            nf = f1 - f0
            # the producer of the conv input (GroupNorm apply in the real group): a row copy
            N.call("sf_copy_rows", D.Rows(src, f0 * HW, HW).view(), D.Rows(xs[k], 0, HW).view(), nf, HW, C, st)
            D.conv2d_tapwise(st, D.Rows(xs[k], 0, HW), D.Rows(out, f0 * HW, HW), nf, H, W, C, CO, prm, ys[k],
                             a.backend)
        for s in streams + [hog_stream]:
            e = torch.cuda.Event()
            e.record(s)
            main.wait_event(e)
        torch.cuda.synchronize()
        return out.clone()

    ref = run(1)
    assert torch.isfinite(ref).all()
    bad = 0
    for r in range(a.reps):
        got = run(S)
        if not torch.equal(got, ref):
            bad += 1
            d = (got != ref).any(dim=1).nonzero().flatten()
            print(f"rep {r}: {d.numel()} rows differ, frames {sorted(set((d // HW).tolist()))}", flush=True)
    print(f"streams={S} backend={a.backend}: {bad} of {a.reps} runs differ", flush=True)


if __name__ == "__main__":
    main()
