"""Race stress for the tcgen05 temporal attention kernels: the fused op (sf_temporal_attention_fused)
and the long-clip core (sf_temporal_attention_core at T > 32), each run many times at several
shapes with a 1 GiB HBM copy on a second stream (slow stores / loads expose missing waits,
profiles finding 30); every repetition must equal the first bit for bit.

    python tools/stress_tattn.py [--reps 50]
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
from paper_2411_01171_b200.device import Rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda")
    torch.manual_seed(0)
    hog_src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    hog_dst = torch.empty_like(hog_src)
    hog = torch.cuda.Stream()
    main_st = torch.cuda.current_stream()
    st = main_st.cuda_stream
    report = {}
    cases = [("fused", 1, 25, 600, 320), ("fused", 1, 25, 9216, 320), ("fused", 2, 64, 300, 320),
             ("fused", 1, 16, 130, 128), ("core", 1, 64, 2304, 640), ("core", 2, 48, 90, 1280)]
    for kind, B, T, P, C in cases:
        rows = B * T * P
        if kind == "fused":
            x = (torch.randn(rows, C, device=dev)).to(torch.bfloat16)
            res = (torch.randn(rows, C, device=dev)).to(torch.bfloat16)
            ws = [torch.randn(C, C, dtype=torch.float64) / C ** 0.5 for _ in range(4)]
            wf = D.temporal_fused_weights(*(w.numpy() for w in ws), dev)

            def launch(out):
                N.call("sf_temporal_attention_fused", Rows(x, 0, P).view(), wf.data_ptr(), Rows(res, 0, P).view(),
                       Rows(out, 0, P).view(), B, T, P, C, st)
        else:
            qkv = (torch.randn(rows, 3 * C, device=dev) * 1.5).to(torch.bfloat16)

            def launch(out):
                N.call("sf_temporal_attention_core", Rows(qkv, 0, P).view(), C, 2 * C, Rows(out, 0, P).view(), B,
                       T, P, C, C ** -0.5, st)
        ref = torch.empty(rows, C, dtype=torch.bfloat16, device=dev)
        launch(ref)
        torch.cuda.synchronize()
        bad = 0
        out = torch.empty_like(ref)
        for _ in range(a.reps):
            out.fill_(float("nan"))
            ev = torch.cuda.Event()
            ev.record(main_st)
            hog.wait_event(ev)
            with torch.cuda.stream(hog):
                hog_dst.copy_(hog_src)
            launch(out)
            torch.cuda.synchronize()
            bad += not torch.equal(out, ref)
        report[f"{kind} B={B} T={T} P={P} C={C}"] = f"{bad} of {a.reps} differ"
        print(kind, B, T, P, C, bad, flush=True)
    print(json.dumps(report))


if __name__ == "__main__":
    main()
