"""Time the spatial attention core alone at a given shape (CUDA events).

    python tools/flash_bench.py [--frames 25] [--hw 9216] [--c 320] [--reps 5]
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200.device import Rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=25)
    ap.add_argument("--hw", type=int, default=9216)
    ap.add_argument("--c", type=int, default=320)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--clocks", action="store_true", help="sample nvidia-smi SM clock / power during the loop")
    a = ap.parse_args()
    F, HW, C = a.frames, a.hw, a.c
    g = torch.Generator(device="cuda").manual_seed(0)
    qk = torch.randn(F * HW, 2 * C, device="cuda", generator=g).to(torch.bfloat16)
    vt = torch.randn(F * C, HW, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty(F * HW, C, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        N.call("sf_spatial_attention_core", Rows(qk, 0, HW).view(), Rows(qk, 0, HW, C).view(), vt.data_ptr(),
               Rows(o, 0, HW).view(), F, HW, C, 1.0 / math.sqrt(C), st)
    run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    smi = None
    if a.clocks:
        import subprocess
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                                "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    s.record()
    for _ in range(a.reps):
        run()
    e.record()
    torch.cuda.synchronize()
    if smi is not None:
        smi.terminate()
        rows = [r.split(",") for r in smi.communicate()[0].strip().splitlines() if r.count(",") == 2]
        mhz = sorted(float(r[0]) for r in rows)
        watts = sorted(float(r[1]) for r in rows)
        if rows:
            print(f"clocks: median {mhz[len(mhz) // 2]:.0f} MHz  power median {watts[len(watts) // 2]:.0f} W  "
                  f"power_cap active in {sum('Active' in r[2] and 'Not' not in r[2] for r in rows)}/{len(rows)}")
    ms = s.elapsed_time(e) / a.reps
    fl = 4.0 * F * HW * HW * C
    if os.environ.get("SF_FA_DBG"):
        import ctypes
        buf = (ctypes.c_ulonglong * 8)()
        fn = N.load().sf_fa3_debug
        if fn is not None:
            fn(buf)
            n_m, n_s = max(buf[1], 1), max(buf[4], 1)
            print(f"dbg: mma-issue loop {buf[0] / n_m / 1e3:.1f} us/CTA  softmax loop {buf[2] / n_s / 1e3:.1f} us/CTA  "
                  f"softmax+last PV {buf[3] / n_s / 1e3:.1f} us/CTA  (ctas {n_m}, {n_s})")
    print(f"flash F={F} HW={HW} C={C}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TF/s  env={os.environ.get('SF_FA_EXP', '0')}")


if __name__ == "__main__":
    main()
