"""Pipeline timeline of the fused temporal attention kernel (CTA 0, -DTA_TRACE build).

    python tools/tattn_trace.py [--T 25] [--P 9216] [--C 320]

Builds a variant library with the trace compiled in (SF_LIB_OUT, not the product .so), runs one
launch at the given shape and prints, per tile of CTA 0, the SM-clock offsets of every pipeline
event of the MMA warp (role 0) and of warps 2 / 6 (column halves 0 / 1).
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT = os.path.join(ROOT, "paper_2411_01171_b200", "_variant_ta_trace.so")
NAMES = {1: "x_full", 2: "A0 issued", 3: "y_free0", 4: "A1 issued", 5: "a_st", 6: "S issued", 7: "p_full",
         9: "B issued", 10: "b_st", 11: "Y0 issued", 12: "Y1 issued",
         20: "a_full", 21: "A packed", 22: "s_full", 23: "max xchg", 24: "P stored", 25: "sums",
         26: "b_full", 27: "B packed", 28: "res loaded", 29: "y_full", 30: "Y stored"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=25)
    ap.add_argument("--P", type=int, default=9216)
    ap.add_argument("--C", type=int, default=320)
    ap.add_argument("--tiles", type=int, default=4)
    a = ap.parse_args()
    env = dict(os.environ, SF_NVCC_EXTRA="-DTA_TRACE", SF_LIB_OUT=VARIANT)
    subprocess.run([sys.executable, "-c", "from paper_2411_01171_b200.build import build; build()"], cwd=ROOT,
                   env=env, check=True, stdout=subprocess.DEVNULL)
    os.environ["SF_LIB"] = VARIANT
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01171_b200 import _native as N
    from paper_2411_01171_b200 import device as D
    from paper_2411_01171_b200.device import Rows
    lib = N.load()
    T, P, C = a.T, a.P, a.C
    dev = torch.device("cuda")
    x = torch.randn(T * P, C, device=dev).to(torch.bfloat16)
    res = torch.randn(T * P, C, device=dev).to(torch.bfloat16)
    y = torch.empty_like(x)
    ws = [torch.randn(C, C, dtype=torch.float64) / C ** 0.5 for _ in range(4)]
    wf = D.temporal_fused_weights(*(w.numpy() for w in ws), dev)
    st = torch.cuda.current_stream().cuda_stream
    host = (ctypes.c_ulonglong * (3 * 1024))()
    cnt = (ctypes.c_uint * 3)()
    for rep in range(2):   # the second launch is the traced one (warm)
        lib.sf_debug_ta_trace(host, cnt)
        N.call("sf_temporal_attention_fused", Rows(x, 0, P).view(), wf.data_ptr(), Rows(res, 0, P).view(),
               Rows(y, 0, P).view(), 1, T, P, C, st)
        torch.cuda.synchronize()
    lib.sf_debug_ta_trace(host, cnt)
    ev = []
    for role in range(3):
        for i in range(min(cnt[role], 1024)):
            v = host[role * 1024 + i]
            ev.append((v >> 8, role, v & 0xFF))
    ev.sort()
    t0 = ev[0][0]
    # split by the MMA warp's x_full events
    starts = [c for c, r, k in ev if r == 0 and k == 1]
    print(f"tiles traced: {len(starts)}; per-tile cycles: "
          f"{[starts[i + 1] - starts[i] for i in range(min(len(starts) - 1, 12))]}")
    for ti in range(1, min(a.tiles + 1, len(starts) - 1)):
        lo, hi = starts[ti], starts[ti + 1]
        print(f"--- tile {ti} ({hi - lo} cycles)")
        for c, r, k in ev:
            if lo <= c < hi:
                print(f"  {c - lo:7d}  role {r}  {NAMES.get(k, k)}")


if __name__ == "__main__":
    main()
