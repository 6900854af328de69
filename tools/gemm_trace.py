"""Pipeline timeline of one tcgen05 GEMM launch (CTA 0), from a -DTC_TRACE build.

    SF_NVCC_EXTRA=-DTC_TRACE python -c "from paper_2411_01171_b200.build import build; build(force=True)"
    cp paper_2411_01171_b200/_sliceflow_b200.so variants/trace.so      # then rebuild the normal library
    SF_LIB=$PWD/variants/trace.so python tools/gemm_trace.py plain 230400 320 960

Events (SM clock): producer 1 = ring slot free; MMA 2 = accumulator free, 3 = stage landed,
4 = tile committed; epilogue half leaders 5 = accumulator full, 6 = TMEM released,
7 = store issued, 8 = tile done.  Prints per-tile gaps, which show where the pipeline waits.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200 import device as D  # noqa: E402
from paper_2411_01171_b200.device import Rows  # noqa: E402


def main():
    mode, m, cin, n = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    res = "--res" in sys.argv
    dev = torch.device("cuda")
    st = torch.cuda.current_stream().cuda_stream
    dims = [int(v) for v in m.split("x")]
    rows = int(np.prod(dims))
    taps = {"plain": 1, "conv": 9, "tconv": 3}[mode]
    x = torch.randn(rows, cin, device=dev).to(torch.bfloat16)
    w = (torch.randn(n, taps * cin, device=dev) * (taps * cin) ** -0.5).to(torch.bfloat16)
    out = torch.empty(rows, n, device=dev, dtype=torch.bfloat16)
    r = torch.randn(rows, n, device=dev).to(torch.bfloat16) if res else None
    kw = dict(cin=cin, n=n, w=w, bias=torch.zeros(n, device=dev))
    if mode == "plain":
        call = lambda: D.gemm(st, mode=N.GEMM_PLAIN, n_outer=1, n_inner=rows, a=Rows(x), out=Rows(out),  # noqa: E731
                              res=Rows(r) if res else None, **kw)
    elif mode == "conv":
        F_, H, W = dims
        call = lambda: D.gemm(st, mode=N.GEMM_CONV3X3, n_outer=F_, n_inner=H * W, H=H, W=W,  # noqa: E731
                              a=Rows(x, 0, H * W), out=Rows(out, 0, H * W), **kw)
    else:
        T, P = dims
        call = lambda: D.gemm(st, mode=N.GEMM_TCONV3, n_outer=T, n_inner=P, T=T, a=Rows(x, 0, P),  # noqa: E731
                              out=Rows(out, 0, P), **kw)
    lib = N.load()
    f = lib.sf_debug_gemm_trace
    f.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    buf = np.zeros((4, 4096), dtype=np.uint64)
    cnt = np.zeros(4, dtype=np.uint32)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    f(buf.ctypes.data, 4096, cnt.ctypes.data)          # reset after warm-up
    call()
    torch.cuda.synchronize()
    f(buf.ctypes.data, 4096, cnt.ctypes.data)
    ev = []
    for role in range(4):
        for v in buf[role, :min(int(cnt[role]), 4096)]:
            ev.append((int(v) >> 4, role, int(v) & 15))
    t0 = min(e[0] for e in ev)
    ev = [(t - t0, r, c) for t, r, c in ev]
    by = {c: [t for t, r, cc in ev if cc == c and (r == 2 or c < 5)] for c in range(1, 9)}
    tiles = len(by[4])
    end = max(e[0] for e in ev)
    print(f"CTA 0: {tiles} tiles, {end} cycles ({end / max(tiles, 1):.0f} per tile)")
    kit = len(by[3]) // max(tiles, 1)
    print("tile  acc_free(2)  first_stage(3)  last_stage  commit(4) | epi: full(5) released(6) stored(7) done(8)")
    for i in range(min(tiles, 14)):
        s3 = by[3][i * kit:(i + 1) * kit]
        row = [by[2][i], s3[0], s3[-1], by[4][i]]
        epi = [by[c][i] if i < len(by[c]) else -1 for c in (5, 6, 7, 8)]
        print(f"{i:4d} " + " ".join(f"{v:10d}" for v in row) + " | " + " ".join(f"{v:10d}" for v in epi))
    # aggregate: where does the MMA wait?
    stage_wait = sum(by[3][i * kit] - by[2][i] for i in range(tiles))
    acc_wait = sum(by[2][i] - by[4][i - 1] for i in range(1, tiles))
    mma_busy = sum(by[4][i] - by[3][i * kit] for i in range(tiles))
    epi_len = [by[6][i] - by[5][i] for i in range(len(by[6]))]
    store = [by[8][i] - by[6][i] for i in range(len(by[8]))]
    print(f"MMA: waiting for accumulator {acc_wait}, first stage after acc {stage_wait}, issuing {mma_busy} cycles")
    print(f"epilogue: TMEM->smem {np.mean(epi_len):.0f} cycles/tile, release->done {np.mean(store):.0f}")


if __name__ == "__main__":
    main()
