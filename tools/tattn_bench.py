"""Time sf_temporal_attention_core alone (CUDA events) at a level's shape, for tuning:

    python tools/tattn_bench.py 25 9216 320      # T, pixels, C   (C3 L0)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200.device import Rows  # noqa: E402


def main():
    T, P, C = (int(v) for v in sys.argv[1:4])
    reps = 50
    dev = torch.device("cuda")
    st = torch.cuda.current_stream().cuda_stream
    qkv = torch.randn(T * P, 3 * C, device=dev).to(torch.bfloat16)
    out = torch.empty(T * P, C, device=dev, dtype=torch.bfloat16)

    def run():
        N.call("sf_temporal_attention_core", Rows(qkv, 0, P).view(), C, 2 * C, Rows(out, 0, P).view(), 1, T, P, C,
               C ** -0.5, st)
    run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        run()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    by = qkv.numel() * 2 + out.numel() * 2
    print(f"temporal attention T={T} P={P} C={C}: {ms * 1e3:.1f} us  {by / ms / 1e6:.0f} GB/s algorithmic")


if __name__ == "__main__":
    main()
