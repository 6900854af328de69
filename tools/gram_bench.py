"""Step Rehash similarity kernel at SVD-XT shape: 25 bf16 probes of 73.7M elements (one K x K map).

    python tools/gram_bench.py [reps]

Prints the device time per map and the achieved HBM rate (K * n * 2 bytes read per map).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200.build import build  # noqa: E402

build()
N.load()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
K, n = 25, 25 * 320 * 72 * 128
probes = torch.randn(K, n, device="cuda").to(torch.bfloat16)
ptrs = torch.tensor([probes[i].data_ptr() for i in range(K)], dtype=torch.int64, device="cuda")
work = torch.empty(N.query("sf_gram_workspace", K, n), dtype=torch.uint8, device="cuda")
out = torch.empty(K * K, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
N.call("sf_gram_bf16", ptrs.data_ptr(), K, n, work.data_ptr(), out.data_ptr(), st)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    N.call("sf_gram_bf16", ptrs.data_ptr(), K, n, work.data_ptr(), out.data_ptr(), st)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(f"gram K={K} n={n}: {ms:.3f} ms per map, {K * n * 2 / (ms * 1e6):.0f} GB/s")
