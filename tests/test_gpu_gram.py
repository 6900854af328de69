"""Step Rehash similarity kernel (sf_gram_bf16, csrc/gram.cu) vs an fp64 torch Gram.  -m gpu.

The kernel reads every probe element once (bf16 mma.sync, exact products, the
tensor core's fp32 accumulation over 256-element partials, flushed to fp64, fixed-order
combine).  Bar against the fp64 Gram of the same bf16 probes (kernels.py:375-390
accumulates in fp64): every Gram entry within 1e-6 of the largest, every cosine within
1e-6 (the C3 schedule's decision margin is 3.7e-4); bit-identical across runs; K from 1
to 40 (two 32-probe blocks), n with a ragged n % 32 tail.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_01171_b200.build import build  # noqa: E402
from paper_2411_01171_b200.rehash import gram_partial  # noqa: E402

build()


@pytest.mark.parametrize("K,n", [(1, 4096), (3, 1000003), (25, 1 << 20), (25, 33 * 16 + 7), (32, 65536), (40, 300017)])
def test_gram_matches_fp64(K, n):
    g = torch.Generator(device="cuda").manual_seed(K * 7 + n)
    base = torch.randn(n, device="cuda", generator=g)
    # nearly parallel probes, like consecutive denoising steps
    probes = [(base + 0.05 * (i + 1) * torch.randn(n, device="cuda", generator=g)).to(torch.bfloat16)
              for i in range(K)]
    G = gram_partial(probes)
    P = torch.stack([p.double() for p in probes])
    R = (P @ P.T).cpu().numpy()
    err = np.abs(G - R) / np.abs(R).max()
    assert err.max() <= 1e-6, err.max()
    d, dr = np.sqrt(np.diag(G)), np.sqrt(np.diag(R))
    assert np.abs(G / np.outer(d, d) - R / np.outer(dr, dr)).max() <= 1e-6
    assert np.array_equal(G, G.T)
    assert np.array_equal(gram_partial(probes), G)


def test_gram_bandwidth_c3_shape():
    """One 25-probe map at SVD-XT shape (73.7M elements each): report the achieved HBM rate."""
    n = 25 * 320 * 72 * 128
    probes = torch.randn(25, n, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    lst = [probes[i] for i in range(25)]
    gram_partial(lst)
    torch.cuda.synchronize()
    from paper_2411_01171_b200 import _native as N
    ptrs = torch.tensor([p.data_ptr() for p in lst], dtype=torch.int64, device="cuda")
    work = torch.empty(N.query("sf_gram_workspace", 25, n), dtype=torch.uint8, device="cuda")
    out = torch.empty(625, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        N.call("sf_gram_bf16", ptrs.data_ptr(), 25, n, work.data_ptr(), out.data_ptr(), st)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    gbs = 25 * n * 2 / (ms * 1e6)
    print(f"gram 25 x {n}: {ms:.3f} ms, {gbs:.0f} GB/s")
    assert gbs > 4000
