"""sf_gemm backends vs a torch fp32 reference of the same contraction (B200 only).

Every implicit-GEMM mode (plain rows, 3x3 conv im2col, 3-tap temporal conv,
batched attention GEMMs, two-level row views, fused epilogue) is run on the
tcgen05/TMA backend and on the mma.sync backend and compared with
torch.float32 math on the same bf16-rounded operands.  Tolerance: max_rel
<= 1e-2 (fp32 accumulation, one bf16 rounding of the output).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.nn.functional as F  # noqa: E402

from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200 import device as D  # noqa: E402
from paper_2411_01171_b200.build import build  # noqa: E402
from paper_2411_01171_b200.device import Rows  # noqa: E402

build()
dev = torch.device("cuda")


def rel(a, b):
    return float((a.float() - b.float()).abs().max() / b.float().abs().max())


def rnd(*shape, scale=1.0):
    return (torch.randn(*shape, device=dev) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("backend", [1, 2])
@pytest.mark.parametrize("M,K,Nn", [(1000, 320, 320), (4096, 640, 1920), (256, 1280, 1280), (77, 64, 96)])
def test_plain(backend, M, K, Nn):
    torch.manual_seed(0)
    a, w = rnd(M, K), rnd(Nn, K, scale=K ** -0.5)
    bias = torch.randn(Nn, device=dev)
    res = rnd(M, Nn)
    out = torch.empty(M, Nn, dtype=torch.bfloat16, device=dev)
    args = D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=M, cin=K, n=Nn,
                  a=Rows(a), w=w, out=Rows(out), bias=bias, res=Rows(res), act=N.ACT_SILU, backend=backend)
    assert N.query("sf_gemm_backend", args) == backend
    ref = F.silu(a.float() @ w.float().T + bias) + res.float()
    assert rel(out, ref) <= 1e-2


@pytest.mark.parametrize("backend", [1, 2])
@pytest.mark.parametrize("F_,H,W,C,Co", [(3, 72, 128, 64, 320), (2, 36, 64, 320, 640), (2, 9, 16, 128, 160),
                                         (1, 16, 16, 64, 64)])
def test_conv3x3(backend, F_, H, W, C, Co):
    torch.manual_seed(1)
    x = rnd(F_, H, W, C)
    w = rnd(Co, C, 3, 3, scale=(9 * C) ** -0.5)
    wk = w.permute(0, 2, 3, 1).reshape(Co, 9 * C).contiguous()
    bias = torch.randn(Co, device=dev)
    emb = torch.randn(Co, device=dev)
    out = torch.empty(F_ * H * W, Co, dtype=torch.bfloat16, device=dev)
    D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_CONV3X3, n_outer=F_, n_inner=H * W, H=H, W=W, cin=C,
           n=Co, a=Rows(x.view(-1, C), 0, H * W), w=wk, out=Rows(out, 0, H * W), bias=bias, rowbias=emb,
           backend=backend)
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float(), bias, padding=1) + emb[None, :, None, None]
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Co)
    assert rel(out, ref) <= 1e-2


@pytest.mark.parametrize("F_,H,W,C,Co", [(25, 9, 16, 128, 256), (5, 18, 32, 64, 128), (10, 9, 16, 64, 64),
                                         (3, 9, 16, 64, 128), (7, 4, 16, 64, 64)])
def test_conv3x3_tail_tiles(F_, H, W, C, Co):
    """Frames whose height is not a multiple of the tile height: the leftover rows of several frames
    share one tile (tcgen05 path), with residual + per-frame bias in the epilogue."""
    torch.manual_seed(6)
    x = rnd(F_, H, W, C)
    w = rnd(Co, C, 3, 3, scale=(9 * C) ** -0.5)
    wk = w.permute(0, 2, 3, 1).reshape(Co, 9 * C).contiguous()
    bias = torch.randn(Co, device=dev)
    emb = torch.randn(F_, Co, device=dev)
    res = rnd(F_ * H * W, Co)
    out = torch.empty(F_ * H * W, Co, dtype=torch.bfloat16, device=dev)
    args = D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_CONV3X3, n_outer=F_, n_inner=H * W, H=H,
                  W=W, cin=C, n=Co, a=Rows(x.view(-1, C), 0, H * W), w=wk, out=Rows(out, 0, H * W), bias=bias,
                  rowbias=emb, rowbias_stride=Co, res=Rows(res, 0, H * W), backend=2)
    assert N.query("sf_gemm_backend", args) == 2
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float(), bias, padding=1) + emb[:, :, None, None]
    ref = ref.permute(0, 2, 3, 1).reshape(-1, Co) + res.float()
    assert rel(out, ref) <= 1e-2
    # fp32 direct-store epilogue over the same tiling
    out32 = torch.empty(F_ * H * W, Co, dtype=torch.float32, device=dev)
    D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_CONV3X3, n_outer=F_, n_inner=H * W, H=H, W=W,
           cin=C, n=Co, a=Rows(x.view(-1, C), 0, H * W), w=wk, out=Rows(out32, 0, H * W), out_fp32=True,
           bias=bias, backend=2)
    ref32 = F.conv2d(x.float().permute(0, 3, 1, 2), w.float(), bias, padding=1).permute(0, 2, 3, 1)
    assert rel(out32, ref32.reshape(-1, Co)) <= 1e-2


@pytest.mark.parametrize("backend", [1, 2])
@pytest.mark.parametrize("F_,H,W,C,Co", [(3, 72, 128, 320, 4), (2, 9, 13, 64, 8), (1, 5, 7, 128, 3)])
def test_conv3x3_tapwise(backend, F_, H, W, C, Co):
    """out_conv path: per-tap projection GEMM + shifted sum, fp32 out, vs torch conv2d."""
    torch.manual_seed(5)
    x = rnd(F_, H, W, C)
    w = rnd(Co, C, 3, 3, scale=(9 * C) ** -0.5)
    bias = torch.randn(Co, device=dev)
    prm = {"w_taps": w.permute(2, 3, 0, 1).reshape(9 * Co, C).contiguous(), "bias": bias}
    ybuf = torch.empty(F_ * H * W, 9 * Co, dtype=torch.float32, device=dev)
    out = torch.empty(F_ * H * W, Co, dtype=torch.float32, device=dev)
    D.conv2d_tapwise(torch.cuda.current_stream().cuda_stream, Rows(x.view(-1, C), 0, H * W), Rows(out, 0, H * W),
                     F_, H, W, C, Co, prm, ybuf, backend=backend)
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float(), bias, padding=1).permute(0, 2, 3, 1).reshape(-1, Co)
    assert rel(out, ref) <= 1e-3


@pytest.mark.parametrize("backend", [2, 2 | N.GEMM_NO_PAIR])
def test_fp32_epilogue_concurrent_streams(backend):
    """fp32-output GEMMs with one 32-column staging chunk per column half (N = 36 -> BN = 64,
    the out_conv's tap projection) on four streams at once, next to a 1 GiB HBM copy on a fifth
    stream, 20 times, against the same GEMMs run one after another: bit-identical.  Regression
    for the staging-buffer reuse that let a tile overwrite the chunk its previous tile's TMA
    store was still reading (profiles finding 30): with the copy slowing the stores, the old
    kernel corrupted rows in 34-38 of 40 such runs (tools/race_tapwise.py --hog-mb)."""
    torch.manual_seed(9)
    HW, C, Nn, S, nf = 9216, 320, 36, 4, 4
    xs = [rnd(nf * HW, C) for _ in range(S)]
    w = rnd(Nn, C, scale=C ** -0.5)
    outs = [torch.empty(nf * HW, Nn, dtype=torch.float32, device=dev) for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    hog = torch.cuda.Stream()
    hog_src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    hog_dst = torch.empty_like(hog_src)

    def launch(k, st):
        D.gemm(st, mode=N.GEMM_PLAIN, n_outer=nf, n_inner=HW, cin=C, n=Nn, a=Rows(xs[k], 0, HW), w=w,
               out=Rows(outs[k], 0, HW), out_fp32=True, backend=backend)

    main = torch.cuda.current_stream()
    for k in range(S):
        launch(k, main.cuda_stream)
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]
    assert rel(ref[0], xs[0].float() @ w.float().t()) <= 1e-2
    for _ in range(20):
        for o in outs:
            o.fill_(float("nan"))
        ev = torch.cuda.Event()
        ev.record(main)
        hog.wait_event(ev)
        with torch.cuda.stream(hog):
            hog_dst.copy_(hog_src)
            hog_dst.copy_(hog_src)
        for k, s in enumerate(streams):
            s.wait_event(ev)
            launch(k, s.cuda_stream)
        torch.cuda.synchronize()
        assert all(torch.equal(o, r) for o, r in zip(outs, ref))


@pytest.mark.parametrize("backend", [1, 2])
@pytest.mark.parametrize("B,T,P,C,band", [(1, 25, 576, 320, None), (1, 25, 144, 128, None), (2, 8, 64, 64, None),
                                          (1, 16, 1024, 64, (100, 612))])
def test_tconv(backend, B, T, P, C, band):
    torch.manual_seed(2)
    x = rnd(B * T * P, C)
    w = rnd(C, C, 3, scale=(3 * C) ** -0.5)
    wk = w.permute(0, 2, 1).reshape(C, 3 * C).contiguous()
    res = rnd(B * T * P, C)
    out = torch.zeros(B * T * P, C, dtype=torch.bfloat16, device=dev)
    p0, p1 = band if band else (0, P)
    D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_TCONV3, n_outer=B * T, n_inner=p1 - p0, T=T, cin=C,
           n=C, a=Rows(x, p0, P), w=wk, out=Rows(out, p0, P), res=Rows(res, p0, P), backend=backend)
    xc = x.float().view(B, T, P, C).permute(0, 2, 3, 1).reshape(B * P, C, T)
    ref = F.conv1d(xc, w.float(), padding=1).reshape(B, P, C, T).permute(0, 3, 1, 2).reshape(-1, C) + res.float()
    got = out.view(B, T, P, C)[:, :, p0:p1].reshape(-1, C)
    assert rel(got, ref.view(B, T, P, C)[:, :, p0:p1].reshape(-1, C)) <= 1e-2


@pytest.mark.parametrize("backend", [1, 2])
@pytest.mark.parametrize("Fr,HW,C", [(2, 2304, 320), (3, 576, 640)])
def test_batched_scores(backend, Fr, HW, C):
    """S = q k^T * alpha per frame straight out of a fused qkv buffer, fp32 out."""
    torch.manual_seed(3)
    qkv = rnd(Fr * HW, 3 * C)
    s = torch.empty(Fr * HW, HW, dtype=torch.float32, device=dev)
    D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=HW, cin=C, n=HW,
           a=Rows(qkv), w=qkv, w_ptr=qkv.data_ptr() + C * 2, w_ld=3 * C, out=Rows(s), out_fp32=True, batch=Fr,
           a_bstride=HW * 3 * C, w_bstride=HW * 3 * C, out_bstride=HW * HW, alpha=0.05, backend=backend)
    q = qkv.float().view(Fr, HW, 3 * C)[..., :C]
    k = qkv.float().view(Fr, HW, 3 * C)[..., C:2 * C]
    ref = (q @ k.transpose(1, 2) * 0.05).reshape(-1, HW)
    assert rel(s, ref) <= 1e-2


@pytest.mark.parametrize("Fr,HW,C", [(2, 9216, 320), (3, 2304, 320), (2, 200, 320), (2, 576, 128), (1, 1000, 192),
                                     (2, 4096, 256), (1, 1000, 128), (2, 296, 256), (1, 136, 320)])
def test_flash_core(Fr, HW, C):
    """Fused tcgen05 attention core vs torch softmax(q k^T / sqrt(C)) v (fp32 math)."""
    if not N.query("sf_flash_supported", HW, C):
        pytest.skip("shape not supported by the fused core")
    torch.manual_seed(4)
    qkv = rnd(Fr * HW, 2 * C, scale=1.5)
    v = rnd(Fr, HW, C)
    vt = v.transpose(1, 2).contiguous()
    o = torch.empty(Fr * HW, C, dtype=torch.bfloat16, device=dev)
    N.call("sf_spatial_attention_core", Rows(qkv, 0, HW).view(), Rows(qkv, 0, HW, C).view(), vt.data_ptr(),
           Rows(o, 0, HW).view(), Fr, HW, C, C ** -0.5, torch.cuda.current_stream().cuda_stream)
    q = qkv.float().view(Fr, HW, 2 * C)[..., :C]
    k = qkv.float().view(Fr, HW, 2 * C)[..., C:]
    ref = torch.softmax(q @ k.transpose(1, 2) * C ** -0.5, dim=-1) @ v.float()
    assert rel(o.view(Fr, HW, C), ref) <= 1.5e-2


@pytest.mark.parametrize("B,T,P,C", [(1, 25, 300, 320), (2, 8, 64, 32), (1, 32, 50, 640), (1, 64, 20, 64),
                                     (1, 16, 40, 1280), (1, 3, 10, 24),
                                     # one warp per pixel (many pixels) and the channel-split block per
                                     # pixel (few pixels: C3 L2 / L3, uneven chunk counts, B = 2)
                                     (1, 25, 2400, 320), (1, 25, 576, 1280), (1, 25, 144, 1280),
                                     (1, 25, 200, 192), (2, 25, 300, 320),
                                     # 32 < T <= 128: the tcgen05 core (BASELINE C4: T = 64 at C = 640 / 1280)
                                     (1, 64, 300, 640), (2, 64, 77, 1280), (1, 48, 90, 320), (1, 100, 9, 128),
                                     (1, 128, 5, 64), (1, 64, 2304, 640)])
def test_temporal_core(B, T, P, C):
    """Per-pixel attention over T frames vs torch (rows o = b*T+t, i = pixel)."""
    torch.manual_seed(5)
    qkv = rnd(B * T * P, 3 * C, scale=1.5)
    o = torch.empty(B * T * P, C, dtype=torch.bfloat16, device=dev)
    N.call("sf_temporal_attention_core", Rows(qkv, 0, P).view(), C, 2 * C, Rows(o, 0, P).view(), B, T, P, C,
           C ** -0.5, torch.cuda.current_stream().cuda_stream)
    x = qkv.float().view(B, T, P, 3 * C).permute(0, 2, 1, 3)
    q, k, v = x[..., :C], x[..., C:2 * C], x[..., 2 * C:]
    ref = (torch.softmax(q @ k.transpose(-1, -2) * C ** -0.5, dim=-1) @ v).permute(0, 2, 1, 3).reshape(-1, C)
    assert rel(o, ref) <= 1.5e-2


@pytest.mark.parametrize("B,T,P,C,res,band", [
    (1, 25, 600, 320, True, None),      # C3 L0 shape: 5 pixels x 25 frames per tile
    (1, 25, 9216, 320, True, None),     # a full C3 L0 frame plane (1844 tiles, persistent grid)
    (2, 25, 333, 320, False, None),     # B = 2, ragged last tile
    (1, 64, 100, 320, True, None),      # C4: T = 64 -> 2 pixels per tile
    (1, 8, 250, 128, True, None), (1, 16, 130, 128, False, None), (1, 25, 77, 192, True, None),
    (1, 5, 90, 256, True, None), (1, 100, 7, 320, True, None),
    (1, 25, 1000, 320, True, (300, 517)),   # a pixel band of a wider plane (row stride 1000)
])
def test_temporal_attention_fused(B, T, P, C, res, band):
    """sf_temporal_attention_fused (x Mqk x^T softmax, (P x) Mvo, + residual) vs torch fp32 of the
    reference's op order: q = x Wq, k = x Wk, v = x Wv, softmax(q k^T / sqrt(C)) v Wo
    (kernels.py:276-308), per pixel over its T frames.  max_rel <= 1.5e-2 (bf16 inputs, one
    bf16 rounding of x Mqk and of P x)."""
    torch.manual_seed(11)
    x = rnd(B * T * P, C, scale=1.0)
    ws = [torch.randn(C, C, device=dev, dtype=torch.float64) * (1.0 / C ** 0.5) for _ in range(4)]
    wq, wk, wv, wo = ws
    wf = D.temporal_fused_weights(*(w.cpu().numpy() for w in ws), dev)
    r = rnd(B * T * P, C) if res else None
    out = torch.full((B * T * P, C), float("nan"), dtype=torch.bfloat16, device=dev)
    p0, p1 = band if band else (0, P)
    n = p1 - p0
    view = lambda t: Rows(t, p0, P)
    N.call("sf_temporal_attention_fused", view(x).view(), wf.data_ptr(), view(r).view() if res else N.View(0, 0, 0),
           view(out).view(), B, T, n, C, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    xs = x.double().view(B, T, P, C)[:, :, p0:p1].permute(0, 2, 1, 3)      # [B, n, T, C]
    q, k, v = xs @ wq, xs @ wk, xs @ wv
    ref = (torch.softmax(q @ k.transpose(-1, -2) / C ** 0.5, dim=-1) @ v) @ wo
    ref = ref.permute(0, 2, 1, 3)
    if res:
        ref = ref + r.double().view(B, T, P, C)[:, :, p0:p1]
    got = out.view(B, T, P, C)[:, :, p0:p1]
    print("fused temporal attention max_rel", rel(got, ref))
    assert rel(got, ref) <= 1.5e-2
    if band:   # rows outside the band untouched
        assert torch.isnan(out.view(B, T, P, C)[:, :, :p0].float()).all()
        assert torch.isnan(out.view(B, T, P, C)[:, :, p1:].float()).all()


@pytest.mark.parametrize("C", [8, 32, 64, 96, 128, 192, 320, 640, 960, 1280, 1920, 2560])
def test_layer_norm_widths(C):
    """sf_layer_norm vs torch layer_norm at every lanes-per-row / vectors-per-lane dispatch."""
    torch.manual_seed(7)
    rows = 333
    x = rnd(rows, C, scale=3.0)
    g = torch.randn(C, device=dev)
    b = torch.randn(C, device=dev)
    y = torch.empty_like(x)
    N.call("sf_layer_norm", Rows(x, 0, rows).view(), Rows(y, 0, rows).view(), 1, rows, C, g.data_ptr(), b.data_ptr(),
           1e-5, N.ACT_NONE, torch.cuda.current_stream().cuda_stream)
    ref = F.layer_norm(x.float(), (C,), g, b, 1e-5)
    assert rel(y, ref) <= 1e-2


@pytest.mark.parametrize("case", ["conv640", "conv640_long", "tconv640", "plain960", "plain640"])
def test_wide_pair_tiles(case):
    """Shapes the tiling model gives 224- or 192-column CTA-pair tiles (N = 640: 224 + 224 + a partial
    192-wide last tile; N = 960: five 192 tiles), with per-frame bias, SiLU and residual in the epilogue."""
    torch.manual_seed(9)
    st = torch.cuda.current_stream().cuda_stream
    if case.startswith("conv"):
        F_, H, W, Co = 25, 36, 64, 640
        C = 1920 if case == "conv640_long" else 640
        x = rnd(F_, H, W, C)
        w = rnd(Co, C, 3, 3, scale=(9 * C) ** -0.5)
        wk = w.permute(0, 2, 3, 1).reshape(Co, 9 * C).contiguous()
        bias, emb = torch.randn(Co, device=dev), torch.randn(F_, Co, device=dev)
        res = rnd(F_ * H * W, Co)
        out = torch.empty(F_ * H * W, Co, dtype=torch.bfloat16, device=dev)
        D.gemm(st, mode=N.GEMM_CONV3X3, n_outer=F_, n_inner=H * W, H=H, W=W, cin=C, n=Co,
               a=Rows(x.view(-1, C), 0, H * W), w=wk, out=Rows(out, 0, H * W), bias=bias, rowbias=emb,
               rowbias_stride=Co, act=N.ACT_SILU, res=Rows(res, 0, H * W), backend=2)
        ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float(), bias, padding=1) + emb[:, :, None, None]
        ref = F.silu(ref.permute(0, 2, 3, 1).reshape(-1, Co)) + res.float()
    elif case == "tconv640":
        T, P, C = 25, 2304, 640
        x = rnd(T * P, C)
        w = rnd(C, C, 3, scale=(3 * C) ** -0.5)
        wk = w.permute(0, 2, 1).reshape(C, 3 * C).contiguous()
        res = rnd(T * P, C)
        out = torch.empty(T * P, C, dtype=torch.bfloat16, device=dev)
        D.gemm(st, mode=N.GEMM_TCONV3, n_outer=T, n_inner=P, T=T, cin=C, n=C, a=Rows(x, 0, P), w=wk,
               out=Rows(out, 0, P), res=Rows(res, 0, P), backend=2)
        xc = x.float().view(T, P, C).permute(1, 2, 0)
        ref = F.conv1d(xc, w.float(), padding=1).permute(2, 0, 1).reshape(-1, C) + res.float()
    else:
        M, K, Nn = (230400, 320, 960) if case == "plain960" else (230400, 320, 640)
        a, w = rnd(M, K), rnd(Nn, K, scale=K ** -0.5)
        bias = torch.randn(Nn, device=dev)
        res = rnd(M, Nn)
        out = torch.empty(M, Nn, dtype=torch.bfloat16, device=dev)
        D.gemm(st, mode=N.GEMM_PLAIN, n_outer=1, n_inner=M, cin=K, n=Nn, a=Rows(a), w=w, out=Rows(out), bias=bias,
               res=Rows(res), backend=2)
        ref = a.float() @ w.float().T + bias + res.float()
    assert rel(out, ref) <= 1e-2


@pytest.mark.parametrize("frames,P,C", [(3, 9216, 320), (2, 2304, 640), (2, 576, 1280), (2, 2056, 320)])
def test_vt_projection(frames, P, C):
    """The spatial-attention v^T projection (device.spatial_attention): v^T[f] = wv^T x[f]^T with the
    weights as a shared A (a_bstride = 0) and each frame's tokens as a K-major B, batched over frames.
    Covers the 160-column tiles picked for it, including a partial last N tile (P = 2056, 9216)."""
    torch.manual_seed(0)
    x, w = rnd(frames * P, C), rnd(C, C, scale=C ** -0.5)
    out = torch.empty(frames * C, P, dtype=torch.bfloat16, device=dev)
    D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=C, cin=C, n=P,
           a=Rows(w), w=out, w_ptr=x.data_ptr(), w_ld=C, out=Rows(out, 0, 0), batch=frames, a_bstride=0,
           w_bstride=P * C, out_bstride=C * P)
    ref = torch.einsum("ck,fpk->fcp", w.float(), x.float().view(frames, P, C)).reshape(frames * C, P)
    assert rel(out, ref) <= 1e-2


@pytest.mark.parametrize("frames,P,C", [(3, 144, 1280), (2, 200, 320), (2, 72, 640)])
def test_partial_k_block_batched_pv(frames, P, C):
    """P.V with a token count that is not a multiple of 64 (C3 L3: 144 tokens) on the tcgen05 backend:
    the last 64-wide K block is partial and loads as zeros past K (TMA OOB fill)."""
    torch.manual_seed(3)
    p = torch.softmax(torch.randn(frames, P, P, device=dev), dim=-1).to(torch.bfloat16)
    vt = rnd(frames, C, P)
    o = torch.empty(frames * P, C, dtype=torch.bfloat16, device=dev)
    args = D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=P, cin=P, n=C,
                  a=Rows(p.view(frames * P, P), 0, 0), w=vt, w_ld=P, out=Rows(o, 0, 0), batch=frames,
                  a_bstride=P * P, w_bstride=C * P, out_bstride=P * C, backend=2)
    assert N.query("sf_gemm_backend", args) == 2
    ref = torch.bmm(p.float(), vt.float().transpose(1, 2)).reshape(frames * P, C)
    assert rel(o, ref) <= 1e-2


@pytest.mark.parametrize("M,K,Nn", [(1000, 200, 320), (4096, 72, 256)])
def test_plain_partial_k_block(M, K, Nn):
    """Plain GEMM + fused epilogue with K % 64 != 0 on tcgen05 (partial last K block)."""
    torch.manual_seed(4)
    a, w = rnd(M, K), rnd(Nn, K, scale=K ** -0.5)
    bias = torch.randn(Nn, device=dev)
    res = rnd(M, Nn)
    out = torch.empty(M, Nn, dtype=torch.bfloat16, device=dev)
    args = D.gemm(torch.cuda.current_stream().cuda_stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=M, cin=K, n=Nn,
                  a=Rows(a), w=w, out=Rows(out), bias=bias, res=Rows(res), act=N.ACT_SILU, backend=2)
    assert N.query("sf_gemm_backend", args) == 2
    ref = F.silu(a.float() @ w.float().T + bias) + res.float()
    assert rel(out, ref) <= 1e-2
