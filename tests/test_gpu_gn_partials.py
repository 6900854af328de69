"""GroupNorm statistics from the conv epilogue (sf_gemm gn_partial) on the B200.

The res-block GroupNorm res.norm2 reads the stored output of res.conv1 (+ step embedding)
(/root/reference/pkg/src/sliceflow/unet.py:186-193); the tcgen05 conv's epilogue emits
per-(frame, split, channel) (sum, sum sq) of exactly the bf16 values it stores, and
sf_group_norm_finalize turns them into the (frame, group) mean / rstd of _group_norm
(kernels.py:228-237).  Checked here:
  * the fused partials equal the separate pass (sf_conv_gn_partials) over the same output bit for
    bit -- same layout, same fp32 summation order -- on main tiles, tail tiles, CTA pairs and
    single-CTA tiles, with residual / per-frame bias epilogues;
  * their per-frame totals equal a torch fp64 reduction of the output (1e-5);
  * finalize(partials) equals the statistics pass (sf_group_norm_stats) on the same tensor;
  * the mma.sync backend (toy widths) produces the same partials through the pass.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_01171_b200 import _native as N  # noqa: E402
from paper_2411_01171_b200 import device as D  # noqa: E402
from paper_2411_01171_b200.build import build  # noqa: E402
from paper_2411_01171_b200.device import Rows  # noqa: E402

build()
dev = torch.device("cuda")


def rnd(*shape, scale=1.0):
    return (torch.randn(*shape, device=dev) * scale).to(torch.bfloat16)


def conv(x, wk, out, F_, H, W, C, Co, backend, part=None, res=None, emb=None, bias=None):
    st = torch.cuda.current_stream().cuda_stream
    return D.gemm(st, mode=N.GEMM_CONV3X3, n_outer=F_, n_inner=H * W, H=H, W=W, cin=C, n=Co,
                  a=Rows(x.view(-1, C), 0, H * W), w=wk, out=Rows(out, 0, H * W), bias=bias, rowbias=emb,
                  rowbias_stride=Co if emb is not None and emb.dim() == 2 else 0,
                  res=Rows(res, 0, H * W) if res is not None else None, backend=backend,
                  gn_partial=part.data_ptr() if part is not None else None)


CASES = [  # frames, H, W, cin, cout  (C3 levels, tail tiles of 64 / 16-row segments, toy widths)
    (3, 72, 128, 320, 320), (2, 36, 64, 320, 640), (5, 18, 32, 640, 1280), (25, 9, 16, 256, 1280),
    (7, 4, 16, 64, 64), (3, 9, 16, 64, 128), (4, 8, 8, 64, 192)]


@pytest.mark.parametrize("backend", [2, 2 | 4])
@pytest.mark.parametrize("F_,H,W,C,Co", CASES)
@pytest.mark.parametrize("epi", ["emb", "res"])
def test_fused_partials_equal_pass(backend, F_, H, W, C, Co, epi):
    torch.manual_seed(3)
    x = rnd(F_, H, W, C)
    wk = rnd(Co, 9 * C, scale=(9 * C) ** -0.5)
    bias = torch.randn(Co, device=dev)
    emb = torch.randn(F_, Co, device=dev) if epi == "emb" else None
    res = rnd(F_ * H * W, Co) if epi == "res" else None
    splits = N.query("sf_conv_gn_splits", H, W)
    part = torch.full((F_, splits, Co, 2), float("nan"), device=dev)
    out = torch.empty(F_ * H * W, Co, dtype=torch.bfloat16, device=dev)
    args = conv(x, wk, out, F_, H, W, C, Co, backend, part=part, res=res, emb=emb, bias=bias)
    assert N.query("sf_gemm_backend", args) == 2
    chk = torch.full_like(part, float("nan"))
    N.call("sf_conv_gn_partials", Rows(out, 0, H * W).view(), F_, H, W, Co, chk.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert not torch.isnan(part).any(), "every (frame, split, channel) written"
    assert torch.equal(part, chk), "fused partials == pass, bit for bit"
    # per-frame totals vs fp64
    y = out.double().view(F_, H * W, Co)
    tot = part.double().sum(1)
    assert torch.allclose(tot[..., 0], y.sum(1), rtol=1e-5, atol=1e-3)
    assert torch.allclose(tot[..., 1], (y * y).sum(1), rtol=1e-5, atol=1e-3)


@pytest.mark.parametrize("F_,H,W,C,Co", [(3, 72, 128, 320, 320), (5, 18, 32, 640, 1280), (25, 9, 16, 256, 1280)])
def test_finalize_matches_stats_pass(F_, H, W, C, Co):
    torch.manual_seed(4)
    groups = 32
    x = rnd(F_, H, W, C)
    wk = rnd(Co, 9 * C, scale=(9 * C) ** -0.5)
    bias = torch.randn(Co, device=dev) + 0.5
    splits = N.query("sf_conv_gn_splits", H, W)
    part = torch.empty((F_, splits, Co, 2), device=dev)
    out = torch.empty(F_ * H * W, Co, dtype=torch.bfloat16, device=dev)
    conv(x, wk, out, F_, H, W, C, Co, 0, part=part, bias=bias)
    st = torch.cuda.current_stream().cuda_stream
    m1, r1 = torch.empty(F_ * groups, device=dev), torch.empty(F_ * groups, device=dev)
    m2, r2 = torch.empty_like(m1), torch.empty_like(r1)
    N.call("sf_group_norm_finalize", part.data_ptr(), F_, splits, H * W, Co, groups, 1e-5, m1.data_ptr(),
           r1.data_ptr(), st)
    work = torch.empty((N.query("sf_group_norm_workspace", F_, H * W, Co) + 3) // 4, device=dev)
    N.call("sf_group_norm_stats", Rows(out, 0, H * W).view(), F_, H * W, Co, groups, 1e-5, work.data_ptr(),
           m2.data_ptr(), r2.data_ptr(), st)
    torch.cuda.synchronize()
    y = out.double().view(F_, H * W, groups, Co // groups)
    mu = y.mean((1, 3)).flatten()
    var = y.var((1, 3), unbiased=False).flatten()
    assert torch.allclose(m1.double(), mu, rtol=1e-5, atol=1e-6)
    assert torch.allclose(r1.double(), 1 / torch.sqrt(var + 1e-5), rtol=1e-5)
    assert torch.allclose(m1, m2, rtol=1e-5, atol=1e-6) and torch.allclose(r1, r2, rtol=1e-5)


@pytest.mark.parametrize("F_,H,W,C,Co", [(2, 16, 16, 16, 24), (3, 8, 8, 8, 8)])
def test_mma_backend_partials(F_, H, W, C, Co):
    """Toy widths run on mma.sync; sf_gemm then produces the partials with the pass."""
    torch.manual_seed(5)
    x = rnd(F_, H, W, C)
    wk = rnd(Co, 9 * C, scale=(9 * C) ** -0.5)
    splits = N.query("sf_conv_gn_splits", H, W)
    part = torch.empty((F_, splits, Co, 2), device=dev)
    out = torch.empty(F_ * H * W, Co, dtype=torch.bfloat16, device=dev)
    args = conv(x, wk, out, F_, H, W, C, Co, 0, part=part)
    assert N.query("sf_gemm_backend", args) == 1
    torch.cuda.synchronize()
    y = out.double().view(F_, H * W, Co)
    assert torch.allclose(part.double().sum(1)[..., 0], y.sum(1), rtol=1e-5, atol=1e-3)


def test_plan_uses_conv_partials_and_matches_stats_path():
    """A tcgen05-width network (base 64): the plan hands res.norm2 its statistics from the conv1
    epilogue; the denoised result stays within bf16 noise of the statistics-pass plan."""
    from paper_2411_01171_b200.executor import ExecConfig
    from paper_2411_01171_b200.harness import Denoiser, initial_latent
    from paper_2411_01171_b200.rehash import StepSchedule
    from paper_2411_01171_b200.unet import UNetConfig
    cfg = UNetConfig(channels=4, frames=4, height=16, width=16, base_channels=64, norm_groups=8, steps=3)
    x0 = initial_latent(cfg)
    sched = StepSchedule([0, 1, 2], 3)
    d1 = Denoiser(cfg, ExecConfig(gn_from_conv=True))
    a = d1.run(x0, sched)
    assert len(d1.plan.gn_feed) == 9 and len(d1.plan.gn_meta) == 16   # + 3 downsamples, 3 concats, in_conv
    d2 = Denoiser(cfg, ExecConfig(gn_from_conv=False), device_weights=d1.model.dw)
    b = d2.run(x0, sched)
    assert not d2.plan.gn_feed and not d2.plan.gn_meta
    assert np.abs(a - b).max() / np.abs(b).max() < 2e-3
    # ragged frame slices on two streams: the partial buffer is indexed by frame, so every slice
    # finalises its own frames (the conv partials do not depend on the slicing)
    d3 = Denoiser(cfg, ExecConfig(gn_from_conv=True, spatial_k=3, temporal_k=2, slice_streams=2),
                  device_weights=d1.model.dw)
    c = d3.run(x0, sched)
    assert np.abs(c - b).max() / np.abs(b).max() < 2e-3
    d4 = Denoiser(cfg, ExecConfig(gn_from_conv=True, spatial_k=3, temporal_k=2, slice_streams=1),
                  device_weights=d1.model.dw)
    assert np.array_equal(c, d4.run(x0, sched))


@pytest.mark.parametrize("F_,H,W,C,splits", [(3, 72, 128, 320, 11), (5, 36, 64, 640, 9), (4, 18, 32, 1280, 3),
                                             (2, 16, 16, 8, 2), (25, 18, 32, 2560, 3)])
def test_downsample_partials(F_, H, W, C, splits):
    """sf_downsample2x_gn: the same pooled output as sf_downsample2x, bit for bit; partials of the stored
    output and of the input (the skip it reads, written at channel offset 0 of a wider concat row)."""
    torch.manual_seed(7)
    st = torch.cuda.current_stream().cuda_stream
    x = (torch.randn(F_ * H * W, C, device=dev) * 2 + 0.5).to(torch.bfloat16)
    y0 = torch.empty(F_ * (H // 2) * (W // 2), C, dtype=torch.bfloat16, device=dev)
    y1 = torch.empty_like(y0)
    ld_in = C + 24
    po = torch.full((F_, splits, C, 2), float("nan"), device=dev)
    pi = torch.full((F_, splits, ld_in, 2), float("nan"), device=dev)
    N.call("sf_downsample2x", Rows(x, 0, H * W).view(), Rows(y0, 0, H * W // 4).view(), F_, H, W, C, st)
    N.call("sf_downsample2x_gn", Rows(x, 0, H * W).view(), Rows(y1, 0, H * W // 4).view(), F_, H, W, C, splits,
           po.data_ptr(), C, pi.data_ptr(), ld_in, st)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    assert not torch.isnan(po).any() and not torch.isnan(pi[:, :, :C]).any()
    assert torch.isnan(pi[:, :, C:]).all(), "only the skip's channel range is written"
    yd = y1.double().view(F_, -1, C)
    xd = x.double().view(F_, -1, C)
    assert torch.allclose(po.double().sum(1)[..., 0], yd.sum(1), rtol=1e-5, atol=1e-3)
    assert torch.allclose(po.double().sum(1)[..., 1], (yd * yd).sum(1), rtol=1e-5, atol=1e-3)
    assert torch.allclose(pi[:, :, :C].double().sum(1)[..., 0], xd.sum(1), rtol=1e-5, atol=1e-3)
    assert torch.allclose(pi[:, :, :C].double().sum(1)[..., 1], (xd * xd).sum(1), rtol=1e-5, atol=1e-3)


@pytest.mark.parametrize("F_,H,W,C,splits,c0", [(3, 36, 64, 640, 11, 320), (4, 9, 16, 1280, 3, 1280),
                                                (2, 8, 8, 8, 2, 16)])
def test_upsample_partials(F_, H, W, C, splits, c0):
    """sf_upsample2x_gn: the same nearest-neighbour copies as sf_upsample2x; partials = the written
    copies' sums (4 x the input's), at channel offset c0 of the concat row."""
    torch.manual_seed(8)
    st = torch.cuda.current_stream().cuda_stream
    x = (torch.randn(F_ * H * W, C, device=dev) - 0.3).to(torch.bfloat16)
    y0 = torch.empty(F_ * 4 * H * W, C, dtype=torch.bfloat16, device=dev)
    y1 = torch.empty_like(y0)
    ld = c0 + C
    pp = torch.full((F_, splits, ld, 2), float("nan"), device=dev)
    N.call("sf_upsample2x", Rows(x, 0, H * W).view(), Rows(y0, 0, 4 * H * W).view(), F_, H, W, C, st)
    N.call("sf_upsample2x_gn", Rows(x, 0, H * W).view(), Rows(y1, 0, 4 * H * W).view(), F_, H, W, C, splits,
           pp.data_ptr(), ld, c0, st)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    assert torch.isnan(pp[:, :, :c0]).all() and not torch.isnan(pp[:, :, c0:]).any()
    yd = y1.double().view(F_, -1, C)
    assert torch.allclose(pp[:, :, c0:].double().sum(1)[..., 0], yd.sum(1), rtol=1e-5, atol=1e-3)
    assert torch.allclose(pp[:, :, c0:].double().sum(1)[..., 1], (yd * yd).sum(1), rtol=1e-5, atol=1e-3)


@pytest.mark.parametrize("F_,HW,C,groups,Nn", [(3, 9216, 320, 32, 36), (2, 1000, 64, 8, 36), (4, 257, 128, 32, 48),
                                               (1, 16, 64, 4, 2), (5, 24, 384, 8, 36)])
def test_group_norm_project(F_, HW, C, groups, Nn):
    """sf_group_norm_project == the GroupNorm apply (+ SiLU, bf16 as stored) followed by an fp32 projection."""
    torch.manual_seed(9)
    st = torch.cuda.current_stream().cuda_stream
    x = (torch.randn(F_ * HW, C, device=dev) * 1.5 + 0.2).to(torch.bfloat16)
    gamma = torch.rand(C, device=dev) + 0.5
    beta = torch.randn(C, device=dev) * 0.1
    w = rnd(Nn, C, scale=C ** -0.5)
    mean = torch.empty(F_ * groups, device=dev)
    rstd = torch.empty_like(mean)
    work = torch.empty((N.query("sf_group_norm_workspace", F_, HW, C) + 3) // 4 + 1, device=dev)
    N.call("sf_group_norm_stats", Rows(x, 0, HW).view(), F_, HW, C, groups, 1e-5, work.data_ptr(), mean.data_ptr(),
           rstd.data_ptr(), st)
    y = torch.empty_like(x)
    N.call("sf_group_norm_apply", Rows(x, 0, HW).view(), Rows(y, 0, HW).view(), F_, HW, C, groups, mean.data_ptr(),
           rstd.data_ptr(), gamma.data_ptr(), beta.data_ptr(), N.ACT_SILU, st)
    ldo = Nn + 4
    out = torch.full((F_ * HW, ldo), float("nan"), device=dev)
    N.call("sf_group_norm_project", Rows(x, 0, HW).view(), F_, HW, C, groups, mean.data_ptr(), rstd.data_ptr(),
           gamma.data_ptr(), beta.data_ptr(), N.ACT_SILU, w.data_ptr(), Nn, out.data_ptr(), ldo, st)
    torch.cuda.synchronize()
    ref = y.double() @ w.double().T
    got = out[:, :Nn].double()
    assert torch.isnan(out[:, Nn:]).all(), "columns past N untouched"
    assert float((got - ref).abs().max() / ref.abs().max()) < 1e-5


def test_out_norm_projection_in_plan(monkeypatch):
    """The plan runs out_norm -> out_conv as statistics + sf_group_norm_project + tap sum (no normalised
    tensor); the network output equals the unfused lowering's within fp32 accumulation-order noise."""
    from paper_2411_01171_b200.executor import ExecConfig
    from paper_2411_01171_b200.harness import Denoiser, initial_latent
    from paper_2411_01171_b200.rehash import StepSchedule
    from paper_2411_01171_b200.unet import UNetConfig
    cfg = UNetConfig(channels=4, frames=4, height=16, width=16, base_channels=64, norm_groups=8, steps=3)
    x0 = initial_latent(cfg)
    sched = StepSchedule([0, 1, 2], 3)
    d1 = Denoiser(cfg, ExecConfig())
    a = d1.run(x0, sched)
    monkeypatch.setenv("SF_GN_PROJECT", "0")
    d2 = Denoiser(cfg, ExecConfig(), device_weights=d1.model.dw)
    b = d2.run(x0, sched)
    assert d1.launches[d1._key(sched, False)] < d2.launches[d2._key(sched, False)]
    assert np.abs(a - b).max() / np.abs(b).max() < 1e-4


@pytest.mark.parametrize("F_,H,W,cout,splits", [(3, 72, 128, 320, 94), (2, 16, 16, 64, 3), (5, 9, 12, 128, 7)])
def test_in_conv_partials(F_, H, W, cout, splits):
    """sf_conv3x3_smallcin_gn: the same in_conv output as sf_conv3x3_smallcin, bit for bit, plus per-(frame,
    split, channel) sums of the stored values (frames whose pixel count is not a multiple of 16 included)."""
    torch.manual_seed(10)
    st = torch.cuda.current_stream().cuda_stream
    cin = 4
    x = torch.randn(F_ * H * W, cin, device=dev)
    w = torch.randn(9, cin, cout, device=dev) * 0.3
    b = torch.randn(cout, device=dev)
    y0 = torch.empty(F_ * H * W, cout, dtype=torch.bfloat16, device=dev)
    y1 = torch.empty_like(y0)
    part = torch.full((F_, splits, cout, 2), float("nan"), device=dev)
    N.call("sf_conv3x3_smallcin", x.data_ptr(), F_, H, W, cin, w.data_ptr(), b.data_ptr(), cout,
           Rows(y0, 0, H * W).view(), st)
    N.call("sf_conv3x3_smallcin_gn", x.data_ptr(), F_, H, W, cin, w.data_ptr(), b.data_ptr(), cout,
           Rows(y1, 0, H * W).view(), splits, part.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    assert not torch.isnan(part).any()
    yd = y1.double().view(F_, H * W, cout)
    assert torch.allclose(part.double().sum(1)[..., 0], yd.sum(1), rtol=1e-5, atol=1e-3)
    assert torch.allclose(part.double().sum(1)[..., 1], (yd * yd).sum(1), rtol=1e-5, atol=1e-3)
