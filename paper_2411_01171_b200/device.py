"""Device-side building blocks: weight upload and per-operator launchers.

Weights are uploaded once, in the layouts the kernels consume:

* conv2d ``(co, ci, 3, 3)`` -> bf16 ``[co][tap][ci]`` (tap = dy*3+dx): the
  K-major B operand of the implicit GEMM, K index = tap*ci + c, taps in the
  reference's row-major (dy, dx) order (kernels.py:172).
* temporal_conv ``(co, ci, 3)`` -> bf16 ``[co][off][ci]``.
* linear ``(f, c)`` -> bf16 ``[f][c]`` (already K-major: y = x W^T).
* attention ``wq, wk, wv, wo`` ``(c, c)``, applied as ``x @ W`` (no transpose,
  kernels.py:285-291) -> one fused bf16 ``[3c][c]`` = [wq^T; wk^T; wv^T] and
  ``wo^T``.
* norm gamma/beta and every bias stay fp32; the latent-edge in_conv (4-8
  input channels) and the step-embedding projections keep fp32 weights only
  (no bf16 copy), every other weight exists once, in bf16.

Every launcher takes :class:`Rows` views (a two-level row view over a torch
tensor, see ``sf_view_t``) and the CUDA stream handle, and goes straight to
the C ABI.  Nothing here computes on the host.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import InvalidParam, ShapeMismatch
from .kinds import OpKind


@dataclass
class Rows:
    """Rows of a 2-D (rows, C>=width) tensor as a two-level view.

    row (o, i) = tensor row  row0 + o*ostride + i ; columns col0 .. col0+width.
    """

    t: torch.Tensor
    row0: int = 0
    ostride: int = 0
    col0: int = 0

    @property
    def ld(self) -> int:
        return self.t.stride(0)

    def view(self) -> N.View:
        es = self.t.element_size()
        ptr = self.t.data_ptr() + (self.row0 * self.t.stride(0) + self.col0) * es
        return N.View(ptr, self.t.stride(0), self.ostride)

    def ptr(self) -> int:
        return self.view().ptr

    def shifted(self, rows: int = 0, cols: int = 0, ostride: int | None = None) -> "Rows":
        return Rows(self.t, self.row0 + rows, self.ostride if ostride is None else ostride, self.col0 + cols)


def bf16(a: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev).to(torch.bfloat16).contiguous()


def f32(a: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev).contiguous()


def attention_weights(prm, dev) -> dict:
    """[wq^T; wk^T; wv^T] and wo^T (bf16) for the projection GEMMs (the reference right-multiplies,
    kernels.py:285-291)."""
    qkv = np.concatenate([np.asarray(prm[n]).T for n in ("wq", "wk", "wv")], axis=0)
    return {"wqkv": bf16(qkv, dev), "wo": bf16(np.asarray(prm["wo"]).T, dev)}


def unfused_weights(prm: dict, dev) -> dict:
    """Make sure a temporal attention's three-launch weights exist (built at plan compile time,
    never during graph capture); returns ``prm``."""
    if "wqkv" not in prm:
        prm.update(attention_weights(prm["host"], dev))
    return prm


def temporal_fused_weights(wq, wk, wv, wo, dev) -> torch.Tensor:
    """[Mqk^T ; Mvo^T] (bf16 [2C][C], K-major B operands) for sf_temporal_attention_fused:
    Mqk = Wq Wk^T log2(e)/sqrt(C) and Mvo = Wv Wo in fp64 (kernels.py:285-292 right-multiplies:
    q = x Wq, ..., out = ctx Wo), so x Mqk x^T is the reference's scaled score in log2 units and
    (P x) Mvo its P (x Wv) Wo."""
    wq, wk, wv, wo = (np.asarray(w, dtype=np.float64) for w in (wq, wk, wv, wo))
    C = wq.shape[0]
    mqk = (wq @ wk.T) * (1.4426950408889634 / math.sqrt(C))
    mvo = wv @ wo
    return bf16(np.concatenate([mqk.T, mvo.T], axis=0), dev)


class DeviceWeights:
    """All parameters of a WeightBundle in kernel layout on one device."""

    def __init__(self, graph, weights, device):
        self.dev = torch.device(device)
        self.p: dict[str, dict[str, torch.Tensor]] = {}
        for node in graph.nodes.values():
            if not node.param_ref:
                continue
            self.p[node.id] = self._convert(node, weights.get(node.param_ref))

    def _convert(self, node, prm) -> dict:
        d = self.dev
        k = node.kind
        if k is OpKind.CONV2D:
            w = np.asarray(prm["weight"], dtype=np.float64)
            co, ci = w.shape[:2]
            out = {"bias": f32(prm["bias"], d)}
            if ci % 8 or tuple(getattr(node, "inputs", ()))[:1] == ("x",):
                # fp32 [tap][ci][co] for sf_conv3x3_smallcin (the latent-edge in_conv)
                out["wt32"] = f32(w.transpose(2, 3, 1, 0).reshape(9, ci, co), d)
            if ci % 8 == 0:
                out["w"] = bf16(w.transpose(0, 2, 3, 1).reshape(co, 9 * ci), d)
                if co < TAPWISE_MAX_COUT:
                    # tap-major [(tap, co)][ci] for conv2d_tapwise (row = tap * co + c)
                    out["w_taps"] = bf16(w.transpose(2, 3, 0, 1).reshape(9 * co, ci), d)
            return out
        if k is OpKind.TEMPORAL_CONV:
            w = np.asarray(prm["weight"], dtype=np.float64)
            co, ci = w.shape[:2]
            return {"w": bf16(w.transpose(0, 2, 1).reshape(co, 3 * ci), d), "bias": f32(prm["bias"], d)}
        if k is OpKind.LINEAR:
            if tuple(getattr(node, "inputs", ())) == ("step_emb",):
                # step-embedding projection: one fp32 gemv per step (executor.emb_launch)
                return {"w32": f32(prm["weight"], d), "bias": f32(prm["bias"], d)}
            return {"w": bf16(prm["weight"], d), "bias": f32(prm["bias"], d)}
        if k in (OpKind.GROUP_NORM, OpKind.LAYER_NORM):
            return {"gamma": f32(prm["gamma"], d), "beta": f32(prm["beta"], d)}
        if k in (OpKind.SPATIAL_ATTENTION, OpKind.TEMPORAL_ATTENTION):
            C = np.asarray(prm["wq"]).shape[0]
            if k is OpKind.TEMPORAL_ATTENTION and C % 64 == 0 and C <= 320:
                # one fused launch (sf_temporal_attention_fused): the projection weights of the
                # three-launch path are uploaded only if a plan needs it (unfused_weights)
                return {"wfused": temporal_fused_weights(prm["wq"], prm["wk"], prm["wv"], prm["wo"], d),
                        "host": {n: np.asarray(prm[n]) for n in ("wq", "wk", "wv", "wo")}}
            return attention_weights(prm, d)
        raise InvalidParam(f"no device layout for {k}")


# ---------------------------------------------------------------------------
# launchers
# ---------------------------------------------------------------------------

def gemm_args(*, mode, n_outer, n_inner, cin, n, a: Rows, w: torch.Tensor, w_ld=None, w_kmajor=True,
              out: Rows, out_fp32=False, bias=None, rowbias=None, rowbias_stride=0, act=N.ACT_NONE,
              res: Rows | None = None, H=0, W=0, T=0, batch=1, a_bstride=0, w_bstride=0, out_bstride=0,
              res_bstride=0, alpha=1.0, backend=0, w_ptr=None, rowstats=None, colvec=None, gn_partial=None):
    args = N.GemmArgs()
    args.mode, args.n_outer, args.n_inner = mode, n_outer, n_inner
    args.H, args.W, args.T = H, W, T
    args.cin, args.N, args.batch = cin, n, batch
    args.a, args.a_bstride = a.view(), a_bstride
    args.w = w_ptr if w_ptr is not None else w.data_ptr()
    args.w_kmajor = 1 if w_kmajor else 0
    args.w_ld = w_ld if w_ld is not None else w.stride(0)
    args.w_bstride = w_bstride
    args.alpha = alpha
    args.bias = bias.data_ptr() if bias is not None else None
    args.rowbias = rowbias.data_ptr() if rowbias is not None else None
    args.rowbias_stride = rowbias_stride
    args.act = act
    args.res = res.view() if res is not None else N.NULL_VIEW
    args.res_bstride = res_bstride
    args.out, args.out_bstride = out.view(), out_bstride
    args.out_fp32 = 1 if out_fp32 else 0
    args.backend = backend
    args.rowstats = rowstats.data_ptr() if rowstats is not None else None
    args.colvec = colvec.data_ptr() if colvec is not None else None
    args.gn_partial = gn_partial
    return args


def gemm(stream, **kw):
    args = gemm_args(**kw)
    N.call("sf_gemm", args, stream)
    return args


class Epilogue:
    """What a GEMM-ending op adds after its bias: SiLU, per-frame bias, residual."""

    def __init__(self, act=N.ACT_NONE, rowbias=None, res: Rows | None = None):
        self.act, self.rowbias, self.res = act, rowbias, res


def conv2d(stream, x: Rows, y: Rows, frames, H, W, cin, cout, prm, epi: Epilogue, backend=0, out_fp32=False,
           gn_partial=None):
    """3x3 conv (kernels.py:181-201) as an implicit GEMM.  ``gn_partial``: device address of
    [frames][sf_conv_gn_splits(H, W)][cout] float2 GroupNorm partials of the stored output."""
    if "w" not in prm:
        raise ShapeMismatch(f"conv2d with cin={cin} needs the small-channel path")
    return gemm(stream, mode=N.GEMM_CONV3X3, n_outer=frames, n_inner=H * W, H=H, W=W, cin=cin, n=cout, a=x,
                w=prm["w"], out=y, out_fp32=out_fp32, bias=prm["bias"], rowbias=epi.rowbias, act=epi.act,
                res=epi.res, backend=backend, gn_partial=gn_partial)


TAPWISE_MAX_COUT = 16


def conv2d_tapwise(stream, x: Rows, out: Rows, frames, H, W, cin, cout, prm, ybuf: torch.Tensor, backend=0):
    """3x3 conv with few output channels (the network's out_conv, 320 -> 4) into fp32 rows.

    A padded-N implicit GEMM would issue 9*cin/16 narrow MMAs per 128 rows for 4 useful
    columns; instead one plain GEMM projects every pixel onto all 9 taps,
    Y[p][tap*cout + c] = x[p] . W_tap[c] (K = cin, N = 9*cout), and sf_conv3x3_tapsum adds the
    9 shifted taps (zero padding) plus the bias: the same sum as kernels.py:181-201 regrouped.
    ``ybuf``: fp32 scratch with >= frames*H*W rows of >= 9*cout columns.
    """
    HW = H * W
    gemm(stream, mode=N.GEMM_PLAIN, n_outer=frames, n_inner=HW, cin=cin, n=9 * cout, a=x, w=prm["w_taps"],
         out=Rows(ybuf, 0, HW), out_fp32=True, backend=backend)
    N.call("sf_conv3x3_tapsum", ybuf.data_ptr(), ybuf.stride(0), frames, H, W, cout, prm["bias"].data_ptr(),
           out.view(), stream)


def temporal_conv(stream, x: Rows, y: Rows, bt, T, n_inner, cin, cout, prm, epi: Epilogue, backend=0):
    return gemm(stream, mode=N.GEMM_TCONV3, n_outer=bt, n_inner=n_inner, T=T, cin=cin, n=cout, a=x, w=prm["w"], out=y,
                bias=prm["bias"], rowbias=epi.rowbias, act=epi.act, res=epi.res, backend=backend)


def linear(stream, x: Rows, y: Rows, n_outer, n_inner, cin, cout, prm, epi: Epilogue, backend=0):
    return gemm(stream, mode=N.GEMM_PLAIN, n_outer=n_outer, n_inner=n_inner, cin=cin, n=cout, a=x, w=prm["w"],
                out=y, bias=prm["bias"], rowbias=epi.rowbias, act=epi.act, res=epi.res, backend=backend)


def group_norm_stats(stream, x: Rows, frames, n_inner, C, groups, eps, work, mean, rstd):
    N.call("sf_group_norm_stats", x.view(), frames, n_inner, C, groups, eps, work.data_ptr(), mean.data_ptr(),
           rstd.data_ptr(), stream)


def group_norm_apply(stream, x: Rows, y: Rows, frames, n_inner, C, groups, mean, rstd, prm, act):
    N.call("sf_group_norm_apply", x.view(), y.view(), frames, n_inner, C, groups, mean.data_ptr(), rstd.data_ptr(),
           prm["gamma"].data_ptr(), prm["beta"].data_ptr(), act, stream)


def layer_norm(stream, x: Rows, y: Rows, n_outer, n_inner, C, prm, eps, act=N.ACT_NONE):
    N.call("sf_layer_norm", x.view(), y.view(), n_outer, n_inner, C, prm["gamma"].data_ptr(), prm["beta"].data_ptr(),
           eps, act, stream)


def spatial_attention(stream, x: Rows, y: Rows, frames, HW, C, prm, epi: Epilogue, scratch, backend=0):
    """Per-frame single-head attention, d = C (kernels.py:295-300).

    qkv = x [wq|wk|wv] (one GEMM, N = 3C); S = q k^T / sqrt(C) per frame (fp32,
    batched GEMM over frames); P = softmax(S) (bf16); o = P v (batched GEMM, v
    read MN-major straight out of qkv); y = o wo (+ residual) in one epilogue.
    ``scratch``: dict with qkv [frames*HW, 3C] bf16, s [frames*HW, HW] fp32,
    p [frames*HW, HW] bf16, o [frames*HW, C] bf16.
    """
    qkv, o = scratch["qkv"], scratch["o"]
    gemm(stream, mode=N.GEMM_PLAIN, n_outer=frames, n_inner=HW, cin=C, n=3 * C if HW <= SMALL_SEQ else 2 * C, a=x,
         w=prm["wqkv"], out=Rows(qkv, 0, HW), backend=backend)
    if HW > SMALL_SEQ and use_flash(HW, C):
        vt = scratch["vt"]
        xv = x.view()
        gemm(stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=C, cin=C, n=HW, a=Rows(prm["wqkv"], 2 * C, 0),
             w=vt, w_ptr=xv.ptr, w_ld=xv.ld, out=Rows(vt, 0, 0), batch=frames, a_bstride=0,
             w_bstride=HW * xv.ld, out_bstride=C * HW, backend=backend)
        N.call("sf_spatial_attention_core", Rows(qkv, 0, HW).view(), Rows(qkv, 0, HW, C).view(), vt.data_ptr(),
               Rows(o, 0, HW).view(), frames, HW, C, 1.0 / math.sqrt(C), stream)
    elif HW <= SMALL_SEQ:
        # short token sequences (deep toy levels): the fused per-sequence core,
        # each frame's HW tokens as one sequence (row b*HW + t, ostride 1)
        N.call("sf_temporal_attention_core", Rows(qkv, 0, 1).view(), C, 2 * C, Rows(o, 0, 1).view(), frames, HW, 1,
               C, 1.0 / math.sqrt(C), stream)
    else:
        # v^T[c][t] = sum_k wv[k][c] x[t][k]: the weights as A (M = C) and the
        # frame's tokens as a K-major B, so P v below is K-major on both sides
        vt = scratch["vt"]
        xv = x.view()
        gemm(stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=C, cin=C, n=HW, a=Rows(prm["wqkv"], 2 * C, 0),
             w=vt, w_ptr=xv.ptr, w_ld=xv.ld, out=Rows(vt, 0, 0), batch=frames, a_bstride=0,
             w_bstride=HW * xv.ld, out_bstride=C * HW, backend=backend)
        _spatial_core_materialized(stream, frames, HW, C, scratch, backend)
    gemm(stream, mode=N.GEMM_PLAIN, n_outer=frames, n_inner=HW, cin=C, n=C, a=Rows(o, 0, HW), w=prm["wo"],
         out=y, rowbias=epi.rowbias, act=epi.act, res=epi.res, backend=backend)


SMALL_SEQ = 64
FLASH = True  # fused tcgen05 attention where supported (tests flip it to compare paths)


def use_flash(HW, C) -> bool:
    return FLASH and HW % 8 == 0 and bool(N.query("sf_flash_supported", HW, C))


def spatial_attention_scratch(rows, HW, C) -> dict:
    """Slice scratch the spatial attention lowering needs: {name: (rows, cols, dtype)}."""
    flash = HW > SMALL_SEQ and use_flash(HW, C)
    # above SMALL_SEQ tokens q|k live in a 2C-wide buffer and V^T in its own (spatial_attention)
    out = {"qkv": (rows, (2 if HW > SMALL_SEQ else 3) * C, torch.bfloat16), "o": (rows, C, torch.bfloat16)}
    frames = rows // HW
    if HW > SMALL_SEQ:
        out["vt"] = (frames * C, HW, torch.bfloat16)
        if not flash:
            out["s"] = (rows, HW, torch.float32)
            out["p"] = (rows, HW, torch.bfloat16)
    return out


def _spatial_core_materialized(stream, frames, HW, C, scratch, backend):
    qkv, s, p, o = scratch["qkv"], scratch["s"], scratch["p"], scratch["o"]
    if HW % 8:
        raise ShapeMismatch(f"spatial attention over {HW} tokens needs a multiple of 8 above {SMALL_SEQ}")
    ld = qkv.stride(0)   # q | k (2C wide)
    gemm(stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=HW, cin=C, n=HW, a=Rows(qkv, 0, 0),
         w=qkv, w_ptr=qkv.data_ptr() + C * qkv.element_size(), w_ld=ld, w_kmajor=True,
         out=Rows(s, 0, 0), out_fp32=True, batch=frames, a_bstride=HW * ld, w_bstride=HW * ld,
         out_bstride=HW * HW, alpha=1.0 / math.sqrt(C), backend=backend)
    N.call("sf_softmax_rows", s.data_ptr(), HW, p.data_ptr(), HW, frames * HW, HW, stream)
    vt = scratch["vt"]
    gemm(stream, mode=N.GEMM_PLAIN, n_outer=1, n_inner=HW, cin=HW, n=C, a=Rows(p, 0, 0),
         w=vt, w_ld=HW, out=Rows(o, 0, 0), batch=frames, a_bstride=HW * HW, w_bstride=C * HW,
         out_bstride=HW * C, backend=backend)


def ln_fold_weights(wqkv: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor) -> dict:
    """A LayerNorm (kernels.py:240-244) folded into the projection that consumes it:
    LN(x)_r . W_n = rstd_r * (x_r . W'_n - mean_r * sum_k W'_nk) + (beta . W_n), W' = W diag(gamma).
    The column sums are taken over the bf16-rounded W' the GEMM multiplies by."""
    w = wqkv.float()
    wf = (w * gamma[None, :]).to(torch.bfloat16).contiguous()
    return {"w": wf, "colsum": wf.float().sum(1).contiguous(), "cb": (w @ beta).contiguous()}


def fused_temporal_ok(prm, T, C, epi=None, backend=0, fold=None) -> bool:
    """Whether the op runs as one sf_temporal_attention_fused launch (tcgen05; C <= 320, T <= 128,
    epilogue = residual only).  ``SF_TATTN_FUSED=0`` keeps the three-launch path (A/B runs)."""
    if os.environ.get("SF_TATTN_FUSED") == "0" or "wfused" not in prm or fold is not None:
        return False
    if (backend & 3) == 1:      # mma.sync forced: no tcgen05 kernels
        return False
    if epi is not None and (epi.rowbias is not None or epi.act):
        return False
    return bool(N.query("sf_temporal_attention_fused_supported", T, C))


def temporal_attention(stream, x: Rows, y: Rows, B, T, n_inner, C, prm, epi: Epilogue, scratch, backend=0,
                       fold=None):
    """Per-pixel single-head attention over T frames (kernels.py:303-308).

    ``fold = (weights from ln_fold_weights, eps)``: ``x`` is the LayerNorm's raw input; one
    statistics pass (mean, rstd per row) replaces the LayerNorm's normalised write + re-read, and
    the QKV GEMM applies it in its epilogue."""
    if fused_temporal_ok(prm, T, C, epi, backend, fold):
        N.call("sf_temporal_attention_fused", x.view(), prm["wfused"].data_ptr(),
               epi.res.view() if epi.res is not None else N.View(0, 0, 0), y.view(), B, T, n_inner, C, stream)
        return
    qkv, o = scratch["qkv"], scratch["o"]
    bt = B * T
    unfused_weights(prm, y.t.device)
    if fold is None:
        gemm(stream, mode=N.GEMM_PLAIN, n_outer=bt, n_inner=n_inner, cin=C, n=3 * C, a=x, w=prm["wqkv"],
             out=Rows(qkv, 0, n_inner), backend=backend)
    else:
        fw, eps = fold
        stats = scratch["lnstats"]
        N.call("sf_layer_norm_stats", x.view(), bt, n_inner, C, eps, stats.data_ptr(), stream)
        gemm(stream, mode=N.GEMM_PLAIN, n_outer=bt, n_inner=n_inner, cin=C, n=3 * C, a=x, w=fw["w"],
             out=Rows(qkv, 0, n_inner), bias=fw["cb"], rowstats=stats, colvec=fw["colsum"], backend=backend)
    N.call("sf_temporal_attention_core", Rows(qkv, 0, n_inner).view(), C, 2 * C, Rows(o, 0, n_inner).view(), B, T,
           n_inner, C, 1.0 / math.sqrt(C), stream)
    gemm(stream, mode=N.GEMM_PLAIN, n_outer=bt, n_inner=n_inner, cin=C, n=C, a=Rows(o, 0, n_inner), w=prm["wo"],
         out=y, rowbias=epi.rowbias, act=epi.act, res=epi.res, backend=backend)
