"""Per-operator entry point on the device: ``apply_kernel``.

Same signature, validation order and errors as the reference
``kernels.apply_kernel`` (``kernels.py:323-368``): static shape rules first
(``output_shape``), then dispatch -- but every kind runs on the sm_100a
kernels.  Host ``Tensor5D`` values are converted at the boundary to bf16
channels-last rows on the device and back to fp32 ``(b,t,c,h,w)``.
"""

from __future__ import annotations

import math
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _native as N
from . import device as D
from .device import Epilogue, Rows
from .errors import InvalidParam, NativeError, ShapeMismatch, ZeroNorm
from .kinds import OpKind, output_shape
from .tensor import Shape5, Tensor5D


def _dev():
    N.load()
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the sliceflow_b200 path has no CPU fallback")
    return torch.device("cuda")


def to_rows(x: Tensor5D, dtype=torch.bfloat16) -> torch.Tensor:
    """(b,t,c,h,w) host -> (b*t*h*w, c) device rows."""
    s = x.shape
    t = torch.from_numpy(np.ascontiguousarray(x.data, dtype=np.float32)).to(_dev())
    return t.permute(0, 1, 3, 4, 2).reshape(s.b * s.t * s.h * s.w, s.c).to(dtype).contiguous()


def from_rows(t: torch.Tensor, s: Shape5) -> Tensor5D:
    a = t.float().reshape(s.b, s.t, s.h, s.w, s.c).permute(0, 1, 4, 2, 3).contiguous().cpu().numpy()
    return Tensor5D(a)


def _req(params, name, kind):
    if params is None or name not in params:
        raise InvalidParam(f"{kind.value} requires parameter {name!r}")
    return params[name]


class _Node:
    def __init__(self, kind, attrs):
        self.kind, self.attrs, self.param_ref, self.id, self.inputs = kind, attrs, "p", "p", ()


def apply_kernel(kind: OpKind, inputs: Sequence[Tensor5D], params: Mapping | None = None,
                 attrs: Mapping | None = None, backend: int = 0) -> Tensor5D:
    """Apply one operator on the GPU; pure (inputs untouched, fresh output)."""
    attrs = attrs or {}
    kind = OpKind(kind)
    out_s = output_shape(kind, [x.shape for x in inputs], attrs)
    dev = _dev()
    st = torch.cuda.current_stream().cuda_stream
    s = inputs[0].shape
    rows, orows = s.b * s.t * s.h * s.w, out_s.b * out_s.t * out_s.h * out_s.w
    frames, hw = s.b * s.t, s.h * s.w
    if kind is OpKind.CONV2D:
        w = np.asarray(_require_shape(_req(params, "weight", kind), (out_s.c, s.c, 3, 3), kind))
        prm = D.DeviceWeights.__new__(D.DeviceWeights)
        prm.dev = dev
        p = prm._convert(_Node(kind, attrs), {"weight": w, "bias": _req(params, "bias", kind)})
        if s.c % 8:
            x = to_rows(inputs[0], torch.float32)
            y = torch.empty(orows, out_s.c, dtype=torch.bfloat16, device=dev)
            N.call("sf_conv3x3_smallcin", x.data_ptr(), frames, s.h, s.w, s.c, p["wt32"].data_ptr(),
                   p["bias"].data_ptr(), out_s.c, Rows(y, 0, hw).view(), st)
            return from_rows(y, out_s)
        x = to_rows(inputs[0])
        if out_s.c % 8:
            y = torch.empty(orows, out_s.c, dtype=torch.float32, device=dev)
            D.conv2d(st, Rows(x, 0, hw), Rows(y, 0, hw), frames, s.h, s.w, s.c, out_s.c, p, Epilogue(), backend,
                     out_fp32=True)
            return from_rows(y, out_s)
        y = torch.empty(orows, out_s.c, dtype=torch.bfloat16, device=dev)
        D.conv2d(st, Rows(x, 0, hw), Rows(y, 0, hw), frames, s.h, s.w, s.c, out_s.c, p, Epilogue(), backend)
        return from_rows(y, out_s)

    x = to_rows(inputs[0])
    y = torch.empty(orows, out_s.c, dtype=torch.bfloat16, device=dev)
    if kind is OpKind.TEMPORAL_CONV:
        _require_shape(_req(params, "weight", kind), (out_s.c, s.c, 3), kind)
        p = _convert(kind, attrs, params, dev)
        D.temporal_conv(st, Rows(x, 0, hw), Rows(y, 0, hw), frames, s.t, hw, s.c, out_s.c, p, Epilogue(), backend)
    elif kind is OpKind.LINEAR:
        _require_shape(_req(params, "weight", kind), (out_s.c, s.c), kind)
        p = _convert(kind, attrs, params, dev)
        D.linear(st, Rows(x), Rows(y), 1, rows, s.c, out_s.c, p, Epilogue(), backend)
    elif kind is OpKind.GROUP_NORM:
        groups = int(attrs.get("groups", 1))
        p = _convert(kind, attrs, params, dev)
        eps = float(attrs.get("eps", 1e-5))
        work = torch.empty(N.query("sf_group_norm_workspace", frames, hw, s.c), dtype=torch.uint8, device=dev)
        mean = torch.empty(frames * groups, dtype=torch.float32, device=dev)
        rstd = torch.empty_like(mean)
        D.group_norm_stats(st, Rows(x, 0, hw), frames, hw, s.c, groups, eps, work, mean, rstd)
        D.group_norm_apply(st, Rows(x, 0, hw), Rows(y, 0, hw), frames, hw, s.c, groups, mean, rstd, p, N.ACT_NONE)
    elif kind is OpKind.LAYER_NORM:
        p = _convert(kind, attrs, params, dev)
        D.layer_norm(st, Rows(x), Rows(y), 1, rows, s.c, p, float(attrs.get("eps", 1e-5)))
    elif kind is OpKind.SILU:
        N.call("sf_silu", Rows(x).view(), Rows(y).view(), 1, rows, s.c, st)
    elif kind in (OpKind.SPATIAL_ATTENTION, OpKind.TEMPORAL_ATTENTION):
        for n in ("wq", "wk", "wv", "wo"):
            _require_shape(_req(params, n, kind), (s.c, s.c), kind)
        p = _convert(kind, attrs, params, dev)
        if kind is OpKind.SPATIAL_ATTENTION:
            sc = {k: torch.empty(r, c, dtype=dt, device=dev)
                  for k, (r, c, dt) in D.spatial_attention_scratch(rows, hw, s.c).items()}
            D.spatial_attention(st, Rows(x, 0, hw), Rows(y, 0, hw), frames, hw, s.c, p, Epilogue(), sc, backend)
        else:
            sc = {"qkv": torch.empty(rows, 3 * s.c, dtype=torch.bfloat16, device=dev),
                  "o": torch.empty(rows, s.c, dtype=torch.bfloat16, device=dev)}
            D.temporal_attention(st, Rows(x, 0, hw), Rows(y, 0, hw), s.b, s.t, hw, s.c, p, Epilogue(), sc, backend)
    elif kind is OpKind.DOWNSAMPLE2X:
        N.call("sf_downsample2x", Rows(x, 0, hw).view(), Rows(y, 0, out_s.h * out_s.w).view(), frames, s.h, s.w,
               s.c, st)
    elif kind is OpKind.UPSAMPLE2X:
        N.call("sf_upsample2x", Rows(x, 0, hw).view(), Rows(y, 0, out_s.h * out_s.w).view(), frames, s.h, s.w, s.c,
               st)
    elif kind is OpKind.ADD:
        b = inputs[1]
        a_s, b_s = inputs[0].shape, b.shape
        if (a_s.h, a_s.w) == (1, 1) and (b_s.h, b_s.w) != (1, 1):
            x, b = to_rows(b), inputs[0]
            a_s, b_s = b_s, a_s
        bt = to_rows(b)
        bcast = (b_s.h, b_s.w) == (1, 1) and (a_s.h, a_s.w) != (1, 1)
        if bcast:
            N.call("sf_add", Rows(x, 0, hw).view(), Rows(bt, 0, 1).view(), Rows(y, 0, hw).view(), frames, hw, s.c, 1,
                   st)
        else:
            N.call("sf_add", Rows(x).view(), Rows(bt).view(), Rows(y).view(), 1, rows, s.c, 0, st)
    elif kind is OpKind.CONCAT:
        off = 0
        for inp in inputs:
            t = to_rows(inp)
            N.call("sf_copy_rows", Rows(t).view(), Rows(y, 0, 0, off).view(), 1, rows, inp.shape.c, st)
            off += inp.shape.c
    elif kind is OpKind.SPLIT:
        sizes = [int(v) for v in attrs["sizes"]]
        off = sum(sizes[:int(attrs["index"])])
        N.call("sf_copy_rows", Rows(x, 0, 0, off).view(), Rows(y).view(), 1, rows, out_s.c, st)
    else:
        raise InvalidParam(f"unknown kind {kind}")
    return from_rows(y, out_s)


def _require_shape(w, shape, kind):
    if tuple(np.shape(w)) != tuple(shape):
        raise InvalidParam(f"{kind.value} weight shape {np.shape(w)} incompatible with {shape}")
    return w


def _convert(kind, attrs, params, dev):
    dw = D.DeviceWeights.__new__(D.DeviceWeights)
    dw.dev = dev
    need = {"gamma", "beta"} if kind in (OpKind.GROUP_NORM, OpKind.LAYER_NORM) else set()
    for n in need:
        _req(params, n, kind)
    return dw._convert(_Node(kind, attrs), params)


def cosine_similarity(a: Tensor5D, b: Tensor5D) -> float:
    """Flattened cosine on the device: bf16 operands, fp64 fixed-order sums (kernels.py:375-390)."""
    if a.shape != b.shape:
        raise ShapeMismatch(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    dev = _dev()
    ta = torch.from_numpy(np.ascontiguousarray(a.data, dtype=np.float32)).to(dev).to(torch.bfloat16).view(-1)
    tb = torch.from_numpy(np.ascontiguousarray(b.data, dtype=np.float32)).to(dev).to(torch.bfloat16).view(-1)
    return cosine_from_device(ta, tb)


def cosine_from_device(ta: torch.Tensor, tb: torch.Tensor) -> float:
    n = ta.numel()
    dev = ta.device
    work = torch.empty(N.query("sf_dot3_workspace", n), dtype=torch.uint8, device=dev)
    out = torch.empty(3, dtype=torch.float64, device=dev)
    N.call("sf_dot3_bf16", ta.data_ptr(), tb.data_ptr(), n, work.data_ptr(), out.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    aa, bb, ab = out.cpu().tolist()
    if aa == 0.0 or bb == 0.0:
        raise ZeroNorm("cosine similarity undefined for an identically-zero tensor")
    return min(1.0, max(-1.0, ab / math.sqrt(aa * bb)))
