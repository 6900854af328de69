"""numpy restatement of the reference operator kernels (test oracle only).

Reference: ``sliceflow/kernels.py:181-390``.  Layout is the reference's
(b, t, c, h, w).  Every kernel returns a fresh array in the input dtype.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2411_01171_b200.errors import InvalidParam, ShapeMismatch, ZeroNorm
from paper_2411_01171_b200.kinds import OpKind, output_shape
from paper_2411_01171_b200.tensor import Shape5


def conv2d(x, weight, bias):
    """3x3 cross-correlation, zero pad 1; taps summed in row-major (dy, dx) order (kernels.py:181-201)."""
    b, t, c, h, w = x.shape
    co = weight.shape[0]
    if weight.shape[1:] != (c, 3, 3):
        raise InvalidParam(f"conv2d weight shape {weight.shape} incompatible with input channels {c}")
    f = x.reshape(b * t, c, h, w).transpose(0, 2, 3, 1)          # frames, h, w, c
    pad = np.zeros((b * t, h + 2, w + 2, c), dtype=x.dtype)
    pad[:, 1:-1, 1:-1] = f
    acc = np.zeros((b * t, h * w, co), dtype=x.dtype)
    for dy in range(3):
        for dx in range(3):
            win = pad[:, dy:dy + h, dx:dx + w].reshape(b * t, h * w, c)
            acc += win @ np.ascontiguousarray(weight[:, :, dy, dx].T).astype(x.dtype)
    acc += bias.astype(x.dtype)
    return np.ascontiguousarray(acc.reshape(b, t, h, w, co).transpose(0, 1, 4, 2, 3))


def temporal_conv(x, weight, bias):
    """Kernel 3 along t, zero pad 1; offset 0 reads t-1 (kernels.py:204-225)."""
    b, t, c, h, w = x.shape
    co = weight.shape[0]
    if weight.shape[1:] != (c, 3):
        raise InvalidParam(f"temporal_conv weight shape {weight.shape} incompatible with input channels {c}")
    cols = x.transpose(0, 3, 4, 1, 2)                              # b, h, w, t, c
    pad = np.zeros((b, h, w, t + 2, c), dtype=x.dtype)
    pad[:, :, :, 1:-1] = cols
    acc = np.zeros((b * h * w, t, co), dtype=x.dtype)
    for off in range(3):
        win = pad[:, :, :, off:off + t].reshape(b * h * w, t, c)
        acc += win @ np.ascontiguousarray(weight[:, :, off].T).astype(x.dtype)
    acc += bias.astype(x.dtype)
    return np.ascontiguousarray(acc.reshape(b, h, w, t, co).transpose(0, 3, 4, 1, 2))


def group_norm(x, gamma, beta, groups, eps):
    """Per (b,t,group) two-pass biased variance (kernels.py:228-237)."""
    b, t, c, h, w = x.shape
    if groups < 1 or c % groups:
        raise InvalidParam(f"group_norm groups={groups} does not divide channels={c}")
    g = x.reshape(b, t, groups, c // groups, h, w)
    mu = g.mean(axis=(3, 4, 5), keepdims=True)
    var = ((g - mu) ** 2).mean(axis=(3, 4, 5), keepdims=True)
    y = ((g - mu) / np.sqrt(var + x.dtype.type(eps))).reshape(x.shape)
    return y * gamma.astype(x.dtype)[:, None, None] + beta.astype(x.dtype)[:, None, None]


def layer_norm(x, gamma, beta, eps):
    """Per (b,t,h,w) over channels (kernels.py:240-244)."""
    mu = x.mean(axis=2, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=2, keepdims=True)
    y = (x - mu) / np.sqrt(var + x.dtype.type(eps))
    return y * gamma.astype(x.dtype)[:, None, None] + beta.astype(x.dtype)[:, None, None]


def silu(x):
    """x * sigmoid(x), never exponentiating a positive argument (kernels.py:247-253)."""
    e = np.exp(-np.abs(x))
    sig = np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))
    return (x * sig).astype(x.dtype, copy=False)


def linear(x, weight, bias):
    """Per token y = x W^T + b (kernels.py:256-266)."""
    b, t, c, h, w = x.shape
    f = weight.shape[0]
    if weight.shape[1] != c:
        raise InvalidParam(f"linear weight shape {weight.shape} incompatible with input channels {c}")
    tok = x.transpose(0, 1, 3, 4, 2).reshape(-1, c)
    y = tok @ weight.T.astype(x.dtype) + bias.astype(x.dtype)
    return np.ascontiguousarray(y.reshape(b, t, h, w, f).transpose(0, 1, 4, 2, 3))


def attention_tokens(tok, wq, wk, wv, wo):
    """Single head, d = C, x @ W (no transpose), scale 1/sqrt(C) (kernels.py:269-292)."""
    dt = tok.dtype
    c = tok.shape[-1]
    if wq.shape != (c, c):
        raise InvalidParam(f"attention weights must be ({c}, {c}), got {wq.shape}")
    q, k, v = (tok @ m.astype(dt) for m in (wq, wk, wv))
    s = (q @ k.transpose(0, 2, 1)) * dt.type(1.0 / math.sqrt(c))
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=-1, keepdims=True)
    return (p @ v) @ wo.astype(dt)


def spatial_attention(x, params):
    """Per frame over h*w tokens (kernels.py:295-300)."""
    b, t, c, h, w = x.shape
    tok = x.reshape(b * t, c, h * w).transpose(0, 2, 1)
    o = attention_tokens(np.ascontiguousarray(tok), params["wq"], params["wk"], params["wv"], params["wo"])
    return np.ascontiguousarray(o.transpose(0, 2, 1).reshape(b, t, c, h, w))


def temporal_attention(x, params):
    """Per pixel over t tokens (kernels.py:303-308)."""
    b, t, c, h, w = x.shape
    tok = np.ascontiguousarray(x.transpose(0, 3, 4, 1, 2)).reshape(b * h * w, t, c)
    o = attention_tokens(tok, params["wq"], params["wk"], params["wv"], params["wo"])
    return np.ascontiguousarray(o.reshape(b, h, w, t, c).transpose(0, 3, 4, 1, 2))


def downsample2x(x):
    """2x2 mean as (x00+x01+x10+x11)*0.25 (kernels.py:311-316)."""
    s = x[..., 0::2, 0::2] + x[..., 0::2, 1::2] + x[..., 1::2, 0::2] + x[..., 1::2, 1::2]
    return (s * x.dtype.type(0.25)).astype(x.dtype, copy=False)


def upsample2x(x):
    """Nearest-neighbour x2 (kernels.py:319-320)."""
    return np.repeat(np.repeat(x, 2, axis=3), 2, axis=4)


def _req(params, name, kind):
    if params is None or name not in params:
        raise InvalidParam(f"{kind.value} requires parameter {name!r}")
    return params[name]


def apply_kernel(kind: OpKind, arrays, params=None, attrs=None):
    """Validate then dispatch on plain arrays (kernels.py:323-368)."""
    attrs = attrs or {}
    output_shape(kind, [Shape5(*a.shape) for a in arrays], attrs)
    x = arrays[0]
    if kind is OpKind.CONV2D:
        out = conv2d(x, _req(params, "weight", kind), _req(params, "bias", kind))
    elif kind is OpKind.TEMPORAL_CONV:
        out = temporal_conv(x, _req(params, "weight", kind), _req(params, "bias", kind))
    elif kind is OpKind.GROUP_NORM:
        out = group_norm(x, _req(params, "gamma", kind), _req(params, "beta", kind),
                         int(attrs.get("groups", 1)), float(attrs.get("eps", 1e-5)))
    elif kind is OpKind.LAYER_NORM:
        out = layer_norm(x, _req(params, "gamma", kind), _req(params, "beta", kind), float(attrs.get("eps", 1e-5)))
    elif kind is OpKind.SILU:
        out = silu(x)
    elif kind is OpKind.LINEAR:
        out = linear(x, _req(params, "weight", kind), _req(params, "bias", kind))
    elif kind is OpKind.SPATIAL_ATTENTION:
        out = spatial_attention(x, params or {})
    elif kind is OpKind.TEMPORAL_ATTENTION:
        out = temporal_attention(x, params or {})
    elif kind is OpKind.DOWNSAMPLE2X:
        out = downsample2x(x)
    elif kind is OpKind.UPSAMPLE2X:
        out = upsample2x(x)
    elif kind is OpKind.ADD:
        a, b = arrays
        out = b + a if (a.shape[3:] == (1, 1) and b.shape[3:] != (1, 1)) else a + b
    elif kind is OpKind.CONCAT:
        out = np.concatenate(arrays, axis=2)
    elif kind is OpKind.SPLIT:
        sizes = [int(s) for s in attrs["sizes"]]
        i = int(attrs["index"])
        off = sum(sizes[:i])
        out = x[:, :, off:off + sizes[i]]
    else:
        raise InvalidParam(f"unknown kind {kind}")
    return np.ascontiguousarray(out)


def cosine_similarity(a, b):
    """Flattened cosine in fp64, clipped to [-1, 1] (kernels.py:375-390)."""
    if a.shape != b.shape:
        raise ShapeMismatch(f"shape mismatch {a.shape} vs {b.shape}")
    af = a.ravel().astype(np.float64)
    bf = b.ravel().astype(np.float64)
    aa, bb = float(af @ af), float(bf @ bf)
    if aa == 0.0 or bb == 0.0:
        raise ZeroNorm("cosine similarity undefined for an identically-zero tensor")
    return min(1.0, max(-1.0, float(af @ bf) / math.sqrt(aa * bb)))
