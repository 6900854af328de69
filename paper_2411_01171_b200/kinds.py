"""Operator kinds, their legality metadata and static shape rules.

Reference: ``sliceflow/kernels.py:35-163``.  Only the *metadata* half of the
reference module lives here (domains, receptive fields, strides, shape rules,
the attention scratch model).  The arithmetic half is the sm_100a CUDA code in
``csrc/`` reached through :mod:`ops`; there is no host implementation of any
kernel in this package.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Mapping, Sequence

from .errors import InvalidParam, ShapeMismatch
from .tensor import Shape5

FULL = math.inf


class Domain(str, Enum):
    SPATIAL = "spatial"
    TEMPORAL = "temporal"
    BOUNDARY = "boundary"


class OpKind(str, Enum):
    CONV2D = "conv2d"
    TEMPORAL_CONV = "temporal_conv"
    GROUP_NORM = "group_norm"
    LAYER_NORM = "layer_norm"
    SILU = "silu"
    LINEAR = "linear"
    SPATIAL_ATTENTION = "spatial_attention"
    TEMPORAL_ATTENTION = "temporal_attention"
    DOWNSAMPLE2X = "downsample2x"
    UPSAMPLE2X = "upsample2x"
    ADD = "add"
    CONCAT = "concat"
    SPLIT = "split"


@dataclass(frozen=True)
class KindInfo:
    domains: frozenset
    arity: int | None
    rf: Mapping[str, float]
    stride: Mapping[str, float] = field(default_factory=lambda: {"h": 1, "w": 1})
    inplace: bool = False


def _rf(**over) -> dict:
    base = {"b": 1, "t": 1, "h": 1, "w": 1}
    base.update(over)
    return base


_S, _T, _B = Domain.SPATIAL, Domain.TEMPORAL, Domain.BOUNDARY

# kernels.py:72-86 -- the receptive-field table is the legality basis for
# slicing (and for sharding across GPUs: an axis with rf 1 can be split).
KIND_INFO: dict[OpKind, KindInfo] = {
    OpKind.CONV2D: KindInfo(frozenset({_S}), 1, _rf(h=3, w=3)),
    OpKind.TEMPORAL_CONV: KindInfo(frozenset({_T}), 1, _rf(t=3)),
    OpKind.GROUP_NORM: KindInfo(frozenset({_S}), 1, _rf(h=FULL, w=FULL), inplace=True),
    OpKind.LAYER_NORM: KindInfo(frozenset({_S, _T}), 1, _rf(), inplace=True),
    OpKind.SILU: KindInfo(frozenset({_S, _T}), 1, _rf(), inplace=True),
    OpKind.LINEAR: KindInfo(frozenset({_S, _T}), 1, _rf()),
    OpKind.SPATIAL_ATTENTION: KindInfo(frozenset({_S}), 1, _rf(h=FULL, w=FULL)),
    OpKind.TEMPORAL_ATTENTION: KindInfo(frozenset({_T}), 1, _rf(t=FULL)),
    OpKind.DOWNSAMPLE2X: KindInfo(frozenset({_S}), 1, _rf(h=2, w=2), stride={"h": 2, "w": 2}),
    OpKind.UPSAMPLE2X: KindInfo(frozenset({_S}), 1, _rf(), stride={"h": 0.5, "w": 0.5}),
    OpKind.ADD: KindInfo(frozenset({_B}), 2, _rf(), inplace=True),
    OpKind.CONCAT: KindInfo(frozenset({_B}), None, _rf()),
    OpKind.SPLIT: KindInfo(frozenset({_B}), 1, _rf()),
}


def scratch_bytes(kind: OpKind, in_shape: Shape5, itemsize: int) -> int:
    """Token-squared score buffer of the attention kinds (kernels.py:89-102)."""
    b, t, _c, h, w = in_shape
    if kind is OpKind.SPATIAL_ATTENTION:
        return b * t * (h * w) ** 2 * itemsize
    if kind is OpKind.TEMPORAL_ATTENTION:
        return b * h * w * t * t * itemsize
    return 0


def output_shape(kind: OpKind, in_shapes: Sequence[Shape5], attrs: Mapping | None = None) -> Shape5:
    """Static output shape; validates arity/extents first (kernels.py:109-163)."""
    attrs = attrs or {}
    info = KIND_INFO[kind]
    n = len(in_shapes)
    if info.arity is None:
        if n < 2:
            raise ShapeMismatch(f"{kind.value} takes at least 2 inputs")
    elif n != info.arity:
        raise ShapeMismatch(f"{kind.value} takes {info.arity} input(s), got {n}")
    s = Shape5(*in_shapes[0])
    if kind in (OpKind.CONV2D, OpKind.TEMPORAL_CONV):
        return s.replace(c=int(attrs["out_channels"]))
    if kind is OpKind.LINEAR:
        return s.replace(c=int(attrs["out_features"]))
    if kind is OpKind.GROUP_NORM:
        g = int(attrs.get("groups", 1))
        if g < 1 or s.c % g:
            raise InvalidParam(f"group_norm groups={g} does not divide channels={s.c}")
        return s
    if kind in (OpKind.LAYER_NORM, OpKind.SILU, OpKind.SPATIAL_ATTENTION, OpKind.TEMPORAL_ATTENTION):
        return s
    if kind is OpKind.DOWNSAMPLE2X:
        if s.h % 2 or s.w % 2:
            raise ShapeMismatch(f"downsample2x needs even h, w; got {s.h}x{s.w}")
        return s.replace(h=s.h // 2, w=s.w // 2)
    if kind is OpKind.UPSAMPLE2X:
        return s.replace(h=2 * s.h, w=2 * s.w)
    if kind is OpKind.ADD:
        a, b = (Shape5(*x) for x in in_shapes)
        if a == b:
            return a
        if a[:3] == b[:3] and (b.h, b.w) == (1, 1):
            return a
        if a[:3] == b[:3] and (a.h, a.w) == (1, 1):
            return b
        raise ShapeMismatch(f"add operands incompatible: {tuple(a)} vs {tuple(b)}")
    if kind is OpKind.CONCAT:
        total = 0
        for sh in in_shapes:
            sh = Shape5(*sh)
            if sh.replace(c=0) != s.replace(c=0):
                raise ShapeMismatch(
                    f"concat operands differ outside channel axis: {tuple(sh)} vs {tuple(s)}")
            total += sh.c
        return s.replace(c=total)
    if kind is OpKind.SPLIT:
        sizes = [int(v) for v in attrs["sizes"]]
        index = int(attrs["index"])
        if sum(sizes) != s.c:
            raise InvalidParam(f"split sizes {sizes} do not sum to channels={s.c}")
        if not 0 <= index < len(sizes):
            raise InvalidParam(f"split index {index} out of range for {len(sizes)} parts")
        return s.replace(c=sizes[index])
    raise InvalidParam(f"unknown kind {kind}")
