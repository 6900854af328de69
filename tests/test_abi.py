"""The C-ABI library loads and exports every symbol include/sliceflow_b200.h declares (CPU)."""

import os
import re

import pytest

from paper_2411_01171_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sliceflow_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(N.EXPORTED)


def test_library_exports_every_symbol():
    if not os.path.exists(N.LIB_PATH):
        from paper_2411_01171_b200.build import build
        build()
    lib = N.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.sf_version() == 1


def test_host_validation_without_gpu():
    """Shape/param validation happens on the host before any launch (kernels.py:327-328)."""
    from paper_2411_01171_b200.errors import InvalidParam, ShapeMismatch
    args = N.GemmArgs()
    args.mode, args.n_outer, args.n_inner, args.cin, args.N, args.batch = 0, 1, 16, 12, 8, 1
    with pytest.raises(ShapeMismatch):
        N.call("sf_gemm", args, None)      # cin % 8 != 0
    args.cin = 16
    with pytest.raises(InvalidParam):
        N.call("sf_gemm", args, None)      # null operands
    with pytest.raises(ShapeMismatch):
        N.call("sf_downsample2x", N.View(None, 8, 0), N.View(None, 8, 0), 1, 3, 4, 8, None)
    with pytest.raises(ShapeMismatch):
        N.call("sf_temporal_attention_core", N.View(None, 8, 0), 8, 16, N.View(None, 8, 0), 1, 65, 4, 8, 1.0, None)


def test_conv_gn_splits_geometry():
    """sf_conv_gn_splits (host-only): two splits per 128-pixel main tile plus one per tail tile, i.e. the
    conv tiling of gemm_tc.cu (w_t = largest power of two <= min(W, 128), tail tiles when H % h_t
    divides h_t) -- the layout the conv epilogue writes and sf_group_norm_finalize reads."""
    if not os.path.exists(N.LIB_PATH):
        from paper_2411_01171_b200.build import build
        build()
    q = lambda h, w: N.query("sf_conv_gn_splits", h, w)   # noqa: E731
    assert q(72, 128) == 144      # C3 L0: 72 one-row tiles
    assert q(36, 64) == 36        # L1: 18 tiles of 2 x 64
    assert q(18, 32) == 9         # L2: 4 tiles of 4 x 32 + a tail tile (rows 16-17 of 2 frames)
    assert q(9, 16) == 3          # L3: 1 tile of 8 x 16 + a tail tile (row 8 of 8 frames)
    assert q(8, 8) == 1           # whole 8x8 frames two to a tile: tail tiles only
    assert q(0, 8) == 0
