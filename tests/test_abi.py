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
