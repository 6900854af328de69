"""ctypes binding of the C ABI in ``include/sliceflow_b200.h``.

The library is loaded once, lazily.  There is no fallback: if the ``.so`` is
missing or fails to load, every compute entry point raises
:class:`NativeError` -- the product path never substitutes host code.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_sliceflow_b200.so")

i32, i64, f32, vp = C.c_int32, C.c_int64, C.c_float, C.c_void_p


class View(C.Structure):
    """sf_view_t: row (o, i) at ptr + (o*ostride + i)*ld elements."""

    _fields_ = [("ptr", vp), ("ld", i64), ("ostride", i64)]


NULL_VIEW = View(None, 0, 0)


class GemmArgs(C.Structure):
    _fields_ = [
        ("mode", i32), ("n_outer", i32), ("n_inner", i32),
        ("H", i32), ("W", i32), ("T", i32),
        ("cin", i32), ("N", i32), ("batch", i32),
        ("a", View), ("a_bstride", i64),
        ("w", vp), ("w_kmajor", i32), ("w_ld", i64), ("w_bstride", i64),
        ("alpha", f32),
        ("bias", vp), ("rowbias", vp), ("rowbias_stride", i64),
        ("act", i32),
        ("res", View), ("res_bstride", i64),
        ("out", View), ("out_bstride", i64),
        ("out_fp32", i32), ("backend", i32),
        ("rowstats", vp), ("colvec", vp),
        ("gn_partial", vp),
    ]


GEMM_PLAIN, GEMM_CONV3X3, GEMM_TCONV3 = 0, 1, 2
GEMM_NO_PAIR = 4          # sf_gemm_args.backend flag: single-CTA tcgen05 tiles only
ACT_NONE, ACT_SILU = 0, 1

# name -> argtypes (restype is sf_status = int unless listed in _RESTYPE)
_PROTOS = {
    "sf_gemm": [C.POINTER(GemmArgs), vp],
    "sf_gemm_backend": [C.POINTER(GemmArgs)],
    "sf_group_norm_workspace": [i32, i32, i32],
    "sf_group_norm_stats": [View, i32, i32, i32, i32, f32, vp, vp, vp, vp],
    "sf_conv_gn_splits": [i32, i32],
    "sf_conv_gn_partials": [View, i32, i32, i32, i32, vp, vp],
    "sf_group_norm_finalize": [vp, i32, i32, i32, i32, i32, f32, vp, vp, vp],
    "sf_group_norm_project": [View, i32, i32, i32, i32, vp, vp, vp, vp, i32, vp, i32, vp, i64, vp],
    "sf_group_norm_apply": [View, View, i32, i32, i32, i32, vp, vp, vp, vp, i32, vp],
    "sf_layer_norm": [View, View, i32, i32, i32, vp, vp, f32, i32, vp],
    "sf_layer_norm_stats": [View, i32, i32, i32, f32, vp, vp],
    "sf_silu": [View, View, i32, i32, i32, vp],
    "sf_add": [View, View, View, i32, i32, i32, i32, vp],
    "sf_copy_rows": [View, View, i32, i32, i32, vp],
    "sf_downsample2x": [View, View, i32, i32, i32, i32, vp],
    "sf_upsample2x": [View, View, i32, i32, i32, i32, vp],
    "sf_downsample2x_gn": [View, View, i32, i32, i32, i32, i32, vp, i32, vp, i32, vp],
    "sf_upsample2x_gn": [View, View, i32, i32, i32, i32, i32, vp, i32, i32, vp],
    "sf_softmax_rows": [vp, i64, vp, i64, i64, i32, vp],
    "sf_flash_supported": [i32, i32],
    "sf_spatial_attention_core": [View, View, vp, View, i32, i32, i32, f32, vp],
    "sf_temporal_attention_core": [View, i32, i32, View, i32, i32, i32, i32, f32, vp],
    "sf_temporal_attention_fused_supported": [i32, i32],
    "sf_temporal_attention_fused": [View, vp, View, View, i32, i32, i32, i32, vp],
    "sf_conv3x3_smallcin": [vp, i32, i32, i32, i32, vp, vp, i32, View, vp],
    "sf_conv3x3_smallcin_gn": [vp, i32, i32, i32, i32, vp, vp, i32, View, i32, vp, vp],
    "sf_conv3x3_tapsum": [vp, i32, i32, i32, i32, i32, vp, View, vp],
    "sf_gemv_f32": [vp, vp, vp, vp, i32, i32, vp],
    "sf_bcthw_to_rows_f32": [vp, vp, i32, i32, i32, vp],
    "sf_rows_to_bcthw_f32": [vp, vp, i32, i32, i32, vp],
    "sf_axpy_f32": [vp, vp, f32, i64, vp],
    "sf_dot3_workspace": [i64],
    "sf_dot3_bf16": [vp, vp, i64, vp, vp, vp],
    "sf_gram_workspace": [i32, i64],
    "sf_gram_bf16": [vp, i32, i64, vp, vp, vp],
    "sf_last_error": [],
    "sf_version": [],
}
_RESTYPE = {
    "sf_group_norm_workspace": i64,
    "sf_dot3_workspace": i64,
    "sf_gram_workspace": i64,
    "sf_gemm_backend": i32,
    "sf_conv_gn_splits": i32,
    "sf_flash_supported": i32,
    "sf_temporal_attention_fused_supported": i32,
    "sf_last_error": C.c_char_p,
    "sf_version": i32,
}
EXPORTED = tuple(_PROTOS)

_lib = None


def load(path: str | None = None) -> C.CDLL:
    """Load (once) and type the library; raises NativeError if absent.

    ``SF_LIB`` names another build of the same library (same-box A/B of kernel variants)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("SF_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise NativeError(f"native library {path} not built; run paper_2411_01171_b200.build.build()")
    try:
        lib = C.CDLL(path)
    except OSError as exc:
        raise NativeError(f"cannot load {path}: {exc}") from exc
    for name, args in _PROTOS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke an sf_* launcher and map its status onto the error hierarchy."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc:
        raise_for_status(rc, name, (lib.sf_last_error() or b"").decode(errors="replace"))


def query(name: str, *args):
    return getattr(load(), name)(*args)
