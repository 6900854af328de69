"""Error taxonomy of the sliceflow path, kept name-for-name with the reference.

Reference: ``sliceflow/errors.py:8-81``.  ``ValidationError`` subclasses are
user-input problems (CLI exit code 2, ``SPEC.md:556``); everything else is a
runtime failure (exit code 1).  The native library reports failures as integer
status codes; :func:`raise_for_status` maps them back onto this hierarchy so a
caller of the CUDA path sees exactly the exceptions the numpy path raises.
"""

from __future__ import annotations


class SliceflowError(Exception):
    """Root of every error raised by this package (errors.py:8)."""


class ValidationError(SliceflowError):
    """Bad user-supplied value (errors.py:12)."""


class ShapeMismatch(SliceflowError):
    """Incompatible operand extents (errors.py:18)."""


class InvalidParam(ValidationError):
    """Structurally invalid kernel parameter/attribute (errors.py:22)."""


class ZeroNorm(SliceflowError):
    """Cosine similarity of an all-zero tensor (errors.py:26)."""


class InvalidGraph(SliceflowError):
    """Graph invariant violated (errors.py:32)."""


class InvalidConfig(ValidationError):
    """Model/run configuration invariant violated (errors.py:36)."""


class NotAChain(SliceflowError):
    """Segment is not a single-input chain (errors.py:40)."""


class ShapeInferenceFailure(SliceflowError):
    """Static shape inference failed (errors.py:44)."""


class BadSliceCount(ValidationError):
    """Slice count out of range (errors.py:50)."""


class PlanShapeMismatch(SliceflowError):
    """Slice plan does not fit the tensor (errors.py:54)."""


class IncompleteCover(SliceflowError):
    """Sub-features leave gaps (errors.py:58)."""


class OverlappingRegions(SliceflowError):
    """Sub-features overlap (errors.py:62)."""


class PipelineStall(SliceflowError):
    """Pipeline stage ran without its input (errors.py:68)."""


class BadThreshold(ValidationError):
    """Similarity threshold outside (0, 1] (errors.py:72)."""


class ScheduleMismatch(SliceflowError):
    """Step schedule does not match the run's step count (errors.py:76)."""


class TargetUnreachable(ValidationError):
    """No threshold yields the requested key-step count (errors.py:80)."""


class NativeError(SliceflowError):
    """CUDA / NCCL / driver failure inside the native library."""


# Status codes returned by every ``sf_*`` entry point of the C ABI
# (include/sliceflow_b200.h).  Keep in sync with SF_STATUS_* there.
STATUS_OK = 0
STATUS_SHAPE = 1
STATUS_PARAM = 2
STATUS_CUDA = 3
STATUS_UNSUPPORTED = 4

_STATUS_CLASS = {
    STATUS_SHAPE: ShapeMismatch,
    STATUS_PARAM: InvalidParam,
    STATUS_CUDA: NativeError,
    STATUS_UNSUPPORTED: InvalidParam,
}


def raise_for_status(code: int, what: str, detail: str = "") -> None:
    """Raise the reference-equivalent exception for a native status code."""
    if code == STATUS_OK:
        return
    cls = _STATUS_CLASS.get(code, NativeError)
    msg = f"{what}: native status {code}"
    if detail:
        msg += f" ({detail})"
    raise cls(msg)
