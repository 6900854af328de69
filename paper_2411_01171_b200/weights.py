"""Named weight arrays per operator plus the SLFW file format.

Reference: ``sliceflow/kernels.py:397-465``.  File layout (little endian):
``b"SLFW"`` | uint32 header length | UTF-8 JSON ``{"entries": [{op, name,
shape, offset}, ...]}`` | raw float32 payload.  Entries are written sorted by
(op, name) so two saves of the same bundle are byte-identical, which lets the
parity tests compare files written by the reference and by this package.
"""

from __future__ import annotations

import json
import struct
from typing import Mapping

import numpy as np

from .errors import InvalidParam
from .tensor import resolve_dtype

MAGIC = b"SLFW"


class WeightBundle:
    """``{param_ref: {name: ndarray}}`` (kernels.py:400-427)."""

    def __init__(self, entries: dict[str, dict[str, np.ndarray]] | None = None):
        self.entries: dict[str, dict[str, np.ndarray]] = entries if entries is not None else {}

    def add(self, key: str, **arrays: np.ndarray) -> None:
        self.entries[key] = {k: np.asarray(v) for k, v in arrays.items()}

    def get(self, key: str) -> Mapping[str, np.ndarray]:
        try:
            return self.entries[key]
        except KeyError:
            raise InvalidParam(f"weight bundle has no entry {key!r}") from None

    def astype(self, dtype) -> "WeightBundle":
        dt = resolve_dtype(dtype)
        return WeightBundle({k: {n: a.astype(dt) for n, a in g.items()} for k, g in self.entries.items()})

    def nbytes(self) -> int:
        return sum(a.nbytes for g in self.entries.values() for a in g.values())

    def param_count(self) -> int:
        return sum(a.size for g in self.entries.values() for a in g.values())

    # -- SLFW ----------------------------------------------------------------

    def to_bytes(self) -> bytes:
        header, chunks, off = [], [], 0
        for op in sorted(self.entries):
            for name in sorted(self.entries[op]):
                arr = np.ascontiguousarray(self.entries[op][name], dtype="<f4")
                header.append({"op": op, "name": name, "shape": list(arr.shape), "offset": off})
                raw = arr.tobytes()
                chunks.append(raw)
                off += len(raw)
        head = json.dumps({"entries": header}).encode("utf-8")
        return MAGIC + struct.pack("<I", len(head)) + head + b"".join(chunks)

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.to_bytes())

    @classmethod
    def from_bytes(cls, blob: bytes) -> "WeightBundle":
        if blob[:4] != MAGIC:
            raise InvalidParam(f"not a weight bundle: bad magic {blob[:4]!r}")
        (hlen,) = struct.unpack_from("<I", blob, 4)
        header = json.loads(blob[8:8 + hlen].decode("utf-8"))
        payload = memoryview(blob)[8 + hlen:]
        out = cls()
        for e in header["entries"]:
            shape = tuple(e["shape"])
            count = int(np.prod(shape)) if shape else 1
            arr = np.frombuffer(payload, dtype="<f4", count=count, offset=e["offset"]).reshape(shape)
            out.entries.setdefault(e["op"], {})[e["name"]] = arr.astype(np.float32)
        return out

    @classmethod
    def load(cls, path) -> "WeightBundle":
        with open(path, "rb") as fh:
            return cls.from_bytes(fh.read())
