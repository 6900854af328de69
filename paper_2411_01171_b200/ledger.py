"""Device memory ledger (SPEC.md:320-323 MemoryLedger, :344-349 export_timeline).

The reference's ledger (``ledger.py:25-71``) is an event sink its CPU executor
charges while it runs.  On the device every allocation is decided before the
run: the arena offsets come from a liveness-interval packing of the schedule
and the slice scratch is one fixed region.  So the ledger here is *derived*
from the compiled plan -- one charge when a stored value is defined, one
release after its last consumer, the scratch charged for the whole
evaluation -- and carries the same invariants: the running total never goes
negative, the peak is the maximum prefix sum, and every charge is released by
the end (``assert_closed``).  Payload bytes only, like the reference
(no allocator fragmentation modelling).
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass


@dataclass(frozen=True)
class LedgerEvent:
    tick: int       # monotonic event index
    delta: int      # signed bytes
    tag: str        # value / region label


class MemoryLedger:
    """Ordered (tick, delta, tag) events with running and peak totals."""

    def __init__(self, summary: dict | None = None):
        self.events: list[LedgerEvent] = []
        self.current_bytes = 0
        self.peak_bytes = 0
        # device facts next to the event model (arena / scratch / torch peak / static model)
        self.summary: dict = dict(summary or {})

    def _push(self, delta: int, tag: str) -> None:
        total = self.current_bytes + delta
        if total < 0:
            raise AssertionError(f"ledger below zero after {tag!r} ({total} bytes)")
        self.current_bytes = total
        self.peak_bytes = max(self.peak_bytes, total)
        self.events.append(LedgerEvent(len(self.events), delta, tag))

    def alloc(self, nbytes: int, tag: str) -> None:
        if nbytes < 0:
            raise ValueError(f"negative allocation for {tag!r}")
        self._push(int(nbytes), tag)

    def free(self, nbytes: int, tag: str) -> None:
        if nbytes < 0:
            raise ValueError(f"negative release for {tag!r}")
        self._push(-int(nbytes), tag)

    def assert_closed(self) -> None:
        if self.current_bytes:
            raise AssertionError(f"ledger not closed: {self.current_bytes} bytes still charged")

    # the executor used to return a plain dict of device byte counts; keep that view
    def __getitem__(self, key):
        return self.summary[key]

    def get(self, key, default=None):
        return self.summary.get(key, default)


def export_timeline(ledger: MemoryLedger) -> str:
    """CSV rows (tick, cumulative_bytes, tag, is_peak); the first row reaching the peak is flagged."""
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(["tick", "cumulative_bytes", "tag", "is_peak"])
    total, seen_peak = 0, False
    for ev in ledger.events:
        total += ev.delta
        hit = not seen_peak and ledger.peak_bytes > 0 and total == ledger.peak_bytes
        seen_peak = seen_peak or hit
        w.writerow([ev.tick, total, ev.tag, int(hit)])
    return out.getvalue()
