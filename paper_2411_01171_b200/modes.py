"""Execution modes (reference ``grouping.py:343`` imports ``executor.ExecMode``;
values from the CLI contract ``SPEC.md:529-536``)."""

from __future__ import annotations

from enum import Enum


class ExecMode(str, Enum):
    REFERENCE = "reference"      # unsliced, ungrouped walk of the topo order
    SLICED_LOOP = "slicedloop"   # grouped, slice-by-slice (paper Fig. 5b)
    PIPELINED = "pipelined"      # grouped, wavefront over slices (paper Fig. 5c)
    NAIVE_CLIP = "naiveclip"     # clip-by-clip baseline (paper §3) -- out of scope here
