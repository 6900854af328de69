"""Memory ledger, pipeline wavefront, NaiveClip chunking and run-report format (CPU).

SPEC.md:320-349 (MemoryLedger, pipeline_schedule, export_timeline) and the
NaiveClip / run-report contracts.  The device
ledger is derived from the compiled plan, so its invariants are checked on
the plan built without a GPU (``plan_memory``).
"""

import csv
import io

import pytest

from paper_2411_01171_b200.errors import InvalidParam
from paper_2411_01171_b200.executor import naive_clip_chunks, pipeline_schedule, plan_memory
from paper_2411_01171_b200.grouping import group_operators
from paper_2411_01171_b200.harness import RunReport
from paper_2411_01171_b200.ledger import MemoryLedger, export_timeline
from paper_2411_01171_b200.slicer import default_temporal_config
from paper_2411_01171_b200.unet import UNetConfig, build_toy_unet


def rows(doc):
    return list(csv.reader(io.StringIO(doc)))


def test_timeline_empty_is_header_only():
    assert rows(export_timeline(MemoryLedger())) == [["tick", "cumulative_bytes", "tag", "is_peak"]]


def test_timeline_single_alloc_free():
    led = MemoryLedger()
    led.alloc(100, "a")
    led.free(100, "a")
    led.assert_closed()
    r = rows(export_timeline(led))
    assert led.peak_bytes == 100
    assert r[1] == ["0", "100", "a", "1"] and r[2] == ["1", "0", "a", "0"]


def test_ledger_rejects_negative_and_unbalanced():
    led = MemoryLedger()
    with pytest.raises(AssertionError):
        led.free(1, "x")
    led = MemoryLedger()
    led.alloc(8, "x")
    with pytest.raises(AssertionError):
        led.assert_closed()
    with pytest.raises(ValueError):
        led.alloc(-1, "y")


@pytest.mark.parametrize("cfg", [
    UNetConfig(channels=4, frames=8, height=32, width=32, base_channels=8, norm_groups=4),
    UNetConfig(channels=4, frames=25, height=72, width=128, base_channels=320, norm_groups=32),
])
def test_plan_ledger_invariants(cfg):
    g, _ = build_toy_unet(cfg)
    gg = group_operators(g, cfg.frames, default_temporal_config(cfg.height, cfg.width))
    mem = plan_memory(g, gg)
    led = mem["ledger"]
    led.assert_closed()
    running, peak = 0, 0
    for i, ev in enumerate(led.events):
        assert ev.tick == i
        running += ev.delta
        assert running >= 0
        peak = max(peak, running)
    assert peak == led.peak_bytes
    # the packed arena can only be at least the live peak
    assert led.peak_bytes <= mem["arena_bytes"]
    # every stored value is charged once and released once
    allocs = [e for e in led.events if e.delta > 0]
    assert len(allocs) == mem["buffers"] and 2 * len(allocs) == len(led.events)


def test_pipeline_schedule_wavefront():
    t = pipeline_schedule(3, 4)
    assert len(t) == 6
    assert t[2] == [(0, 2), (1, 1), (2, 0)]
    assert pipeline_schedule(1, 5) == [[(0, i)] for i in range(5)]
    assert pipeline_schedule(4, 1) == [[(j, 0)] for j in range(4)]
    # the dependency contract: a slice enters stage j+1 only after stage j
    seen = {}
    for tick, pairs in enumerate(pipeline_schedule(5, 7)):
        for j, i in pairs:
            if j:
                assert seen[(j - 1, i)] < tick
            seen[(j, i)] = tick
    with pytest.raises(InvalidParam):
        pipeline_schedule(0, 3)


def test_naive_clip_chunks():
    assert naive_clip_chunks(25, 8) == [(0, 8), (8, 16), (16, 24), (24, 25)]
    assert naive_clip_chunks(8, 2) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    for bad in (0, 8, 9):
        with pytest.raises(InvalidParam):
            naive_clip_chunks(8, bad)


def test_run_report_json_fields():
    rep = RunReport(peak_bytes=10, arena_bytes=4, scratch_bytes=3, wall_ms=1.5, output_checksum=0.25,
                    op_counts={}, schedule=None, similarity_summary=None, mode="naiveclip", static_model_bytes=9,
                    ledger_peak_bytes=7, ticks=12)
    d = rep.to_json_dict()
    for k in ("mode", "peak_bytes", "ticks", "wall_ms", "output_checksum"):
        assert k in d
    assert d["mode"] == "naiveclip" and d["static_model_bytes"] == 9
