"""Measured clock on CPU with a recorder data path: per-member durations come
from the device, and swaps share one host link (FIFO channel, SURVEY.md 8(f)
item 2): a swap starts when the previous one has finished, so transfer
intervals never overlap, and each completes after its own measured time.
With the serial cost model members are launched one at a time (ADVICE r1:
overlapping batch-relative times must never be chained)."""

import scenarios
from recorder import Recorder
from paper_2512_14142_b200 import plugin, reference

ref = reference.load()
_, GpuEngine = plugin.engine_classes()


class LinkRecorder(Recorder):
    def __init__(self, **kw):
        super().__init__(batch_seconds=0.05, **kw)
        self.swaps = []


class RecordingEngine(GpuEngine):
    def _link_delay(self, state, direction):
        d = super()._link_delay(state, direction)
        self.datapath.swaps.append((self.now, d))
        return d


def test_measured_swaps_share_one_fifo_link():
    wl, pol, pred, mem, cfg = scenarios.build(ref, "c1b200/6000")
    dp = LinkRecorder()
    rep = RecordingEngine(wl, pol, pred, mem, cfg, dp, clock="measured").run()
    assert len(dp.swaps) > 20
    end_prev = 0.0
    for now, delay in dp.swaps:
        end = now + delay
        start = end - dp.swap_s
        assert start >= now - 1e-12                       # never before it was issued
        assert start >= end_prev - 1e-9                   # never overlaps the previous transfer
        assert abs(start - max(now, end_prev)) < 1e-9     # starts as soon as the link is free
        end_prev = end
    assert any(delay > dp.swap_s + 1e-9 for _, delay in dp.swaps)   # some swaps did queue
    assert ref.audit_time_decomposition(rep) <= 1e-9
    assert plugin.requests_per_second(rep) > 0


def test_model_clock_ignores_device_durations():
    """Model clock: the recorder's durations are never consulted (decisions stay the reference's)."""
    wl, pol, pred, mem, cfg = scenarios.build(ref, "c1b200/6000")
    rep = RecordingEngine(wl, pol, pred, mem, cfg, LinkRecorder(), clock="model").run()
    assert rep.to_json() == scenarios.run_scenario(ref, "c1b200/6000").to_json()


def test_serial_measured_launches_members_one_by_one():
    wl, pol, pred, mem, cfg = scenarios.build(ref, "decomp/fcfs/serial/adaptive/40000")
    dp = LinkRecorder()
    rep = RecordingEngine(wl, pol, pred, mem, cfg, dp, clock="measured").run()
    batches = [e for e in dp.log if e[0] == "batch"]
    assert batches and all(len(b) == 2 for b in batches)     # one member per launch
    # serial: spans of one batch abut (start_i+1 == end_i), each as long as its own launch
    computes = [s for s in rep.gantt if s.kind == "compute"]
    assert all(abs((s.end - s.start) - 0.05) < 1e-9 for s in computes)
    assert ref.audit_time_decomposition(rep) <= 1e-9
