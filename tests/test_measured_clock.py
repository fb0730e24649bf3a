"""Measured-clock engine on CPU with a stub data path: per-member durations
come from the device, and swaps share one host link (FIFO channel, SURVEY.md
8(f) item 2): a swap starts when the previous one has finished, so transfer
intervals never overlap, and each completes after its own measured time."""

import scenarios
from paper_2512_14142_b200 import host
from paper_2512_14142_b200.gpu.engine import GpuEngine


class StubDataPath:
    """Device seams of KvDataPath with fixed durations (no GPU)."""

    def __init__(self, batch_s=0.05, swap_s=0.2):
        self.measure = False
        self.batch_s, self.swap_s = batch_s, swap_s
        self.swaps = []   # (issue time, delay returned) per swap

    def launch_batch(self, members):
        return [self.batch_s * (1 + i % 3) for i, _ in enumerate(members)] if self.measure else None

    def swap_seconds(self, state, direction):
        return self.swap_s

    def audit(self, states):
        pass

    def synchronize(self):
        pass

    def summary(self):
        return {}

    def drop(self, state):
        pass

    def swap_out_begin(self, state):
        pass

    def swap_out_done(self, state):
        pass

    def swap_in_begin(self, state):
        pass

    def swap_in_done(self, state):
        pass

    def release(self, state, where):
        pass


class RecordingEngine(GpuEngine):
    def _swap_delay(self, state, direction):
        d = super()._swap_delay(state, direction)
        self.datapath.swaps.append((self.now, d))
        return d


def test_measured_swaps_share_one_fifo_link():
    wl, pol, pred, mem, cfg = scenarios.build(host, "c1b200/6000")
    dp = StubDataPath()
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
    assert host.audit_time_decomposition(rep) <= 1e-9
    assert rep.requests_per_second() > 0


def test_model_clock_ignores_device_durations():
    """Model clock: the stub's durations are never consulted (decisions stay the reference's)."""
    wl, pol, pred, mem, cfg = scenarios.build(host, "c1b200/6000")
    dp = StubDataPath()
    rep = RecordingEngine(wl, pol, pred, mem, cfg, dp, clock="model").run()
    ref = scenarios.run_scenario(host, "c1b200/6000")
    assert rep.to_json() == ref.to_json()
