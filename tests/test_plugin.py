"""The plugin seam on the unmodified reference (CPU, the device is a
recorder; tests/test_gpu_plugin.py runs the real data path): attaching a
device leaves the reference's report bytes unchanged, and the device sees a
well-formed transition sequence -- every swap-out completes before its
swap-in, every request is released exactly once, and each batch carries the
members' pre-admission cache locations."""

import collections

import pytest

import scenarios
from recorder import Recorder
from paper_2512_14142_b200 import plugin, reference

ref = reference.load()


@pytest.mark.parametrize("name", ["c1b200/6000", "c1/stateful-mlfq/3600/adaptive", "hetero/1/stateful-mlfq",
                                  "fig2/fcfs", "aging/5.0"])
def test_plugin_leaves_reference_bytes_unchanged(name):
    plain = scenarios.run_scenario(ref, name)
    wl, pol, pred, mem, cfg = scenarios.build(ref, name)
    rec = Recorder()
    rep = plugin.run_on_gpu(wl, pol, pred, mem, cfg, rec)
    assert rep.to_json() == plain.to_json()
    assert rep.device["clock"] == "model" and rep.device["batches"] > 0

    state = collections.defaultdict(lambda: "none")   # device-side location per request
    released = collections.Counter()
    for e in rec.log:
        if e[0] == "batch":
            for rid, seg, loc, kv in e[1:]:
                assert loc == state[rid], (rid, loc, state[rid])
                assert (loc == "gpu") == (kv > 0) or loc == "gpu"
                state[rid] = "gpu"
        elif e[0] == "drop":
            assert state[e[1]] == "gpu"
            state[e[1]] = "dropped"
        elif e[0] == "swap_out_begin":
            assert state[e[1]] == "gpu"
            state[e[1]] = "out"
        elif e[0] == "swap_out_done":
            assert state[e[1]] == "out"
            state[e[1]] = "host"
        elif e[0] == "swap_in_begin":
            assert state[e[1]] == "host"
            state[e[1]] = "in"
        elif e[0] == "swap_in_done":
            assert state[e[1]] == "in"
            state[e[1]] = "gpu"
        elif e[0] == "release":
            released[e[1]] += 1
            state[e[1]] = "released"
    assert set(released) == {r.id for r in wl} and set(released.values()) == {1}


def test_no_restated_scheduler_in_the_package():
    """north_star: the scheduler, classification and KV policy remain the
    reference's host code -- the package subclasses it, it does not copy it."""
    from pathlib import Path
    pkg = Path(plugin.__file__).resolve().parent
    assert not (pkg / "host").exists()
    _, eng = plugin.engine_classes()
    assert eng.__mro__[1] is ref.Engine
    for src in pkg.rglob("*.py"):
        text = src.read_text()
        for sym in ("def hrrn_score", "def estimate_waste", "def _pack_greedy", "def execute_batch",
                    "class StatefulMlfqPolicy", "class MemoryModel"):
            assert sym not in text, (src, sym)


def test_pool_size_check_bounds_by_capacity_and_trace():
    """The block-feasibility check (GpuEngine.__init__) needs ceil(peak/16)
    + one partial block per request, peak = min(capacity, the whole trace's
    context): fig2 (capacity 1e6, 12 tokens of context) fits 512 blocks, as
    __graft_entry__.smoke() runs it; a pool short of a block is refused."""
    import math
    import types
    wl, pol, pred, mem, cfg = scenarios.build(ref, "fig2/fcfs")
    rec = Recorder()
    GpuEngine = plugin.engine_classes(ref)[1]
    rec.pool = types.SimpleNamespace(num_blocks=512)
    GpuEngine(wl, pol, pred, mem, cfg, rec)   # accepted
    wl, pol, pred, mem, cfg = scenarios.build(ref, "c1b200/6000")
    peak = min(mem.capacity_tokens, sum(s.n_in + s.n_gen for r in wl for s in r.segments))
    rec.pool = types.SimpleNamespace(num_blocks=math.ceil(peak / 16) + len(wl) - 1)
    with pytest.raises(ref.ConfigError):
        GpuEngine(wl, pol, pred, mem, cfg, rec)
    rec.pool.num_blocks += 1
    wl, pol, pred, mem, cfg = scenarios.build(ref, "c1b200/6000")
    GpuEngine(wl, pol, pred, mem, cfg, rec)


def test_report_with_device_audits_loads_in_the_reference():
    """Opt-in export: the device counters under
    audits["device"]; the reference's RunReport.from_dict and compare()
    accept it, and everything but that key equals the default bytes."""
    import json
    name = "c1b200/6000"
    wl, pol, pred, mem, cfg = scenarios.build(ref, name)
    rep = plugin.run_on_gpu(wl, pol, pred, mem, cfg, Recorder())
    js = plugin.report_json_with_device(rep)
    d = json.loads(js)
    assert d["audits"]["device"]["batches"] == rep.device["batches"]
    back = ref.RunReport.from_dict(d)
    assert back.audits["device"]["clock"] == "model"
    del d["audits"]["device"]
    assert ref.RunReport.from_dict(d).to_json() == rep.to_json()
    table = ref.compare({"b200": back, "reference": scenarios.run_scenario(ref, name)}, baseline="reference")
    assert table is not None


def test_calibrated_prefill_profile_is_valid_for_the_reference():
    """Launch-bound prefill points can measure out of order; the calibration
    keeps the running maximum so the reference's PrefillProfile (which
    requires non-decreasing latencies, predictor.py:47-57) accepts them."""
    from paper_2512_14142_b200.gpu import calibrate
    raw = [[32, 3.4e-4], [64, 3.3e-4], [128, 5.7e-3], [256, 5.6e-3], [512, 9.0e-3]]
    prof = calibrate.monotone_profile(raw)
    assert [n for n, _ in prof] == [32, 64, 128, 256, 512]
    assert all(a[1] <= b[1] for a, b in zip(prof, prof[1:]))
    assert prof[1][1] == 3.4e-4 and prof[4][1] == 9.0e-3
    cal = {"predictor": {"prefill_profile": prof, "decode_seconds_per_token": 3.1e-3, "api_latency_means": None}}
    pred = calibrate.predictor_from_calibration(ref, cal)
    assert pred.prefill_seconds(64) == pytest.approx(3.4e-4)
    with pytest.raises(ref.ConfigError):
        calibrate.predictor_from_calibration(ref, {"predictor": dict(cal["predictor"], prefill_profile=raw)})
