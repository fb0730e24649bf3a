"""The plugin seam on the unmodified reference: attaching a device to the
reference's own Engine/KvCacheManager (paper_2512_14142_b200.plugin) drives
exactly the same sequence of device transitions as this package's engine,
and leaves the reference's report bytes unchanged. CPU-only: the device is a
recorder here; tests/test_gpu_plugin.py runs the real data path."""

import hashlib
import sys
from pathlib import Path

import pytest

import scenarios
from paper_2512_14142_b200 import host, plugin


def _reference():
    for cand in ("/root/reference/pkg/src", str(Path(__file__).resolve().parent.parent / "baseline" / "_ref")):
        if Path(cand, "agentsched").exists():
            if cand not in sys.path:
                sys.path.insert(0, cand)
            import agentsched
            return agentsched
    pytest.skip("reference package not available")


class Recorder:
    def __init__(self):
        self.log = []

    def _rec(self, name, st, *extra):
        self.log.append((name, st.spec.id, st.kv_tokens) + extra)

    def drop(self, st):
        self._rec("drop", st)

    def swap_out_begin(self, st):
        self._rec("swap_out_begin", st)

    def swap_out_done(self, st):
        self._rec("swap_out_done", st)

    def swap_in_begin(self, st):
        self._rec("swap_in_begin", st)

    def swap_in_done(self, st):
        self._rec("swap_in_done", st)

    def release(self, st, where):
        self._rec("release", st, where.value)

    def launch_batch(self, members):
        self.log.append(("batch",) + tuple((m.state.spec.id, m.segment_index, m.prior_location.value,
                                            m.prior_kv_tokens) for m in members))

    def synchronize(self):
        pass

    def audit(self, states):
        pass


class HostWithDevice(host.Engine):
    def _launch_batch(self, members):
        self.device.launch_batch(members)
        return None


@pytest.mark.parametrize("name", ["c1b200/6000", "c1/stateful-mlfq/3600/adaptive", "hetero/1/stateful-mlfq"])
def test_reference_engine_with_plugin_matches_ours(name, golden):
    ref = _reference()
    wl, pol, pred, mem, cfg = scenarios.build(ref, name)
    rec_ref = Recorder()
    rep_ref = plugin.run_reference_on_gpu(ref, rec_ref, wl, pol, pred, mem, cfg)
    assert hashlib.sha256(rep_ref.to_json().encode()).hexdigest() == golden[name]["sha256"]

    wl, pol, pred, mem, cfg = scenarios.build(host, name)
    rec_ours = Recorder()
    rep = HostWithDevice(wl, pol, pred, mem, cfg, device=rec_ours).run()
    assert rep.to_json() == rep_ref.to_json()
    assert rec_ours.log == rec_ref.log
    kinds = {e[0] for e in rec_ref.log}
    assert "batch" in kinds and "release" in kinds
