"""The B200 data path behind the reference's own engine (the product path).

The reference (``agentsched``, pkg/src/agentsched) exposes a duck-typed plugin
API and no FFI. :func:`engine_classes` builds two subclasses
of *its* classes, overriding only documented seams; everything else --
event loop, policies, KV policy, memory model, report -- is the reference's
code, imported unmodified (``reference.load()``):

* ``KvCacheManager`` (kvcache.py:152-292): every transition first runs the
  reference method unchanged, then forwards to the device (``KvDataPath``),
  i.e. the eight transitions of SURVEY.md Appendix C. In the measured clock
  ``swap_out_seconds`` / ``swap_in_seconds`` (kvcache.py:227-228, 252-253)
  return the measured K1/K2 time on a FIFO host link instead of
  ``tokens / bandwidth``.
* ``Engine`` (simulator.py:101-481): ``policy.build_next_batch`` (called
  first in ``_try_start_batch``, simulator.py:340-342) is wrapped to record
  the plan; ``_actual_seconds`` (simulator.py:329-337) is called once per
  plan entry *before* any member's location flips, so on its first call the
  whole batch -- with every member's pre-admission cache location -- is
  launched on the device. Model clock: the reference's durations are
  returned (report bytes unchanged). Measured clock: the CUDA-event time from
  the batch start to the decode step that retires each member.

Clock modes:
  ``model``     the virtual clock advances by the reference cost model while
                the GPU executes every plan; decisions and ``RunReport`` bytes
                are identical to the reference's.
  ``measured``  segment and swap durations come from the device; API waits
                stay virtual. Swaps share one host link: a transfer starts
                when the previous one has finished (the FIFO channel
                SPEC.md:323 promises), as the data
                path runs them on its one swap stream. With the ``serial``
                cost model (simulator.py:90-95) members run one after another,
                so each is launched as its own batch in plan order and its
                own time is chained; ``parallel-max`` launches one batch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Any, Optional

from . import reference

CLOCKS = ("model", "measured")


@dataclass(frozen=True)
class AdmittedMember:
    """What the device needs to run one member of a batch: the state (still
    pre-admission), its segment and its cache location / tokens before the
    admission flip (simulator.py:365-369)."""

    state: Any
    segment_index: int
    prior_location: Any
    prior_kv_tokens: int


def requests_per_second(report) -> float:
    """Completed requests over (last finish - first arrival). The reference
    defines no throughput metric."""
    first = min(r.arrival for r in report.per_request)
    last = max(r.finish for r in report.per_request)
    return len(report.per_request) / (last - first) if last > first else math.inf


_CLASSES: dict = {}


def engine_classes(ns=None):
    """``(GpuKvCacheManager, GpuEngine)`` built on namespace ``ns`` (default:
    the reference package). Cached per namespace."""
    ns = ns or reference.load()
    hit = _CLASSES.get(id(ns))
    if hit is not None:
        return hit
    Phase = ns.scheduler.Phase
    SERIAL = ns.SERIAL

    class GpuKvCacheManager(ns.KvCacheManager):
        device = None    # KvDataPath (or any object with the same seams)
        engine = None    # the GpuEngine owning the clock

        def on_api_yield(self, state, predicted_api_seconds, batch_demand_tokens, now):
            action = super().on_api_yield(state, predicted_api_seconds, batch_demand_tokens, now)
            if action is ns.CacheAction.DISCARD:
                self.device.drop(state)
            elif action is ns.CacheAction.SWAP:
                self.device.swap_out_begin(state)
            return action

        def swap_out_seconds(self, state):
            if self.engine is not None and self.engine.clock == "measured":
                return self.engine._link_delay(state, "out")
            return super().swap_out_seconds(state)

        def complete_swap_out(self, state):
            super().complete_swap_out(state)
            self.device.swap_out_done(state)

        def try_begin_swap_in(self, state):
            ok = super().try_begin_swap_in(state)
            if ok:
                self.device.swap_in_begin(state)
            return ok

        def swap_in_seconds(self, state):
            if self.engine is not None and self.engine.clock == "measured":
                return self.engine._link_delay(state, "in")
            return super().swap_in_seconds(state)

        def complete_swap_in(self, state):
            super().complete_swap_in(state)
            self.device.swap_in_done(state)

        def release_request(self, state):
            where = state.cache_location
            super().release_request(state)
            self.device.release(state, where)

        def force_discard(self, state, now):
            super().force_discard(state, now)
            self.device.drop(state)

    class GpuEngine(ns.Engine):
        def __init__(self, workload, policy, predictor, memory, config, datapath, clock: str = "model",
                     device_audit: bool = True):
            if clock not in CLOCKS:
                raise ns.ConfigError(f"unknown clock {clock!r}; choose from {CLOCKS}")
            super().__init__(workload, policy, predictor, memory, config)
            pool = getattr(datapath, "pool", None)
            if pool is not None:
                # token-exact admission must always be block-feasible: every
                # resident request may round up to one partial block. Resident
                # tokens never exceed the capacity nor the whole trace's context.
                trace_tokens = sum(s.n_in + s.n_gen for r in self.workload for s in r.segments)
                peak = min(memory.capacity_tokens, trace_tokens)
                need = math.ceil(peak / 16) + len(self.workload)
                if pool.num_blocks < need:
                    raise ns.ConfigError(f"KV pool of {pool.num_blocks} blocks cannot back "
                                         f"{peak} resident tokens (capacity {memory.capacity_tokens}) with "
                                         f"{len(self.workload)} requests (needs {need})")
            self.manager = GpuKvCacheManager(memory, predictor, mode=config.cache_mode)
            self.manager.device = datapath
            self.manager.engine = self
            self.datapath = datapath
            self.clock = clock
            self.device_audit = device_audit
            datapath.measure = clock == "measured"
            self.device_report: Optional[dict] = None
            self._link_free = 0.0     # measured clock: when the host link finishes its queued swaps
            self._plan_entries = ()
            self._entry = 0
            self._durations = None
            build = policy.build_next_batch

            def recorded(free_tokens, now, max_segments=None):
                plan = build(free_tokens, now, max_segments)
                self._plan_entries = plan.entries
                self._entry = 0
                self._durations = None
                return plan

            policy.build_next_batch = recorded

        # -- seams -------------------------------------------------------------

        def _launch_plan(self):
            members = []
            for request_id, segment_index in self._plan_entries:
                st = self.states[request_id]
                if st.phase is not Phase.WAITING_READY or st.current_segment != segment_index:
                    return None   # the reference raises ProtocolError on this entry; launch nothing
                members.append(AdmittedMember(st, segment_index, st.cache_location, st.kv_tokens))
            if self.clock == "measured" and self.config.cost_model == SERIAL and len(members) > 1:
                return [self.datapath.launch_batch([m])[0] for m in members]
            out = self.datapath.launch_batch(members)
            return out if self.clock == "measured" else None

        def _actual_seconds(self, state):
            seconds = super()._actual_seconds(state)
            if self._entry == 0:
                self._durations = self._launch_plan()
            i = self._entry
            self._entry += 1
            return self._durations[i] if self._durations is not None else seconds

        def _link_delay(self, state, direction):
            start = max(self.now, self._link_free)
            self._link_free = start + self.datapath.swap_seconds(state, direction)
            return self._link_free - self.now

        def _try_start_batch(self):
            super()._try_start_batch()
            if self.device_audit and self._active_batch is not None:
                self.datapath.audit(self.states.values())

        def run(self):
            report = super().run()
            self.datapath.synchronize()
            if self.device_audit:
                self.datapath.audit(self.states.values())
            self.device_report = dict(self.datapath.summary(), clock=self.clock)
            report.device = self.device_report   # an attribute only: to_json() stays the reference's
            return report

    _CLASSES[id(ns)] = (GpuKvCacheManager, GpuEngine)
    return GpuKvCacheManager, GpuEngine


def report_json_with_device(report) -> str:
    """RunReport v1 JSON (metrics.py:115-126) with the device counters under
    ``audits["device"]`` -- opt-in: the default
    ``report.to_json()`` stays byte-identical to the reference, this one
    still loads with the reference's ``RunReport.from_dict`` so its
    ``gantt`` / ``compare`` tooling (cli.py:561-721) works on B200 runs."""
    import json
    d = report.to_dict()
    dev = getattr(report, "device", None)
    if dev is not None:
        d["audits"] = dict(d["audits"], device=dict(dev))
    return json.dumps(d, sort_keys=True, indent=2)


def run_on_gpu(workload, policy, predictor, memory, config, datapath, clock: str = "model", ns=None):
    """The reference's ``run()`` (simulator.py:484-494) with the B200 data
    path attached."""
    _, engine = engine_classes(ns)
    return engine(workload, policy, predictor, memory, config, datapath, clock).run()


def run_reference_on_gpu(agentsched, datapath, workload, policy, predictor, memory, config, clock="model"):
    """Same as :func:`run_on_gpu` with an explicit reference module."""
    return run_on_gpu(workload, policy, predictor, memory, config, datapath, clock, ns=agentsched)
