"""Global multi-replica scheduler (8(e)).

The reference runs ONE engine over one memory model (simulator.py:101-481)
and lists cross-GPU placement as a non-goal. This module gives
N replicas -- one B200 each -- one scheduling view: every request is placed
at its arrival instant on the replica with the most free KV tokens net of
commitments -- ``MemoryModel.free_tokens`` (kvcache.py:110-112) minus the
``kv_demand`` (scheduler.py:123-132) of the replica's unfinished requests,
i.e. the caches it must still bring back from the host, recompute or grow
(ties: fewer unfinished requests, then the lower replica index; plain free
tokens let a replica whose caches sit swapped out look empty and pile up
requests, tools/placement_probe.py) -- and from then on it is scheduled by
that replica's own, unmodified reference policy, KV policy and memory model.

The replicas advance in lockstep on one virtual clock, so a placement sees
every replica's state at the arrival instant. Each replica is the
reference's ``Engine`` (or the plugin's ``GpuEngine`` when a data path is
attached) with its event loop (simulator.py:144-181) split into steps:

* before placing the arrivals of time t, every replica has processed all of
  its events before t; the arrivals of t are pushed into their replicas'
  queues and processed with the replica's other events of t, in the
  reference's tie order (simulator.py:55-61);
* arrivals are global events: a replica does not break a memory deadlock
  (``_force_progress``, simulator.py:387-421) while arrivals remain to be
  placed anywhere, as the single engine does not while an arrival is queued;
  once the last arrival is placed an idle, deadlocked replica resolves at
  that instant.

With N = 1 this is exactly the reference's ``run()``: same event order,
report bytes identical (tests/test_cluster.py). Decisions depend only on
the virtual clock, so every process of a multi-GPU job can run the same
cluster schedule on the host and execute only its own replica's batches on
its GPU (``device_for``); no collective is needed (bench.py).
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

from . import reference

PLACEMENTS = ("free-tokens", "least-requests", "round-robin")


def _step_class(base):
    """``base`` (the reference Engine or the plugin's GpuEngine) with its
    event loop split into steps."""

    class Replica(base):
        def begin(self):
            self.workload = []            # the requests placed here, in (arrival, id) order
            self.more_arrivals = True

        def admit(self, spec):
            ns = self._ns
            self.states[spec.id] = ns.RequestState(spec=spec)
            self.workload.append(spec)
            self._push(spec.arrival_time, ns.simulator.EventKind.ARRIVAL, spec.id)

        def next_time(self):
            return self._heap[0][0] if self._heap else math.inf

        def step(self):
            """One iteration of Engine.run's loop (simulator.py:147-179)."""
            ns = self._ns
            EK = ns.simulator.EventKind
            time = self._heap[0][0]
            self.now = time
            while self._heap and self._heap[0][0] == time:
                _, kind_value, request_id, _, payload = heapq.heappop(self._heap)
                self._events_processed += 1
                kind = EK(kind_value)
                if kind is EK.ARRIVAL:
                    self._on_arrival(request_id)
                elif kind is EK.SEGMENT_DONE:
                    self._on_segment_done(request_id, payload)
                elif kind is EK.BATCH_DONE:
                    self._on_batch_done()
                elif kind is EK.API_RETURN:
                    self._on_api_return(request_id)
                elif kind is EK.SWAP_DONE:
                    self._on_swap_done(request_id, payload)
            self._settle()

        def _settle(self):
            self._drain_resume_queue()
            if self._active_batch is None:
                self._try_start_batch()
            if self._active_batch is None and not self._heap and not self.more_arrivals:
                self._force_progress()
            if self.config.audit_memory:
                self._ns.kvcache.audit_conservation(self.memory, self.states.values())

        def deadlocked(self):
            return (self._active_batch is None and not self._heap
                    and any(not st.done for st in self.states.values()))

        def poke(self, now):
            """The last arrival has been placed (elsewhere): an idle replica
            with unfinished requests settles at that instant."""
            self.now = max(self.now, now)
            self._settle()

        def finish(self):
            """The end of Engine.run (simulator.py:181-193) and of the
            plugin's GpuEngine.run; None for a replica that got no request."""
            ns = self._ns
            if not self.workload:
                return None
            stuck = sorted(st.spec.id for st in self.states.values() if not st.done)
            if stuck:
                raise ns.SimulationError(
                    f"replica drained with {len(stuck)} unfinished requests: {stuck[:10]}")
            if self.memory.resident_tokens != 0 or self.memory.host_tokens != 0:
                raise ns.SimulationError(
                    f"token leak at end of run: resident={self.memory.resident_tokens} "
                    f"host={self.memory.host_tokens}")
            report = self._build_report()
            dp = getattr(self, "datapath", None)
            if dp is not None:
                dp.synchronize()
                if self.device_audit:
                    dp.audit(self.states.values())
                self.device_report = dict(dp.summary(), clock=self.clock)
                report.device = self.device_report
            return report

    return Replica


_STEP: dict = {}


def replica_class(ns, gpu: bool):
    key = (id(ns), gpu)
    cls = _STEP.get(key)
    if cls is None:
        if gpu:
            from .plugin import engine_classes
            base = engine_classes(ns)[1]
        else:
            base = ns.Engine
        cls = _step_class(base)
        cls._ns = ns
        _STEP[key] = cls
    return cls


@dataclass
class ClusterReport:
    replicas: list                       # RunReport per replica (its placed requests)
    placement: dict                      # request id -> replica index
    placement_rule: str
    per_replica_requests: list = field(default_factory=list)

    def jcts(self):
        return [r.jct for rep in self.replicas if rep is not None for r in rep.per_request]

    def aggregates(self) -> dict:
        """Whole-cluster avg / p99 JCT and requests/s (metrics.py:104-113
        over every replica's records; req/s over first arrival .. last
        finish across the cluster)."""
        ns = reference.load()
        recs = [r for rep in self.replicas if rep is not None for r in rep.per_request]
        jcts = [r.jct for r in recs]
        first = min(r.arrival for r in recs)
        last = max(r.finish for r in recs)
        return {"count": len(recs), "avg_jct": sum(jcts) / len(jcts), "p99_jct": ns.percentile(jcts, 99),
                "req_per_s": len(recs) / (last - first) if last > first else math.inf,
                "per_replica": list(self.per_replica_requests)}


class ClusterScheduler:
    """N replicas under one placement view.

    ``make_replica(i) -> (policy, predictor, memory, config)``: replica i's
    reference objects (fresh per replica: policies are single-use).
    ``device_for(i) -> KvDataPath | None``: the data path executing replica
    i's batches (None: host-only replica, e.g. another process's GPU).
    """

    def __init__(self, ns, workload: Sequence, n_replicas: int, make_replica: Callable,
                 device_for: Optional[Callable] = None, placement: str = "free-tokens",
                 clock: str = "model"):
        if n_replicas < 1:
            raise ns.ConfigError("a cluster needs at least one replica")
        if placement not in PLACEMENTS:
            raise ns.ConfigError(f"unknown placement {placement!r}; choose from {PLACEMENTS}")
        if clock != "model" and n_replicas > 1:
            # measured durations differ per process: placements would diverge
            raise ns.ConfigError("a multi-replica cluster runs on the model clock")
        self.ns = ns
        self.workload = sorted(workload, key=lambda r: (r.arrival_time, r.id))
        self.placement_rule = placement
        self.replicas = []
        for i in range(n_replicas):
            policy, predictor, memory, config = make_replica(i)
            dp = device_for(i) if device_for else None
            if dp is not None:
                eng = replica_class(ns, True)(self.workload, policy, predictor, memory, config, dp, clock)
            else:
                eng = replica_class(ns, False)(self.workload, policy, predictor, memory, config)
            eng.begin()
            self.replicas.append(eng)
        self.placement: dict = {}
        self._rr = 0

    def _place(self, spec) -> int:
        if self.placement_rule == "round-robin":
            k = self._rr % len(self.replicas)
            self._rr += 1
            return k

        kv_demand = self.ns.scheduler.kv_demand

        def key(i):
            eng = self.replicas[i]
            live = [st for st in eng.states.values() if not st.done]
            # free tokens net of what the replica's unfinished requests must
            # still make resident (swapped-out, dropped and queued caches)
            free = eng.memory.free_tokens - sum(kv_demand(st) for st in live)
            if self.placement_rule == "least-requests":
                return (len(live), -free, i)
            return (-free, len(live), i)

        return min(range(len(self.replicas)), key=key)

    def run(self) -> ClusterReport:
        arrivals = self.workload
        n, ai = len(arrivals), 0
        reps = self.replicas
        while True:
            t_arr = arrivals[ai].arrival_time if ai < n else math.inf
            k = min(range(len(reps)), key=lambda i: (reps[i].next_time(), i))
            if reps[k].next_time() < t_arr:
                reps[k].step()
                continue
            if ai >= n:
                break
            # every replica is past the events before t_arr: place its arrivals
            while ai < n and arrivals[ai].arrival_time == t_arr:
                spec = arrivals[ai]
                dest = self._place(spec)
                self.placement[spec.id] = dest
                reps[dest].admit(spec)
                ai += 1
            if ai >= n:
                for eng in reps:
                    eng.more_arrivals = False
                for eng in reps:
                    if eng.deadlocked():
                        eng.poke(t_arr)
        reports = [eng.finish() for eng in reps]
        return ClusterReport(reports, self.placement, self.placement_rule,
                             [len(r.per_request) if r is not None else 0 for r in reports])
