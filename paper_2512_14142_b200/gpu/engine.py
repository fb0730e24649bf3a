"""GpuEngine: the reference's event loop with the B200 data path plugged in.

Subclasses ``host.engine.Engine`` (the reference contract of
simulator.py:101-481) and fills its seams:

* ``_launch_batch`` -> ``KvDataPath.launch_batch``: allocate blocks, (re)prefill,
  decode loop (simulator.py:339-385);
* the manager's ``device`` mirror -> discard / swap / release on the pool
  (CS3-CS5, kvcache.py:173-292);
* ``_swap_delay`` -> measured gather/scatter time in ``measured`` mode.

Clock modes
  ``model``     the virtual clock advances by the reference cost model while
                the GPU really executes every plan; decisions (and the
                RunReport bytes) are identical to the reference's.
  ``measured``  the clock advances by CUDA-event durations of each member's
                segment (batch start -> the decode step that retires it) and
                of each swap; API waits stay virtual. This gives JCT and req/s
                of the B200 data path under the same scheduler. Swaps share
                one host link: they complete in issue order, each after the
                previous one (a FIFO channel -- SPEC.md:323 promises it, the
                reference's independent delays lack it),
                exactly as the data path runs them on its one swap stream.
"""

from __future__ import annotations

from ..host.engine import Engine
from ..host.errors import ConfigError

CLOCKS = ("model", "measured")


class GpuEngine(Engine):
    def __init__(self, workload, policy, predictor, memory, config, datapath, clock: str = "model",
                 device_audit: bool = True):
        if clock not in CLOCKS:
            raise ConfigError(f"unknown clock {clock!r}; choose from {CLOCKS}")
        super().__init__(workload, policy, predictor, memory, config, device=datapath)
        datapath.measure = clock == "measured"
        self.clock = clock
        self.datapath = datapath
        self.device_audit = device_audit
        self._link_free = 0.0   # measured clock: when the host link finishes its queued swaps

    def _launch_batch(self, members):
        measured = self.datapath.launch_batch(members)
        return measured if self.clock == "measured" else None

    def _swap_delay(self, state, direction):
        if self.clock == "measured":
            # FIFO host link: this transfer starts when the previous one ends
            start = max(self.now, self._link_free)
            self._link_free = start + self.datapath.swap_seconds(state, direction)
            return self._link_free - self.now
        return super()._swap_delay(state, direction)

    def _try_start_batch(self):
        super()._try_start_batch()
        if self.device_audit and self._active is not None:
            self.datapath.audit(self.states.values())

    def run(self):
        report = super().run()
        self.datapath.synchronize()
        if self.device_audit:
            self.datapath.audit(self.states.values())
        report.device = self.datapath.summary()
        report.device["clock"] = self.clock
        return report


def run_on_gpu(workload, policy, predictor, memory, config, datapath, clock="model"):
    """GPU counterpart of the reference's ``run()`` entry point."""
    return GpuEngine(workload, policy, predictor, memory, config, datapath, clock).run()
