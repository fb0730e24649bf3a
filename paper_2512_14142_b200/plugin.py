"""Plug the B200 data path into the *unmodified* reference package.

``agentsched`` (the reference, pkg/src/agentsched) exposes a duck-typed
plugin API but no FFI. ``attach(agentsched)`` builds two subclasses of its
own classes, overriding only documented seams, so a maintainer can run the
reference's scheduler with real device work:

* ``KvCacheManager`` (kvcache.py:152-292): every transition first runs the
  reference method unchanged, then forwards to ``KvDataPath``;
* ``Engine`` (simulator.py:101-481): the plan returned by
  ``policy.build_next_batch`` (called first in ``_try_start_batch``,
  simulator.py:340-342) is recorded, and ``_actual_seconds``
  (simulator.py:329-337, called once per plan entry *before* the location
  flip) collects each member's pre-admission cache location; after the last
  entry the whole batch is launched on the device. Durations stay the
  reference's (model clock), so its report bytes are unchanged.

No reference code is copied: the subclasses call ``super()`` for all
semantics. See INTEGRATION.md for the ctypes-level binding.
"""

from __future__ import annotations

from .host.engine import AdmittedMember


def attach(agentsched, datapath):
    """Return (GpuKvCacheManager, GpuEngine) subclasses of the reference's classes."""

    class GpuKvCacheManager(agentsched.KvCacheManager):
        device = datapath

        def on_api_yield(self, state, predicted_api_seconds, batch_demand_tokens, now):
            action = super().on_api_yield(state, predicted_api_seconds, batch_demand_tokens, now)
            if action is agentsched.CacheAction.DISCARD:
                self.device.drop(state)
            elif action is agentsched.CacheAction.SWAP:
                self.device.swap_out_begin(state)
            return action

        def complete_swap_out(self, state):
            super().complete_swap_out(state)
            self.device.swap_out_done(state)

        def try_begin_swap_in(self, state):
            ok = super().try_begin_swap_in(state)
            if ok:
                self.device.swap_in_begin(state)
            return ok

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

    class GpuEngine(agentsched.Engine):
        def __init__(self, workload, policy, predictor, memory, config):
            super().__init__(workload, policy, predictor, memory, config)
            self.manager = GpuKvCacheManager(memory, predictor, mode=config.cache_mode)
            self._plan_entries = ()
            self._pending = []
            build = policy.build_next_batch

            def recorded(free_tokens, now, max_segments=None):
                plan = build(free_tokens, now, max_segments)
                self._plan_entries = plan.entries
                self._pending = []
                return plan

            policy.build_next_batch = recorded

        def _actual_seconds(self, state):
            seconds = super()._actual_seconds(state)
            self._pending.append(AdmittedMember(state, state.current_segment, state.cache_location,
                                                state.kv_tokens))
            if len(self._pending) == len(self._plan_entries):
                datapath.launch_batch(self._pending)
                self._pending = []
            return seconds

        def run(self):
            report = super().run()
            datapath.synchronize()
            datapath.audit(self.states.values())
            return report

    return GpuKvCacheManager, GpuEngine


def run_reference_on_gpu(agentsched, datapath, workload, policy, predictor, memory, config):
    """The reference's ``run()`` with the B200 data path attached."""
    _, engine_cls = attach(agentsched, datapath)
    return engine_cls(workload, policy, predictor, memory, config).run()
