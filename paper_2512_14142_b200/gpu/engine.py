"""``GpuEngine``: the reference's own event loop (simulator.py:101-481) with
the B200 data path attached -- see ``paper_2512_14142_b200.plugin`` for the
seams and the clock modes. Importing this module imports the reference."""

from __future__ import annotations

from ..plugin import CLOCKS, AdmittedMember, engine_classes, requests_per_second, run_on_gpu  # noqa: F401

GpuKvCacheManager, GpuEngine = engine_classes()
