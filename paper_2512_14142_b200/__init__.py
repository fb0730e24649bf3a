"""B200-native GPU data path for Astraea's state-aware agent scheduler.

``host``  -- the reference's plugin API (policies, KV policy, event loop).
``gpu``   -- the device data path behind it: paged KV pool, swap, decode
             attention, recompute prefill, all through ``libastraea_b200.so``
             (C ABI declared in ``include/astraea_b200.h``).
"""

__version__ = "0.1.0"
