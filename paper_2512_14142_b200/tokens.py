"""Token ids for the synthetic traces.

The reference's traces carry token *counts* only (``SegmentSpec.n_in``,
workload.py:57-76); the data path needs ids. They come from a SHA-256-seeded
stream, so any process (any replica, any rerun, a recompute after a discard)
reconstructs the same context.
"""

from __future__ import annotations

import hashlib
import random


def segment_token_ids(request_id: str, segment_index: int, n: int, vocab: int, seed: int = 0):
    digest = hashlib.sha256(f"{seed}:{request_id}:{segment_index}".encode()).digest()
    rng = random.Random(int.from_bytes(digest[:8], "little"))
    return [rng.randrange(vocab) for _ in range(n)]
