"""Shared helpers for the GPU tests (data path construction)."""

import math

from paper_2512_14142_b200.gpu.datapath import KvDataPath
from paper_2512_14142_b200.gpu.model import PRESETS


def datapath_for(memory_capacity_tokens, model="tiny", max_requests=256, **kw):
    blocks = math.ceil(memory_capacity_tokens / 16) + max_requests + 16
    return KvDataPath(PRESETS[model], num_blocks=blocks, **kw)
