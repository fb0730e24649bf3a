"""K1/K2 swap under decode load, swept over the SM path's grid size
(ASTRAEA_SWAP_CTAS) and the copy-engine (DMA) mode: the swap stream runs
swap-out/in round trips of C tokens while the compute stream runs decode
steps of the Llama-3-8B shape at batch B, sized so both take about as long;
reports swap GB/s alone / under load and the decode step alone / under load.

    python tools/swap_load.py --ctas 8 16 32 64 296 --tokens 673 --batch 4
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvDataPath
from paper_2512_14142_b200.gpu.model import PRESETS

ap = argparse.ArgumentParser()
ap.add_argument("--ctas", type=int, nargs="+", default=[8, 16, 32, 64, 296])
ap.add_argument("--tokens", type=int, default=673)
ap.add_argument("--batch", type=int, default=4)
ap.add_argument("--ctx", type=int, default=673)
ap.add_argument("--swaps", type=int, default=4)
a = ap.parse_args()

cfg = PRESETS["llama3-8b"]
nb = (a.tokens + 15) // 16
dnb = (a.ctx + 16) // 16
dp = KvDataPath(cfg, num_blocks=a.batch * dnb + 2 * nb + 8)
B = a.batch
table = torch.arange(B * dnb, dtype=torch.int32, device="cuda").view(B, dnb)
src = list(range(B * dnb, B * dnb + nb))
dst = list(range(B * dnb + nb, B * dnb + 2 * nb))
tok = torch.zeros(B, dtype=torch.int32, device="cuda")
pos = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
slots = table[:, a.ctx // 16] * 16 + a.ctx % 16
ctxd = torch.full((B,), a.ctx + 1, dtype=torch.int32, device="cuda")
keys = torch.zeros(B, dtype=torch.int64, device="cuda")
bpt = dp.pool.bytes_per_token
slot = torch.empty(a.tokens * bpt, dtype=torch.uint8, pin_memory=True)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def decode_loop(steps):
    x, y = ev(), ev()
    x.record(dp.compute)
    for _ in range(steps):
        dp.runner.decode(tok, pos, slots, table, ctxd, stream=dp.compute, keys_out=keys)
    y.record(dp.compute)
    return x, y


def swap_loop(mode):
    x, y = ev(), ev()
    x.record(dp.swapper)
    for _ in range(a.swaps):
        ops.swap_out(dp.pool.geo, dp.pool.data, src, a.tokens, slot, mode, dp.swapper)
        ops.swap_in(dp.pool.geo, dp.pool.data, dst, a.tokens, slot, mode, dp.swapper)
    y.record(dp.swapper)
    return x, y


decode_loop(5)
torch.cuda.synchronize()
x, y = decode_loop(20)
torch.cuda.synchronize()
dec_alone = x.elapsed_time(y) / 20
moved = 2 * a.swaps * a.tokens * bpt
out = {"tokens": a.tokens, "bytes_per_swap": a.tokens * bpt, "decode_batch": B, "decode_ctx": a.ctx,
       "decode_step_ms_alone": dec_alone, "modes": []}
for c in a.ctas + ["dma", "staged"]:
    mode = {"dma": L.SWAP_DMA, "staged": L.SWAP_STAGED}.get(c, L.SWAP_KERNEL)
    if isinstance(c, int):
        os.environ["ASTRAEA_SWAP_CTAS"] = str(c)
    swap_loop(mode)
    torch.cuda.synchronize()
    x, y = swap_loop(mode)
    torch.cuda.synchronize()
    alone_ms = x.elapsed_time(y)
    steps = max(2, int(alone_ms / dec_alone))   # decode for about as long as the swaps take
    sx, sy = swap_loop(mode)
    dx, dy = decode_loop(steps)
    torch.cuda.synchronize()
    loaded_ms = sx.elapsed_time(sy)
    dec_loaded = dx.elapsed_time(dy) / steps
    out["modes"].append({"ctas": c, "swap_gbs_alone": moved / alone_ms / 1e6,
                         "swap_gbs_under_decode": moved / loaded_ms / 1e6, "decode_steps": steps,
                         "decode_step_ms_under_swap": dec_loaded, "decode_slowdown": dec_loaded / dec_alone})
    print(json.dumps(out["modes"][-1]), flush=True)
print(json.dumps(out))
