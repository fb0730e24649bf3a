"""Short, ncu-friendly workload: Llama-3-8B decode steps at a small batch and
one prefill chunk, through the same LlamaRunner the engine uses.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        python tools/profile_step.py --batch 3 --ctx 900 --steps 3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--batch", type=int, default=3)
ap.add_argument("--ctx", type=int, default=900)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--prefill", type=int, default=512)
a = ap.parse_args()
cfg = PRESETS[a.model]
B, ctx = a.batch, a.ctx
nb = (ctx + 16) // 16
w = LlamaWeights(cfg)
pool = KvPool(cfg, B * nb + nb + 4)
r = LlamaRunner(w, pool)
d = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
tok = torch.zeros(B, dtype=torch.int32, device="cuda")
pos = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
slots = table[:, ctx // 16] * 16 + ctx % 16
ctxd = torch.full((B,), ctx + 1, dtype=torch.int32, device="cuda")
out = torch.zeros(B, dtype=torch.int64, device="cuda")
for _ in range(a.steps):
    r.decode(tok, pos, slots, table, ctxd, keys_out=out)
if a.prefill:
    T = a.prefill
    blocks = list(range(B * nb, B * nb + (T + 15) // 16))
    r.prefill(d(list(range(T))), d(list(range(T))), d([blocks[p // 16] * 16 + p % 16 for p in range(T)]),
              d([0, T]), d([blocks]).view(1, -1), d([T]), torch.tensor([T - 1], device="cuda"), T)
torch.cuda.synchronize()
print("done")
