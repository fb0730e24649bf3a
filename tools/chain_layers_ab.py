"""Decode step with one vs two decoder layers per chained launch
(LlamaRunner.chain_layers), Llama-3-8B, ctx 540, CUDA events over 20 steps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

cfg = PRESETS["llama3-8b"]
w = LlamaWeights(cfg, seed=0)
C = 540
nb = (C + 16) // 16
pool = KvPool(cfg, 32 * nb + 8)
r = LlamaRunner(w, pool)
for rep in range(2):
    for B in (1, 2, 4, 16):
        table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
        tok = torch.zeros(B, dtype=torch.int32, device="cuda")
        pos = torch.full((B,), C - 1, dtype=torch.int32, device="cuda")
        slots = table[:, (C - 1) // 16] * 16 + (C - 1) % 16
        ctx = torch.full((B,), C, dtype=torch.int32, device="cuda")
        keys = torch.zeros(B, dtype=torch.int64, device="cuda")
        out = []
        for cl in (1, 2):
            r.chain_layers = cl
            for _ in range(3):
                r.decode(tok, pos, slots, table, ctx, keys_out=keys)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                r.decode(tok, pos, slots, table, ctx, keys_out=keys)
            e1.record()
            e1.synchronize()
            out.append(e0.elapsed_time(e1) / 20)
        print(f"B={B}: one layer/launch {out[0]:.3f} ms, two {out[1]:.3f} ms", flush=True)
