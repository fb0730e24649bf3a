"""Decode-step time of Llama-3-8B at a given batch/context: chained launches
carrying 1 or 2 layers each, optionally the one-launch step kernel (several
L2 look-ahead depths).
Prints one JSON line per variant with ms/step and HBM GB/s (weights + KV)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--batch", type=int, nargs="+", default=[1, 4, 16])
ap.add_argument("--ctx", type=int, default=900)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--l2", type=int, nargs="*", default=[])
ap.add_argument("--chain-layers", type=int, nargs="+", default=[1, 2])
a = ap.parse_args()
cfg = PRESETS[a.model]
w = LlamaWeights(cfg)
maxB = max(a.batch)
nb = (a.ctx + 16) // 16
pool = KvPool(cfg, maxB * nb + 4)
pool.data.normal_(0, 0.5)
r = LlamaRunner(w, pool)
for B in a.batch:
    table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
    tok = torch.randint(0, cfg.vocab, (B,), dtype=torch.int32, device="cuda")
    pos = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
    slots = table[:, a.ctx // 16] * 16 + a.ctx % 16
    ctxd = torch.full((B,), a.ctx + 1, dtype=torch.int32, device="cuda")
    keys = torch.zeros(B, dtype=torch.int64, device="cuda")
    variants = ([(f"chain_{c}", False, 0, c) for c in a.chain_layers] +
                [(f"step_l2_{l}", True, l, 1) for l in a.l2])
    for name, step_kernel, l2, cl in variants:
        r.use_step_kernel = step_kernel
        r.l2_ahead = l2
        r.chain_layers = cl
        for _ in range(3):
            r.decode(tok, pos, slots, table, ctxd, keys_out=keys)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            r.decode(tok, pos, slots, table, ctxd, keys_out=keys)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        by = cfg.decode_weight_bytes + B * (a.ctx + 1) * cfg.kv_bytes_per_token
        print(json.dumps({"B": B, "ctx": a.ctx, "variant": name, "ms": round(ms, 4),
                          "hbm_gbs": round(by / ms / 1e6, 1)}), flush=True)
