"""Short workload for profiling the decode-step kernel (ncu): Llama-3-8B,
B rows at context C, a few decode steps through LlamaRunner.decode."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--ctx", type=int, default=900)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--layers-path", action="store_true", help="per-layer launches instead of the step kernel")
a = ap.parse_args()
cfg = PRESETS[a.model]
B, nb = a.batch, (a.ctx + 16) // 16
w = LlamaWeights(cfg)
pool = KvPool(cfg, B * nb + 4)
r = LlamaRunner(w, pool)
r.use_step_kernel = not a.layers_path
table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
tok = torch.zeros(B, dtype=torch.int32, device="cuda")
pos = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
slots = table[:, a.ctx // 16] * 16 + a.ctx % 16
ctxd = torch.full((B,), a.ctx + 1, dtype=torch.int32, device="cuda")
keys = torch.zeros(B, dtype=torch.int64, device="cuda")
for _ in range(a.steps):
    r.decode(tok, pos, slots, table, ctxd, keys_out=keys)
torch.cuda.synchronize()
print("done")
