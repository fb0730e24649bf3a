"""Workload for ncu captures of the main kernels (Llama-3-8B, one GPU):
  chain    one layer's chained decode GEMMs at batch B (3 launches)
  attn     paged decode attention at batch B, context C (3 launches)
  prefill  a T-token prefill forward (gemm_rows_kernel + prefill attention)
  swap     K1 gather / K2 scatter of C tokens (kernel mode)
    python tools/prof_kernels.py chain --batch 1
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import bench
from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvDataPath
from paper_2512_14142_b200.gpu.model import PRESETS

ap = argparse.ArgumentParser()
ap.add_argument("what", choices=["chain", "attn", "prefill", "swap"])
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--ctx", type=int, default=900)
ap.add_argument("--tokens", type=int, default=1024)
a = ap.parse_args()
cfg = PRESETS["llama3-8b"]
B, C = a.batch, a.ctx
nb = (C + 16) // 16
dp = KvDataPath(cfg, num_blocks=max(B * nb + 8, (a.tokens + 15) // 16 + 8))
dp.pool.data.normal_(0, 0.5)
if a.what == "chain":
    bench.chain_kernel_time(dp, cfg, B, C, reps=3)
elif a.what == "attn":
    qd = cfg.num_q_heads * cfg.head_dim
    q = torch.randn(B, qd, device="cuda").bfloat16()
    out = torch.empty(B, qd, device="cuda").bfloat16()
    table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
    ctx = torch.full((B,), C, dtype=torch.int32, device="cuda")
    ws = ops.decode_workspace(B, cfg.num_q_heads, cfg.head_dim, nb, "cuda")
    for _ in range(3):
        ops.decode_attention(dp.pool.geo, dp.pool.data, 0, q, qd, B, cfg.num_q_heads, table, ctx,
                             dp.runner.scale, out, ws)
elif a.what == "prefill":
    T = a.tokens
    d = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
    blocks = list(range((T + 15) // 16))
    dp.runner.prefill(d([i % cfg.vocab for i in range(T)]), d(list(range(T))),
                      d([blocks[p // 16] * 16 + p % 16 for p in range(T)]), d([0, T]), d([blocks]).view(1, -1),
                      d([T]), torch.tensor([T - 1], device="cuda"), T)
else:
    ids = list(range((C + 15) // 16))
    slot = torch.empty(C * dp.pool.bytes_per_token, dtype=torch.uint8, pin_memory=True)
    ops.swap_out(dp.pool.geo, dp.pool.data, ids, C, slot, L.SWAP_KERNEL)
    ops.swap_in(dp.pool.geo, dp.pool.data, ids, C, slot, L.SWAP_KERNEL)
torch.cuda.synchronize()
print("done", a.what)
