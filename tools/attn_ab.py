"""Decode attention A/B on the Llama-3-8B shape: for each batch B at context
C, (1) the standalone paged decode attention kernel alone (one layer, CUDA
events over repetitions) vs its algorithmic bytes (B x C x 4 KiB K+V pages
per layer at 8 kv heads of 128), and (2) the whole decode step with the
attention fused into the layer chain vs the standalone kernel + chain.
The kernel is chosen by ASTRAEA_DECODE_ATTN (t = TMA-staged, m = one page
per warp), so run it once per value.

    ASTRAEA_DECODE_ATTN=t python tools/attn_ab.py --batch 1 4 8 16 32 --ctx 673
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, nargs="+", default=[1, 4, 8, 16, 32])
ap.add_argument("--ctx", type=int, default=673)
ap.add_argument("--no-step", action="store_true")
ap.add_argument("--no-step-standalone", action="store_true", help="only the fused step")
a = ap.parse_args()
cfg = PRESETS["llama3-8b"]
hbm = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0
w = LlamaWeights(cfg, seed=0)
C = a.ctx
nb = (C + 16) // 16
pool = KvPool(cfg, max(a.batch) * nb + 8)
pool.data.normal_(0, 1)
runner = LlamaRunner(w, pool)
qd = cfg.num_q_heads * cfg.head_dim
mode = os.environ.get("ASTRAEA_DECODE_ATTN", "t")


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


for B in a.batch:
    table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
    q = torch.randn(B, qd, device="cuda").to(torch.bfloat16)
    out = torch.empty(B, qd, dtype=torch.bfloat16, device="cuda")
    ctxd = torch.full((B,), C, dtype=torch.int32, device="cuda")
    ws = runner._dec_ws(B, nb)
    res = {"mode": mode, "batch": B, "ctx": C}
    layers = [0, 7, 15, 23, 31]
    li = [0]

    def attn():
        li[0] = (li[0] + 1) % len(layers)   # rotate layers: K/V pages not L2-resident
        ops.decode_attention(pool.geo, pool.data, layers[li[0]], q, qd, B, cfg.num_q_heads, table, ctxd,
                             runner.scale, out, ws)

    ms = timed(attn, 50)
    by = B * C * 2 * cfg.num_kv_heads * cfg.head_dim * 2
    res["attn_us"] = ms * 1e3
    res["attn_gbs"] = by / (ms / 1e3) / 1e9
    res["attn_frac"] = res["attn_gbs"] / hbm
    if not a.no_step:
        tok = torch.zeros(B, dtype=torch.int32, device="cuda")
        pos = torch.full((B,), C - 1, dtype=torch.int32, device="cuda")
        slots = table[:, (C - 1) // 16] * 16 + (C - 1) % 16
        keys = torch.zeros(B, dtype=torch.int64, device="cuda")
        for fuse in ((True,) if a.no_step_standalone else (True, False)):
            runner.fuse_attention = fuse
            runner.fuse_max_batch = 64
            ms = timed(lambda: runner.decode(tok, pos, slots, table, ctxd, keys_out=keys), 10)
            step_by = cfg.decode_weight_bytes + B * C * cfg.kv_bytes_per_token
            res["step_ms_" + ("fused" if fuse else "standalone")] = ms
            res["step_frac_" + ("fused" if fuse else "standalone")] = step_by / (ms / 1e3) / 1e9 / hbm
        runner.fuse_attention = True
    print(json.dumps(res), flush=True)
