"""Per-CTA timeline of the decode GEMM chain of one layer (O -> GU -> Down ->
next QKV) from %globaltimer stamps (astraea_debug_gemm_trace).

For each phase: when its activations were released to the producer
(phase barrier / PDL), and when each CTA's epilogue finished the phase,
as [min, median, max] microseconds after the chain's first CTA entry."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

B = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = PRESETS["llama3-8b"]
w = LlamaWeights(cfg)
pool = KvPool(cfg, 64)
r = LlamaRunner(w, pool)
dev = "cuda"
d, F, qd = cfg.hidden, cfg.ffn, cfg.num_q_heads * cfg.head_dim
lw, lw1 = w.layers[0], w.layers[1]
ws = r.gemm_ws
x = torch.randn(B, d, device=dev).bfloat16()
att = torch.randn(B, qd, device=dev).bfloat16()
h = torch.empty(B, F, device=dev).bfloat16()
q = torch.empty(B, qd, device=dev).bfloat16()
s1 = torch.empty(d // 128, B, device=dev)
s2 = torch.empty(d // 128, B, device=dev)
pos = torch.full((B,), 100, dtype=torch.int32, device=dev)
slots = torch.arange(B, dtype=torch.int32, device=dev)
cs = ops.rope_table(pos, cfg.head_dim, cfg.rope_theta)
phases = [dict(a=att, w=lw["wo"], out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s1),
          dict(a=x, w=lw["wgu"], out=h, kind=L.EPI_SILU, ssq_in=s1, rms_dim=d, rms_eps=cfg.eps),
          dict(a=h, w=lw["wdown"], out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s2),
          dict(a=x, w=lw1["wqkv"], out=q, kind=L.EPI_QKV_ROPE, ssq_in=s2, rms_dim=d, rms_eps=cfg.eps,
               pool=pool.data, geo=pool.geo, layer=1, num_q_heads=cfg.num_q_heads, positions=pos, slots=slots,
               rope_theta=cfg.rope_theta, rope_table=cs)]
for _ in range(3):
    ops.gemm_chain(phases, ws)
torch.cuda.synchronize()
reps = 3
lib = L.load()
buf = torch.zeros(reps, 148 * 32, dtype=torch.int64, device=dev)
lib.astraea_debug_gemm_trace(buf.data_ptr(), reps, 148 * 32)
for _ in range(reps):
    ops.gemm_chain(phases, ws)
torch.cuda.synchronize()
lib.astraea_debug_gemm_trace(None, 0, 0)
t = buf.view(reps, 148, 32).cpu().double()
names = ["o", "gu", "down", "qkv"]


def mmm(col, base):
    col = col[col > 0]
    return [round(float(col.min() - base) / 1000, 2), round(float(col.median() - base) / 1000, 2),
            round(float(col.max() - base) / 1000, 2)]


for rr in range(reps):
    s = t[rr]
    base = s[:, 0].min()
    row = {"rep": rr, "entry": mmm(s[:, 0], base)}
    for p, n in enumerate(names):
        row[n + "_x_released"] = mmm(s[:, 1 + p], base)
        row[n + "_epi_done"] = mmm(s[:, 5 + p], base)
    row["mma_done"] = mmm(s[:, 9], base)
    row["exit"] = mmm(s[:, 10], base)
    print(json.dumps(row))
by = {n: ph["w"].numel() * 2 for n, ph in zip(names, phases)}
print(json.dumps({"weight_MB": {k: round(v / 1e6, 1) for k, v in by.items()},
                  "ideal_us_at_6.5TBps": {k: round(v / 6.5e6, 1) for k, v in by.items()}}))
