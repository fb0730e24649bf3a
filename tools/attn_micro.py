"""The step kernel's attention phase in isolation: a 2-phase program
[QKV(layer 0), ATTN(layer 0)] for Llama-3-8B at batch B / context C; prints
the per-warp attention stamps (see astraea_debug_step_trace)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

cfg = PRESETS["llama3-8b"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
C = int(sys.argv[2]) if len(sys.argv) > 2 else 900
w = LlamaWeights(cfg)
nb = (C + 16) // 16
pool = KvPool(cfg, B * nb + 4)
pool.data.normal_(0, 0.3)
r = LlamaRunner(w, pool)
d, qd = cfg.hidden, cfg.num_q_heads * cfg.head_dim
x = torch.randn(B, d, device="cuda").bfloat16()
q = torch.empty(B, qd, device="cuda").bfloat16()
att = torch.empty(B, qd, device="cuda").bfloat16()
ssq = (x.float() ** 2).sum(1).view(1, B).contiguous()
table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
pos = torch.full((B,), C, dtype=torch.int32, device="cuda")
slots = table[:, C // 16] * 16 + C % 16
ctx = torch.full((B,), C + 1, dtype=torch.int32, device="cuda")
cs = ops.rope_table(pos, cfg.head_dim, cfg.rope_theta)
ph = [dict(kind="gemm", a=x, w=w.layers[0]["wqkv"], out=q, epi=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=d,
           rms_eps=cfg.eps, pool=pool.data, geo=pool.geo, layer=0, num_q_heads=cfg.num_q_heads, positions=pos,
           slots=slots, rope_theta=cfg.rope_theta, rope_table=cs, a_from=-1, epi_from=-1),
      dict(kind="attn", pool=pool.data, geo=pool.geo, layer=0, num_q_heads=cfg.num_q_heads, q=q, q_stride=qd,
           table=table, ctx=ctx, scale=r.scale, out=att, qkv_from=0)]
prog = ops.StepProgram(B, ph, ops.StepWorkspace())
for _ in range(3):
    prog.launch()
torch.cuda.synchronize()
G = torch.cuda.get_device_properties(0).multi_processor_count
nph = 2
buf = torch.zeros(G * nph * 8 + G + G * 64, dtype=torch.int64, device="cuda")
L.load().astraea_debug_step_trace(buf.data_ptr())
prog.launch()
torch.cuda.synchronize()
L.load().astraea_debug_step_trace(None)
t = buf.cpu().double()
entry = t[G * nph * 8: G * nph * 8 + G]
base = entry.min()
atr = t[G * nph * 8 + G:].view(G * 4, 16)
act = atr[atr[:, 0] > 0]
st = t[: G * nph * 8].view(G, nph, 8)
qkv_done = st[:, 0, 2]
print(json.dumps({"B": B, "ctx": C, "qkv_epi_done_max": round(float(qkv_done.max() - base) / 1000, 1),
                  "attn_warps": int(act.shape[0]),
                  "median_us": [round(float(c[c > 0].median() - base) / 1000, 1) if (c > 0).any() else None
                                for c in act.T],
                  "max_us": [round(float(c[c > 0].max() - base) / 1000, 1) if (c > 0).any() else None for c in act.T]}))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    prog.launch()
e1.record()
e1.synchronize()
print(json.dumps({"us_per_launch": e0.elapsed_time(e1) / 20 * 1000}))
