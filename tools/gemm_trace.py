"""Per-CTA timeline of the decode (stream-K) GEMMs of one layer, from
%globaltimer stamps (astraea_debug_gemm_trace). Runs a layer's 4 GEMMs
back to back a few times (PDL chain) and reports, per GEMM, the spread of
CTA entry, dependency release, first MMA, last MMA, epilogue end and exit,
relative to the previous GEMM's last exit."""
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
lw = w.layers[0]
ws = r.gemm_ws
x = torch.randn(B, d, device=dev).bfloat16()
att = torch.randn(B, qd, device=dev).bfloat16()
h = torch.randn(B, F, device=dev).bfloat16()
q = torch.empty(B, cfg.qkv_dim, device=dev).bfloat16()
ssq = (x.float().pow(2).view(B, -1, 128).sum(-1)).T.contiguous()
ssq2 = torch.empty_like(ssq)
gu = torch.empty(B, F, device=dev).bfloat16()
seq = [("qkv", lambda: ops.gemm(x, lw["wqkv"], out=q, workspace=ws)),
       ("o", lambda: ops.gemm_ex(att, lw["wo"], x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq2, workspace=ws)),
       ("gu", lambda: ops.gemm_ex(x, lw["wgu"], gu, kind=L.EPI_SILU, ssq_in=ssq2, rms_dim=d, rms_eps=1e-5, workspace=ws)),
       ("down", lambda: ops.gemm_ex(h, lw["wdown"], x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq, workspace=ws))]
reps = 3
for _ in range(2):
    for _, f in seq:
        f()
torch.cuda.synchronize()
lib = L.load()
buf = torch.zeros(reps * len(seq), 148 * 8, dtype=torch.int64, device=dev)
lib.astraea_debug_gemm_trace(buf.data_ptr(), reps * len(seq), 148 * 8)
for _ in range(reps):
    for _, f in seq:
        f()
torch.cuda.synchronize()
lib.astraea_debug_gemm_trace(None, 0, 0)
t = buf.view(reps * len(seq), 148, 8).cpu().double()
out = []
prev_exit = None
for i in range(reps * len(seq)):
    name = seq[i % len(seq)][0]
    s = t[i]
    base = prev_exit if prev_exit is not None else s[:, 0].min()
    row = {"gemm": name}
    for j, lab in enumerate(["entry", "dep", "first_mma", "last_mma", "epi_done", "exit"]):
        col = s[:, j]
        col = col[col > 0]
        if len(col):
            row[lab] = [round(float(col.min() - base) / 1000, 2), round(float(col.median() - base) / 1000, 2),
                        round(float(col.max() - base) / 1000, 2)]
    prev_exit = s[:, 5].max()
    out.append(row)
print(json.dumps(out[len(seq):], indent=0))
