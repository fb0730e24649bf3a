"""Per-CTA timeline of one short-prefill GEMM on the one-CTA (rows) kernel:
entry, setup done, first stage landed, last MMA done, split partial
published, split sum done, epilogue done (us after the first CTA entered;
min / median / max over CTAs), for the Llama-3-8B projections at T tokens.

    python tools/rows_trace.py --tokens 128 --op o qkv gu down
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=128)
ap.add_argument("--op", nargs="+", default=["qkv", "o", "gu", "down"])
ap.add_argument("--per-cta", action="store_true")
a = ap.parse_args()
cfg = PRESETS["llama3-8b"]
T = a.tokens
w = LlamaWeights(cfg, seed=0)
pool = KvPool(cfg, (T + 15) // 16 + 8)
r = LlamaRunner(w, pool)
dev = "cuda"
qd = cfg.num_q_heads * cfg.head_dim
pos = torch.arange(T, dtype=torch.int32, device=dev)
x = torch.randn(T, cfg.hidden, device=dev).to(torch.bfloat16)
q = torch.empty(T, qd, dtype=torch.bfloat16, device=dev)
att = torch.randn(T, qd, device=dev).to(torch.bfloat16)
h = torch.randn(T, cfg.ffn, device=dev).to(torch.bfloat16)
ssq = torch.full((r.parts, T), cfg.hidden / r.parts, dtype=torch.float32, device=dev)  # x ~ N(0, 1): sum x^2 = d
cs = ops.rope_table(pos, cfg.head_dim, cfg.rope_theta)
ws = r.gemm_ws
lw = w.layers[3]
calls = {
    "qkv": lambda: ops.gemm_ex(x, lw["wqkv"], q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=cfg.hidden, rms_eps=cfg.eps,
                               pool=pool.data, geo=pool.geo, layer=0, num_q_heads=cfg.num_q_heads, positions=pos,
                               slots=pos, rope_theta=cfg.rope_theta, rope_table=cs, workspace=ws),
    "o": lambda: ops.gemm_ex(att, lw["wo"], x, kind=L.EPI_RESIDUAL, residual=x, workspace=ws),
    "gu": lambda: ops.gemm_ex(x, lw["wgu"], h, kind=L.EPI_SILU, ssq_in=ssq, rms_dim=cfg.hidden, rms_eps=cfg.eps,
                              workspace=ws),
    "down": lambda: ops.gemm_ex(h, lw["wdown"], x, kind=L.EPI_RESIDUAL, residual=x, workspace=ws),
}
lib = L.load()
NW = 1024 * 16
buf = torch.zeros(NW, dtype=torch.int64, device=dev)
names = ["entry", "setup", "first_stage", "mma_done", "published", "summed", "epi_done", None,
         "wake_w2", "wake_w3", "wake_w4", "wake_w5", "epi_staged", "epi_computed", "epi_bar2"]
for op in a.op:
    for _ in range(3):
        calls[op]()
    torch.cuda.synchronize()
    buf.zero_()
    lib.astraea_debug_gemm_trace(buf.data_ptr(), 1, NW)
    calls[op]()
    torch.cuda.synchronize()
    lib.astraea_debug_gemm_trace(None, 0, 0)
    t = buf.view(-1, 16).cpu()
    live = t[:, 0] > 0
    t = t[live]
    base = t[:, 0].min()
    res = {"op": op, "tokens": T, "ctas": int(live.sum())}
    for k, nm in enumerate(names):
        if nm is None:
            continue
        col = t[:, k]
        col = col[col > 0]
        if col.numel():
            v = (col - base).double() / 1000
            res[nm] = [round(float(v.min()), 2), round(float(v.median()), 2), round(float(v.max()), 2)]
    res["span_us"] = round(float((t[:, 6].max() - base)) / 1000, 2)
    sms = (t[:, 7] & 0xFFFF)
    res["distinct_sms"] = int(torch.unique(sms).numel())
    print(json.dumps(res), flush=True)
    if a.per_cta:
        for i in range(t.shape[0]):
            row = [round(float(t[i, k] - base) / 1000, 2) if t[i, k] > 0 else None for k in range(7)]
            print(i, int(t[i, 7] & 0xFFFF), int((t[i, 7] >> 16) & 0x7FFF), int(t[i, 7] >> 31), row)
