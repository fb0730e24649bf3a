"""Per-CTA timeline of the tcgen05 prefill attention (astraea_debug_prefill_trace):
startup (entry -> first scores), per-KV-tile time, tail (last P -> exit),
for one layer's attention at T tokens on the Llama-3-8B shape.

    python tools/prefill_trace.py --tokens 2048 [--ctx-before 0]
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
from paper_2512_14142_b200.gpu.model import PRESETS

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=2048)
ap.add_argument("--ctx-before", type=int, default=0)
a = ap.parse_args()
cfg = PRESETS["llama3-8b"]
T, c0 = a.tokens, a.ctx_before
ctx = T + c0
nb = (ctx + 15) // 16
pool = KvPool(cfg, nb + 4)
pool.data.normal_()
qd = cfg.num_q_heads * cfg.head_dim
q = torch.randn(T, qd, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
d = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
args = (pool.geo, pool.data, 0, q, qd, d([0, T]), 1, T, cfg.num_q_heads, d([list(range(nb))]), d([ctx]),
        1 / 128 ** 0.5, out)
for _ in range(3):
    ops.prefill_attention(*args)
torch.cuda.synchronize()
QT = 128 // (cfg.num_q_heads // cfg.num_kv_heads)
grid = ((T + QT - 1) // QT) * cfg.num_kv_heads
buf = torch.zeros(grid, 16, dtype=torch.int64, device="cuda")
lib = L.load()
lib.astraea_debug_prefill_trace(buf.data_ptr())
ops.prefill_attention(*args)
torch.cuda.synchronize()
lib.astraea_debug_prefill_trace(None)
t = buf.cpu().double()
base = t[:, 0].min()
life = (t[:, 7] - t[:, 0]) / 1e3
tiles = t[:, 3]
start = (t[:, 2] - t[:, 0]) / 1e3
per_tile = (t[:, 4] - t[:, 2]) / 1e3 / (tiles - 1).clamp(min=1)
tail = (t[:, 7] - t[:, 4]) / 1e3
q_seen = (t[:, 1] - t[:, 0]) / 1e3
kv_first = (t[:, 8] - t[:, 0]) / 1e3


def st(x):
    return {"min": round(float(x.min()), 2), "median": round(float(x.median()), 2), "max": round(float(x.max()), 2)}


m = tiles > 5
if bool(m.any()):
    tt = t[m]
    rel = lambda k: (tt[:, k] - tt[:, 10]) / 1e3  # noqa: E731
    print(json.dumps({"tile4_from_issue_us": {"landed": st(rel(11)), "scores_seen": st(rel(12)),
                                             "p_published": st(rel(13)), "p_seen_by_mma": st(rel(14))}}))
print(json.dumps({"tokens": T, "ctx_before": c0, "ctas": grid, "span_us": round(float((t[:, 7].max() - base) / 1e3), 1),
                  "lifetime_us": st(life), "tiles": st(tiles), "startup_us": st(start), "q_seen_us": st(q_seen),
                  "kv_first_issue_us": st(kv_first), "per_tile_us": st(per_tile[tiles > 1]), "tail_us": st(tail)}))
