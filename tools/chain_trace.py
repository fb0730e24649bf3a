"""Per-layer timeline of a decode step on the per-layer path (fused
attention + chained GEMMs): for each traced launch, [median, max] over CTAs
of entry, attention done, each phase's activations released and epilogue
done, and exit, in microseconds after the first launch's first CTA entered."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--ctx", type=int, default=900)
ap.add_argument("--layers", type=int, nargs="+", default=[0, 1, 2, 16, 31])
ap.add_argument("--no-fuse", action="store_true")
ap.add_argument("--per-cta", action="store_true")
ap.add_argument("--chain-layers", type=int, default=1)
a = ap.parse_args()
cfg = PRESETS["llama3-8b"]
w = LlamaWeights(cfg)
B, nb = a.batch, (a.ctx + 16) // 16
pool = KvPool(cfg, B * nb + 4)
r = LlamaRunner(w, pool)
r.fuse_attention = not a.no_fuse
r.chain_layers = a.chain_layers
table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
tok = torch.zeros(B, dtype=torch.int32, device="cuda")
pos = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
slots = table[:, a.ctx // 16] * 16 + a.ctx % 16
ctxd = torch.full((B,), a.ctx + 1, dtype=torch.int32, device="cuda")
keys = torch.zeros(B, dtype=torch.int64, device="cuda")
for _ in range(3):
    r.decode(tok, pos, slots, table, ctxd, keys_out=keys)
torch.cuda.synchronize()
G = torch.cuda.get_device_properties(0).multi_processor_count
n = cfg.num_layers + 1
buf = torch.zeros(n, G * 32, dtype=torch.int64, device="cuda")
lib = L.load()
lib.astraea_debug_gemm_trace(buf.data_ptr(), n, G * 32)
r.decode(tok, pos, slots, table, ctxd, keys_out=keys)
torch.cuda.synchronize()
lib.astraea_debug_gemm_trace(None, 0, 0)
t = buf.view(n, G, 32).cpu().double()
base = t[0, :, 0][t[0, :, 0] > 0].min()


def mm(col):
    col = col[col > 0]
    if col.numel() == 0:
        return None
    return [round(float(col.median() - base) / 1000, 1), round(float(col.max() - base) / 1000, 1)]


names = ["o", "gu", "down", "qkv"]
for i in range(n):
    li = i - 1   # launch 0 = layer 0's QKV
    if i > 0 and li not in a.layers:
        continue
    s = t[i]
    row = {"launch": i, "layer": li, "entry": mm(s[:, 0]), "attn_done": mm(s[:, 15])}
    for p, nm in enumerate(names):
        row[nm + "_rel"] = mm(s[:, 1 + p])
        row[nm + "_done"] = mm(s[:, 5 + p])
    row["exit"] = mm(s[:, 10])
    print(json.dumps(row))
    if i > 0:
        att = {k: mm(s[:, 16 + j]) for j, k in enumerate(
            ["a_entry", "a_flags", "a_q", "a_pages", "a_part", "a_merged", "a_out", "a_exit",
             "it_start", "it_k", "it_scores", "it_softmax", "it_pv", "m_group0_ready"])}
        sp = s[:, 16 + 14]
        att["m_group0_spins_max"] = int(sp.max())
        print(json.dumps({"layer": li, "attention_warp0_first_piece": att}))

# split-tile finishers of phase ASTRAEA_TRACE_PHASE (default 2, down): collect / own MMAs / epilogue
import os
tp = int(os.environ.get("ASTRAEA_TRACE_PHASE", "2"))
i = a.layers[-1] + 1
s = t[i]
fm = s[:, 11] > 0
if bool(fm.any()):
    f = s[fm]
    d = lambda k1, k0: round(float((f[:, k1] - f[:, k0]).median()) / 1000, 2)  # noqa: E731
    print(json.dumps({"phase": tp, "finishers": int(fm.sum()), "epilogue_us": d(14, 13),
                      "tmem_ld_us": d(30, 13), "acc_add_us": d(31, 30), "to_mark0_us": d(28, 31),
                      "mark0_to_mark1_us": d(29, 28), "tail_us": d(14, 29)}))
if bool(fm.any()) and os.environ.get("TRACE_FINISHERS"):
    base14 = float(s[:, 1 + tp][s[:, 1 + tp] > 0].median()) if tp < 4 else float(s[fm][:, 13].min())
    idx = torch.nonzero(fm).view(-1).tolist()
    rows = sorted(((int(c), [round(float(s[c, k] - base14) / 1000, 2) for k in (11, 12, 13, 28, 29, 14)]) for c in idx),
                  key=lambda r: -r[1][-1])
    print(json.dumps({"phase": tp, "finishers_by_done (cta, [collect_start, collect_done, own_mma, mark0, mark1, done])": rows[:10] + rows[-3:]}))
if bool(fm.any()) and tp < 4:
    rel = float(s[:, 1 + tp][s[:, 1 + tp] > 0].median())   # the phase's activations released
    f = s[fm]
    g = lambda k: [round(float((f[:, k] - rel).median()) / 1000, 2), round(float((f[:, k] - rel).max()) / 1000, 2)]  # noqa: E731
    print(json.dumps({"phase": tp, "finishers": int(fm.sum()), "collect_start": g(11), "collect_done": g(12),
                      "own_mma_done": g(13), "xch_done": g(30), "stores_done": g(31), "epilogue_done": g(14),
                      "others_done_median": round(float((s[~fm][:, 5 + tp] - rel).median()) / 1000, 2),
                      "all_done_max": round(float((s[:, 5 + tp] - rel).max()) / 1000, 2)}))

if a.per_cta:
    # per-CTA phase completion (relative to the phase's activation release) of one launch
    i = a.layers[-1] + 1
    s = t[i]
    for p, nm in enumerate(names):
        rel = float(s[:, 1 + p][s[:, 1 + p] > 0].median())
        done = (s[:, 5 + p] - rel) / 1000
        order = torch.argsort(done, descending=True)[:12]
        print(json.dumps({"phase": nm, "median_us": round(float(done.median()), 2),
                          "slowest": [[int(c), round(float(done[c]), 2)] for c in order]}))
