"""Per-phase timeline of one decode-step launch (astraea_debug_step_trace):
for each phase, [median, max] over CTAs of when the weight producer / the
activation producer started it, when the MMA warp and the epilogue finished
it, in microseconds after the first CTA entered."""
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
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--ctx", type=int, default=900)
ap.add_argument("--l2", type=int, default=0)
ap.add_argument("--layers", type=int, nargs="+", default=[0, 1, 15, 31])
a = ap.parse_args()
cfg = PRESETS[a.model]
w = LlamaWeights(cfg)
B, nb = a.batch, (a.ctx + 16) // 16
pool = KvPool(cfg, B * nb + 4)
r = LlamaRunner(w, pool)
r.l2_ahead = a.l2
table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
tok = torch.zeros(B, dtype=torch.int32, device="cuda")
pos = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
slots = table[:, a.ctx // 16] * 16 + a.ctx % 16
ctxd = torch.full((B,), a.ctx + 1, dtype=torch.int32, device="cuda")
keys = torch.zeros(B, dtype=torch.int64, device="cuda")
for _ in range(3):
    r.decode(tok, pos, slots, table, ctxd, keys_out=keys)
torch.cuda.synchronize()
nph = r.last_program.n
G = torch.cuda.get_device_properties(0).multi_processor_count
buf = torch.zeros(G * nph * 8 + G + G * 64, dtype=torch.int64, device="cuda")
lib = L.load()
lib.astraea_debug_step_trace(buf.data_ptr())
r.decode(tok, pos, slots, table, ctxd, keys_out=keys)
torch.cuda.synchronize()
lib.astraea_debug_step_trace(None)
t = buf.cpu().double()
entry = t[G * nph * 8: G * nph * 8 + G]
atr = t[G * nph * 8 + G:].view(G * 4, 16)
base = entry.min()
st = t[: G * nph * 8].view(G, nph, 8)
names = ["qkv0"] + [n for _ in range(cfg.num_layers) for n in ("attn", "o", "gu", "down", "qkv")]
names[-1] = "lm"


def mm(col):
    col = col[col > 0]
    if col.numel() == 0:
        return None
    return [round(float(col.median() - base) / 1000, 1), round(float(col.max() - base) / 1000, 1)]


print(json.dumps({"entry": mm(entry), "nph": nph}))
for p in range(nph):
    layer = (p - 1) // 5 if p else 0
    if layer not in a.layers and p != nph - 1:
        continue
    print(json.dumps({"p": p, "name": names[p] if p < len(names) else "?", "layer": layer,
                      "w_start": mm(st[:, p, 0]), "x_start": mm(st[:, p, 1]), "mma_done": mm(st[:, p, 3]),
                      "epi_done": mm(st[:, p, 2])}))
act = atr[atr[:, 0] > 0]
rowsel = act[:, 7].argmax()
print(json.dumps({"attn_layer0_warps": int(act.shape[0]),
                  "slowest_warp_us": [round(float(v - base) / 1000, 1) if v > 0 else None for v in act[rowsel]],
                  "median_us": [round(float(c[c > 0].median() - base) / 1000, 1) if (c > 0).any() else None
                                for c in act.T]}))
end = st[:, :, 2].max()
print(json.dumps({"total_us": round(float(end - base) / 1000, 1)}))
