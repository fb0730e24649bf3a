"""One Llama-3-8B prefill forward of T tokens after warm-up, bracketed by
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures exactly its
launches; summarise the launch list with --summarise <csv>.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        --log-file gpurun_out/pf.csv python tools/prefill_launches.py --tokens 2048
    python tools/prefill_launches.py --summarise gpurun_out/pf.csv
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=2048)
ap.add_argument("--summarise", default=None)
a = ap.parse_args()

if a.summarise:
    import csv
    from collections import defaultdict
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in csv.DictReader(l for l in open(a.summarise) if l.startswith('"')):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:70]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1000 if unit in ("ns", "nsecond") else (v * 1000 if unit in ("ms", "msecond") else v)
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{tot[k]:10.1f} us  {100 * tot[k] / total:5.1f}%  x{cnt[k]:4d}  {k}")
    print(f"{total:10.1f} us  total (serialised, cold-cache)")
    sys.exit(0)

import torch

from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

cfg = PRESETS["llama3-8b"]
T = a.tokens
w = LlamaWeights(cfg, seed=0)
nb = (T + 15) // 16 + 1
pool = KvPool(cfg, nb + 8)
r = LlamaRunner(w, pool)
d = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
ids = d([(7 * i) % cfg.vocab for i in range(T)])
pos = d(list(range(T)))
table = d([list(range(nb))])
args = (ids, pos, pos, d([0, T]), table, d([T]), torch.tensor([T - 1], device="cuda"), T)
for _ in range(2):
    r.prefill(*args)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r.prefill(*args)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
