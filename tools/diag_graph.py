"""Locate the first batch where CUDA-graph decode and eager decode diverge:
per batch, generated tokens and a checksum of the KV pool, for
eager / graphs / graphs re-captured every batch."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import scenarios  # noqa: E402
from gpu_util import datapath_for  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402
host = reference.load()   # the unmodified reference package
from paper_2512_14142_b200.gpu.datapath import KvDataPath  # noqa: E402
from paper_2512_14142_b200.gpu.engine import GpuEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1b200/6000"


def run(mode):
    wl, pol, pred, mem, cfg = scenarios.build(host, name)
    dp = datapath_for(mem.capacity_tokens)
    dp.use_graphs = mode != "eager"
    log = []
    orig = dp.launch_batch

    def lb(members):
        if mode == "fresh":
            dp._graphs.clear()
        r = orig(members)
        torch.cuda.synchronize()
        rows = [(m.state.spec.id, m.segment_index, str(m.prior_location)) for m in members]
        log.append((rows, dp.results[-1][1].tolist(), float(dp.pool.data.double().sum())))
        return r

    dp.launch_batch = lb
    GpuEngine(wl, pol, pred, mem, cfg, dp).run()
    return log


logs = {m: run(m) for m in ("eager", "graphs", "fresh")}
for m in ("graphs", "fresh"):
    first = None
    for i, (a, b) in enumerate(zip(logs["eager"], logs[m])):
        if a[1] != b[1] or a[2] != b[2]:
            first = i
            break
    print(m, "first differing batch:", first)
    if first is not None:
        a, b = logs["eager"][first], logs[m][first]
        print("  rows", a[0])
        print("  pool sum eager", a[2], m, b[2], "tokens equal", a[1] == b[1])
        for r, (x, y) in enumerate(zip(a[1], b[1])):
            if x != y:
                k = next(i for i, (u, v) in enumerate(zip(x, y)) if u != v)
                print("  row", r, "pos", k, "eager", x[max(0, k - 3):k + 3], m, y[max(0, k - 3):k + 3])
        if first:
            print("  previous batch pool sums", logs["eager"][first - 1][2], logs[m][first - 1][2])
