"""Decode determinism check: run one GPU-engine scenario under several
launch variants (CUDA graphs on/off, chained decode GEMMs on/off) twice
each, and report whether the generated tokens are identical.

    python tools/diag_determinism.py [--scenario c1b200/6000] [--model tiny]
(set ASTRAEA_PDL=0 in the environment to disable programmatic dependent launch)
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import scenarios  # noqa: E402
from gpu_util import datapath_for  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402
host = reference.load()   # the unmodified reference package
from paper_2512_14142_b200.gpu.engine import GpuEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scenario", default="c1b200/6000")
ap.add_argument("--model", default="tiny")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()


def run(graphs, chain):
    wl, pol, pred, mem, cfg = scenarios.build(host, a.scenario)
    dp = datapath_for(mem.capacity_tokens, model=a.model)
    dp.use_graphs = graphs
    dp.runner.use_chain = chain
    GpuEngine(wl, pol, pred, mem, cfg, dp).run()
    return [h.cpu().tolist() for _, h in dp.results]


def first_diff(x, y):
    for bi, (bx, by) in enumerate(zip(x, y)):
        if bx != by:
            for ri, (rx, ry) in enumerate(zip(bx, by)):
                if rx != ry:
                    k = next(i for i, (u, v) in enumerate(zip(rx, ry)) if u != v)
                    return {"batch": bi, "row": ri, "pos": k}
            return {"batch": bi}
    return None


res = {}
for graphs in (True, False):
    for chain in (True, False):
        outs = [run(graphs, chain) for _ in range(a.reps)]
        key = f"graphs={int(graphs)} chain={int(chain)}"
        res[key] = outs[0]
        print(key, "self-consistent:", all(o == outs[0] for o in outs),
              [first_diff(outs[0], o) for o in outs[1:]], flush=True)
base = res["graphs=0 chain=0"]
for k, v in res.items():
    print(k, "vs graphs=0 chain=0:", first_diff(base, v))
print("PDL", os.environ.get("ASTRAEA_PDL", "1"))
