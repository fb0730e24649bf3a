"""Mean decode batch the reference scheduler (stateful-MLFQ, adaptive KV,
parallel-max) forms on the reference trace generator, host only: one line
per (cost tables, requests, qps, capacity). Why the C2 bench runs at a mean
decode batch near 1: a batch closes at its longest member (parallel-max)
and requests spend most of their life in API waits, so few are ready at
once -- raising qps or the request count does not change that.

    python tools/batch_probe.py > profiles/r2_c2_batch_probe.txt
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import bench  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402

ns = reference.load()
print("tables requests qps capacity batches mean_decode_batch max_members decode_steps avg_jct_s")
for tables in ["calibrated", "reference"]:
    for n, qps in [(64, 2), (64, 8), (64, 32), (256, 4), (256, 8), (512, 8), (512, 16), (1024, 16)]:
        for cap in [12000, 40000]:
            args = bench.parse(["--qps", str(qps), "--capacity", str(cap), "--requests", str(n),
                                "--cost-tables", tables])
            shard, pred = bench.build_workload(args, 0, 1)
            batches, rep = bench.work_profile(ns, shard, pred, args, 131072)
            s = bench.summarize(batches, 0, len(batches))
            mx = max(b["members"] for b in batches)
            print(tables, n, qps, cap, len(batches), round(s["mean_batch"], 2), mx, s["decode_steps"],
                  round(rep.aggregates()["avg_jct"], 1), flush=True)
