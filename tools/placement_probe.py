"""Cluster JCT under free-token vs round-robin placement (host only, model
clock, the bench's C2 configuration scaled to N replicas): one JSON line per
(N, placement). python tools/placement_probe.py --capacity 12000"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import bench  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402
from paper_2512_14142_b200.cluster import ClusterScheduler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--capacity", type=int, default=12000)
ap.add_argument("--qps", type=float, default=2.0)
ap.add_argument("--cost-tables", default="calibrated")
a = ap.parse_args()
ns = reference.load()
for world in (1, 2, 4, 8):
    args = bench.parse(["--gpus", str(world), "--capacity", str(a.capacity), "--qps", str(a.qps),
                        "--cost-tables", a.cost_tables, "--placement", "round-robin"])
    full = []
    for r in range(world):
        full += bench.build_workload(args, r, world)[0]
    pred = bench.build_workload(args, 0, world)[1]

    def make(i):
        pol, mem, cfg = bench.make_run(ns, None, pred, args, 131072)
        return pol, pred, mem, cfg

    for placement in ("free-tokens", "least-requests", "round-robin"):
        rep = ClusterScheduler(ns, full, world, make, placement=placement).run()
        agg = rep.aggregates()
        print(json.dumps({"replicas": world, "placement": placement, "capacity": a.capacity, "qps_per_replica": a.qps,
                          "tables": a.cost_tables, **{k: agg[k] for k in ("count", "avg_jct", "p99_jct", "req_per_s",
                                                                          "per_replica")}}), flush=True)
