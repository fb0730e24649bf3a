"""Memory-pressure (C3) and request-rate (C4) sweeps of the B200 data path.

For each cell: the reference scheduler (the unmodified reference, decisions byte-identical
to the reference -- asserted against a host-only run) drives the Llama-3-8B
data path; the clock advances by B200-measured batch and swap durations
(``clock="measured"``; API waits stay virtual). Reported per cell: avg / p99
JCT, req/s, and the KV actions the adaptive policy chose (preserve / swap /
discard, with the decision reasons), plus the same for the model clock.

    python tools/sweep.py pressure --out gpurun_out/sweep_pressure.json
    python tools/sweep.py rate     --out gpurun_out/sweep_rate.json
"""
import argparse
import json
import sys
import time
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import scenarios  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402
host = reference.load()   # the unmodified reference package
from paper_2512_14142_b200.gpu.datapath import KvDataPath  # noqa: E402
from paper_2512_14142_b200 import plugin  # noqa: E402
from paper_2512_14142_b200.gpu.engine import GpuEngine  # noqa: E402
from paper_2512_14142_b200.gpu.model import PRESETS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("kind", choices=["pressure", "rate"])
ap.add_argument("--requests", type=int, default=64, help="C2 trace length (64 in the survey's C2/C3)")
ap.add_argument("--base", type=int, default=40_000, help="C3: capacity x {0.3, 0.5, 0.7, 0.9} (SURVEY 8(d))")
ap.add_argument("--rate-capacity", type=int, default=12_000)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = PRESETS["llama3-8b"]


def trace(qps, n):
    full = host.generate(host.WorkloadConfig(seed=0, qps=qps, duration=4.0 * n / qps + 60.0))[:n]
    return sorted(full, key=lambda r: (r.arrival_time, r.id))


def cell(wl, capacity, tables, dp):
    if tables == "calibrated":
        pred, cal = scenarios.calibrated_predictor(host, ROOT / "profiles" / "r2_b200_cost_tables.json")
        bw = float(cal["swap_bandwidth_tokens_per_s"])
    else:
        pred, bw = host.ServiceTimePredictor(), 20_000.0
    def parts():
        return (host.make_policy("stateful-mlfq", pred, host.MlfqConfig()), pred,
                host.MemoryModel(capacity_tokens=capacity, bytes_per_token=float(cfg.kv_bytes_per_token),
                                 swap_bandwidth_tokens_per_s=bw),
                host.SimConfig(cost_model="parallel-max", cache_mode="adaptive"))
    ref = host.run(wl, *parts())
    t0 = time.time()
    dev0 = dict(dp.stats)
    model = GpuEngine(wl, *parts(), dp, clock="model").run()
    assert model.to_json() == ref.to_json(), "device run diverged from the host schedule"
    measured = GpuEngine(wl, *parts(), dp, clock="measured").run()
    acts = Counter(f"{e['chosen']}:{e['reason']}" for e in json.loads(model.to_json())["audits"]["waste_log"])
    agg_m, agg_s = measured.aggregates(), model.aggregates()
    return {"capacity_tokens": capacity, "cost_tables": tables, "requests": len(wl),
            "kv_actions": dict(acts),
            "measured_clock": {"avg_jct_s": agg_m["avg_jct"], "p99_jct_s": agg_m["p99_jct"],
                               "req_per_s": plugin.requests_per_second(measured)},
            "model_clock": {"avg_jct_s": agg_s["avg_jct"], "p99_jct_s": agg_s["p99_jct"],
                            "req_per_s": plugin.requests_per_second(model)},
            # device work of the measured-clock run (same plans as the model-clock run)
            "device": {k: (measured.device[k] - dev0[k]) // 2 for k in
                       ("batches", "prefill_tokens", "decode_steps", "swap_outs", "swap_ins", "discards",
                        "recompute_tokens")},
            "wall_s": round(time.time() - t0, 1)}


rows = []
n = a.requests
if a.kind == "pressure":
    wl = trace(2.0, n)
    base = a.base   # x {0.3 .. 0.9} (cli.py:41-47, 245-256)
    dp = KvDataPath(cfg, num_blocks=base // 16 + 2 * n + 64)
    for tables in ("calibrated", "reference-default"):
        for frac in (0.3, 0.5, 0.7, 0.9):
            rows.append(cell(wl, int(base * frac), tables, dp))
            print(json.dumps(rows[-1]), flush=True)
else:
    dp = KvDataPath(cfg, num_blocks=a.rate_capacity // 16 + 2 * n + 64)
    for qps in (1.0, 2.0, 4.0, 8.0):
        r = cell(trace(qps, n), a.rate_capacity, "calibrated", dp)
        r["qps"] = qps
        rows.append(r)
        print(json.dumps(r), flush=True)
if a.out:
    Path(a.out).write_text(json.dumps(rows, indent=1))
