"""Parity scenarios, built against *any* module exposing the reference API.

``build(ns, name)`` returns ``(workload, policy, predictor, memory, config)``
using the classes of namespace ``ns`` -- either the reference package
(``agentsched``, only when generating golden fixtures in the build
container) or ``paper_2512_14142_b200.host``. The same scenario therefore
runs through both implementations and the reports are compared byte for
byte.

Scenario families:

* ``fig2/<policy>``           -- Figure-2 demo, serial, batch 1, preserve
                                 (reference tests/conftest.py:24-31).
* ``c1/<policy>/<cap>/<mode>`` -- config C1: ``generate(seed=0, qps=1,
                                 4 segments)[:64]``, parallel-max.
* ``c1b200/<cap>``             -- C1 with B200-like cost tables (swap-heavy).
* ``c2/<cap>``                 -- C2 trace (default segment mix, qps 2).
* ``hetero/<seed>/<policy>``   -- the reference's bimodal ``hetero_workload``
                                 at qps 3 (test_acceptance.py:81-122), which
                                 exercises discard.
* ``decomp/...``               -- criterion-4 grid (test_acceptance.py:239-263).
* ``aging/<tau>``              -- aging scenario (test_acceptance.py:125-159).
* ``noise``                    -- predictor noise sigma 0.3.
* ``c1cal/<cap>``              -- C1 with the cost tables *measured* on the B200
                                 (profiles/r1_b200_cost_tables.json, written by
                                 tools/calibrate.py).
"""

from __future__ import annotations

import json
import random
from pathlib import Path

CALIBRATION = Path(__file__).resolve().parent.parent / "profiles" / "r1_b200_cost_tables.json"

POLICY_NAMES = ("stateful-mlfq", "fcfs", "sjf-segment", "sjf-request", "las")

# Swap-heavy tables: prefill ~40k tok/s, decode 6 ms/token, swap 380k tok/s,
# Llama-3-8B KV bytes per token (probe p4).
B200_LIKE_PREFILL = ((128, 0.0052), (256, 0.0084), (512, 0.0148), (1024, 0.0276), (2048, 0.0532))


def c1_trace(ns, n=64):
    cfg = ns.WorkloadConfig(seed=0, qps=1.0, duration=10_000.0,
                            segment_count_distribution={4: 1.0})
    return ns.generate(cfg)[:n]


def c2_trace(ns, n=64, qps=2.0, seed=0):
    return ns.generate(ns.WorkloadConfig(seed=seed, qps=qps, duration=10_000.0))[:n]


def hetero_workload(ns, seed, qps, duration=40.0):
    """Bimodal mix: one-shot prompts plus long tool-calling chains."""
    heavy = ((ns.ApiCategory.CHAT, 28.6, 0.35), (ns.ApiCategory.IMAGE_GEN, 20.03, 0.4),
             (ns.ApiCategory.TTS, 10.0, 0.25))
    rng = random.Random(seed)
    cats = [c for c, _, _ in heavy]
    weights = [w for _, _, w in heavy]
    means = {c: m for c, m, _ in heavy}
    out = []
    t = 0.0
    while True:
        t += rng.expovariate(qps)
        if t >= duration:
            return out
        if rng.random() < 0.55:
            segs = (ns.SegmentSpec(1, rng.randint(400, 800), rng.randint(180, 260)),)
        else:
            count = rng.randint(3, 5)
            parts = []
            for j in range(1, count + 1):
                n_in = rng.randint(60, 160)
                n_gen = rng.randint(30, 70)
                if j == count:
                    parts.append(ns.SegmentSpec(j, n_in, n_gen))
                else:
                    cat = rng.choices(cats, weights=weights)[0]
                    api_s = means[cat] * rng.lognormvariate(-0.03125, 0.25)
                    parts.append(ns.SegmentSpec(j, n_in, n_gen, cat, api_s))
            segs = tuple(parts)
        out.append(ns.RequestSpec(id=f"h{len(out):05d}", arrival_time=t, segments=segs))


def aging_workload(ns):
    long_req = ns.RequestSpec(
        id="long", arrival_time=0.0,
        segments=(ns.SegmentSpec(1, 1, 1, direct_compute_time=10.0),
                  ns.SegmentSpec(2, 0, 1, direct_compute_time=5.0)))
    stream = [ns.RequestSpec(id=f"s{k:03d}", arrival_time=0.5 + 0.9 * k,
                             segments=(ns.SegmentSpec(1, 1, 1, direct_compute_time=1.0),))
              for k in range(200)]
    return [long_req] + stream


def b200_like_predictor(ns):
    return ns.ServiceTimePredictor(profile=ns.PrefillProfile(B200_LIKE_PREFILL),
                                   decode=ns.DecodeModel(0.006))


def calibrated_predictor(ns, path=None):
    """ServiceTimePredictor from B200-measured tables (default: the round-1
    tables the c1cal goldens were generated with)."""
    cal = json.loads((path or CALIBRATION).read_text())
    cfg = dict(cal["predictor"])
    cfg["api_latency_means"] = ns.ServiceTimePredictor().to_config()["api_latency_means"]
    return ns.ServiceTimePredictor.from_config(cfg), cal


def scenario_names():
    names = [f"fig2/{p}" for p in POLICY_NAMES]
    for p in POLICY_NAMES:
        for cap in (40_000, 12_000, 6_000, 3_600):
            for mode in ("adaptive", "preserve"):
                names.append(f"c1/{p}/{cap}/{mode}")
    names += [f"c1b200/{cap}" for cap in (12_000, 6_000, 3_600)]
    names += [f"c1cal/{cap}" for cap in (12_000, 6_000, 3_600)]
    names += [f"c2/{cap}" for cap in (40_000, 12_000)]
    for seed in (0, 1):
        for p in ("stateful-mlfq", "fcfs", "sjf-segment"):
            names.append(f"hetero/{seed}/{p}")
    for p in ("stateful-mlfq", "fcfs"):
        for cm in ("serial", "parallel-max"):
            for mode in ("adaptive", "preserve"):
                for cap in (8_000, 40_000):
                    names.append(f"decomp/{p}/{cm}/{mode}/{cap}")
    names += ["aging/5.0", "aging/none", "noise", "spill/2"]
    return names


def build(ns, name):
    parts = name.split("/")
    fam = parts[0]
    if fam == "fig2":
        pred = ns.figure2_predictor()
        return (ns.figure2_workload(), ns.make_policy(parts[1], pred), pred,
                ns.MemoryModel(capacity_tokens=1_000_000),
                ns.SimConfig(cost_model="serial", max_batch_segments=1, cache_mode="preserve"))
    if fam == "c1":
        pred = ns.ServiceTimePredictor()
        return (c1_trace(ns), ns.make_policy(parts[1], pred, ns.MlfqConfig()), pred,
                ns.MemoryModel(capacity_tokens=int(parts[2])),
                ns.SimConfig(cost_model="parallel-max", cache_mode=parts[3]))
    if fam == "c1b200":
        pred = b200_like_predictor(ns)
        return (c1_trace(ns), ns.make_policy("stateful-mlfq", pred, ns.MlfqConfig()), pred,
                ns.MemoryModel(capacity_tokens=int(parts[1]), bytes_per_token=131072.0,
                               swap_bandwidth_tokens_per_s=380_000.0),
                ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive"))
    if fam == "c1cal":
        pred, cal = calibrated_predictor(ns)
        return (c1_trace(ns), ns.make_policy("stateful-mlfq", pred, ns.MlfqConfig()), pred,
                ns.MemoryModel(capacity_tokens=int(parts[1]), bytes_per_token=float(cal["bytes_per_token"]),
                               swap_bandwidth_tokens_per_s=float(cal["swap_bandwidth_tokens_per_s"])),
                ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive"))
    if fam == "c2":
        pred = ns.ServiceTimePredictor()
        return (c2_trace(ns), ns.make_policy("stateful-mlfq", pred, ns.MlfqConfig()), pred,
                ns.MemoryModel(capacity_tokens=int(parts[1]), bytes_per_token=131072.0),
                ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive"))
    if fam == "hetero":
        pred = ns.ServiceTimePredictor()
        return (hetero_workload(ns, int(parts[1]), 3.0),
                ns.make_policy(parts[2], pred, ns.MlfqConfig()), pred,
                ns.MemoryModel(capacity_tokens=int(12_000 * 0.3)),
                ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive",
                             max_batch_segments=2))
    if fam == "decomp":
        pred = ns.ServiceTimePredictor()
        wl = ns.generate(ns.WorkloadConfig(seed=11, qps=1.0, duration=30.0))
        return (wl, ns.make_policy(parts[1], pred, ns.MlfqConfig()), pred,
                ns.MemoryModel(capacity_tokens=int(parts[4])),
                ns.SimConfig(cost_model=parts[2], cache_mode=parts[3]))
    if fam == "aging":
        tau = None if parts[1] == "none" else float(parts[1])
        pred = ns.figure2_predictor()
        pol = ns.make_policy("stateful-mlfq", pred,
                             ns.MlfqConfig(num_queues=2, token_thresholds=(5.0,), aging_threshold=tau))
        return (aging_workload(ns), pol, pred, ns.MemoryModel(capacity_tokens=100_000),
                ns.SimConfig(cost_model="serial", max_batch_segments=1, cache_mode="preserve"))
    if fam == "noise":
        pred = ns.ServiceTimePredictor(noise_sigma=0.3, noise_seed=7)
        return (c1_trace(ns), ns.make_policy("stateful-mlfq", pred, ns.MlfqConfig()), pred,
                ns.MemoryModel(capacity_tokens=6_000),
                ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive"))
    if fam == "spill":
        pred = ns.ServiceTimePredictor()
        pol = ns.make_policy("stateful-mlfq", pred, ns.MlfqConfig(spillover=True))
        return (c2_trace(ns, qps=4.0), pol, pred, ns.MemoryModel(capacity_tokens=12_000),
                ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive",
                             max_batch_segments=int(parts[1])))
    raise KeyError(name)


def run_scenario(ns, name):
    wl, pol, pred, mem, cfg = build(ns, name)
    return ns.run(wl, pol, pred, mem, cfg)
