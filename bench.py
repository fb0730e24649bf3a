"""Benchmark: Astraea's scheduler driving the B200 data path (BASELINE.json C2).

Workload (``config.workload``): C2 -- Llama-3-8B shape (random init, bf16);
the 64-request synthetic agent trace of the reference generator
(``generate(WorkloadConfig(seed=0, qps=2))[:64]``, default segment and
category mix, workload.py:390-433); Stateful-MLFQ + adaptive Preserve/Swap/
Discard, KV capacity 12,000 tokens per GPU (the 0.3 level of the survey's
40,000-token grid, 131,072 B/token), parallel-max; cost tables measured on the
B200 (profiles/r2_b200_cost_tables.json). The scheduler, KV policy and event
loop are the unmodified reference (``agentsched``), with the device attached
through ``paper_2512_14142_b200.plugin``; model clock, so every decision is
the reference's and the replay's report bytes are asserted equal to the
reference's own ``run()``.

One *step* = one scheduled batch of that replay: block allocation, the
members' (re)prefill, the decode loop until the last member's n_gen, and the
swap-outs/ins and discards the KV policy issues before the next batch. The
replay is deterministic; a window of K consecutive batches centred in it is
timed (the batches before it are the warm-up steps, >= W), bracketed by a
barrier + device synchronize on both sides, max over ranks.

  value      request-equivalents/s over the timed window: each completed
             segment counts 1/num_segments of its request (summed over a whole
             replay this is exactly the request count), device time (CUDA
             events on the data path's streams), prompt ids resident in HBM;
  replay     the whole 64-request replay, device-timed: requests/s;
  e2e        the same window through the public API (GpuEngine.run) on the
             host clock, prompt ids uploaded from pinned host memory per batch
             and generated tokens read back per batch (bytes reported);
  roofline   the dominant kernel (one decoder layer's fused launch: paged
             attention + the chained tcgen05 GEMMs) at the window's mean
             decode batch and context, vs measured HBM bandwidth;
  jct_measured_clock  avg/p99 JCT and req/s with B200-measured durations;
  reference_scheduler the reference's own CPU path (``agentsched.run``) on the
             same trace: wall time, events/s, decision time, simulated JCT;
  cpu_baseline  the CPU port (oracle/cpu_baseline.py, fp32, all host cores)
             on a bounded sample of the same window.

Multi-GPU: one process per GPU (torchrun); the trace is partitioned
round-robin over (arrival, id) order with qps scaled by N ("weak"); no
collective on the data path; timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "avg/p99 JCT and req/s on synthetic agent trace; KV swap GB/s; decode HBM GB/s"
# cost tables measured on the B200 with this round's kernels (tools/calibrate.py)
CAL_TABLES = ROOT / "profiles" / "r2_b200_cost_tables.json"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10, help="timed steps (scheduled batches)")
    ap.add_argument("--warmup", type=int, default=3, help="untimed batches before the window (at least)")
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--requests", type=int, default=64, help="requests per rank (C2: 64)")
    ap.add_argument("--qps", type=float, default=2.0, help="arrival rate per rank")
    ap.add_argument("--capacity", type=int, default=12000, help="KV capacity (tokens) per GPU")
    ap.add_argument("--swap-mode", choices=("kernel", "dma", "staged"), default="staged",
                    help="K1/K2 path (tools/swap_load.py: staged keeps the host link at ~54 GB/s and slows a "
                         "concurrent decode by ~4%%; the zero-copy SM kernel slows it 2x)")
    ap.add_argument("--cost-tables", choices=("calibrated", "b200-like", "reference"), default="calibrated",
                    help="scheduler cost tables: measured on the B200 (profiles/r2_b200_cost_tables.json), "
                         "the survey's B200-like guess, or the reference defaults")
    ap.add_argument("--placement", choices=("free-tokens", "round-robin"), default="free-tokens",
                    help="multi-GPU: requests placed at arrival on the replica with the most free KV "
                         "tokens (the global scheduler, cluster.py), or round-robin over (arrival, id)")
    ap.add_argument("--measured-runs", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip roofline sweep / swap-under-load legs")
    return ap.parse_args(argv)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------------------- workload

def build_workload(args, rank, world):
    """The rank's shard of the C2 trace and the scheduler's cost tables."""
    from paper_2512_14142_b200 import reference
    import scenarios
    ns = reference.load()
    need = args.requests * world
    duration = 2.0 * need / (args.qps * world) + 60.0
    while True:  # the first n arrivals do not depend on the horizon once it covers them
        full = ns.generate(ns.WorkloadConfig(seed=0, qps=args.qps * world, duration=duration))
        if len(full) >= need:
            break
        duration *= 2
    full = full[:need]
    full.sort(key=lambda r: (r.arrival_time, r.id))
    tables = getattr(args, "cost_tables", "calibrated")
    if tables == "calibrated":
        pred, cal = scenarios.calibrated_predictor(ns, CAL_TABLES)
        args.swap_tokens_per_s = float(cal["swap_bandwidth_tokens_per_s"])
    elif tables == "b200-like":
        pred = scenarios.b200_like_predictor(ns)
        args.swap_tokens_per_s = 380_000.0
    else:
        pred = ns.ServiceTimePredictor()
        args.swap_tokens_per_s = 20_000.0
    placement = getattr(args, "placement", "round-robin")
    if world == 1 or placement == "round-robin":
        shard = full[rank::world]
    else:
        # the global scheduler (cluster.py) on the host: every rank computes
        # the same placement by free KV tokens and replays its own replica
        # (a replica's report is the reference run of its requests)
        from paper_2512_14142_b200.cluster import ClusterScheduler

        def make(i):
            pol, mem, cfg = make_run(ns, None, pred, args, 131072)
            return pol, pred, mem, cfg

        placed = ClusterScheduler(ns, full, world, make, placement=placement).run().placement
        shard = [r for r in full if placed[r.id] == rank]
    return shard, pred


def make_run(ns, shard, pred, args, bytes_per_token):
    policy = ns.make_policy("stateful-mlfq", pred, ns.MlfqConfig())
    memory = ns.MemoryModel(capacity_tokens=args.capacity, bytes_per_token=float(bytes_per_token),
                            swap_bandwidth_tokens_per_s=getattr(args, "swap_tokens_per_s", 380_000.0))
    config = ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive")
    return policy, memory, config


class WorkProbe:
    """CPU stand-in for the data path: records each scheduled batch's exact
    work (what the device executes for it) without a GPU."""

    measure = False

    def __init__(self):
        self.batches = []

    def launch_batch(self, members):
        n = [m.state.current_seg.n_gen for m in members]
        pre = ctx_rows = 0
        for m in members:
            seg = m.state.current_seg
            extra = m.state.context_before_current if m.prior_location.value == "dropped" else 0
            pre += seg.n_in + extra
            ctx_rows += m.state.context_after(m.segment_index) * seg.n_gen
        self.batches.append(dict(members=len(members), decode_steps=max(n), row_steps=sum(n),
                                 prefill_tokens=pre, mean_ctx=ctx_rows / max(1, sum(n)),
                                 req_equiv=sum(1.0 / m.state.spec.num_segments for m in members)))

    def drop(self, st):
        pass

    def swap_out_begin(self, st):
        pass

    def swap_out_done(self, st):
        pass

    def swap_in_begin(self, st):
        pass

    def swap_in_done(self, st):
        pass

    def release(self, st, where):
        pass

    def synchronize(self):
        pass

    def audit(self, states):
        pass

    def summary(self):
        return {}


def work_profile(ns, shard, pred, args, bytes_per_token):
    """Per-batch work of the replay (the reference engine + a CPU probe) and
    the report, which must equal the reference's own ``run()`` bytes."""
    from paper_2512_14142_b200 import plugin
    probe = WorkProbe()
    pol, mem, cfg = make_run(ns, shard, pred, args, bytes_per_token)
    rep = plugin.run_on_gpu(shard, pol, pred, mem, cfg, probe)
    pol, mem, cfg = make_run(ns, shard, pred, args, bytes_per_token)
    plain = ns.run(shard, pol, pred, mem, cfg)
    assert rep.to_json() == plain.to_json(), "plugin engine diverged from the reference run()"
    return probe.batches, rep


def window_start(n_batches, steps, warmup):
    """First timed batch: the K-batch window centred in the replay, after at
    least W warm-up batches."""
    if n_batches < warmup + steps:
        raise SystemExit(f"the replay has {n_batches} batches; --warmup {warmup} + --steps {steps} do not fit")
    return max(warmup, (n_batches - steps) // 2)


def summarize(batches, s, k):
    win = batches[s:s + k]
    dsteps = sum(b["decode_steps"] for b in win)
    rows = sum(b["row_steps"] for b in win)
    return dict(batches=len(win), decode_steps=dsteps, row_steps=rows,
                mean_batch=rows / max(1, dsteps),
                mean_ctx=sum(b["mean_ctx"] * b["row_steps"] for b in win) / max(1, rows),
                prefill_tokens=sum(b["prefill_tokens"] for b in win),
                req_equiv=sum(b["req_equiv"] for b in win),
                members=sum(b["members"] for b in win))


def reference_scheduler(ns, shard, pred, args, bytes_per_token, reps=7):
    """The reference's own CPU path on the same trace:
    ``agentsched.run`` with the shipped audits on, best of ``reps`` wall
    times, events/s, ``build_next_batch`` decision time, and its simulated
    outcome (with the bench's cost tables and with the reference defaults)."""
    from paper_2512_14142_b200 import plugin
    walls, decisions = [], []
    rep = None
    for _ in range(reps):
        pol, mem, cfg = make_run(ns, shard, pred, args, bytes_per_token)
        inner = pol.build_next_batch
        ts = []

        def timed(*a, _f=inner, _ts=ts, **kw):
            t = time.perf_counter()
            out = _f(*a, **kw)
            _ts.append(time.perf_counter() - t)
            return out

        pol.build_next_batch = timed
        t0 = time.perf_counter()
        rep = ns.run(shard, pol, pred, mem, cfg)
        walls.append(time.perf_counter() - t0)
        decisions = ts
    agg = rep.aggregates()
    dpred = ns.ServiceTimePredictor()
    pol = ns.make_policy("stateful-mlfq", dpred, ns.MlfqConfig())
    mem = ns.MemoryModel(capacity_tokens=args.capacity, bytes_per_token=float(bytes_per_token))
    drep = ns.run(shard, pol, dpred, mem, ns.SimConfig(cost_model="parallel-max", cache_mode="adaptive"))
    dagg = drep.aggregates()
    ev = rep.audits["events_processed"]
    return {"impl": "agentsched.run (unmodified reference, 1 Python thread)",
            "cores": 1, "wall_ms": min(walls) * 1e3, "events": ev, "events_per_s": ev / min(walls),
            "build_next_batch_us_mean": statistics.mean(decisions) * 1e6,
            "build_next_batch_us_p50": statistics.median(decisions) * 1e6,
            "simulated": {"tables": args.cost_tables, "avg_jct_s": agg["avg_jct"], "p99_jct_s": agg["p99_jct"],
                          "req_per_s": plugin.requests_per_second(rep)},
            "simulated_reference_tables": {"avg_jct_s": dagg["avg_jct"], "p99_jct_s": dagg["p99_jct"],
                                           "req_per_s": plugin.requests_per_second(drep)}}


class ClockSampler:
    def __init__(self, enabled, idx):
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"clocks_{os.getpid()}.csv"
        if enabled:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={idx}",
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "200"],
                    stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except OSError:
                self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = [l.split(", ") for l in self.path.read_text().splitlines() if l.strip()]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        if not sm:
            return None
        mx = float(rows[0][1])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 3 + i and r[3 + i].strip() == "Active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons, "samples": len(sm)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: run every rank on one device over gloo (NCCL needs one GPU per rank)
    if os.environ.get("ASTRAEA_BENCH_SHARE_GPU") == "1":
        local = 0
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local) if torch.cuda.is_available() else None
        backend = "gloo" if (os.environ.get("ASTRAEA_BENCH_SHARE_GPU") == "1" or not torch.cuda.is_available()) \
            else "nccl"
        dist.init_process_group(backend)
    return rank, world, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def min_over_ranks(x, world):
    return -max_over_ranks(-x, world)


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def roofline_sweep(dp, cfg, ctx, hbm, batches=(1, 4, 8, 16, 32)):
    """The dominant kernel and the whole decode step at several batch sizes
    (same context), vs measured HBM: where the step leaves the roofline."""
    out = []
    for B in batches:
        ms, by, c = chain_kernel_time(dp, cfg, B, ctx, reps=30)
        sg, sms = decode_step_gbs(dp, cfg, B, ctx)
        out.append({"batch": B, "ctx": c, "chain_us": ms * 1e3, "chain_frac": by / (ms / 1000.0) / 1e9 / hbm,
                    "step_ms": sms, "step_frac": sg / hbm})
    return out


def swap_under_load(dp, cfg, tokens, batch=4, steps=40, swaps=8):
    """K1/K2 while the decode loop runs (SURVEY.md hard part 3): decode steps
    on the compute stream and swap-out/in round trips of ``tokens`` tokens on
    the swap stream, launched together; per mode: swap GB/s alone and under
    load, decode step alone and under load."""
    import torch
    from paper_2512_14142_b200.gpu import lib as L
    from paper_2512_14142_b200.gpu import ops
    nb = (tokens + 15) // 16
    ctx = min(tokens, 2048)
    dnb = (ctx + 16) // 16
    assert batch * dnb + 2 * nb <= dp.pool.num_blocks
    table = torch.arange(batch * dnb, dtype=torch.int32, device="cuda").view(batch, dnb)
    src = list(range(batch * dnb, batch * dnb + nb))
    dst = list(range(batch * dnb + nb, batch * dnb + 2 * nb))
    tok = torch.zeros(batch, dtype=torch.int32, device="cuda")
    pos = torch.full((batch,), ctx, dtype=torch.int32, device="cuda")
    slots = table[:, ctx // 16] * 16 + ctx % 16
    ctxd = torch.full((batch,), ctx + 1, dtype=torch.int32, device="cuda")
    keys = torch.zeros(batch, dtype=torch.int64, device="cuda")
    slot = torch.empty(tokens * dp.pool.bytes_per_token, dtype=torch.uint8, pin_memory=True)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def decode_loop():
        a, b = ev(), ev()
        a.record(dp.compute)
        for _ in range(steps):
            dp.runner.decode(tok, pos, slots, table, ctxd, stream=dp.compute, keys_out=keys)
        b.record(dp.compute)
        return a, b

    def swap_loop(mode):
        a, b = ev(), ev()
        a.record(dp.swapper)
        for _ in range(swaps):
            ops.swap_out(dp.pool.geo, dp.pool.data, src, tokens, slot, mode, dp.swapper)
            ops.swap_in(dp.pool.geo, dp.pool.data, dst, tokens, slot, mode, dp.swapper)
        b.record(dp.swapper)
        return a, b

    res = {"tokens": tokens, "bytes_per_swap": tokens * dp.pool.bytes_per_token, "decode_batch": batch,
           "decode_ctx": ctx}
    decode_loop()
    torch.cuda.synchronize()
    a, b = decode_loop()
    torch.cuda.synchronize()
    alone_dec = a.elapsed_time(b) / steps
    res["decode_step_ms_alone"] = alone_dec
    moved = 2 * swaps * tokens * dp.pool.bytes_per_token
    for name, mode in (("kernel", L.SWAP_KERNEL), ("dma", L.SWAP_DMA), ("staged", L.SWAP_STAGED)):
        swap_loop(mode)
        torch.cuda.synchronize()
        a, b = swap_loop(mode)
        torch.cuda.synchronize()
        alone = a.elapsed_time(b)
        torch.cuda.synchronize()
        sa, sb = swap_loop(mode)
        da, db = decode_loop()
        torch.cuda.synchronize()
        loaded_swap = sa.elapsed_time(sb)
        loaded_dec = da.elapsed_time(db) / steps
        res[name] = {"swap_gbs_alone": moved / (alone / 1000.0) / 1e9,
                     "swap_gbs_under_decode": moved / (loaded_swap / 1000.0) / 1e9,
                     "decode_step_ms_under_swap": loaded_dec,
                     "decode_slowdown": loaded_dec / alone_dec}
    return res


# --------------------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's CPU implementation of the path on the host cores: the
    CPU port (oracle/cpu_baseline.py, fp32, every host thread) sampled on the
    same window of scheduled batches the GPU arm times; plus the reference's
    own scheduler path (``agentsched.run``). Rank 0 only."""
    rank, world, _ = dist_setup(args)
    if rank != 0:
        barrier(world)
        return
    from oracle.cpu_baseline import CpuLlama, batch_sample
    from paper_2512_14142_b200 import reference
    from paper_2512_14142_b200.gpu.model import PRESETS
    ns = reference.load()
    cfg = PRESETS[args.model]
    shard, pred = build_workload(args, 0, world)
    batches, rep = work_profile(ns, shard, pred, args, cfg.kv_bytes_per_token)
    s = window_start(len(batches), args.steps, args.warmup)
    model = CpuLlama(cfg)
    for b in batches[s - args.warmup: s]:
        batch_sample(model, b)                         # warm-up steps
    samples = [batch_sample(model, b) for b in batches[s: s + args.steps]]
    win = summarize(batches, s, args.steps)
    cpu_s = sum(x["batch_cpu_s"] for x in samples)
    value = win["req_equiv"] / cpu_s
    sample_ms = statistics.mean(x["sample_s"] for x in samples) * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": "req/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sample_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": config_block(args, shard, world, batches, s),
        "cpu_baseline": {"value": value, "unit": "req/s", "cores": model.threads, "kind": "port",
                         "sample": cpu_sample_text(args.steps, samples)},
        "e2e": {"value": value, "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "window": win,
        "reference_scheduler": reference_scheduler(ns, shard, pred, args, cfg.kv_bytes_per_token),
    }
    print(json.dumps(line))
    barrier(world)


def cpu_sample_text(k, samples):
    pre = statistics.median(x["prefill_chunk_s"] / x["prefill_chunk"] for x in samples if x["prefill_chunk_s"])
    dec = statistics.median(x["decode_step_s"] for x in samples)
    return (f"{k} window batches; per batch one full-model (32 layers, fp32) prefill chunk of <= 128 of its "
            f"prefill tokens and one decode step with its rows, timed; batch time = its prefill tokens x "
            f"measured s/token (median {pre * 1e3:.1f} ms/token) + its decode steps x measured step "
            f"(median {dec * 1e3:.0f} ms)")


def config_block(args, shard, world, batches, s):
    return {"workload": f"C2 {args.model} random-init, reference trace generate(seed 0, qps {args.qps}/rank)"
                        f"[:{args.requests * world}], {len(shard)} requests on this rank, stateful-mlfq + adaptive KV, "
                        f"capacity {args.capacity} tok/GPU, parallel-max, model clock, {args.cost_tables} "
                        f"cost tables; step = one scheduled batch, window = batches {s}..{s + args.steps - 1} "
                        f"of {len(batches)}",
            "global_requests": args.requests * world, "parallelism": f"replicas x{world}",
            "placement": "single replica" if world == 1 else f"{args.placement} (cluster.py)",
            "l2": "weights (15 GB) stream every decode step: inputs >> L2 (126 MB)",
            "replay_batches": len(batches), "window_start": s, "swap_mode": args.swap_mode}


# --------------------------------------------------------------------------- our arm

class StopReplay(Exception):
    pass


class Window:
    """Step hook: called before each batch launch; brackets batches
    [s, s + k) with barrier + synchronize + events (and the host clock)."""

    def __init__(self, dp, s, k, world, stop_after=False):
        self.dp, self.s, self.k, self.world, self.stop_after = dp, s, k, world, stop_after
        self.i = 0
        self.e0 = self.e1 = None
        self.wall = None
        self.launches = 0
        self.req_equiv = 0.0
        self.results = []

    def open(self):
        import torch
        from paper_2512_14142_b200.gpu import ops
        barrier(self.world)
        torch.cuda.synchronize()
        self.dp.drain_results()
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e0.record(self.dp.compute)
        self.t0 = time.perf_counter()
        self.l0 = ops.LAUNCHES[0]

    def close(self):
        import torch
        from paper_2512_14142_b200.gpu import ops
        self.dp.compute.wait_stream(self.dp.swapper)
        self.e1 = torch.cuda.Event(enable_timing=True)
        self.e1.record(self.dp.compute)
        for ev, _ in self.dp.results:   # the window's generated tokens are on the host
            ev.synchronize()
        torch.cuda.synchronize()
        self.wall = time.perf_counter() - self.t0
        self.launches = ops.LAUNCHES[0] - self.l0
        self.results = self.dp.drain_results()
        barrier(self.world)

    def __call__(self, engine):
        if self.i == self.s:
            self.open()
        if self.i == self.s + self.k:
            self.close()
            if self.stop_after:
                raise StopReplay
        if self.s <= self.i < self.s + self.k:
            self.req_equiv += sum(1.0 / engine.states[r].spec.num_segments for r, _ in engine._plan_entries)
        self.i += 1

    def finish(self):
        if self.e1 is None and self.e0 is not None:
            self.close()

    @property
    def device_ms(self):
        return self.e0.elapsed_time(self.e1)


def bench_engine():
    from paper_2512_14142_b200 import plugin
    _, gpu_engine = plugin.engine_classes()

    class BenchEngine(gpu_engine):
        hook = None

        def _launch_plan(self):
            if self.hook is not None:
                self.hook(self)
            return super()._launch_plan()

    return BenchEngine


def main():
    args = parse()
    if os.environ.get("ASTRAEA_BENCH_TRACEBACK_S"):   # diagnostics: dump every thread's stack on a hang
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["ASTRAEA_BENCH_TRACEBACK_S"]), exit=True)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    rank, world, local = dist_setup(args)
    torch.cuda.set_device(local)
    from paper_2512_14142_b200 import plugin, reference
    from paper_2512_14142_b200.gpu import lib as L
    from paper_2512_14142_b200.gpu.datapath import KvDataPath
    from paper_2512_14142_b200.gpu.model import PRESETS

    ns = reference.load()
    cfg = PRESETS[args.model]
    shard, pred = build_workload(args, rank, world)
    batches, ref_rep = work_profile(ns, shard, pred, args, cfg.kv_bytes_per_token)
    n_b = int(min_over_ranks(len(batches), world))
    s = window_start(n_b, args.steps, args.warmup)
    win = summarize(batches, s, args.steps)
    blocks = max(math.ceil(args.capacity / 16) + 2 * len(shard) + 64, 32 * 72)   # sweep room: B 32 x 1.1k ctx
    dp = KvDataPath(cfg, num_blocks=blocks, swap_mode={"kernel": L.SWAP_KERNEL, "dma": L.SWAP_DMA,
                                                             "staged": L.SWAP_STAGED}[args.swap_mode])
    Engine = bench_engine()

    def replay(hook=None, clock="model"):
        pol, mem, scfg = make_run(ns, shard, pred, args, cfg.kv_bytes_per_token)
        eng = Engine(shard, pol, pred, mem, scfg, dp, clock=clock)
        eng.hook = hook
        return eng.run()

    # ---- warm-up replay (graph capture, every kernel instantiation) + parity
    dp.prestage(shard)
    rep = replay()
    assert rep.to_json() == ref_rep.to_json(), "B200 replay diverged from the reference run()"
    dp.drain_results()

    # ---- value: the K-batch window, inputs resident in HBM, device-timed;
    # the whole replay is device-timed too
    clocks = ClockSampler(not args.no_clocks and rank == 0, local)
    w = Window(dp, s, args.steps, world)
    torch.cuda.synchronize()
    r0 = torch.cuda.Event(enable_timing=True)
    r0.record(dp.compute)
    rep = replay(hook=w)
    w.finish()
    dp.compute.wait_stream(dp.swapper)
    r1 = torch.cuda.Event(enable_timing=True)
    r1.record(dp.compute)
    r1.synchronize()
    clk = clocks.stop()
    assert rep.to_json() == ref_rep.to_json()
    dp.drain_results()
    ms = max_over_ranks(w.device_ms, world)
    value = sum_over_ranks(w.req_equiv, world) / (ms / 1000.0)
    replay_ms = max_over_ranks(r0.elapsed_time(r1), world)
    device = dict(rep.device)

    # ---- e2e: the same window through the public API, host buffers, host clock
    dp.staged = {}
    s0 = dict(dp.stats)
    we = Window(dp, s, args.steps, world, stop_after=True)
    try:
        replay(hook=we)
    except StopReplay:
        pass
    we.finish()
    dp.reset()
    e2e_s = max_over_ranks(we.wall, world)
    e2e = sum_over_ranks(we.req_equiv, world) / e2e_s
    h2d = (dp.stats["h2d_bytes"] - s0["h2d_bytes"])
    d2h = (dp.stats["d2h_bytes"] - s0["d2h_bytes"])
    dp.prestage(shard)

    # ---- measured-clock JCT (same scheduler, B200 durations, virtual API waits);
    # median of runs by avg JCT: the schedule reacts to run-to-run timing noise
    mruns = []
    for _ in range(args.measured_runs):
        r_ = replay(clock="measured")
        dp.drain_results()
        mruns.append((r_.aggregates(), plugin.requests_per_second(r_)))
    mruns.sort(key=lambda x: x[0]["avg_jct"])
    agg, m_rps = mruns[len(mruns) // 2]

    # ---- dominant kernel at the window's mean decode batch and context
    hbm, peak_kind = peaks()
    B = max(1, int(round(win["mean_batch"])))
    ctx = int(win["mean_ctx"])
    chain_ms, chain_bytes, chain_ctx = chain_kernel_time(dp, cfg, B, ctx)
    gemm_gbs = chain_bytes / (chain_ms / 1000.0) / 1e9
    step_gbs, step_ms = decode_step_gbs(dp, cfg, B, ctx)
    swap = swap_gbs(dp, cfg, ctx)
    line = {
        "metric": METRIC, "value": value, "unit": "req/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, reference trace generator)",
        "config": config_block(args, shard, world, batches, s),
        "e2e": {"value": e2e, "unit": "req/s", "h2d_bytes_per_step": int(h2d // args.steps),
                "d2h_bytes_per_step": int(d2h // args.steps)},
        "gpu_launches": int(w.launches),
        "roofline": {"bound": "hbm", "achieved": gemm_gbs, "peak": hbm, "unit": "GB/s", "frac": gemm_gbs / hbm,
                     "traffic": profiled_traffic(B),
                     "kernel": f"gemm_chain_kernel (layer: paged attention -> O -> GU -> Down -> next QKV, "
                               f"tcgen05 stream-K), M={B} (window mean decode batch "
                               f"{win['mean_batch']:.2f}), ctx={chain_ctx}",
                     "algorithmic_bytes_per_launch": chain_bytes, "launch_ms": chain_ms,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, copy burst)"},
        "window": win,
        "replay": {"requests": args.requests * world, "device_ms": replay_ms,
                   "req_per_s": args.requests * world / (replay_ms / 1000.0), "batches": len(batches),
                   "decode_steps": sum(b["decode_steps"] for b in batches),
                   "mean_decode_batch": sum(b["row_steps"] for b in batches) / max(1, sum(b["decode_steps"]
                                                                                        for b in batches))},
        "jct_measured_clock": {"avg_s": agg["avg_jct"], "p99_s": agg["p99_jct"], "req_per_s": m_rps,
                               "runs_avg_s": [r[0]["avg_jct"] for r in mruns],
                               "note": f"median of {len(mruns)} runs"},
        "decode_step": {"batch": B, "ms": step_ms, "hbm_gbs": step_gbs, "frac": step_gbs / hbm},
        "kv_swap": swap,
        "device": {k: device[k] for k in ("batches", "prefill_tokens", "decode_steps", "swap_outs", "swap_ins",
                                          "discards", "recompute_tokens")},
    }
    if not args.no_extras:
        line["roofline_sweep"] = roofline_sweep(dp, cfg, ctx, hbm)
        line["kv_swap"]["under_load"] = swap_under_load(dp, cfg, ctx)
    if clk:
        line["clocks"] = clk
    if rank == 0:
        line["reference_scheduler"] = reference_scheduler(ns, shard, pred, args, cfg.kv_bytes_per_token)
        if world > 1:
            line["cluster"] = cluster_outcome(ns, args, world, pred, cfg.kv_bytes_per_token)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, batches, s, min(args.steps, 3))
        print(json.dumps(line))
    barrier(world)


def cluster_outcome(ns, args, world, pred, bytes_per_token):
    """Whole-cluster avg / p99 JCT and req/s of the global schedule on the
    model clock (every rank executed its replica's batches of exactly this
    schedule), next to round-robin placement."""
    from paper_2512_14142_b200.cluster import ClusterScheduler
    full = []
    rr = argparse.Namespace(**dict(vars(args), placement="round-robin"))
    for r in range(world):
        full += build_workload(rr, r, world)[0]

    def make(i):
        pol, mem, cfg = make_run(ns, None, pred, args, bytes_per_token)
        return pol, pred, mem, cfg

    out = {}
    for rule in (args.placement, "round-robin"):
        agg = ClusterScheduler(ns, full, world, make, placement=rule).run().aggregates()
        out[rule] = {k: agg[k] for k in ("avg_jct", "p99_jct", "req_per_s", "per_replica")}
    return {"placement": args.placement, "clock": "model", **out}


def cpu_baseline(cfg, batches, s, k):
    """The CPU port on a bounded sample: the first k batches of the window."""
    from oracle.cpu_baseline import CpuLlama, batch_sample
    model = CpuLlama(cfg)
    batch_sample(model, batches[s])   # warm-up
    samples = [batch_sample(model, b) for b in batches[s: s + k]]
    win = summarize(batches, s, k)
    value = win["req_equiv"] / sum(x["batch_cpu_s"] for x in samples)
    return {"value": value, "unit": "req/s", "cores": model.threads, "kind": "port",
            "sample": cpu_sample_text(k, samples)}


def chain_kernel_time(dp, cfg, B, ctx, reps=50):
    """One decoder layer's fused launch exactly as LlamaRunner.decode issues
    it: the paged decode attention (B rows x ctx tokens) followed by the
    chained O + residual, gate/up + SiLU, down + residual and next layer's
    QKV + RoPE + KV append, one persistent tcgen05 kernel. Returns (ms per
    launch, algorithmic bytes per launch = the four weight matrices + the
    layer's K/V pages + activations in/out, context actually used)."""
    import torch
    from paper_2512_14142_b200.gpu import lib as L
    from paper_2512_14142_b200.gpu import ops
    w, pool, r = dp.weights, dp.pool, dp.runner
    d, F, qd = cfg.hidden, cfg.ffn, cfg.num_q_heads * cfg.head_dim
    lw, lw1 = w.layers[0], w.layers[1 % cfg.num_layers]
    dev = "cuda"
    nb = (ctx + 16) // 16
    if B * nb > pool.num_blocks:   # the bench's pool is sized for its capacity: shorten the context
        nb = max(1, pool.num_blocks // B)
        ctx = nb * 16 - 1
    x = torch.randn(B, d, device=dev).bfloat16()
    q = (torch.randn(B, qd, device=dev) * 0.5).bfloat16()
    att = torch.empty(B, qd, device=dev).bfloat16()
    h = torch.empty(B, F, device=dev).bfloat16()
    s1 = torch.empty(-(-d // 128), B, device=dev)
    s2 = torch.empty(-(-d // 128), B, device=dev)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    slots = torch.full((B,), -1, dtype=torch.int32, device=dev)   # no KV written: every launch reads the same
    table = torch.arange(B * nb, dtype=torch.int32, device=dev).view(B, nb)
    ctxd = torch.full((B,), ctx + 1, dtype=torch.int32, device=dev)
    cs = ops.rope_table(pos, cfg.head_dim, cfg.rope_theta)
    phases = [dict(a=att, w=lw["wo"], out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s1),
              dict(a=x, w=lw["wgu"], out=h, kind=L.EPI_SILU, ssq_in=s1, rms_dim=d, rms_eps=cfg.eps),
              dict(a=h, w=lw["wdown"], out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s2),
              dict(a=x, w=lw1["wqkv"], out=q, kind=L.EPI_QKV_ROPE, ssq_in=s2, rms_dim=d, rms_eps=cfg.eps,
                   pool=pool.data, geo=pool.geo, layer=1 % cfg.num_layers, num_q_heads=cfg.num_q_heads,
                   positions=pos, slots=slots, rope_theta=cfg.rope_theta, rope_table=cs)]
    attn = (dict(pool=pool.data, geo=pool.geo, layer=0, num_q_heads=cfg.num_q_heads, q=q, q_stride=qd,
                 table=table, ctx=ctxd, scale=r.scale, out=att) if r.fuse_attention and r._attn_fusable() else None)
    ws = r.gemm_ws
    s = torch.cuda.current_stream()
    for _ in range(3):
        ops.gemm_chain(phases, ws, stream=s, attn=attn)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        ops.gemm_chain(phases, ws, stream=s, attn=attn)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    wbytes = sum(ph["w"].numel() * 2 for ph in phases)
    act = 2 * B * (qd + d + d + F + F + d + d + qd)   # A in + C out per phase
    kv = B * (ctx + 1) * cfg.kv_bytes_per_token // cfg.num_layers if attn else 0
    return ms, wbytes + act + kv, ctx


def profiled_traffic(B):
    """DRAM bytes (read + write) per chain launch from the committed ncu
    --set full capture of the same kernel (profiles/), or None."""
    p = ROOT / "profiles" / "r2_ncu_chain_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(str(B), d.get("1"))


def decode_step_gbs(dp, cfg, B, ctx):
    import torch
    from paper_2512_14142_b200.gpu import ops
    nb = (ctx + 16) // 16
    if nb * B > dp.pool.num_blocks:
        B = max(1, dp.pool.num_blocks // nb)
    table = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
    tok = torch.zeros(B, dtype=torch.int32, device="cuda")
    pos = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    slots = table[:, ctx // 16] * 16 + ctx % 16
    ctxd = torch.full((B,), ctx + 1, dtype=torch.int32, device="cuda")
    out = torch.zeros(B, dtype=torch.int64, device="cuda")
    for _ in range(3):
        dp.runner.decode(tok, pos, slots, table, ctxd, keys_out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        dp.runner.decode(tok, pos, slots, table, ctxd, keys_out=out)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    by = cfg.decode_weight_bytes + B * (ctx + 1) * cfg.kv_bytes_per_token
    return by / (ms / 1000.0) / 1e9, ms


def swap_gbs(dp, cfg, tokens):
    import torch
    from paper_2512_14142_b200.gpu import lib as L
    from paper_2512_14142_b200.gpu import ops
    nb = (tokens + 15) // 16
    ids = list(range(nb))
    slot = torch.empty(tokens * dp.pool.bytes_per_token, dtype=torch.uint8, pin_memory=True)
    res = {"tokens": tokens, "bytes": tokens * dp.pool.bytes_per_token}
    for name, mode in (("kernel", L.SWAP_KERNEL), ("dma", L.SWAP_DMA), ("staged", L.SWAP_STAGED)):
        for direction in ("out", "in"):
            fn = ops.swap_out if direction == "out" else ops.swap_in
            fn(dp.pool.geo, dp.pool.data, ids, tokens, slot, mode)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 5
            e0.record()
            for _ in range(n):
                fn(dp.pool.geo, dp.pool.data, ids, tokens, slot, mode)
            e1.record()
            e1.synchronize()
            res[f"{name}_{direction}_gbs"] = res["bytes"] * n / (e0.elapsed_time(e1) / 1000.0) / 1e9
    # host-link reference: one contiguous pinned copy of the same size each way
    dev = torch.empty(res["bytes"], dtype=torch.uint8, device="cuda")
    for direction in ("d2h", "h2d"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            (slot.copy_(dev, non_blocking=True) if direction == "d2h" else dev.copy_(slot, non_blocking=True))
        e1.record()
        e1.synchronize()
        res[f"memcpy_{direction}_gbs"] = res["bytes"] * 5 / (e0.elapsed_time(e1) / 1000.0) / 1e9
    best_out = max(res["kernel_out_gbs"], res["dma_out_gbs"], res["staged_out_gbs"])
    best_in = max(res["kernel_in_gbs"], res["dma_in_gbs"], res["staged_in_gbs"])
    res["frac_out_vs_memcpy"] = best_out / res["memcpy_d2h_gbs"]
    res["frac_in_vs_memcpy"] = best_in / res["memcpy_h2d_gbs"]
    return res


if __name__ == "__main__":
    main()
