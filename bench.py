"""Benchmark: Astraea's scheduler driving the B200 data path (BASELINE.json C2).

Workload (``config.workload``): Llama-3-8B shape (random init, bf16), a
synthetic agent trace from the reference generator (seed 0, default segment
and category mix), Stateful-MLFQ + adaptive Preserve/Swap/Discard KV policy,
parallel-max batches, model clock (so every decision equals the
reference's). One *step* = one full replay of the rank's trace shard: every
scheduled batch's prefill / recompute-prefill and decode loop plus every
swap-out/in the KV policy orders, executed on the GPU.

  value      requests/s over the device-timed replay (CUDA events on the
             data path's streams), prompt ids pre-staged in HBM;
  e2e        requests/s through the public API (GpuEngine.run) timed on the
             host clock, prompt ids uploaded from pinned host memory per batch
             and generated tokens read back per batch (bytes reported);
  roofline   the dominant kernel (one decoder layer's fused launch: paged
             attention + the chained tcgen05 GEMMs, weight + KV stream)
             against measured HBM bandwidth;
  cpu_baseline  the CPU port (oracle/cpu_baseline.py) on a bounded sample.

Multi-GPU: one process per GPU (torchrun), the trace is partitioned
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--requests", type=int, default=12, help="requests per rank")
    ap.add_argument("--qps", type=float, default=4.0, help="arrival rate per rank")
    ap.add_argument("--capacity", type=int, default=3000,
                    help="KV capacity (tokens) per GPU; 3000 puts the 12-request shard under memory pressure "
                         "(preserve, swap and forced discard all occur)")
    ap.add_argument("--swap-mode", choices=("kernel", "dma"), default="kernel")
    ap.add_argument("--cost-tables", choices=("calibrated", "b200-like"), default="calibrated",
                    help="scheduler cost tables: measured on the B200 by tools/calibrate.py "
                         "(profiles/r1_b200_cost_tables.json), or the survey's B200-like guess")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def build_workload(args, rank, world):
    from paper_2512_14142_b200 import host
    import scenarios
    need = args.requests * world
    duration = 2.0 * need / (args.qps * world) + 60.0
    while True:  # the first n arrivals do not depend on the horizon once it covers them
        full = host.generate(host.WorkloadConfig(seed=0, qps=args.qps * world, duration=duration))
        if len(full) >= need:
            break
        duration *= 2
    full = full[:need]
    full.sort(key=lambda r: (r.arrival_time, r.id))
    shard = full[rank::world]
    if getattr(args, "cost_tables", "calibrated") == "calibrated":
        pred, cal = scenarios.calibrated_predictor(host)
        args.swap_tokens_per_s = float(cal["swap_bandwidth_tokens_per_s"])
    else:
        pred = scenarios.b200_like_predictor(host)
        args.swap_tokens_per_s = 380_000.0
    return shard, pred


def make_run(host, shard, pred, args, bytes_per_token):
    policy = host.make_policy("stateful-mlfq", pred, host.MlfqConfig())
    memory = host.MemoryModel(capacity_tokens=args.capacity, bytes_per_token=float(bytes_per_token),
                              swap_bandwidth_tokens_per_s=getattr(args, "swap_tokens_per_s", 380_000.0))
    config = host.SimConfig(cost_model="parallel-max", cache_mode="adaptive")
    return policy, memory, config


def work_profile(host, shard, pred, args, bytes_per_token):
    """Exact prefill tokens / decode steps the schedule implies (host only)."""

    class Probe(host.Engine):
        def _launch_batch(self, members):
            n = [m.state.current_seg.n_gen for m in members]
            self.w["decode_steps"] += max(n)
            self.w["row_steps"] += sum(n)
            self.w["batches"] += 1
            for m in members:
                seg = m.state.current_seg
                extra = m.state.context_before_current if m.prior_location is host.CacheLocation.DROPPED else 0
                self.w["prefill_tokens"] += seg.n_in + extra
                self.w["ctx_sum"] += m.state.context_after(m.segment_index) * seg.n_gen
            return None

    pol, mem, cfg = make_run(host, shard, pred, args, bytes_per_token)
    e = Probe(shard, pol, pred, mem, cfg)
    e.w = dict(decode_steps=0, row_steps=0, batches=0, prefill_tokens=0, ctx_sum=0)
    rep = e.run()
    w = e.w
    w["mean_batch"] = w["row_steps"] / max(1, w["decode_steps"])
    w["mean_ctx"] = w["ctx_sum"] / max(1, w["row_steps"])
    return w, rep


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


# --------------------------------------------------------------------------- reference arm

def run_reference(args):
    """CPU port of the path on the host cores (oracle/cpu_baseline.py)."""
    rank, world, _ = dist_setup(args)
    if rank != 0:
        barrier(world)
        return
    from oracle.cpu_baseline import CpuLayerSample, estimate_replay_seconds
    from paper_2512_14142_b200 import host
    from paper_2512_14142_b200.gpu.model import PRESETS
    cfg = PRESETS[args.model]
    shard, pred = build_workload(args, 0, world)
    work, rep = work_profile(host, shard, pred, args, cfg.kv_bytes_per_token)
    sample = CpuLayerSample(cfg)
    times = []
    est = None
    for i in range(args.warmup + args.steps):
        est = estimate_replay_seconds(sample, work, budget_s=8.0)
        if i >= args.warmup:
            times.append(est["replay_seconds"])
    t = statistics.mean(times)
    value = len(shard) / t
    line = {
        "metric": METRIC, "value": value, "unit": "req/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1000.0, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"C2 {args.model} random-init, trace seed 0 {len(shard)} req @ qps {args.qps}, "
                               f"stateful-mlfq adaptive KV, capacity {args.capacity} tok",
                   "kind": "CPU port (oracle/cpu_baseline.py): 1 layer x num_layers + lm_head, extrapolated"},
        "cpu_baseline": {"value": value, "unit": "req/s", "cores": est["threads"], "kind": "port",
                         "sample": f"prefill {est['prefill_chunk_tokens']} tok + decode steps at batch "
                                   f"{est['decode_step_batch']}, 1 layer applied x{cfg.num_layers}; "
                                   f"extrapolated to {work['prefill_tokens']} prefill tok + "
                                   f"{work['decode_steps']} decode steps"},
        "e2e": {"value": value, "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    barrier(world)


# --------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    rank, world, local = dist_setup(args)
    torch.cuda.set_device(local)
    from paper_2512_14142_b200 import host
    from paper_2512_14142_b200.gpu import lib as L
    from paper_2512_14142_b200.gpu import ops
    from paper_2512_14142_b200.gpu.datapath import KvDataPath
    from paper_2512_14142_b200.gpu.engine import GpuEngine
    from paper_2512_14142_b200.gpu.model import PRESETS

    cfg = PRESETS[args.model]
    shard, pred = build_workload(args, rank, world)
    work, ref_rep = work_profile(host, shard, pred, args, cfg.kv_bytes_per_token)
    blocks = math.ceil(args.capacity / 16) + 2 * len(shard) + 64
    dp = KvDataPath(cfg, num_blocks=blocks, swap_mode=L.SWAP_KERNEL if args.swap_mode == "kernel" else L.SWAP_DMA)

    def replay():
        pol, mem, scfg = make_run(host, shard, pred, args, cfg.kv_bytes_per_token)
        return GpuEngine(shard, pol, pred, mem, scfg, dp, clock="model").run()

    # ---- value: inputs resident in HBM, device-timed
    dp.prestage(shard)
    for _ in range(args.warmup):
        rep = replay()
    assert rep.to_json() == ref_rep.to_json(), "GPU engine diverged from the host schedule"
    clocks = ClockSampler(not args.no_clocks and rank == 0, local)
    spans = []
    launches0 = ops.LAUNCHES[0]
    barrier(world)
    torch.cuda.synchronize()
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(dp.compute)
        replay()
        dp.compute.wait_stream(dp.swapper)
        e1.record(dp.compute)
        e1.synchronize()
        spans.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier(world)
    launches = (ops.LAUNCHES[0] - launches0) // args.steps
    clk = clocks.stop()
    ms = max_over_ranks(statistics.mean(spans), world)
    value = len(shard) * world / (ms / 1000.0)

    # ---- e2e: public API, host buffers, wall clock
    dp.staged = {}
    s0 = dict(dp.stats)
    barrier(world)
    torch.cuda.synchronize()
    walls = []
    reports = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = replay()
        for ev, host_buf in dp.results:
            ev.synchronize()       # generated tokens are on the host
        dp.results.clear()
        walls.append(time.perf_counter() - t0)
        reports.append(r)
    barrier(world)
    e2e_s = max_over_ranks(statistics.mean(walls), world)
    e2e = len(shard) * world / e2e_s
    h2d = (dp.stats["h2d_bytes"] - s0["h2d_bytes"]) // args.steps
    d2h = (dp.stats["d2h_bytes"] - s0["d2h_bytes"]) // args.steps

    # ---- measured-clock JCT (same scheduler, B200 durations, virtual API waits)
    # three runs, median by avg JCT: the measured-clock schedule reacts to
    # run-to-run timing noise (an arrival before or after a batch boundary
    # changes later decisions), so one run can sit +-30% from another
    mruns = []
    for _ in range(3):
        pol, mem, scfg = make_run(host, shard, pred, args, cfg.kv_bytes_per_token)
        r_ = GpuEngine(shard, pol, pred, mem, scfg, dp, clock="measured").run()
        mruns.append((r_.aggregates(), r_.requests_per_second()))
    mruns.sort(key=lambda x: x[0]["avg_jct"])
    agg, m_rps = mruns[1]

    # ---- dominant kernel: one decoder layer's fused launch (paged attention ->
    # O -> gate/up -> down -> next QKV in one persistent tcgen05 kernel) at the
    # replay's mean batch and context, timed with CUDA events on its stream;
    # algorithmic bytes = the four weight matrices + the layer's K/V pages +
    # activations in/out per launch
    hbm, peak_kind = peaks()
    B = max(1, int(round(work["mean_batch"])))
    chain_ms, chain_bytes, chain_ctx = chain_kernel_time(dp, cfg, B, int(work["mean_ctx"]))
    gemm_gbs = chain_bytes / (chain_ms / 1000.0) / 1e9
    traffic = profiled_traffic(B)

    # ---- decode step (weights + KV) and swap bandwidth
    step_gbs, step_ms = decode_step_gbs(dp, cfg, B, int(work["mean_ctx"]))
    swap = swap_gbs(dp, cfg, int(work["mean_ctx"]))

    line = {
        "metric": METRIC, "value": value, "unit": "req/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, generated trace)",
        "config": {"workload": f"C2 {args.model} random-init, trace seed 0, {len(shard)} req/rank @ qps "
                               f"{args.qps}/rank, stateful-mlfq + adaptive KV, capacity {args.capacity} "
                               f"tok/GPU, parallel-max, model clock, {args.cost_tables} cost tables",
                   "global_requests": len(shard) * world, "parallelism": f"replicas x{world}",
                   "l2": "weights (15 GB) stream every decode step: inputs >> L2",
                   "decode_steps_per_step": work["decode_steps"], "prefill_tokens_per_step": work["prefill_tokens"],
                   "swap_mode": args.swap_mode},
        "e2e": {"value": e2e, "unit": "req/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": gemm_gbs, "peak": hbm, "unit": "GB/s", "frac": gemm_gbs / hbm,
                     "traffic": traffic,
                     "kernel": f"gemm_chain_kernel (layer: paged attention -> O -> GU -> Down -> next QKV, "
                               f"tcgen05 stream-K), M={B}, ctx={chain_ctx}",
                     "algorithmic_bytes_per_launch": chain_bytes, "launch_ms": chain_ms,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, copy burst)"},
        "jct_measured_clock": {"avg_s": agg["avg_jct"], "p99_s": agg["p99_jct"], "req_per_s": m_rps,
                               "runs_avg_s": [r[0]["avg_jct"] for r in mruns], "note": "median of 3 runs"},
        "decode_step": {"batch": B, "ms": step_ms, "hbm_gbs": step_gbs, "frac": step_gbs / hbm},
        "kv_swap": swap,
        "kv_decisions": {k: v for k, v in json.loads(ref_rep.to_json())["audits"].items() if k == "events_processed"},
        "device": {k: reports[-1].device[k] for k in ("batches", "prefill_tokens", "decode_steps", "swap_outs",
                                                       "swap_ins", "discards", "recompute_tokens")},
    }
    if clk:
        line["clocks"] = clk
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, work, len(shard))
    if rank == 0:
        print(json.dumps(line))
    barrier(world)


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
    p = ROOT / "profiles" / "r1_ncu_chain_traffic.json"
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
    for name, mode in (("kernel", L.SWAP_KERNEL), ("dma", L.SWAP_DMA)):
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
    best_out = max(res["kernel_out_gbs"], res["dma_out_gbs"])
    best_in = max(res["kernel_in_gbs"], res["dma_in_gbs"])
    res["frac_out_vs_memcpy"] = best_out / res["memcpy_d2h_gbs"]
    res["frac_in_vs_memcpy"] = best_in / res["memcpy_h2d_gbs"]
    return res


def cpu_baseline(cfg, work, n_req):
    from oracle.cpu_baseline import CpuLayerSample, estimate_replay_seconds
    est = estimate_replay_seconds(CpuLayerSample(cfg), work, budget_s=10.0)
    return {"value": n_req / est["replay_seconds"], "unit": "req/s", "cores": est["threads"], "kind": "port",
            "sample": f"prefill {est['prefill_chunk_tokens']} tok + decode at batch {est['decode_step_batch']}, "
                      f"1 layer x{cfg.num_layers} + lm_head, extrapolated to the replay"}


if __name__ == "__main__":
    main()
