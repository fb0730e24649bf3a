"""Calibrate the scheduler's cost model on the B200 (the
paper's "offline profiling of the target hardware").

The reference's engine advances its clock with ServiceTimePredictor tables
(predictor.py:47-66: a piecewise-linear prefill profile, seconds per decoded
token) and MemoryModel.swap_bandwidth_tokens_per_s (kvcache.py:136-137).
This module measures those quantities on the device with the data path's
own kernels and emits them in the reference's formats
(ServiceTimePredictor.to_config(), predictor.py:169-176), so the unmodified
scheduler can make its decisions with B200-true costs:
  prefill_profile            [[n, seconds]] for a single n-token prefill
  decode_seconds_per_token   one decode step at batch 1 (the DecodeModel is
                             batch-independent; steps at larger batches are
                             reported alongside for reference)
  swap_bandwidth_tokens_per_s  K1 gather + K2 scatter round trip / 2
Every duration is a CUDA-event measurement (median of `reps`).
"""

from __future__ import annotations

import statistics

import torch

from . import lib as L
from . import ops


def _time(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1) / 1000.0)
    return statistics.median(out)


def monotone_profile(points):
    """The reference's PrefillProfile requires non-decreasing latencies
    (predictor.py:47-57): launch-bound small points can measure out of order
    within noise, so keep the running maximum."""
    out = [[int(n), float(t)] for n, t in points]
    for i in range(1, len(out)):
        out[i][1] = max(out[i][1], out[i - 1][1])
    return out


def calibrate(dp, prefill_points=(128, 256, 512, 1024, 2048), decode_batches=(1, 2, 4, 8, 16), decode_ctx=512,
              swap_tokens=1024, reps=3) -> dict:
    cfg, runner, pool = dp.cfg, dp.runner, dp.pool
    dev = "cuda"

    def d(v):
        return torch.tensor(v, dtype=torch.int32, device=dev)

    need = max(max(prefill_points), max(decode_batches) * (decode_ctx + 16), swap_tokens) // 16 + 8
    if pool.num_blocks < need:
        raise ValueError(f"calibration needs a pool of >= {need} blocks")
    prefill = []
    for n in prefill_points:
        blocks = list(range((n + 15) // 16))
        ids = d([(7 * i + 1) % cfg.vocab for i in range(n)])
        pos = d(list(range(n)))
        slots = d([blocks[p // 16] * 16 + p % 16 for p in range(n)])
        table = d([blocks]).view(1, -1)
        args = (ids, pos, slots, d([0, n]), table, d([n]), torch.tensor([n - 1], device=dev), n)
        prefill.append([n, _time(lambda: runner.prefill(*args), max(reps, 5), warm=2)])
    prefill = monotone_profile(prefill)
    decode = {}
    nb = (decode_ctx + 16) // 16
    # two passes over the batch sizes, the faster kept: the first decode timed
    # right after the prefill points runs while clocks recover from the
    # tensor-heavy prefills (batch 1 read 3.40 ms in one pass, 3.15 in the next)
    for B in list(decode_batches) * 2:
        table = torch.arange(B * nb, dtype=torch.int32, device=dev).view(B, nb)
        tok = torch.zeros(B, dtype=torch.int32, device=dev)
        pos = torch.full((B,), decode_ctx, dtype=torch.int32, device=dev)
        slots = table[:, decode_ctx // 16] * 16 + decode_ctx % 16
        ctx = torch.full((B,), decode_ctx + 1, dtype=torch.int32, device=dev)
        keys = torch.zeros(B, dtype=torch.int64, device=dev)
        # the data path replays decode steps from CUDA graphs: time a graph
        # replay (an eager call also times the host launching ~35 kernels)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                runner.decode(tok, pos, slots, table, ctx, stream=side, keys_out=keys)
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            runner.decode(tok, pos, slots, table, ctx, stream=side, keys_out=keys)
        t = _time(graph.replay, max(reps, 10), warm=3)
        decode[B] = min(t, decode.get(B, t))
        del graph
    ids = list(range((swap_tokens + 15) // 16))
    slot = torch.empty(swap_tokens * pool.bytes_per_token, dtype=torch.uint8, pin_memory=True)
    t_out = _time(lambda: ops.swap_out(pool.geo, pool.data, ids, swap_tokens, slot, dp.swap_mode), reps)
    t_in = _time(lambda: ops.swap_in(pool.geo, pool.data, ids, swap_tokens, slot, dp.swap_mode), reps)
    return {
        "model": cfg.name,
        "predictor": {"prefill_profile": prefill, "decode_seconds_per_token": decode[min(decode)],
                      "api_latency_means": None},
        "swap_bandwidth_tokens_per_s": 2 * swap_tokens / (t_out + t_in),
        "bytes_per_token": pool.bytes_per_token,
        "decode_step_seconds_by_batch": {str(k): v for k, v in decode.items()},
        "decode_ctx": decode_ctx,
        "swap": {"tokens": swap_tokens, "out_s": t_out, "in_s": t_in,
                 "mode": {L.SWAP_KERNEL: "kernel", L.SWAP_DMA: "dma", L.SWAP_STAGED: "staged"}[dp.swap_mode]},
    }


def predictor_from_calibration(ns, cal: dict):
    """A reference ServiceTimePredictor with the measured tables (API means keep the
    reference defaults: API latency is the environment's, not the GPU's)."""
    cfg = dict(cal["predictor"])
    cfg["api_latency_means"] = ns.ServiceTimePredictor().to_config()["api_latency_means"]
    return ns.ServiceTimePredictor.from_config(cfg)
