"""Host launch cost vs device time of the short-prefill ops (Llama-3-8B
shapes): for each op, CUDA-event time of back-to-back calls (what
tools/prefill_ops.py reports), the host time per call (perf_counter, no
sync), and the device time of the same call replayed from a CUDA graph
(no host in the loop). Then the whole prefill forward: host time per
forward vs device time.

    python tools/prefill_host.py --tokens 128 512
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, nargs="+", default=[128, 512])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
cfg = PRESETS["llama3-8b"]
dev = "cuda"
w = LlamaWeights(cfg, seed=0)
nb = (max(a.tokens) + 15) // 16 + 1
pool = KvPool(cfg, nb + 8)
runner = LlamaRunner(w, pool)
qd = cfg.num_q_heads * cfg.head_dim


def ev_time(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def host_time(fn, reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / reps * 1e6


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for T in a.tokens:
    d = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
    pos_t = d(list(range(T)))
    slots_t = d(list(range(T)))
    table = d([list(range(nb))])
    x = torch.randn(T, cfg.hidden, device=dev).to(torch.bfloat16)
    q = torch.empty(T, qd, dtype=torch.bfloat16, device=dev)
    att = torch.randn(T, qd, device=dev).to(torch.bfloat16)
    h = torch.randn(T, cfg.ffn, device=dev).to(torch.bfloat16)
    ssq = torch.full((runner.parts, T), cfg.hidden / runner.parts, dtype=torch.float32, device=dev)  # x ~ N(0, 1): sum x^2 = d
    cs = ops.rope_table(pos_t, cfg.head_dim, cfg.rope_theta)
    ws = runner.gemm_ws
    res = {"tokens": T}
    for li_name, mk in (
        ("qkv", lambda lw: lambda: ops.gemm_ex(x, lw["wqkv"], q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=cfg.hidden,
                                               rms_eps=cfg.eps, pool=pool.data, geo=pool.geo, layer=0,
                                               num_q_heads=cfg.num_q_heads, positions=pos_t, slots=slots_t,
                                               rope_theta=cfg.rope_theta, rope_table=cs, workspace=ws)),
        ("o", lambda lw: lambda: ops.gemm_ex(att, lw["wo"], x, kind=L.EPI_RESIDUAL, residual=x, workspace=ws)),
        ("gu", lambda lw: lambda: ops.gemm_ex(x, lw["wgu"], h, kind=L.EPI_SILU, ssq_in=ssq, rms_dim=cfg.hidden,
                                              rms_eps=cfg.eps, workspace=ws)),
        ("down", lambda lw: lambda: ops.gemm_ex(h, lw["wdown"], x, kind=L.EPI_RESIDUAL, residual=x, workspace=ws)),
    ):
        fn = mk(w.layers[0])
        layers = [mk(lw) for lw in w.layers]   # rotate layers: weights not L2-resident
        k = [0]

        def rot():
            k[0] = (k[0] + 1) % len(layers)
            layers[k[0]]()

        res[li_name] = {"events_us": round(ev_time(fn, a.reps), 1), "host_us": round(host_time(fn, a.reps), 1),
                        "graph_us": round(graph_time(fn, a.reps), 1), "graph_rot_us": round(graph_time(rot, 32), 1)}
    ids = d([(7 * i) % cfg.vocab for i in range(T)])
    cu_t, ctx_t, last_t = d([0, T]), d([T]), torch.tensor([T - 1], device=dev)
    fwd = lambda: runner.prefill(ids, pos_t, slots_t, cu_t, table, ctx_t, last_t, T)  # noqa: E731
    res["forward"] = {"events_ms": round(ev_time(fwd, 5) / 1e3, 3), "host_ms": round(host_time(fwd, 5) / 1e3, 3)}
    try:
        res["forward"]["graph_ms"] = round(graph_time(fwd, 1) / 1e3, 3)
    except Exception as ex:   # noqa: BLE001
        res["forward"]["graph_ms"] = repr(ex)[:120]
    print(json.dumps(res), flush=True)
