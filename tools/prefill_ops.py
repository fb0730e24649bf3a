"""Per-op timing of the Llama-3-8B prefill (recompute-on-resume) at T tokens:
one layer's QKV GEMM (+RoPE +KV append), paged prefill attention, O, gate/up
and down GEMMs (CUDA events over back-to-back repetitions), and the whole
32-layer prefill forward with sampling. Prints one JSON line per T.

    python tools/prefill_ops.py --tokens 128 512 2048 [--ctx-before 0]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, nargs="+", default=[128, 512, 2048])
ap.add_argument("--ctx-before", type=int, default=0, help="resident context before the new tokens")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--seqs", type=int, default=1, help="sequences sharing the T tokens (varlen)")
a = ap.parse_args()

cfg = PRESETS["llama3-8b"]
dev = "cuda"
w = LlamaWeights(cfg, seed=0)
TMAX = max(a.tokens) + a.ctx_before
nb = (TMAX + 15) // 16 + 1
pool = KvPool(cfg, nb * a.seqs + 8)
runner = LlamaRunner(w, pool)
d = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
qd = cfg.num_q_heads * cfg.head_dim
peak_tf = 1640.0


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


for T in a.tokens:
    S = a.seqs
    per = T // S
    c0 = a.ctx_before
    pos, slots, cu, ctxs, last = [], [], [0], [], []
    tables = []
    for s in range(S):
        blocks = list(range(s * nb, (s + 1) * nb))
        tables.append(blocks)
        n = per if s < S - 1 else T - per * (S - 1)
        pos += list(range(c0, c0 + n))
        slots += [blocks[p // 16] * 16 + p % 16 for p in range(c0, c0 + n)]
        cu.append(cu[-1] + n)
        ctxs.append(c0 + n)
        last.append(cu[-1] - 1)
    ids = d([(7 * i) % cfg.vocab for i in range(T)])
    pos_t, slots_t, cu_t, ctx_t = d(pos), d(slots), d(cu), d(ctxs)
    table = d(tables)
    last_t = torch.tensor(last, device=dev)
    x = torch.randn(T, cfg.hidden, device=dev).to(torch.bfloat16)
    q = torch.empty(T, qd, dtype=torch.bfloat16, device=dev)
    att = torch.randn(T, qd, device=dev).to(torch.bfloat16)
    h = torch.randn(T, cfg.ffn, device=dev).to(torch.bfloat16)
    ssq = torch.full((runner.parts, T), cfg.hidden / runner.parts, dtype=torch.float32, device=dev)  # x ~ N(0, 1): sum x^2 = d
    cs = ops.rope_table(pos_t, cfg.head_dim, cfg.rope_theta)
    lw = w.layers[0]
    ws = runner.gemm_ws
    dd, eps = cfg.hidden, cfg.eps
    res = {"tokens": T, "seqs": S, "ctx_before": c0}
    res["qkv_us"] = timed(lambda: ops.gemm_ex(x, lw["wqkv"], q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=dd,
                                              rms_eps=eps, pool=pool.data, geo=pool.geo, layer=0,
                                              num_q_heads=cfg.num_q_heads, positions=pos_t, slots=slots_t,
                                              rope_theta=cfg.rope_theta, rope_table=cs, workspace=ws), a.reps)
    res["attn_us"] = timed(lambda: ops.prefill_attention(pool.geo, pool.data, 0, q, qd, cu_t, S, max(cu[i + 1] - cu[i] for i in range(S)),
                                                         cfg.num_q_heads, table, ctx_t, runner.scale, att), a.reps)
    res["o_us"] = timed(lambda: ops.gemm_ex(att, lw["wo"], x, kind=L.EPI_RESIDUAL, residual=x, workspace=ws), a.reps)
    res["gu_us"] = timed(lambda: ops.gemm_ex(x, lw["wgu"], h, kind=L.EPI_SILU, ssq_in=ssq, rms_dim=dd, rms_eps=eps,
                                             workspace=ws), a.reps)
    res["down_us"] = timed(lambda: ops.gemm_ex(h, lw["wdown"], x, kind=L.EPI_RESIDUAL, residual=x, workspace=ws),
                           a.reps)
    res["layer_sum_us"] = res["qkv_us"] + res["attn_us"] + res["o_us"] + res["gu_us"] + res["down_us"]
    fl_lin = 2.0 * T * cfg.linear_params_per_token / cfg.num_layers
    fl_att = sum(4.0 * (ctxs[s] - (cu[s + 1] - cu[s])) * (cu[s + 1] - cu[s]) * cfg.head_dim * cfg.num_q_heads
                 + 2.0 * (cu[s + 1] - cu[s]) * (cu[s + 1] - cu[s] + 1) * cfg.head_dim * cfg.num_q_heads
                 for s in range(S))
    res["attn_tflops"] = fl_att / (res["attn_us"] * 1e-6) / 1e12
    gemm_us = res["layer_sum_us"] - res["attn_us"]
    res["gemm_tflops"] = fl_lin / (gemm_us * 1e-6) / 1e12
    wbytes = 2 * (cfg.qkv_dim * dd + dd * qd + 3 * cfg.ffn * dd)
    res["gemm_hbm_floor_us"] = wbytes / 6.5e12 * 1e6
    res["gemm_tensor_floor_us"] = fl_lin / (peak_tf * 1e12) * 1e6
    res["forward_ms"] = timed(lambda: runner.prefill(ids, pos_t, slots_t, cu_t, table, ctx_t, last_t,
                                                     max(cu[i + 1] - cu[i] for i in range(S))), max(3, a.reps // 4)) / 1e3
    print(json.dumps(res), flush=True)
