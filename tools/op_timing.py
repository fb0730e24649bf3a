"""In-application per-op timing of one Llama decode layer (CUDA events,
back-to-back repetitions so PDL overlap is representative), plus the full
decode step. ncu serialises kernels and cannot show PDL overlap; this can.

    python tools/op_timing.py --batch 3 --ctx 900
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


GRAPH = True


def timed(fn, reps=50):
    """Microseconds per call: reps back-to-back calls captured in one CUDA
    graph (pure device time, PDL edges kept); eager if capture fails."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GRAPH:
        try:
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for _ in range(reps):
                        fn()
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            return e0.elapsed_time(e1) * 1000.0 / reps
        except Exception as exc:  # noqa: BLE001
            print("graph capture failed:", exc, file=sys.stderr)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / reps   # microseconds


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--batch", type=int, default=3)
    ap.add_argument("--ctx", type=int, default=900)
    a = ap.parse_args()
    cfg = PRESETS[a.model]
    B, ctx = a.batch, a.ctx
    nb = (ctx + 16) // 16
    w = LlamaWeights(cfg)
    pool = KvPool(cfg, B * nb + 4)
    r = LlamaRunner(w, pool)
    dev = "cuda"
    d, F, qd = cfg.hidden, cfg.ffn, cfg.num_q_heads * cfg.head_dim
    lw = w.layers[0]
    ws = r.gemm_ws
    x = torch.randn(B, d, device=dev).bfloat16()
    q = torch.empty(B, qd, device=dev, dtype=torch.bfloat16)
    att = torch.randn(B, qd, device=dev).bfloat16()
    h = torch.randn(B, F, device=dev).bfloat16()
    ssq = (x.float().pow(2).view(B, -1, 128).sum(-1)).T.contiguous()
    ssq2 = torch.empty_like(ssq)
    table = torch.arange(B * nb, dtype=torch.int32, device=dev).view(B, nb)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    slots = table[:, ctx // 16] * 16 + ctx % 16
    ctxd = torch.full((B,), ctx + 1, dtype=torch.int32, device=dev)
    dws = r._dec_ws(B, nb)
    cs = ops.rope_table(pos, cfg.head_dim, cfg.rope_theta)
    res = {}
    res["qkv_rope_gemm"] = timed(lambda: ops.gemm_ex(x, lw["wqkv"], q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=d,
                                                     rms_eps=cfg.eps, pool=pool.data, geo=pool.geo, layer=0,
                                                     num_q_heads=cfg.num_q_heads, positions=pos, slots=slots,
                                                     rope_theta=cfg.rope_theta, rope_table=cs, workspace=ws))
    res["qkv_plain_gemm"] = timed(lambda: ops.gemm(x, lw["wqkv"], workspace=ws))
    res["attention"] = timed(lambda: ops.decode_attention(pool.geo, pool.data, 0, q, qd, B, cfg.num_q_heads, table,
                                                          ctxd, r.scale, att, dws))
    res["o_resid_gemm"] = timed(lambda: ops.gemm_ex(att, lw["wo"], x, kind=L.EPI_RESIDUAL, residual=x,
                                                    ssq_out=ssq2, workspace=ws))
    res["o_plain_gemm"] = timed(lambda: ops.gemm(att, lw["wo"], workspace=ws))
    res["gu_silu_gemm"] = timed(lambda: ops.gemm_ex(x, lw["wgu"], h, kind=L.EPI_SILU, ssq_in=ssq, rms_dim=d,
                                                    rms_eps=cfg.eps, workspace=ws))
    res["gu_plain_gemm"] = timed(lambda: ops.gemm(x, lw["wgu"], workspace=ws))
    res["down_resid_gemm"] = timed(lambda: ops.gemm_ex(h, lw["wdown"], x, kind=L.EPI_RESIDUAL, residual=x,
                                                       ssq_out=ssq2, workspace=ws))
    res["down_plain_gemm"] = timed(lambda: ops.gemm(h, lw["wdown"], workspace=ws))
    res["lm_head_gemm"] = timed(lambda: ops.gemm(x, w.lm_head, workspace=ws), reps=20)
    def layer_seq():
        ops.gemm_ex(x, lw["wqkv"], q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=d, rms_eps=cfg.eps, pool=pool.data,
                    geo=pool.geo, layer=0, num_q_heads=cfg.num_q_heads, positions=pos, slots=slots,
                    rope_theta=cfg.rope_theta, rope_table=cs, workspace=ws)
        ops.decode_attention(pool.geo, pool.data, 0, q, qd, B, cfg.num_q_heads, table, ctxd, r.scale, att, dws)
        ops.gemm_ex(att, lw["wo"], x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq2, workspace=ws)
        ops.gemm_ex(x, lw["wgu"], h, kind=L.EPI_SILU, ssq_in=ssq2, rms_dim=d, rms_eps=cfg.eps, workspace=ws)
        ops.gemm_ex(h, lw["wdown"], x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq, workspace=ws)

    res["layer_seq"] = timed(layer_seq, reps=32)
    tokv = torch.zeros(B, dtype=torch.int32, device=dev)
    res["embedding"] = timed(lambda: ops.embedding(tokv, w.embed, ssq_out=torch.empty(1, B, device=dev)))
    res["rope_table"] = timed(lambda: ops.rope_table(pos, cfg.head_dim, cfg.rope_theta))
    lg = torch.randn(B, cfg.vocab, device=dev).bfloat16()
    res["argmax"] = timed(lambda: ops.argmax(lg))
    tok = torch.zeros(B, dtype=torch.int32, device=dev)
    out = torch.zeros(B, dtype=torch.int64, device=dev)
    res["decode_step"] = timed(lambda: r.decode(tok, pos, slots, table, ctxd, keys_out=out), reps=10)
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        r.decode(tok, pos, slots, table, ctxd, keys_out=out)
    t_host = (time.perf_counter() - t0) / 10 * 1e6
    torch.cuda.synchronize()
    res["decode_step_host_issue"] = t_host
    layer = res["qkv_rope_gemm"] + res["attention"] + res["o_resid_gemm"] + res["gu_silu_gemm"] + res["down_resid_gemm"]
    res["layer_sum"] = layer
    res["step_estimate"] = layer * cfg.num_layers + res["lm_head_gemm"]
    by = {"qkv": lw["wqkv"].numel() * 2, "o": lw["wo"].numel() * 2, "gu": lw["wgu"].numel() * 2,
          "down": lw["wdown"].numel() * 2, "lm": w.lm_head.numel() * 2}
    gbs = {k: by[k.split("_")[0]] / (v * 1e-6) / 1e9 for k, v in res.items()
           if k.split("_")[0] in by and k.endswith("gemm")}
    print(json.dumps({"us": {k: round(v, 2) for k, v in res.items()},
                      "weight_GBps": {k: round(v) for k, v in gbs.items()},
                      "weight_bytes_per_step": cfg.weight_bytes}, indent=1))


if __name__ == "__main__":
    main()
