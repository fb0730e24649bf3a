"""Weight-streaming efficiency of the step kernel's GEMM machinery alone:
one layer's O -> gate/up -> down -> QKV as (a) a 4-phase step program and
(b) the per-layer chain kernel, M = batch rows; GB/s of weight bytes."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu import ops
from paper_2512_14142_b200.gpu.datapath import KvPool
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaRunner, LlamaWeights

cfg = PRESETS["llama3-8b"]
w = LlamaWeights(cfg)
pool = KvPool(cfg, 64)
r = LlamaRunner(w, pool)
d, F, qd = cfg.hidden, cfg.ffn, cfg.num_q_heads * cfg.head_dim
lw, lw1 = w.layers[0], w.layers[1]
wbytes = sum(t.numel() * 2 for t in (lw["wo"], lw["wgu"], lw["wdown"], lw1["wqkv"]))
for B in [int(x) for x in (sys.argv[1:] or ["1", "16"])]:
    x = torch.randn(B, d, device="cuda").bfloat16()
    att = torch.randn(B, qd, device="cuda").bfloat16()
    h = torch.empty(B, F, device="cuda").bfloat16()
    q = torch.empty(B, qd, device="cuda").bfloat16()
    s1 = torch.empty(d // 128, B, device="cuda")
    s2 = torch.empty(d // 128, B, device="cuda")
    pos = torch.full((B,), 100, dtype=torch.int32, device="cuda")
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    cs = ops.rope_table(pos, cfg.head_dim, cfg.rope_theta)
    ph = [dict(a=att, w=lw["wo"], out=x, epi=L.EPI_RESIDUAL, residual=x, ssq_out=s1),
          dict(a=x, w=lw["wgu"], out=h, epi=L.EPI_SILU, ssq_in=s1, rms_dim=d, rms_eps=cfg.eps),
          dict(a=h, w=lw["wdown"], out=x, epi=L.EPI_RESIDUAL, residual=x, ssq_out=s2),
          dict(a=x, w=lw1["wqkv"], out=q, epi=L.EPI_QKV_ROPE, ssq_in=s2, rms_dim=d, rms_eps=cfg.eps,
               pool=pool.data, geo=pool.geo, layer=1, num_q_heads=cfg.num_q_heads, positions=pos, slots=slots,
               rope_theta=cfg.rope_theta, rope_table=cs)]
    step = [dict(kind="gemm", **ph[0], a_from=-1, epi_from=-1), dict(kind="gemm", **ph[1], a_from=0, epi_from=0),
            dict(kind="gemm", **ph[2], a_from=1, epi_from=0), dict(kind="gemm", **ph[3], a_from=2, epi_from=2)]
    prog = ops.StepProgram(B, step, ops.StepWorkspace())
    chain = [{("kind" if k == "epi" else k): v for k, v in p.items()} for p in ph]

    def t(fn, n=30):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / n * 1000

    if B == 1:
        G = torch.cuda.get_device_properties(0).multi_processor_count
        buf = torch.zeros(G * 4 * 8 + G, dtype=torch.int64, device="cuda")
        L.load().astraea_debug_step_trace(buf.data_ptr())
        prog.launch()
        torch.cuda.synchronize()
        L.load().astraea_debug_step_trace(None)
        tt = buf.cpu().double()
        base = tt[G * 32:].min()
        st = tt[: G * 32].view(G, 4, 8)
        for p_ in range(4):
            row = {}
            for k, nm in enumerate(["w_start", "x_start", "epi_done", "mma_done", "epi_begin", "parts_seen",
                                    "last_acc", "last_finish"]):
                c = st[:, p_, k]
                c = c[c > 0]
                row[nm] = [round(float(c.median() - base) / 1000, 1), round(float(c.max() - base) / 1000, 1)] \
                    if c.numel() else None
            print(json.dumps({"phase": ["o", "gu", "down", "qkv"][p_], **row}))
            if p_ in (0, 2):
                ep = st[:, p_, 2]
                order = ep.argsort(descending=True)[:8]
                print(json.dumps({"slowest_ctas (cta, k=0..7)": [[int(c)] + [round(float(st[c, p_, k] - base) / 1000, 1)
                                                    if st[c, p_, k] > 0 else None for k in range(8)] for c in order]}))
    for name, fn in [("step_program", lambda: prog.launch()), ("step_program_l2_16", lambda: prog.launch(l2_ahead=16)),
                     ("chain", lambda: ops.gemm_chain(chain, r.gemm_ws))]:
        us = t(fn)
        print(json.dumps({"B": B, "variant": name, "lib": L.LIB_PATH.parent.name, "us": round(us, 1),
                          "weight_gbs": round(wbytes / us / 1e3, 1)}), flush=True)
