"""Prefill-GEMM throughput (tcgen05) at Llama-3-8B projection shapes:
TFLOP/s per (M, N, K) with CUDA events around a CUDA graph of 20 launches. ASTRAEA_GEMM_PAIR=0 selects the
one-CTA kernel instead of the CTA-pair kernel."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2512_14142_b200.gpu import lib as L, ops

shapes = [(6144, 4096, "qkv"), (4096, 4096, "o"), (28672, 4096, "gate_up"), (4096, 14336, "down")]
Ms = [int(x) for x in (sys.argv[1:] or ["256", "1024", "2048", "4096"])]
for M in Ms:
    for N, K, name in shapes:
        a = torch.randn(M, K, device="cuda").bfloat16()
        w = torch.randn(N, K, device="cuda").bfloat16() * 0.02
        out = torch.empty(M, N, device="cuda").bfloat16()
        need = L.require_cuda().astraea_gemm_workspace_bytes(M, N, K)
        ws = torch.zeros(need // 4 + 1, dtype=torch.float32, device="cuda") if need else None
        for _ in range(3):
            ops.gemm(a, w, out, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        # n back-to-back launches in one CUDA graph: device time, not the
        # host's per-call launch overhead (which alone is ~25 us per call)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(n):
                ops.gemm(a, w, out, workspace=ws)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) / n * 1000
        rows = torch.arange(0, M, 7, device="cuda")
        ref = (a[rows].float() @ w.float().T)
        err = float((out[rows].float() - ref).norm() / ref.norm())
        print(json.dumps({"pair": os.environ.get("ASTRAEA_GEMM_PAIR", "1"),
                          "splitk": os.environ.get("ASTRAEA_PAIR_SPLITK", "0"), "M": M, "shape": name, "N": N, "K": K,
                          "us": round(us, 1), "tflops": round(2 * M * N * K / us / 1e6, 1), "rel_err": err}),
              flush=True)
