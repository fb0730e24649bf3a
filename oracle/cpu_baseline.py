"""CPU port of the data path, for the bench's ``cpu_baseline`` leg and the
``--impl reference`` arm -- TEST/BASELINE INFRASTRUCTURE ONLY (see
oracle/__init__).

The reference executes no model (every GPU action is a delay,
simulator.py:329-337), so "the reference's CPU implementation of the path"
is this restatement: the whole Llama-3 model (all ``num_layers`` layers
materialised, fp32 weights, fp32 math) on the host cores with torch's
threads, a contiguous per-row KV cache, and the batch shapes the reference
scheduler produces (``bench.work_profile``).

Timed sample per scheduled batch (``batch_sample``): one full-model prefill
chunk of up to ``PREFILL_CHUNK`` of the batch's prefill tokens against its
mean context, and one full-model decode step with the batch's rows at their
context. Every input (activations, KV caches, weights) is created before the
timed region; nothing random happens inside it. A batch's CPU time is then
``prefill_tokens / chunk x t_chunk + decode_steps x t_step`` -- the batch's
exact work counts times the measured per-unit costs (prefill is linear in
tokens at these sizes, and a decode step's cost on the CPU is the weight
stream, independent of how many of the batch's rows are still active).

Weights: N(0, 0.02) blocks tiled over each matrix (fp32 dense GEMM cost does
not depend on the values; tiling keeps the 8B model's 32 GB init to seconds).
"""

from __future__ import annotations

import os
import time

import torch
import torch.nn.functional as F

PREFILL_CHUNK = 128


def _tiled(shape, g, block=1 << 22):
    t = torch.empty(shape)
    flat = t.view(-1)
    src = torch.randn(min(block, flat.numel()), generator=g) * 0.02
    n = src.numel()
    full = flat.numel() // n
    if full:
        flat[: full * n].view(full, n).copy_(src.expand(full, n))
    rest = flat.numel() - full * n
    if rest:
        flat[full * n:].copy_(src[:rest])
    return t


class CpuLlama:
    """fp32 Llama-3 decoder (RMSNorm, RoPE, GQA, SwiGLU) on the host cores."""

    def __init__(self, cfg, seed: int = 0, threads: int | None = None):
        torch.set_num_threads(threads or os.cpu_count() or 1)
        g = torch.Generator().manual_seed(seed)
        d, qd = cfg.hidden, cfg.num_q_heads * cfg.head_dim
        self.cfg = cfg
        self.layers = [dict(wqkv=_tiled((cfg.qkv_dim, d), g), wo=_tiled((d, qd), g),
                            wgu=_tiled((2 * cfg.ffn, d), g), wdown=_tiled((d, cfg.ffn), g))
                       for _ in range(cfg.num_layers)]
        self.lm = _tiled((cfg.vocab, d), g)
        self.inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.head_dim, 2).float() / cfg.head_dim))
        self._kv = {}

    @property
    def threads(self) -> int:
        return torch.get_num_threads()

    def _rope(self, x, pos):   # x [T, H, D], NeoX half split
        ang = pos.float()[:, None] * self.inv[None, :]
        cos, sin = ang.cos()[:, None, :], ang.sin()[:, None, :]
        h = x.shape[-1] // 2
        return torch.cat([x[..., :h] * cos - x[..., h:] * sin, x[..., h:] * cos + x[..., :h] * sin], -1)

    def _norm(self, x):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.cfg.eps)

    def _caches(self, rows, ctx):
        """Per-layer K/V caches [rows, Hkv, ctx, D], filled once (untimed)."""
        key = (rows, ctx)
        if key not in self._kv:
            c = self.cfg
            g = torch.Generator().manual_seed(rows * 100003 + ctx)
            kv = torch.randn(2, rows, c.num_kv_heads, ctx, c.head_dim, generator=g)
            self._kv = {key: kv}    # keep one shape resident at a time
        return self._kv[key]

    def forward(self, x, pos, kv, causal_from):
        """x [R, T, d] (R rows of T new tokens) attending the rows' cached
        ``kv`` ([2, R, Hkv, C, D], same cache reused by every layer: the cost
        is identical) plus the new tokens causally. Returns last-token logits."""
        c = self.cfg
        R, T, d = x.shape
        Hq, Hkv, D = c.num_q_heads, c.num_kv_heads, c.head_dim
        for lw in self.layers:
            h = self._norm(x).view(R * T, d)
            qkv = h @ lw["wqkv"].T
            q = qkv[:, : Hq * D].view(R * T, Hq, D)
            k = qkv[:, Hq * D: (Hq + Hkv) * D].view(R * T, Hkv, D)
            v = qkv[:, (Hq + Hkv) * D:].view(R * T, Hkv, D)
            q = self._rope(q, pos).view(R, T, Hq, D).transpose(1, 2)
            k = self._rope(k, pos).view(R, T, Hkv, D).transpose(1, 2)
            v = v.view(R, T, Hkv, D).transpose(1, 2)
            kk = torch.cat([kv[0], k], 2)
            vv = torch.cat([kv[1], v], 2)
            mask = None
            if T > 1:
                C = kk.shape[2]
                mask = torch.ones(T, C, dtype=torch.bool).tril(C - T)
            a = F.scaled_dot_product_attention(q, kk, vv, attn_mask=mask, enable_gqa=True)
            x = x + (a.transpose(1, 2).reshape(R * T, Hq * D) @ lw["wo"].T).view(R, T, d)
            h = self._norm(x).view(R * T, d)
            gu = h @ lw["wgu"].T
            m = F.silu(gu[:, : c.ffn]) * gu[:, c.ffn:]
            x = x + (m @ lw["wdown"].T).view(R, T, d)
        return self._norm(x[:, -1]) @ self.lm.T

    def time_prefill(self, tokens: int, ctx: int) -> float:
        kv = self._caches(1, ctx)
        x = torch.randn(1, tokens, self.cfg.hidden) * 0.1
        pos = torch.arange(ctx, ctx + tokens)
        t0 = time.perf_counter()
        self.forward(x, pos, kv, ctx)
        return time.perf_counter() - t0

    def time_decode(self, rows: int, ctx: int) -> float:
        kv = self._caches(rows, ctx)
        x = torch.randn(rows, 1, self.cfg.hidden) * 0.1
        pos = torch.full((rows,), ctx)
        t0 = time.perf_counter()
        self.forward(x, pos, kv, ctx)
        return time.perf_counter() - t0


def batch_sample(model: CpuLlama, b: dict) -> dict:
    """Time one scheduled batch's bounded sample; ``b`` is a
    ``bench.work_profile`` batch record. Returns the measured sample times and
    the batch's CPU time (its exact work counts x the measured unit costs)."""
    chunk = max(1, min(PREFILL_CHUNK, b["prefill_tokens"]))
    ctx = max(1, int(b["mean_ctx"]))
    t0 = time.perf_counter()
    t_pre = model.time_prefill(chunk, max(0, ctx - chunk)) if b["prefill_tokens"] else 0.0
    t_dec = model.time_decode(b["members"], ctx)
    sample = time.perf_counter() - t0
    est = (b["prefill_tokens"] / chunk) * t_pre + b["decode_steps"] * t_dec
    return {"sample_s": sample, "prefill_chunk": chunk, "prefill_chunk_s": t_pre, "decode_step_s": t_dec,
            "batch_cpu_s": est}
