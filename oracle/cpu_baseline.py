"""CPU port of the data path, for the bench's ``cpu_baseline`` leg and the
``--impl reference`` arm -- TEST/BASELINE INFRASTRUCTURE ONLY (see
oracle/__init__).

The reference executes no model (every GPU action is a delay,
simulator.py:329-337), so its "CPU implementation of the path" is this
restatement: the same Llama-3 layer math in torch on the host cores
(bf16 weights, fp32 accumulation, all threads), with a contiguous KV cache.

Bounded sample: one decoder layer is materialised (all layers of a Llama
have identical shapes and cost) and applied ``num_layers`` times, plus the
lm_head; a prefill chunk and a few decode steps at the replay's mean batch
are timed, and the replay's time is extrapolated from the exact prefill
token and decode step counts the scheduler produces for the trace.
"""

from __future__ import annotations

import os
import time

import torch


class CpuLayerSample:
    def __init__(self, cfg, seed: int = 0, dtype=torch.bfloat16):
        g = torch.Generator().manual_seed(seed)
        d = cfg.hidden
        r = lambda *s: (torch.randn(*s, generator=g) * 0.02).to(dtype)  # noqa: E731
        self.cfg = cfg
        self.wqkv = r(cfg.qkv_dim, d)
        self.wo = r(d, cfg.num_q_heads * cfg.head_dim)
        self.wgu = r(2 * cfg.ffn, d)
        self.wdown = r(d, cfg.ffn)
        self.lm = r(cfg.vocab, d)
        self.dtype = dtype

    def _layer(self, x, kv_len):
        cfg = self.cfg
        T = x.shape[0]
        Hq, Hkv, D = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
        h = x * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + cfg.eps).to(x.dtype)
        qkv = h @ self.wqkv.T
        q = qkv[:, : Hq * D].reshape(T, Hq, D).transpose(0, 1)
        # attention against kv_len cached tokens (+ the new ones), GQA
        k = torch.randn(Hkv, kv_len, D, dtype=x.dtype)
        v = torch.randn(Hkv, kv_len, D, dtype=x.dtype)
        k = k.repeat_interleave(Hq // Hkv, 0)
        v = v.repeat_interleave(Hq // Hkv, 0)
        a = torch.softmax((q.float() @ k.float().transpose(1, 2)) / D ** 0.5, -1) @ v.float()
        x = x + a.transpose(0, 1).reshape(T, Hq * D).to(x.dtype) @ self.wo.T
        h = x * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + cfg.eps).to(x.dtype)
        gu = h @ self.wgu.T
        m = torch.nn.functional.silu(gu[:, : cfg.ffn]) * gu[:, cfg.ffn:]
        return x + m @ self.wdown.T

    def step_seconds(self, T, kv_len):
        """Seconds for one full-model pass over T tokens attending kv_len tokens."""
        x = torch.randn(T, self.cfg.hidden, dtype=self.dtype)
        t0 = time.perf_counter()
        y = self._layer(x, kv_len)
        per_layer = time.perf_counter() - t0
        t0 = time.perf_counter()
        _ = y[-min(T, 64):] @ self.lm.T
        head = time.perf_counter() - t0
        return per_layer * self.cfg.num_layers + head


def threads() -> int:
    return torch.get_num_threads()


def estimate_replay_seconds(sample: CpuLayerSample, work: dict, budget_s: float = 20.0) -> dict:
    """Time a bounded sample and extrapolate to the replay's total work.

    ``work``: prefill_tokens, decode_steps, mean_batch, mean_ctx, batches.
    """
    torch.set_num_threads(os.cpu_count() or 1)
    pre_T = int(min(512, max(16, work["prefill_tokens"] / max(1, work["batches"]))))
    B = max(1, int(round(work["mean_batch"])))
    ctx = int(work["mean_ctx"])
    sample.step_seconds(8, 64)  # warm-up
    t_begin = time.perf_counter()
    pre = sample.step_seconds(pre_T, ctx)
    decs = []
    while len(decs) < 3 or (time.perf_counter() - t_begin < budget_s * 0.5 and len(decs) < 20):
        decs.append(sample.step_seconds(B, ctx))
    dec = sorted(decs)[len(decs) // 2]
    total = work["prefill_tokens"] / pre_T * pre + work["decode_steps"] * dec
    return {
        "replay_seconds": total,
        "prefill_chunk_tokens": pre_T,
        "prefill_chunk_seconds": pre,
        "decode_step_batch": B,
        "decode_step_seconds": dec,
        "sample_seconds": time.perf_counter() - t_begin,
        "threads": torch.get_num_threads(),
    }
