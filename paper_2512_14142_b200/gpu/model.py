"""Llama-3-shaped decoder executed entirely by the sm_100a kernels.

The reference has no model; its cost model stands in
for one (predictor.py:47-66). This module is the real computation behind
those delays: the recompute-on-resume prefill and the paged decode step.
Weights are random-init N(0, 0.02) with unit norms -- the
data path's cost does not depend on the values.

Per layer (bf16 activations, fp32 accumulation everywhere):
  h   = rmsnorm(x)                                  K8
  qkv = h @ Wqkv^T                                  K6/K9 tcgen05 GEMM
  rope(q, k); append k, v to pool slots             K5
  a   = paged attention (prefill K7 | decode K4)
  x   = a @ Wo^T + x                                GEMM, residual fused in epilogue
  h   = rmsnorm(x)
  gu  = h @ Wgu^T ; m = silu(g) * u                 GEMM + K8
  x   = m @ Wdown^T + x                             GEMM, residual fused
then logits = rmsnorm(x_last) @ Wlm^T and greedy argmax.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import lib as L
from . import ops


@dataclass(frozen=True)
class LlamaConfig:
    name: str
    num_layers: int
    hidden: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float = 500000.0
    eps: float = 1e-5

    @property
    def qkv_dim(self) -> int:
        return (self.num_q_heads + 2 * self.num_kv_heads) * self.head_dim

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.num_layers * self.num_kv_heads * self.head_dim * 2

    @property
    def weight_bytes(self) -> int:
        d, L = self.hidden, self.num_layers
        per_layer = (self.qkv_dim * d + d * self.num_q_heads * self.head_dim
                     + 2 * self.ffn * d + d * self.ffn + 2 * d)
        return 2 * (L * per_layer + 2 * self.vocab * d + d)

    @property
    def linear_params_per_token(self) -> int:
        """Multiply-adds per token in the layer projections (prefill FLOPs / 2)."""
        d = self.hidden
        return self.num_layers * (self.qkv_dim * d + d * self.num_q_heads * self.head_dim
                                  + 3 * self.ffn * d)


PRESETS = {
    # unit-test sized
    "tiny": LlamaConfig("tiny", 2, 256, 4, 2, 64, 512, 1024),
    # small random-init model for C1 numerics (2,048 B/token)
    "small": LlamaConfig("small", 4, 512, 8, 2, 64, 1536, 32000),
    "llama3-8b": LlamaConfig("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256),
    # one tensor-parallel rank of Llama-3-70B at TP=8 (40,960 B/token/GPU)
    "llama3-70b-tp8": LlamaConfig("llama3-70b-tp8", 80, 8192, 8, 1, 128, 3584, 128256),
}


class LlamaWeights:
    """Device-resident bf16 weights; deterministic for a (config, seed)."""

    def __init__(self, cfg: LlamaConfig, device="cuda", seed: int = 0, std: float = 0.02):
        self.cfg = cfg
        g = torch.Generator(device=device)
        g.manual_seed(seed)

        def w(*shape):
            t = torch.empty(*shape, dtype=torch.bfloat16, device=device)
            t.normal_(0.0, std, generator=g)
            return t

        d = cfg.hidden
        self.embed = w(cfg.vocab, d)
        self.layers = []
        for _ in range(cfg.num_layers):
            self.layers.append({
                "attn_norm": torch.ones(d, dtype=torch.bfloat16, device=device),
                "wqkv": w(cfg.qkv_dim, d),
                "wo": w(d, cfg.num_q_heads * cfg.head_dim),
                "mlp_norm": torch.ones(d, dtype=torch.bfloat16, device=device),
                "wgu": w(2 * cfg.ffn, d),          # rows [0, F) gate, [F, 2F) up
                "wdown": w(d, cfg.ffn),
            })
        self.final_norm = torch.ones(d, dtype=torch.bfloat16, device=device)
        self.lm_head = w(cfg.vocab, d)

    def to_cpu_dict(self) -> dict:
        return {
            "embed": self.embed.cpu(),
            "layers": [{k: v.cpu() for k, v in lw.items()} for lw in self.layers],
            "final_norm": self.final_norm.cpu(),
            "lm_head": self.lm_head.cpu(),
        }


class LlamaRunner:
    """Runs prefill / decode passes of one model against one KV pool."""

    def __init__(self, weights: LlamaWeights, pool, max_tokens: int = 8192, max_rows: int = 64):
        self.w = weights
        self.cfg = weights.cfg
        self.pool = pool
        dev = weights.embed.device
        cfg = self.cfg
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        # split-K workspace for decode GEMMs (M <= 64): partials + arrival
        # counters; zero-filled once, the kernel resets its counters.
        d = cfg.hidden
        shapes = [(cfg.qkv_dim, d), (d, cfg.num_q_heads * cfg.head_dim), (2 * cfg.ffn, d), (d, cfg.ffn),
                  (cfg.vocab, d)]
        lib = L.load()
        need = max(lib.astraea_gemm_workspace_bytes(64, n, k) for n, k in shapes)
        self.gemm_ws = torch.zeros(need // 4 + 64, dtype=torch.float32, device=dev)
        self.max_rows = max_rows
        self.dec_ws = None
        self.dec_ws_key = None
        self.device = dev

    def _dec_ws(self, B, max_blocks):
        need = L.load().astraea_decode_workspace_bytes(B, self.cfg.num_q_heads, self.cfg.head_dim, max_blocks)
        if self.dec_ws is None or self.dec_ws.numel() * 4 < need:
            self.dec_ws = ops.decode_workspace(B, self.cfg.num_q_heads, self.cfg.head_dim, max_blocks,
                                               self.device)
        return self.dec_ws

    def _layers(self, x, positions, slots, attend, stream=None):
        cfg, w, pool = self.cfg, self.w, self.pool
        T = x.shape[0]
        qd = cfg.num_q_heads * cfg.head_dim
        for li, lw in enumerate(w.layers):
            h = ops.rmsnorm(x, lw["attn_norm"], cfg.eps, stream=stream)
            qkv = ops.gemm(h, lw["wqkv"], workspace=self.gemm_ws, stream=stream)
            ops.rope_kv_append(pool.geo, pool.data, li, qkv, cfg.num_q_heads, positions, slots,
                               cfg.rope_theta, stream=stream)
            att = torch.empty(T, qd, dtype=torch.bfloat16, device=x.device)
            attend(li, qkv, att)
            ops.gemm(att, lw["wo"], out=x, residual=x, workspace=self.gemm_ws, stream=stream)
            h = ops.rmsnorm(x, lw["mlp_norm"], cfg.eps, stream=stream)
            gu = ops.gemm(h, lw["wgu"], workspace=self.gemm_ws, stream=stream)
            m = ops.silu_mul(gu, stream=stream)
            ops.gemm(m, lw["wdown"], out=x, residual=x, workspace=self.gemm_ws, stream=stream)
        return x

    def _sample(self, x_rows, stream=None, want_logits=False, ids_out=None):
        cfg = self.cfg
        h = ops.rmsnorm(x_rows, self.w.final_norm, cfg.eps, stream=stream)
        logits = ops.gemm(h, self.w.lm_head, workspace=self.gemm_ws, stream=stream)
        ids = ops.argmax(logits, out=ids_out, stream=stream)
        return (ids, logits) if want_logits else ids

    def prefill(self, ids, positions, slots, cu_q, table, ctx, last_rows, max_q_len, stream=None,
                want_logits=False):
        """Varlen prefill of S sequences; returns the greedy next token of each."""
        cfg = self.cfg
        S = ctx.shape[0]
        x = ops.embedding(ids, self.w.embed, stream=stream)

        def attend(li, qkv, out):
            ops.prefill_attention(self.pool.geo, self.pool.data, li, qkv, cfg.qkv_dim, cu_q, S, max_q_len,
                                  cfg.num_q_heads, table, ctx, self.scale, out, stream=stream)

        self._layers(x, positions, slots, attend, stream)
        return self._sample(x.index_select(0, last_rows), stream, want_logits)

    def decode(self, tokens, positions, slots, table, ctx, stream=None, want_logits=False, ids_out=None):
        """One decode step for B rows (retired rows: slot -1, ctx 0)."""
        cfg = self.cfg
        B = tokens.shape[0]
        x = ops.embedding(tokens, self.w.embed, stream=stream)
        ws = self._dec_ws(B, table.shape[1])

        def attend(li, qkv, out):
            ops.decode_attention(self.pool.geo, self.pool.data, li, qkv, cfg.qkv_dim, B, cfg.num_q_heads,
                                 table, ctx, self.scale, out, ws, stream=stream)

        self._layers(x, positions, slots, attend, stream)
        return self._sample(x, stream, want_logits, ids_out)
