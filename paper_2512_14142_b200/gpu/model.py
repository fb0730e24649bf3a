"""Llama-3-shaped decoder executed entirely by the sm_100a kernels.

The reference has no model; its cost model stands in
for one (predictor.py:47-66). This module is the real computation behind
those delays: the recompute-on-resume prefill and the paged decode step.
Weights are random-init N(0, 0.02) with unit norms -- the
data path's cost does not depend on the values.

Per layer (bf16 activations, fp32 accumulation everywhere), five launches:
  q, k, v = rmsnorm(x) @ Wqkv^T ; rope ; k, v -> pool   one GEMM (K6/K9 + K5 fused)
  a       = paged attention (prefill K7 | decode K4)
  x       = a @ Wo^T + x                                 GEMM, residual + norm statistics fused
  m       = silu(g) * u,  [g|u] = rmsnorm(x) @ Wgu^T     GEMM, RMS scale + SiLU fused (K8)
  x       = m @ Wdown^T + x                              GEMM, residual + norm statistics fused
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
    def decode_weight_bytes(self) -> int:
        """Weight bytes one decode step must read: every layer, the final norm
        and lm_head; of the embedding table only the B gathered rows (not
        counted here)."""
        d, L = self.hidden, self.num_layers
        per_layer = (self.qkv_dim * d + d * self.num_q_heads * self.head_dim
                     + 2 * self.ffn * d + d * self.ffn + 2 * d)
        return 2 * (L * per_layer + self.vocab * d + d)

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


def interleave_gate_up(w_gu: torch.Tensor, ffn: int) -> torch.Tensor:
    """[gate F | up F] rows -> [64 gate | 64 up] per 128 rows (SILU epilogue layout)."""
    d = w_gu.shape[1]
    g = w_gu[:ffn].view(ffn // 64, 64, d)
    u = w_gu[ffn:].view(ffn // 64, 64, d)
    return torch.stack([g, u], dim=1).reshape(2 * ffn, d)


def deinterleave_gate_up(w: torch.Tensor, ffn: int) -> torch.Tensor:
    d = w.shape[1]
    v = w.view(ffn // 64, 2, 64, d)
    return torch.cat([v[:, 0].reshape(ffn, d), v[:, 1].reshape(ffn, d)], dim=0)


class LlamaWeights:
    """Device-resident bf16 weights in the fused-epilogue layout.

    Deterministic for a (config, seed). RMSNorm weights are folded into the
    following projection (x*w @ W^T == x @ (W diag w)^T), and the gate/up
    rows are interleaved per 64 for the SILU epilogue. ``to_cpu_dict``
    returns the logical (textbook) weights for the oracle.
    """

    def __init__(self, cfg: LlamaConfig, device="cuda", seed: int = 0, std: float = 0.02, embed_vocab: int = 0):
        """``embed_vocab``: embedding rows when it differs from cfg.vocab (a
        tensor-parallel rank keeps the whole embedding but a vocab slice of
        the lm_head)."""
        self.cfg = cfg
        g = torch.Generator(device=device)
        g.manual_seed(seed)

        def w(*shape):
            t = torch.empty(*shape, dtype=torch.bfloat16, device=device)
            t.normal_(0.0, std, generator=g)
            return t

        def fold(weight, norm):
            return (weight.float() * norm.float()[None, :]).to(torch.bfloat16)

        d = cfg.hidden
        ones = torch.ones(d, dtype=torch.bfloat16, device=device)
        self.embed = w(embed_vocab or cfg.vocab, d)
        self.layers = []
        for _ in range(cfg.num_layers):
            attn_norm, mlp_norm = ones.clone(), ones.clone()
            wqkv = w(cfg.qkv_dim, d)
            wo = w(d, cfg.num_q_heads * cfg.head_dim)
            wgu = w(2 * cfg.ffn, d)
            wdown = w(d, cfg.ffn)
            self.layers.append({
                "attn_norm": attn_norm,
                "mlp_norm": mlp_norm,
                "wqkv": fold(wqkv, attn_norm) if not bool((attn_norm == 1).all()) else wqkv,
                "wo": wo,
                "wgu": interleave_gate_up(fold(wgu, mlp_norm) if not bool((mlp_norm == 1).all()) else wgu, cfg.ffn),
                "wdown": wdown,
            })
        self.final_norm = ones.clone()
        self.lm_head = w(cfg.vocab, d)

    @classmethod
    def from_logical(cls, cfg: LlamaConfig, wd: dict, device="cuda") -> "LlamaWeights":
        """Device weights from logical ones (the to_cpu_dict format): norms
        folded into the following projection, gate/up interleaved."""
        self = cls.__new__(cls)
        self.cfg = cfg

        def dv(t):
            return t.to(device=device, dtype=torch.bfloat16).contiguous()

        def fold(weight, norm):
            return (weight.float() * norm.float()[None, :]).to(torch.bfloat16)

        self.embed = dv(wd["embed"])
        self.layers = []
        for lw in wd["layers"]:
            self.layers.append({
                "attn_norm": dv(lw["attn_norm"]), "mlp_norm": dv(lw["mlp_norm"]),
                "wqkv": dv(fold(lw["wqkv"], lw["attn_norm"])),
                "wo": dv(lw["wo"]),
                "wgu": dv(interleave_gate_up(fold(lw["wgu"], lw["mlp_norm"]), cfg.ffn)),
                "wdown": dv(lw["wdown"]),
            })
        self.final_norm = dv(wd["final_norm"])
        self.lm_head = dv(fold(wd["lm_head"], wd["final_norm"]))
        return self

    def to_cpu_dict(self, device="cpu") -> dict:
        """Logical weights: un-interleaved gate/up, norms separate (the
        stored projections are W diag(norm); with unit norms that is W).
        ``device``: where the copies live (the oracle runs there)."""

        def unfold(weight, norm):
            return (weight.float() / norm.float()[None, :]).to(torch.bfloat16).to(device)

        layers = []
        for lw in self.layers:
            layers.append({
                "attn_norm": lw["attn_norm"].to(device),
                "mlp_norm": lw["mlp_norm"].to(device),
                "wqkv": unfold(lw["wqkv"], lw["attn_norm"]),
                "wo": lw["wo"].to(device),
                "wgu": unfold(deinterleave_gate_up(lw["wgu"], self.cfg.ffn), lw["mlp_norm"]),
                "wdown": lw["wdown"].to(device),
            })
        return {"embed": self.embed.to(device), "layers": layers, "final_norm": self.final_norm.to(device),
                "lm_head": unfold(self.lm_head, self.final_norm)}


class LlamaRunner:
    """Runs prefill / decode passes of one model against one KV pool.

    Per layer, five launches: QKV GEMM (RMS scale + RoPE + KV append fused),
    paged attention, O GEMM (+ residual, emits the next norm's statistics),
    gate/up GEMM (RMS scale + SiLU*up fused), down GEMM (+ residual,
    statistics). RMSNorm never runs as its own kernel: every GEMM that
    consumes a normalised input scales its accumulator by rsqrt(mean x^2 +
    eps) computed from per-128-column sums of squares its producer wrote.
    """

    def __init__(self, weights: LlamaWeights, pool, max_tokens: int = 8192, max_rows: int = 64):
        self.w = weights
        self.cfg = weights.cfg
        self.pool = pool
        dev = weights.embed.device
        cfg = self.cfg
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        d = cfg.hidden
        shapes = [(cfg.qkv_dim, d), (d, cfg.num_q_heads * cfg.head_dim), (2 * cfg.ffn, d), (d, cfg.ffn),
                  (cfg.vocab, d)]
        lib = L.load()
        # decode (M <= 64: stream-K partials) and short prefills (CTA-pair K-split partials)
        need = max(lib.astraea_gemm_workspace_bytes(m, n, k) for n, k in shapes
                   for m in (64, 65, 128, 192, 256, 384, 512, 768, 1024))
        # (a chain's workspace is the max over its phases: the same bound)
        # split-K workspace (partials + arrival counters): zero-filled once,
        # the kernel resets its counters.
        self.gemm_ws = torch.zeros(need // 4 + 64, dtype=torch.float32, device=dev)
        self.max_rows = max_rows
        self.dec_ws = None
        self._old_ws = []
        self.device = dev
        self.parts = -(-d // 128)
        self.use_chain = True   # decode GEMMs as one persistent chain per layer (False: one launch each)
        # decoder layers per chain launch (with fused attention; 1 or 2). 2
        # measured equal at batch 1-16 (the launch boundary costs what an
        # in-kernel phase barrier costs under PDL), so 1 keeps the launches small
        self.chain_layers = 1
        # decode step as ONE persistent kernel (astraea_step_launch). Off by
        # default: on B200 it matches the per-layer chain at batch 1 and trails
        # it at larger batches ("decode-step kernel")
        self.use_step_kernel = False
        # the layer's decode attention runs inside its chained-GEMM launch
        # (astraea_gemm_chain_attn) instead of as a separate kernel
        self.fuse_attention = True
        # above this batch the layer's attention runs as its own TMA-staged
        # kernel before the chain (more pages in flight than the chain's
        # epilogue warps can keep; tools/attn_ab.py)
        self.fuse_max_batch = 64
        self.l2_ahead = 0
        self._mk = None
        self._programs: dict = {}
        self.last_program = None
        self.step_ws = ops.StepWorkspace()

    def _dec_ws(self, B, max_blocks):
        need = L.load().astraea_decode_workspace_bytes(B, self.cfg.num_q_heads, self.cfg.head_dim, max_blocks)
        if self.dec_ws is None or self.dec_ws.numel() * 4 < need:
            # superseded buffers stay alive: captured CUDA graphs may still use them
            if self.dec_ws is not None:
                self._old_ws.append(self.dec_ws)
            self.dec_ws = ops.decode_workspace(B, self.cfg.num_q_heads, self.cfg.head_dim, max_blocks,
                                               self.device)
        return self.dec_ws

    def _embed(self, ids, stream):
        T = ids.shape[0]
        ssq = torch.empty(1, T, dtype=torch.float32, device=self.device)
        x = ops.embedding(ids, self.w.embed, ssq_out=ssq, stream=stream)
        return x, ssq

    def _layers(self, x, ssq, positions, slots, attend, stream=None):
        cfg, w, pool = self.cfg, self.w, self.pool
        T = x.shape[0]
        dev = x.device
        qd = cfg.num_q_heads * cfg.head_dim
        q = torch.empty(T, qd, dtype=torch.bfloat16, device=dev)
        att = torch.empty(T, qd, dtype=torch.bfloat16, device=dev)
        h = torch.empty(T, cfg.ffn, dtype=torch.bfloat16, device=dev)
        ssq_mid = torch.empty(self.parts, T, dtype=torch.float32, device=dev)
        ssq_out = torch.empty(self.parts, T, dtype=torch.float32, device=dev)
        ws = self.gemm_ws
        d, eps = cfg.hidden, cfg.eps
        cs = ops.rope_table(positions, cfg.head_dim, cfg.rope_theta, stream=stream)
        for li, lw in enumerate(w.layers):
            ops.gemm_ex(x, lw["wqkv"], q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=d, rms_eps=eps, pool=pool.data,
                        geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads, positions=positions, slots=slots,
                        rope_theta=cfg.rope_theta, rope_table=cs, workspace=ws, stream=stream)
            attend(li, q, att)
            ops.gemm_ex(att, lw["wo"], x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq_mid, workspace=ws,
                        stream=stream)
            ops.gemm_ex(x, lw["wgu"], h, kind=L.EPI_SILU, ssq_in=ssq_mid, rms_dim=d, rms_eps=eps, workspace=ws,
                        stream=stream)
            ops.gemm_ex(h, lw["wdown"], x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq_out, workspace=ws,
                        stream=stream)
            ssq = ssq_out
        return x, ssq

    def _sample(self, x_rows, ssq_rows, stream=None, want_logits=False, keys_out=None):
        """Final norm + lm_head + greedy argmax in one GEMM (ARGMAX epilogue).

        With ``keys_out`` (int64, zeroed) the packed argmax keys stay on the
        device for ``decode_advance``; otherwise token ids are returned.
        """
        cfg = self.cfg
        rows = x_rows.shape[0]
        keys = keys_out if keys_out is not None else torch.zeros(rows, dtype=torch.int64, device=x_rows.device)
        logits = (torch.empty(rows, cfg.vocab, dtype=torch.bfloat16, device=x_rows.device)
                  if want_logits else None)
        ops.gemm_ex(x_rows, self.w.lm_head, logits, kind=L.EPI_ARGMAX, ssq_in=ssq_rows, rms_dim=cfg.hidden,
                    rms_eps=cfg.eps, argmax_keys=keys, workspace=self.gemm_ws, stream=stream)
        if keys_out is not None:
            return (keys_out, logits) if want_logits else keys_out
        ids = ops.keys_to_ids(keys)
        return (ids, logits) if want_logits else ids

    def prefill(self, ids, positions, slots, cu_q, table, ctx, last_rows, max_q_len, stream=None,
                want_logits=False):
        """Varlen prefill of S sequences; returns the greedy next token of each."""
        cfg = self.cfg
        S = ctx.shape[0]
        x, ssq = self._embed(ids, stream)
        qd = cfg.num_q_heads * cfg.head_dim

        def attend(li, q, out):
            ops.prefill_attention(self.pool.geo, self.pool.data, li, q, qd, cu_q, S, max_q_len,
                                  cfg.num_q_heads, table, ctx, self.scale, out, stream=stream)

        x, ssq = self._layers(x, ssq, positions, slots, attend, stream)
        return self._sample(x.index_select(0, last_rows), ssq.index_select(1, last_rows).contiguous(), stream,
                            want_logits)

    def decode(self, tokens, positions, slots, table, ctx, stream=None, want_logits=False, keys_out=None):
        """One decode step for B rows (retired rows: slot -1, ctx 0). With
        ``keys_out`` the sampled tokens stay on the device as argmax keys.

        Launches: embedding, RoPE table, layer 0's QKV GEMM, then per
        ``chain_layers`` (1) layer(s) ONE kernel running, for each layer, the
        paged attention and the chained GEMMs O-proj -> gate/up -> down ->
        next layer's QKV (the last layer ends with lm_head + argmax
        instead); with fuse_attention off the attention is a separate
        launch and each chain carries one layer."""
        if self.cfg.num_layers < 1 or tokens.shape[0] > 64:
            return self._decode_unchained(tokens, positions, slots, table, ctx, stream, want_logits, keys_out)
        if self.use_step_kernel and self._step_supported():
            return self._decode_step_kernel(tokens, positions, slots, table, ctx, stream, keys_out, want_logits)
        if not self.use_chain:
            return self._decode_unchained(tokens, positions, slots, table, ctx, stream, want_logits, keys_out)
        cfg, w, pool = self.cfg, self.w, self.pool
        B = tokens.shape[0]
        dev = tokens.device
        x, ssq0 = self._embed(tokens, stream)
        dws = self._dec_ws(B, table.shape[1])
        qd = cfg.num_q_heads * cfg.head_dim
        d, eps = cfg.hidden, cfg.eps
        ws = self.gemm_ws
        q = torch.empty(B, qd, dtype=torch.bfloat16, device=dev)
        att = torch.empty(B, qd, dtype=torch.bfloat16, device=dev)
        h = torch.empty(B, cfg.ffn, dtype=torch.bfloat16, device=dev)
        ssq_mid = torch.empty(self.parts, B, dtype=torch.float32, device=dev)
        ssq = torch.empty(self.parts, B, dtype=torch.float32, device=dev)
        keys = keys_out if keys_out is not None else torch.zeros(B, dtype=torch.int64, device=dev)
        # the last layer's chain ends with lm_head + argmax; it also writes the
        # logits when asked (same epilogue, C non-null)
        logits = torch.empty(B, cfg.vocab, dtype=torch.bfloat16, device=dev) if want_logits else None
        cs = ops.rope_table(positions, cfg.head_dim, cfg.rope_theta, stream=stream)

        def qkv(li, ssq_in):
            return dict(a=x, w=w.layers[li]["wqkv"], out=q, kind=L.EPI_QKV_ROPE, ssq_in=ssq_in, rms_dim=d,
                        rms_eps=eps, pool=pool.data, geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads,
                        positions=positions, slots=slots, rope_theta=cfg.rope_theta, rope_table=cs)

        ops.gemm_ex(**qkv(0, ssq0), workspace=ws, stream=stream)
        fuse = self.fuse_attention and self._attn_fusable() and B <= self.fuse_max_batch
        per = self.chain_layers if fuse else 1
        for l0 in range(0, cfg.num_layers, per):
            phases, attns = [], []
            for li in range(l0, min(l0 + per, cfg.num_layers)):
                lw = w.layers[li]
                if fuse:
                    attns.append(dict(pool=pool.data, geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads, q=q,
                                      q_stride=qd, table=table, ctx=ctx, scale=self.scale, out=att,
                                      before=len(phases)))
                else:
                    ops.decode_attention(pool.geo, pool.data, li, q, qd, B, cfg.num_q_heads, table, ctx,
                                         self.scale, att, dws, stream=stream)
                phases += [
                    dict(a=att, w=lw["wo"], out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq_mid),
                    dict(a=x, w=lw["wgu"], out=h, kind=L.EPI_SILU, ssq_in=ssq_mid, rms_dim=d, rms_eps=eps),
                    dict(a=h, w=lw["wdown"], out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq),
                ]
                if li + 1 < cfg.num_layers:
                    phases.append(qkv(li + 1, ssq))
                else:
                    phases.append(dict(a=x, w=w.lm_head, out=logits, kind=L.EPI_ARGMAX, ssq_in=ssq, rms_dim=d,
                                       rms_eps=eps, argmax_keys=keys))
            ops.gemm_chain(phases, ws, stream=stream, attn=attns or None)
        if keys_out is not None:
            return (keys_out, logits) if want_logits else keys_out
        ids = ops.keys_to_ids(keys)
        return (ids, logits) if want_logits else ids

    def _attn_fusable(self) -> bool:
        cfg = self.cfg
        G = cfg.num_q_heads // cfg.num_kv_heads
        return (cfg.head_dim, G) in ((128, 4), (64, 2), (64, 4), (128, 8))

    def _step_supported(self) -> bool:
        cfg = self.cfg
        G = cfg.num_q_heads // cfg.num_kv_heads
        return (cfg.head_dim, G) in ((128, 4), (64, 2), (64, 4))

    def _mk_bufs(self):
        """Persistent activation buffers of the step kernel (max_rows rows):
        the program's TMA descriptors point at them, so they never move."""
        if self._mk is None:
            cfg, R, dev = self.cfg, self.max_rows, self.device
            qd = cfg.num_q_heads * cfg.head_dim
            bf = dict(dtype=torch.bfloat16, device=dev)
            self._mk = {
                "x": torch.zeros(R, cfg.hidden, **bf), "q": torch.zeros(R, qd, **bf),
                "att": torch.zeros(R, qd, **bf), "h": torch.zeros(R, cfg.ffn, **bf),
                "ssq0": torch.zeros(1, R, dtype=torch.float32, device=dev),
                "ssq_mid": torch.zeros(self.parts, R, dtype=torch.float32, device=dev),
                "ssq": torch.zeros(self.parts, R, dtype=torch.float32, device=dev),
                "cs": torch.zeros(R, cfg.head_dim // 2, 2, dtype=torch.float32, device=dev),
            }
        return self._mk

    def step_phases(self, B, positions, slots, table, ctx, keys, logits=None):
        """The decode step as a phase program (see ops.StepProgram): per layer
        QKV(+RoPE+append) -> ATTN -> O(+residual) -> gate/up(+SiLU) ->
        down(+residual), the last layer's down feeding lm_head + argmax."""
        cfg, w, pool = self.cfg, self.w, self.pool
        mb = self._mk_bufs()
        x, q, att, h = mb["x"][:B], mb["q"][:B], mb["att"][:B], mb["h"][:B]
        P = self.parts
        ssq0 = mb["ssq0"].view(-1)[:B].view(1, B)
        ssq_mid = mb["ssq_mid"].view(-1)[:P * B].view(P, B)
        ssq = mb["ssq"].view(-1)[:P * B].view(P, B)
        cs = mb["cs"][:B]
        d, eps, qd = cfg.hidden, cfg.eps, cfg.num_q_heads * cfg.head_dim
        phases = []

        def qkv(li, ssq_in, a_from):
            phases.append(dict(kind="gemm", a=x, w=w.layers[li]["wqkv"], out=q, epi=L.EPI_QKV_ROPE, a_from=a_from,
                               epi_from=a_from, ssq_in=ssq_in, rms_dim=d,
                               rms_eps=eps, pool=pool.data, geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads,
                               positions=positions, slots=slots, rope_theta=cfg.rope_theta, rope_table=cs))
            return len(phases) - 1

        i_qkv = qkv(0, ssq0, -1)
        i_down = -1
        for li, lw in enumerate(w.layers):
            phases.append(dict(kind="attn", pool=pool.data, geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads,
                               q=q, q_stride=qd, table=table, ctx=ctx, scale=self.scale, out=att, qkv_from=i_qkv))
            i_att = len(phases) - 1
            phases.append(dict(kind="gemm", a=att, w=lw["wo"], out=x, epi=L.EPI_RESIDUAL, residual=x,
                               ssq_out=ssq_mid, a_from=i_att, epi_from=i_down))
            i_o = len(phases) - 1
            phases.append(dict(kind="gemm", a=x, w=lw["wgu"], out=h, epi=L.EPI_SILU, ssq_in=ssq_mid, rms_dim=d,
                               rms_eps=eps, a_from=i_o, epi_from=i_o))
            i_gu = len(phases) - 1
            phases.append(dict(kind="gemm", a=h, w=lw["wdown"], out=x, epi=L.EPI_RESIDUAL, residual=x,
                               ssq_out=ssq, a_from=i_gu, epi_from=i_o))
            i_down = len(phases) - 1
            if li + 1 < cfg.num_layers:
                i_qkv = qkv(li + 1, ssq, i_down)
        phases.append(dict(kind="gemm", a=x, w=w.lm_head, out=logits, epi=L.EPI_ARGMAX, ssq_in=ssq, rms_dim=d,
                           rms_eps=eps, argmax_keys=keys, a_from=i_down, epi_from=i_down))
        return phases

    def _decode_step_kernel(self, tokens, positions, slots, table, ctx, stream=None, keys_out=None,
                            want_logits=False):
        """Embedding + RoPE table + ONE persistent launch for every layer and
        the sampling (astraea_step_launch)."""
        cfg = self.cfg
        B = tokens.shape[0]
        dev = tokens.device
        mb = self._mk_bufs()
        keys = keys_out if keys_out is not None else torch.zeros(B, dtype=torch.int64, device=dev)
        ops.embedding(tokens, self.w.embed, out=mb["x"][:B], ssq_out=mb["ssq0"].view(-1)[:B], stream=stream)
        ops.rope_table(positions, cfg.head_dim, cfg.rope_theta, out=mb["cs"][:B], stream=stream)
        logits = None
        if want_logits:
            if "logits" not in mb:
                mb["logits"] = torch.zeros(self.max_rows, cfg.vocab, dtype=torch.bfloat16, device=dev)
            logits = mb["logits"][:B]
        key = (B, positions.data_ptr(), slots.data_ptr(), table.data_ptr(), table.shape[1], ctx.data_ptr(),
               keys.data_ptr(), want_logits)
        prog = self._programs.get(key)
        if prog is None:
            s = stream if stream is not None else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                prog = ops.StepProgram(B, self.step_phases(B, positions, slots, table, ctx, keys, logits),
                                       self.step_ws)
            if len(self._programs) >= 16:
                self._programs.pop(next(iter(self._programs)))
            self._programs[key] = prog
        self.last_program = prog
        prog.launch(stream, self.l2_ahead)
        if want_logits:
            ids = ops.keys_to_ids(keys)
            return ids, logits.clone()
        if keys_out is not None:
            return keys_out
        return ops.keys_to_ids(keys)

    def _decode_unchained(self, tokens, positions, slots, table, ctx, stream=None, want_logits=False,
                          keys_out=None):
        """Same step, one launch per GEMM (reference path for the chained one)."""
        cfg = self.cfg
        B = tokens.shape[0]
        x, ssq = self._embed(tokens, stream)
        ws = self._dec_ws(B, table.shape[1])
        qd = cfg.num_q_heads * cfg.head_dim

        def attend(li, q, out):
            ops.decode_attention(self.pool.geo, self.pool.data, li, q, qd, B, cfg.num_q_heads,
                                 table, ctx, self.scale, out, ws, stream=stream)

        x, ssq = self._layers(x, ssq, positions, slots, attend, stream)
        return self._sample(x, ssq, stream, want_logits, keys_out)
