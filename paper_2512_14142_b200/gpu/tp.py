"""Tensor parallelism for the large-model configuration (BASELINE.json C5:
Llama-3-70B shape, TP=8 over NVLink), SURVEY.md 8(e).

One process per GPU. Rank r of T holds, per layer,
  Wqkv rows of its Hq/T q heads and Hkv/T kv heads (its KV pool holds only
        those kv heads, so a swap moves 1/T of the token's KV),
  Wo   columns of its q heads          -> partial sums, all-reduce,
  Wgu  rows of its F/T gate and up features,
  Wdown columns of its F/T features    -> partial sums, all-reduce,
and the lm_head rows of its V/T vocabulary slice; the embedding and norm
weights are replicated. The residual stream is replicated after each
all-reduce, so RMSNorm statistics are recomputed locally (astraea_row_ssq).
Greedy sampling needs no logits exchange: each rank's ARGMAX epilogue packs
(value, global column) keys and one max-all-reduce of the keys picks the
token. Collectives go through torch.distributed (NCCL on the GPU box, gloo in
the CPU tests); the reference has no parallelism at all.
"""

from __future__ import annotations

import dataclasses

import torch

from . import lib as L
from . import ops
from .model import LlamaConfig, LlamaRunner, LlamaWeights


def shard_config(cfg: LlamaConfig, world: int) -> LlamaConfig:
    """The per-rank shape (vocab = the rank's lm_head slice)."""
    if cfg.num_q_heads % world or cfg.num_kv_heads % world or cfg.ffn % world or cfg.vocab % world:
        raise ValueError(f"{cfg.name} does not shard {world} ways")
    return dataclasses.replace(cfg, name=f"{cfg.name}-tp{world}", num_q_heads=cfg.num_q_heads // world,
                               num_kv_heads=cfg.num_kv_heads // world, ffn=cfg.ffn // world,
                               vocab=cfg.vocab // world)


def shard_logical(wd: dict, cfg: LlamaConfig, rank: int, world: int) -> dict:
    """Rank `rank`'s slice of logical (textbook-layout) weights
    (LlamaWeights.to_cpu_dict() format: wqkv [(Hq+2Hkv)D][d] as q|k|v heads,
    wgu [2F][d] as gate rows then up rows)."""
    Hq, Hkv, D, F, V = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.ffn, cfg.vocab
    hq, hk, f, v = Hq // world, Hkv // world, F // world, V // world
    layers = []
    for lw in wd["layers"]:
        q = lw["wqkv"][rank * hq * D:(rank + 1) * hq * D]
        k = lw["wqkv"][Hq * D + rank * hk * D:Hq * D + (rank + 1) * hk * D]
        vv = lw["wqkv"][(Hq + Hkv) * D + rank * hk * D:(Hq + Hkv) * D + (rank + 1) * hk * D]
        gate = lw["wgu"][rank * f:(rank + 1) * f]
        up = lw["wgu"][F + rank * f:F + (rank + 1) * f]
        layers.append({
            "attn_norm": lw["attn_norm"], "mlp_norm": lw["mlp_norm"],
            "wqkv": torch.cat([q, k, vv]).contiguous(),
            "wo": lw["wo"][:, rank * hq * D:(rank + 1) * hq * D].contiguous(),
            "wgu": torch.cat([gate, up]).contiguous(),
            "wdown": lw["wdown"][:, rank * f:(rank + 1) * f].contiguous(),
        })
    return {"embed": wd["embed"], "layers": layers, "final_norm": wd["final_norm"],
            "lm_head": wd["lm_head"][rank * v:(rank + 1) * v].contiguous()}


class TpLlamaRunner(LlamaRunner):
    """LlamaRunner for one tensor-parallel rank: the same kernels and fused
    epilogues, with the all-reduces after the O and down projections and a
    max-all-reduce of the sampling keys. Rank 0 adds the residual inside its
    projection epilogue; the other ranks contribute the bare partial sums."""

    def __init__(self, weights: LlamaWeights, pool, rank: int, world: int, group=None, max_tokens: int = 8192,
                 max_rows: int = 64):
        super().__init__(weights, pool, max_tokens=max_tokens, max_rows=max_rows)
        self.rank, self.world, self.group = rank, world, group
        self.use_chain = True     # decode: two chained launches per layer around the all-reduces
        self.use_step_kernel = False
        self.hidden = weights.embed.shape[1]

    def _allreduce(self, t, op=None, stream=None):
        """In-place all-reduce of ``t``, ordered on ``stream`` (the stream the
        kernels producing and consuming ``t`` run on): torch.distributed
        enqueues on the current stream."""
        if self.world == 1:
            return t
        import contextlib

        import torch.distributed as dist
        ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
        with ctx:
            dist.all_reduce(t, op=op or dist.ReduceOp.SUM, group=self.group)
        return t

    def _residual_pair(self, T, dev):
        """Ping-pong buffers for the replicated residual stream: a projection
        writes its partial sums (rank 0: + residual) into the buffer the
        residual does not occupy, the all-reduce runs in place there, and that
        buffer becomes the residual -- no copy after a collective."""
        d = self.hidden
        return [torch.empty(T, d, dtype=torch.bfloat16, device=dev) for _ in range(2)]

    def _layers(self, x, ssq, positions, slots, attend, stream=None):
        cfg, w, pool = self.cfg, self.w, self.pool
        T = x.shape[0]
        dev = x.device
        d, eps = self.hidden, cfg.eps
        qd = cfg.num_q_heads * cfg.head_dim
        q = torch.empty(T, qd, dtype=torch.bfloat16, device=dev)
        att = torch.empty(T, qd, dtype=torch.bfloat16, device=dev)
        h = torch.empty(T, cfg.ffn, dtype=torch.bfloat16, device=dev)
        pair = self._residual_pair(T, dev)
        ws = self.gemm_ws
        cs = ops.rope_table(positions, cfg.head_dim, cfg.rope_theta, stream=stream)
        lead = self.rank == 0
        for li, lw in enumerate(w.layers):
            ops.gemm_ex(x, lw["wqkv"], q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=d, rms_eps=eps, pool=pool.data,
                        geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads, positions=positions, slots=slots,
                        rope_theta=cfg.rope_theta, rope_table=cs, workspace=ws, stream=stream)
            attend(li, q, att)
            part = pair[1] if x is pair[0] else pair[0]
            ops.gemm_ex(att, lw["wo"], part, kind=L.EPI_RESIDUAL if lead else L.EPI_NONE,
                        residual=x if lead else None, workspace=ws, stream=stream)
            x = self._allreduce(part, stream=stream)
            ssq_mid = ops.row_ssq(x, stream=stream)
            ops.gemm_ex(x, lw["wgu"], h, kind=L.EPI_SILU, ssq_in=ssq_mid, rms_dim=d, rms_eps=eps, workspace=ws,
                        stream=stream)
            part = pair[1] if x is pair[0] else pair[0]
            ops.gemm_ex(h, lw["wdown"], part, kind=L.EPI_RESIDUAL if lead else L.EPI_NONE,
                        residual=x if lead else None, workspace=ws, stream=stream)
            x = self._allreduce(part, stream=stream)
            ssq = ops.row_ssq(x, stream=stream)
        return x, ssq

    def _sample(self, x_rows, ssq_rows, stream=None, want_logits=False, keys_out=None):
        import torch.distributed as dist
        cfg = self.cfg
        rows = x_rows.shape[0]
        keys = keys_out if keys_out is not None else torch.zeros(rows, dtype=torch.int64, device=x_rows.device)
        logits = (torch.empty(rows, cfg.vocab, dtype=torch.bfloat16, device=x_rows.device)
                  if want_logits else None)
        ops.gemm_ex(x_rows, self.w.lm_head, logits, kind=L.EPI_ARGMAX, ssq_in=ssq_rows, rms_dim=self.hidden,
                    rms_eps=cfg.eps, argmax_keys=keys, argmax_col_offset=self.rank * cfg.vocab,
                    workspace=self.gemm_ws, stream=stream)
        if self.world > 1:
            import contextlib
            ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
            with ctx:   # the key and logits exchange run on the kernels' stream
                # keys are order-preserving unsigned (value, ~column) pairs: as int64 they compare like
                # the unsigned keys only when the top bit agrees, so reduce the bit-flipped signed view
                flipped = keys ^ torch.iinfo(torch.int64).min
                dist.all_reduce(flipped, op=dist.ReduceOp.MAX, group=self.group)
                keys.copy_(flipped ^ torch.iinfo(torch.int64).min)
                if want_logits:
                    parts = [torch.empty_like(logits) for _ in range(self.world)]
                    dist.all_gather(parts, logits, group=self.group)
                    logits = torch.cat(parts, dim=1)
        if keys_out is not None:
            return (keys_out, logits) if want_logits else keys_out
        ids = ops.keys_to_ids(keys)
        return (ids, logits) if want_logits else ids

    def decode(self, tokens, positions, slots, table, ctx, stream=None, want_logits=False, keys_out=None):
        """One decode step of this rank: per layer two chained launches around
        the two all-reduces -- [QKV (RoPE + KV append) -> paged attention ->
        O partials] and [gate/up -> down partials] -- each partial written
        straight into the buffer the all-reduce then reduces in place; the
        RMSNorm statistics of the reduced residual come from one row_ssq."""
        if not self.use_chain or not self._attn_fusable() or tokens.shape[0] > 64:
            return self._decode_unchained(tokens, positions, slots, table, ctx, stream, want_logits, keys_out)
        cfg, w, pool = self.cfg, self.w, self.pool
        B = tokens.shape[0]
        dev = tokens.device
        d, eps = self.hidden, cfg.eps
        qd = cfg.num_q_heads * cfg.head_dim
        x, ssq = self._embed(tokens, stream)
        q = torch.empty(B, qd, dtype=torch.bfloat16, device=dev)
        att = torch.empty(B, qd, dtype=torch.bfloat16, device=dev)
        h = torch.empty(B, cfg.ffn, dtype=torch.bfloat16, device=dev)
        pair = self._residual_pair(B, dev)
        ws = self.gemm_ws
        cs = ops.rope_table(positions, cfg.head_dim, cfg.rope_theta, stream=stream)
        lead = self.rank == 0
        for li, lw in enumerate(w.layers):
            part = pair[1] if x is pair[0] else pair[0]
            ops.gemm_chain([
                dict(a=x, w=lw["wqkv"], out=q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=d, rms_eps=eps,
                     pool=pool.data, geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads, positions=positions,
                     slots=slots, rope_theta=cfg.rope_theta, rope_table=cs),
                dict(a=att, w=lw["wo"], out=part, kind=L.EPI_RESIDUAL if lead else L.EPI_NONE,
                     residual=x if lead else None),
            ], ws, stream=stream, attn=[dict(pool=pool.data, geo=pool.geo, layer=li, num_q_heads=cfg.num_q_heads,
                                             q=q, q_stride=qd, table=table, ctx=ctx, scale=self.scale, out=att,
                                             before=1)])
            x = self._allreduce(part, stream=stream)
            ssq_mid = ops.row_ssq(x, stream=stream)
            part = pair[1] if x is pair[0] else pair[0]
            ops.gemm_chain([
                dict(a=x, w=lw["wgu"], out=h, kind=L.EPI_SILU, ssq_in=ssq_mid, rms_dim=d, rms_eps=eps),
                dict(a=h, w=lw["wdown"], out=part, kind=L.EPI_RESIDUAL if lead else L.EPI_NONE,
                     residual=x if lead else None),
            ], ws, stream=stream)
            x = self._allreduce(part, stream=stream)
            ssq = ops.row_ssq(x, stream=stream)
        return self._sample(x, ssq, stream, want_logits, keys_out)
