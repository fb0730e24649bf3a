"""fp32 CPU restatement of the Llama-3 decoder the data path runs (test oracle).

Pinned to transformers' LlamaForCausalLM (tests/test_oracle_pin.py); the
reference itself has no model (see oracle/__init__). This is
the textbook Llama-3 block -- RMSNorm, RoPE (NeoX half split, theta
500000), grouped-query attention, SwiGLU MLP -- over a contiguous causal
sequence, i.e. *without* paging, so the device's paged KV, block tables,
swap and recompute are all checked against a layout-free computation.

``bf16_points=True`` rounds tensors to bf16 at the points where the device
materialises bf16 (projection outputs, RoPE outputs, SiLU, the residual
stream; the normalised activations are never materialised on the device --
the norm is applied to the fp32 accumulators -- so they are not rounded
here either), which removes the storage-precision part of the difference
and leaves accumulation order.
"""

import torch


def _r(x, on):
    return x.bfloat16().float() if on else x


def rmsnorm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def rope(x, positions, theta):
    D = x.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, D, 2, dtype=torch.float32, device=x.device) / D))
    ang = positions.float().unsqueeze(1) * inv.unsqueeze(0)
    cos, sin = ang.cos().unsqueeze(1), ang.sin().unsqueeze(1)
    x1, x2 = x[..., : D // 2], x[..., D // 2:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def forward(w, cfg, ids, bf16_points=True, last_only=False):
    """Logits [T, vocab] (fp32) for one sequence of token ids starting at position 0
    (``last_only``: [1, vocab], the last position's). Runs on the device the
    weights ``w`` live on (CPU for the unit tests; the 8B-shape GPU tests keep
    the same fp32 arithmetic on the GPU with TF32 off)."""
    T = len(ids)
    Hq, Hkv, D = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
    G = Hq // Hkv
    r = lambda t: _r(t, bf16_points)  # noqa: E731
    dev = w["embed"].device
    pos = torch.arange(T, device=dev)
    x = w["embed"][torch.as_tensor(ids, dtype=torch.long, device=dev)].float()
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=dev), 1)
    for lw in w["layers"]:
        h = rmsnorm(x, lw["attn_norm"].float(), cfg.eps)
        qkv = r(h @ lw["wqkv"].float().T)
        q = qkv[:, : Hq * D].view(T, Hq, D)
        k = qkv[:, Hq * D: (Hq + Hkv) * D].view(T, Hkv, D)
        v = qkv[:, (Hq + Hkv) * D:].view(T, Hkv, D)
        q = r(rope(q, pos, cfg.rope_theta))
        k = r(rope(k, pos, cfg.rope_theta))
        kk = k.repeat_interleave(G, dim=1)
        vv = v.repeat_interleave(G, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, kk) / (D ** 0.5)
        s = s.masked_fill(mask.unsqueeze(0), float("-inf"))
        a = r(torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), vv).reshape(T, Hq * D))
        x = r(a @ lw["wo"].float().T + x)
        h = rmsnorm(x, lw["mlp_norm"].float(), cfg.eps)
        gu = r(h @ lw["wgu"].float().T)
        g, u = gu[:, : cfg.ffn], gu[:, cfg.ffn:]
        m = r(r(torch.nn.functional.silu(g)) * u)
        x = r(m @ lw["wdown"].float().T + x)
    if last_only:
        x = x[-1:]
    h = rmsnorm(x, w["final_norm"].float(), cfg.eps)
    return h @ w["lm_head"].float().T


def greedy_continue(w, cfg, ids, n_steps, bf16_points=True):
    """Greedy decode n_steps tokens after ``ids`` (full recompute each step)."""
    seq = list(ids)
    out = []
    for _ in range(n_steps):
        nxt = int(forward(w, cfg, seq, bf16_points)[-1].argmax())
        out.append(nxt)
        seq.append(nxt)
    return out


def forward_tp(w, cfg, ids, rank, world, all_reduce, all_gather, bf16_points=True):
    """Tensor-parallel restatement (paper_2512_14142_b200.gpu.tp): `w` is this
    rank's shard (tp.shard_logical) of a model with full config `cfg`. The O
    and down projections produce partial sums (rank 0 adds the residual) that
    are all-reduced; the lm_head logits slices are all-gathered. Returns the
    full logits [T, vocab] on every rank."""
    T = len(ids)
    Hq, Hkv, D = cfg.num_q_heads // world, cfg.num_kv_heads // world, cfg.head_dim
    G = Hq // Hkv
    r = lambda t: _r(t, bf16_points)  # noqa: E731
    pos = torch.arange(T)
    x = w["embed"][torch.as_tensor(ids, dtype=torch.long)].float()
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool), 1)
    for lw in w["layers"]:
        h = rmsnorm(x, lw["attn_norm"].float(), cfg.eps)
        qkv = r(h @ lw["wqkv"].float().T)
        q = qkv[:, : Hq * D].view(T, Hq, D)
        k = qkv[:, Hq * D: (Hq + Hkv) * D].view(T, Hkv, D)
        v = qkv[:, (Hq + Hkv) * D:].view(T, Hkv, D)
        q = r(rope(q, pos, cfg.rope_theta))
        k = r(rope(k, pos, cfg.rope_theta))
        s = torch.einsum("qhd,khd->hqk", q, k.repeat_interleave(G, dim=1)) / (D ** 0.5)
        s = s.masked_fill(mask.unsqueeze(0), float("-inf"))
        a = r(torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v.repeat_interleave(G, dim=1)).reshape(T, Hq * D))
        part = r(a @ lw["wo"].float().T + (x if rank == 0 else 0.0))
        all_reduce(part)
        x = r(part)
        h = rmsnorm(x, lw["mlp_norm"].float(), cfg.eps)
        gu = r(h @ lw["wgu"].float().T)
        f = gu.shape[1] // 2
        m = r(r(torch.nn.functional.silu(gu[:, :f])) * gu[:, f:])
        part = r(m @ lw["wdown"].float().T + (x if rank == 0 else 0.0))
        all_reduce(part)
        x = r(part)
    h = rmsnorm(x, w["final_norm"].float(), cfg.eps)
    local = (h @ w["lm_head"].float().T).contiguous()
    parts = [torch.empty_like(local) for _ in range(world)]
    all_gather(parts, local)
    return torch.cat(parts, dim=1)
