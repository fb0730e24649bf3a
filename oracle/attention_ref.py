"""fp32 CPU restatement of paged decode / prefill attention (test oracle).

Pinned to transformers' Llama attention through its cached K/V
(tests/test_oracle_pin.py); the reference has no model (oracle/__init__).
Follows the standard scaled-dot-product attention with GQA and causal
masking on absolute positions, reading K/V through the same block table the
CUDA kernels read.
"""

import torch


def _pool5(pool, L, Hkv, D, BS=16):
    return pool.float().reshape(-1, L, 2, Hkv, BS, D)


def gather(pool, table_row, ctx, layer, L, Hkv, D, BS=16):
    pv = _pool5(pool, L, Hkv, D, BS)
    nb = (ctx + BS - 1) // BS
    ids = [int(x) for x in table_row[:nb]]
    pages = pv[ids, layer]                                   # [nb, 2, Hkv, BS, D]
    k = pages[:, 0].permute(0, 2, 1, 3).reshape(-1, Hkv, D)[:ctx]
    v = pages[:, 1].permute(0, 2, 1, 3).reshape(-1, Hkv, D)[:ctx]
    return k, v


def decode_ref(pool, layer, q, table, ctx, scale, L, Hkv, D, BS=16):
    """q [B, Hq, D] -> out [B, Hq, D] (fp32)."""
    B, Hq, _ = q.shape
    G = Hq // Hkv
    out = torch.zeros(B, Hq, D, dtype=torch.float32)
    for b in range(B):
        c = int(ctx[b])
        if c == 0:
            continue
        k, v = gather(pool, table[b], c, layer, L, Hkv, D, BS)
        kk = k.repeat_interleave(G, dim=1)                   # [c, Hq, D]
        vv = v.repeat_interleave(G, dim=1)
        s = torch.einsum("hd,thd->ht", q[b].float(), kk) * scale
        p = torch.softmax(s, dim=-1)
        out[b] = torch.einsum("ht,thd->hd", p, vv)
    return out


def prefill_ref(pool, layer, q, cu_q, table, ctx, scale, L, Hkv, D, BS=16):
    """q [T, Hq, D] (rows of sequence s at positions ctx[s]-len_s ..) -> [T, Hq, D]."""
    T, Hq, _ = q.shape
    G = Hq // Hkv
    out = torch.zeros(T, Hq, D, dtype=torch.float32)
    for s in range(len(ctx)):
        a, b = int(cu_q[s]), int(cu_q[s + 1])
        n = b - a
        if n == 0:
            continue
        c = int(ctx[s])
        k, v = gather(pool, table[s], c, layer, L, Hkv, D, BS)
        kk = k.repeat_interleave(G, dim=1)
        vv = v.repeat_interleave(G, dim=1)
        sc = torch.einsum("qhd,thd->hqt", q[a:b].float(), kk) * scale
        pos = torch.arange(c - n, c).unsqueeze(1)
        mask = torch.arange(c).unsqueeze(0) > pos            # [n, c]
        sc = sc.masked_fill(mask.unsqueeze(0), float("-inf"))
        p = torch.softmax(sc, dim=-1)
        out[a:b] = torch.einsum("hqt,thd->qhd", p, vv)
    return out


def rope_ref(x, positions, theta):
    """NeoX half-split RoPE in fp32, x [T, H, D]."""
    D = x.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, D, 2, dtype=torch.float32) / D))
    ang = positions.float().unsqueeze(1) * inv.unsqueeze(0)  # [T, D/2]
    cos, sin = ang.cos().unsqueeze(1), ang.sin().unsqueeze(1)
    x1, x2 = x[..., : D // 2].float(), x[..., D // 2:].float()
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)
