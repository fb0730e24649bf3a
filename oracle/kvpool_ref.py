"""numpy restatement of the paged KV pool's byte movement (test oracle).

Layout contract (include/astraea_b200.h):
  pool[num_blocks][L][2][Hkv][BS][D]  (bf16, handled here as uint16)
  slot[L][2][Hkv][n_tokens][D]         token-compact host slot
Reference seams: swap delay kvcache.py:136-137, transitions kvcache.py:230-258.
"""

import numpy as np


def pool_view(pool_u16: np.ndarray, L, Hkv, D, BS=16) -> np.ndarray:
    return pool_u16.reshape(-1, L, 2, Hkv, BS, D)


def swap_out_ref(pool_u16, block_ids, n_tokens, L, Hkv, D, BS=16) -> np.ndarray:
    """Gather the first n_tokens of the request's blocks into a compact slot."""
    pv = pool_view(pool_u16, L, Hkv, D, BS)
    pages = pv[np.asarray(block_ids)]                       # [nb, L, 2, Hkv, BS, D]
    seq = np.moveaxis(pages, 0, 3).reshape(L, 2, Hkv, len(block_ids) * BS, D)
    return np.ascontiguousarray(seq[:, :, :, :n_tokens, :])


def swap_in_ref(pool_u16, block_ids, n_tokens, slot, L, Hkv, D, BS=16) -> np.ndarray:
    """Scatter a compact slot back into (possibly different) blocks; returns a new pool."""
    out = pool_u16.copy()
    pv = pool_view(out, L, Hkv, D, BS)
    for i, b in enumerate(block_ids):
        t0 = i * BS
        t1 = min(n_tokens, t0 + BS)
        pv[b, :, :, :, : t1 - t0, :] = slot[:, :, :, t0:t1, :]
    return out


def table_build_ref(csr_ptr, csr_ids, rows, ctx_src, max_blocks):
    B = len(rows)
    table = np.full((B, max_blocks), -1, dtype=np.int32)
    ctx = np.zeros(B, dtype=np.int32)
    for b, r in enumerate(rows):
        ids = csr_ids[csr_ptr[r]:csr_ptr[r + 1]]
        table[b, : len(ids)] = ids
        ctx[b] = ctx_src[r]
    return table, ctx


def slot_of(block_list, pos, BS=16) -> int:
    return block_list[pos // BS] * BS + pos % BS


def gather_kv(pool_f32, block_list, n_tokens, layer, Hkv, D, BS=16):
    """K, V [n_tokens, Hkv, D] of one request from a float pool view."""
    pv = pool_f32.reshape(-1, pool_f32.shape[1], 2, Hkv, BS, D)
    pages = pv[list(block_list), layer]                     # [nb, 2, Hkv, BS, D]
    k = pages[:, 0].transpose(0, 2, 1, 3).reshape(-1, Hkv, D)[:n_tokens]
    v = pages[:, 1].transpose(0, 2, 1, 3).reshape(-1, Hkv, D)[:n_tokens]
    return k, v
