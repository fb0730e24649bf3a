"""Oracle self-checks on CPU (the oracle is the checker, so pin it first)."""

import numpy as np
import pytest
import torch

from oracle import attention_ref, kvpool_ref, llama_ref
from paper_2512_14142_b200.gpu.model import PRESETS


def _pool(nb, L, Hkv, D, seed=0):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 65535, size=nb * L * 2 * Hkv * 16 * D, dtype=np.uint16)


@pytest.mark.parametrize("n_tokens", [1, 15, 16, 17, 100, 257])
def test_swap_round_trip_is_identity_on_valid_tokens(n_tokens):
    L, Hkv, D = 3, 2, 64
    pool = _pool(64, L, Hkv, D)
    nb = (n_tokens + 15) // 16
    src = [5, 9, 2, 40, 33, 11, 60, 1, 17, 23, 8, 50, 30, 31, 32, 3, 4][:nb]
    slot = kvpool_ref.swap_out_ref(pool, src, n_tokens, L, Hkv, D)
    assert slot.shape == (L, 2, Hkv, n_tokens, D)
    dst = [i for i in range(64) if i not in src][:nb]
    pool2 = kvpool_ref.swap_in_ref(pool, dst, n_tokens, slot, L, Hkv, D)
    assert np.array_equal(kvpool_ref.swap_out_ref(pool2, dst, n_tokens, L, Hkv, D), slot)
    # blocks outside dst untouched
    pv, pv2 = kvpool_ref.pool_view(pool, L, Hkv, D), kvpool_ref.pool_view(pool2, L, Hkv, D)
    others = [i for i in range(64) if i not in dst]
    assert np.array_equal(pv[others], pv2[others])


def test_slot_bytes_are_exactly_algorithmic():
    L, Hkv, D = 32, 8, 128
    assert L * 2 * Hkv * D * 2 == 131072


def test_table_build_ref():
    ptr = [0, 2, 5, 5]
    ids = [7, 8, 1, 2, 3]
    t, c = kvpool_ref.table_build_ref(ptr, ids, [2, 0, 1], [10, 20, 30], 4)
    assert t.tolist() == [[-1] * 4, [7, 8, -1, -1], [1, 2, 3, -1]]
    assert c.tolist() == [30, 10, 20]


def test_decode_ref_matches_dense_softmax():
    torch.manual_seed(0)
    L, Hkv, D, Hq = 2, 2, 64, 8
    nb = 8
    pool = torch.randn(nb * L * 2 * Hkv * 16 * D)
    table = torch.tensor([[3, 5, 1, -1]])
    q = torch.randn(1, Hq, D)
    out = attention_ref.decode_ref(pool, 1, q, table, [40], 0.125, L, Hkv, D)
    k, v = attention_ref.gather(pool, table[0], 40, 1, L, Hkv, D)
    h = 5
    s = (q[0, h] @ k[:, h // 4].T) * 0.125
    assert torch.allclose(out[0, h], torch.softmax(s, 0) @ v[:, h // 4], atol=1e-5)


def test_prefill_ref_last_row_equals_decode_ref():
    torch.manual_seed(1)
    L, Hkv, D, Hq = 1, 2, 64, 4
    pool = torch.randn(6 * L * 2 * Hkv * 16 * D)
    table = torch.tensor([[0, 4, 2, -1]])
    q = torch.randn(5, Hq, D)
    pre = attention_ref.prefill_ref(pool, 0, q, [0, 5], table, [37], 0.1, L, Hkv, D)
    dec = attention_ref.decode_ref(pool, 0, q[-1:], table, [37], 0.1, L, Hkv, D)
    assert torch.allclose(pre[-1], dec[0], atol=1e-5)


def test_rope_is_a_rotation():
    x = torch.randn(7, 3, 64)
    y = attention_ref.rope_ref(x, torch.arange(7) * 100, 500000.0)
    assert torch.allclose(x.norm(dim=-1), y.norm(dim=-1), atol=1e-4)
    assert torch.allclose(attention_ref.rope_ref(x, torch.zeros(7), 500000.0), x)


def test_llama_ref_is_causal_and_deterministic():
    cfg = PRESETS["tiny"]
    g = torch.Generator().manual_seed(0)
    d = cfg.hidden
    rnd = lambda *s: (torch.randn(*s, generator=g) * 0.02).bfloat16()  # noqa: E731
    w = {"embed": rnd(cfg.vocab, d), "final_norm": torch.ones(d).bfloat16(), "lm_head": rnd(cfg.vocab, d),
         "layers": [{"attn_norm": torch.ones(d).bfloat16(), "wqkv": rnd(cfg.qkv_dim, d),
                     "wo": rnd(d, cfg.num_q_heads * cfg.head_dim), "mlp_norm": torch.ones(d).bfloat16(),
                     "wgu": rnd(2 * cfg.ffn, d), "wdown": rnd(d, cfg.ffn)} for _ in range(cfg.num_layers)]}
    ids = [3, 17, 200, 999, 5, 6]
    full = llama_ref.forward(w, cfg, ids)
    pre = llama_ref.forward(w, cfg, ids[:4])
    assert torch.allclose(full[:4], pre, atol=1e-5)  # later tokens do not change earlier logits
    assert llama_ref.greedy_continue(w, cfg, ids, 3) == llama_ref.greedy_continue(w, cfg, ids, 3)
