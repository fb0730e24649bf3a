"""Pin the numerics oracle to a published implementation.

The reference has no model, so ``oracle/llama_ref.py``
restates Llama-3. Here it is checked against Hugging Face transformers'
``LlamaForCausalLM`` (the image's transformers 5.5.0, fp32, CPU) on the same
weights: Llama-3's rope_theta 500000, GQA, SwiGLU, RMSNorm with non-unit
weights, untied lm_head. ``bf16_points=False`` makes the oracle pure fp32, so
the two must agree to fp32 rounding. The paged-attention oracle
(``attention_ref``) is pinned to the same model through its decode of the
HF prefix's cached K/V, and the tensor-parallel restatement to the dense one.
"""

import pytest
import torch

from oracle import attention_ref, llama_ref
from paper_2512_14142_b200.gpu.model import LlamaConfig, PRESETS

transformers = pytest.importorskip("transformers")

CONFIGS = [
    LlamaConfig("pin-gqa4", 2, 256, 8, 2, 32, 512, 1000),           # GQA 4:1 like Llama-3-8B (32:8)
    LlamaConfig("pin-8b-heads", 1, 512, 32, 8, 16, 768, 512),        # Llama-3-8B head counts, narrow heads
    LlamaConfig("pin-d128", 1, 512, 4, 1, 128, 1024, 700),           # D=128 as in 8B/70B, 70B/TP8 head split
]


def _weights(cfg, seed):
    g = torch.Generator().manual_seed(seed)
    d, qd = cfg.hidden, cfg.num_q_heads * cfg.head_dim
    r = lambda *s, sc=0.05: torch.randn(*s, generator=g) * sc  # noqa: E731
    layers = [{"attn_norm": 1 + r(d, sc=0.2), "mlp_norm": 1 + r(d, sc=0.2), "wqkv": r(cfg.qkv_dim, d),
               "wo": r(d, qd), "wgu": r(2 * cfg.ffn, d), "wdown": r(d, cfg.ffn)} for _ in range(cfg.num_layers)]
    return {"embed": r(cfg.vocab, d, sc=1.0), "layers": layers, "final_norm": 1 + r(d, sc=0.2),
            "lm_head": r(cfg.vocab, d)}


def _hf(cfg, w):
    from transformers import LlamaConfig as HfConfig
    from transformers import LlamaForCausalLM
    hc = HfConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
                  num_hidden_layers=cfg.num_layers, num_attention_heads=cfg.num_q_heads,
                  num_key_value_heads=cfg.num_kv_heads, head_dim=cfg.head_dim, rope_theta=cfg.rope_theta,
                  rms_norm_eps=cfg.eps, tie_word_embeddings=False, max_position_embeddings=8192,
                  attention_bias=False, mlp_bias=False)
    hc._attn_implementation = "eager"
    m = LlamaForCausalLM(hc).float().eval()
    Hq, Hkv, D, F = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.ffn
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"], "lm_head.weight": w["lm_head"]}
    for i, lw in enumerate(w["layers"]):
        p = f"model.layers.{i}."
        sd[p + "self_attn.q_proj.weight"] = lw["wqkv"][: Hq * D]
        sd[p + "self_attn.k_proj.weight"] = lw["wqkv"][Hq * D: (Hq + Hkv) * D]
        sd[p + "self_attn.v_proj.weight"] = lw["wqkv"][(Hq + Hkv) * D:]
        sd[p + "self_attn.o_proj.weight"] = lw["wo"]
        sd[p + "mlp.gate_proj.weight"] = lw["wgu"][:F]
        sd[p + "mlp.up_proj.weight"] = lw["wgu"][F:]
        sd[p + "mlp.down_proj.weight"] = lw["wdown"]
        sd[p + "input_layernorm.weight"] = lw["attn_norm"]
        sd[p + "post_attention_layernorm.weight"] = lw["mlp_norm"]
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    return m


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: c.name)
def test_llama_ref_matches_transformers(cfg):
    w = _weights(cfg, 1)
    m = _hf(cfg, w)
    ids = torch.randint(0, cfg.vocab, (57,), generator=torch.Generator().manual_seed(2)).tolist()
    with torch.no_grad():
        want = m(torch.tensor([ids])).logits[0]
    got = llama_ref.forward(w, cfg, ids, bf16_points=False)
    err = float((got - want).norm() / want.norm())
    assert err < 1e-5, err
    assert torch.equal(got.argmax(-1), want.argmax(-1))


def test_greedy_continuation_matches_transformers():
    cfg = CONFIGS[0]
    w = _weights(cfg, 3)
    m = _hf(cfg, w)
    ids = torch.randint(0, cfg.vocab, (20,), generator=torch.Generator().manual_seed(4)).tolist()
    with torch.no_grad():
        hf = m.generate(torch.tensor([ids]), max_new_tokens=12, do_sample=False, min_new_tokens=12)[0, 20:].tolist()
    assert llama_ref.greedy_continue(w, cfg, ids, 12, bf16_points=False) == hf


def test_paged_decode_oracle_matches_transformers_kv():
    """attention_ref.decode_ref over a paged pool holding HF's cached K/V (in
    scattered blocks) reproduces HF's attention output for the next token."""
    cfg = CONFIGS[0]
    w = _weights(cfg, 5)
    m = _hf(cfg, w)
    T = 37
    ids = torch.randint(0, cfg.vocab, (T + 1,), generator=torch.Generator().manual_seed(6))
    with torch.no_grad():
        out = m(ids[None, :T], use_cache=True)
        cache = out.past_key_values
    L, Hkv, D, Hq = cfg.num_layers, cfg.num_kv_heads, cfg.head_dim, cfg.num_q_heads
    blocks = [9, 2, 14]                       # non-contiguous pages
    pool = torch.zeros(16, L, 2, Hkv, 16, D)
    for layer in range(L):
        k = cache.layers[layer].keys[0]       # [Hkv, T, D], RoPE applied
        v = cache.layers[layer].values[0]
        for p in range(T):
            pool[blocks[p // 16], layer, 0, :, p % 16] = k[:, p]
            pool[blocks[p // 16], layer, 1, :, p % 16] = v[:, p]
    # the query of the next position through the oracle's own layer-0 math
    lw = w["layers"][0]
    x = w["embed"][ids[T]][None]
    h = llama_ref.rmsnorm(x, lw["attn_norm"], cfg.eps)
    q = (h @ lw["wqkv"].T)[:, : Hq * D].view(1, Hq, D)
    q = llama_ref.rope(q, torch.tensor([T]), cfg.rope_theta)
    # K/V of the new token itself go to slot T
    kv = (h @ lw["wqkv"].T)[:, Hq * D:]
    knew = llama_ref.rope(kv[:, : Hkv * D].view(1, Hkv, D), torch.tensor([T]), cfg.rope_theta)[0]
    pool[blocks[T // 16], 0, 0, :, T % 16] = knew
    pool[blocks[T // 16], 0, 1, :, T % 16] = kv[0, Hkv * D:].view(Hkv, D)
    table = torch.tensor([blocks])
    got = attention_ref.decode_ref(pool.reshape(-1), 0, q, table, [T + 1], D ** -0.5, L, Hkv, D)
    # HF: run the full T+1 sequence and read layer 0's attention output before o_proj
    captured = {}
    hook = m.model.layers[0].self_attn.o_proj.register_forward_hook(
        lambda mod, inp, outp: captured.setdefault("a", inp[0][0, -1]))
    with torch.no_grad():
        m(ids[None, : T + 1])
    hook.remove()
    want = captured["a"].view(Hq, D)
    assert float((got[0] - want).norm() / want.norm()) < 1e-5


def test_tp_restatement_equals_dense():
    """forward_tp over 2 simulated ranks == forward (the TP oracle is pinned
    through the dense one, which is pinned to transformers above)."""
    from paper_2512_14142_b200.gpu import tp
    cfg = CONFIGS[0]
    w = _weights(cfg, 7)
    ids = list(range(3, 30))
    want = llama_ref.forward(w, cfg, ids, bf16_points=False)
    world = 2
    shards = [tp.shard_logical(w, cfg, r, world) for r in range(world)]
    # run the ranks in lockstep: collectives are sums / concatenations
    import threading
    outs, parts = [None] * world, {}
    bar = threading.Barrier(world)

    def run(r):
        def all_reduce(t):
            key = ("ar", run.count[r])
            slot = parts.setdefault(key, [None] * world)
            slot[r] = t.clone()
            bar.wait()
            t.copy_(sum(slot))
            bar.wait()
            run.count[r] += 1

        def all_gather(lst, t):
            slot = parts.setdefault(("ag",), [None] * world)
            slot[r] = t.clone()
            bar.wait()
            for i in range(world):
                lst[i].copy_(slot[i])
            bar.wait()
        outs[r] = llama_ref.forward_tp(shards[r], cfg, ids, r, world, all_reduce, all_gather, bf16_points=False)

    run.count = [0] * world
    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    for o in outs:
        assert float((o - want).norm() / want.norm()) < 1e-5
