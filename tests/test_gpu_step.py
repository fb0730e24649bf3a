"""The decode step as one persistent kernel (astraea_step_launch): logits
against the fp32 oracle and the per-layer launch path, bit-identical KV
appends, retired rows, contexts long enough to split attention across
warps, repeated launches (epoch flags) and several batch widths."""

import pytest
import torch

from conftest import cuda_available
from oracle import llama_ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a B200")]

from paper_2512_14142_b200.gpu.datapath import KvPool  # noqa: E402
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaConfig, LlamaRunner, LlamaWeights  # noqa: E402
from paper_2512_14142_b200.tokens import segment_token_ids  # noqa: E402

DEV = "cuda"
# head_dim 128 with 4 q heads per kv head (the Llama-3-8B attention shape) at
# a size the CPU oracle runs in seconds
D128 = LlamaConfig("d128", 2, 512, 4, 1, 128, 512, 1000)
CFGS = dict(PRESETS, d128=D128)


def d(v):
    return torch.tensor(v, dtype=torch.int32, device=DEV)


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return float((a - b).norm() / b.norm())


def _check_kv(pool, kv_ref, cfg):
    """Layer 0's appended K/V comes from the same tcgen05 projection in both
    paths (only the order of the split-K partial sums differs); deeper layers
    also inherit the attention's different summation order."""
    nb = pool.num_blocks
    a = pool.data.view(nb, cfg.num_layers, -1)
    b = kv_ref.view(nb, cfg.num_layers, -1)
    assert rel(a[:, 0], b[:, 0]) < 2e-3, "layer-0 KV appended by the step kernel differs"
    assert rel(a, b) < 1e-2


def _setup(cfg, w, lens, retired=()):
    """Prefill every row's prompt into its own blocks; returns runner-independent
    decode inputs and the per-row histories."""
    pool = KvPool(cfg, sum((n + 17) // 16 + 1 for n in lens) + 8)
    runner = LlamaRunner(w, pool)
    runner.use_step_kernel = False
    nb = max((n + 17) // 16 for n in lens)
    table, seqs, nxt, nxt_blk = [], [], [], 0
    for b, n in enumerate(lens):
        blocks = list(range(nxt_blk, nxt_blk + (n + 17) // 16))
        nxt_blk += len(blocks)
        ids = segment_token_ids(f"s{b}", 1, n, cfg.vocab)
        pos = list(range(n))
        slots = [blocks[p // 16] * 16 + p % 16 for p in pos]
        tok = runner.prefill(d(ids), d(pos), d(slots), d([0, n]), d([blocks]).view(1, -1), d([n]),
                             torch.tensor([n - 1], device=DEV), n)
        seqs.append(ids + [int(tok[0])])
        table.append(blocks + [-1] * (nb - len(blocks)))
        nxt.append(int(tok[0]))
    torch.cuda.synchronize()
    B = len(lens)
    toks = d(nxt)
    posv = [len(s) - 1 for s in seqs]
    slots = [table[b][p // 16] * 16 + p % 16 for b, p in enumerate(posv)]
    ctx = [p + 1 for p in posv]
    for b in retired:
        slots[b], ctx[b] = -1, 0
    return pool, runner, dict(tokens=toks, positions=d(posv), slots=d(slots), table=d(table), ctx=d(ctx)), seqs


@pytest.mark.parametrize("model,lens,retired", [
    ("tiny", [33], ()),
    ("d128", [900], ()),
    ("d128", [3, 700, 64, 1500, 129], (3,)),
    ("small", [5, 300, 17, 64, 900], (2,)),
    ("small", [40 + 13 * i for i in range(23)], (0, 7)),
    ("tiny", [200 + 9 * i for i in range(48)], ()),
])
def test_step_kernel_logits_match_oracle_and_launch_path(model, lens, retired):
    cfg = CFGS[model]
    w = LlamaWeights(cfg, seed=5)
    wc = w.to_cpu_dict()
    pool, runner, inp, seqs = _setup(cfg, w, lens, retired)
    base = pool.data.clone()
    # per-layer launch path
    ids_ref, lg_ref = runner.decode(**inp, want_logits=True)
    torch.cuda.synchronize()
    kv_ref = pool.data.clone()
    pool.data.copy_(base)
    runner.use_step_kernel = True
    ids, lg = runner.decode(**inp, want_logits=True)
    torch.cuda.synchronize()
    _check_kv(pool, kv_ref, cfg)
    live = [b for b in range(len(lens)) if b not in retired]
    for b in live:
        assert rel(lg[b], lg_ref[b]) < 1e-2, b
    for b in live[:3] if model != "tiny" else live[:1]:
        ref = llama_ref.forward(wc, cfg, seqs[b])[-1]
        assert rel(lg[b], ref) < 1e-2, b
        assert int(ids[b]) == int(lg[b].float().argmax())


def test_step_kernel_repeated_launches_are_deterministic():
    """Same inputs, many launches (the epoch advances each time): identical
    tokens and logits every time, and the same as a fresh runner."""
    cfg = PRESETS["small"]
    w = LlamaWeights(cfg, seed=6)
    pool, runner, inp, _ = _setup(cfg, w, [100, 250, 7, 31])
    runner.use_step_kernel = True
    base = pool.data.clone()
    outs = []
    for _ in range(5):
        pool.data.copy_(base)
        ids, lg = runner.decode(**inp, want_logits=True)
        torch.cuda.synchronize()
        outs.append((ids.cpu(), lg.cpu()))
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1])


def test_step_kernel_multi_step_greedy_matches_oracle():
    cfg = PRESETS["tiny"]
    w = LlamaWeights(cfg, seed=7)
    wc = w.to_cpu_dict()
    lens = [20, 47]
    pool, runner, inp, seqs = _setup(cfg, w, lens)
    runner.use_step_kernel = True
    table = inp["table"].cpu().tolist()
    for step in range(6):
        ids = runner.decode(**inp).cpu().tolist()
        for b in range(len(lens)):
            ref = llama_ref.forward(wc, cfg, seqs[b])[-1]
            assert ids[b] == int(ref.argmax()), (step, b)
            seqs[b].append(ids[b])
        posv = [len(s) - 1 for s in seqs]
        inp = dict(tokens=d(ids), positions=d(posv), table=inp["table"],
                   slots=d([table[b][p // 16] * 16 + p % 16 for b, p in enumerate(posv)]),
                   ctx=d([p + 1 for p in posv]))


@pytest.mark.parametrize("B", [1, 3, 20, 64])
def test_step_kernel_llama3_8b_matches_launch_path(B):
    """Llama-3-8B shape (no CPU oracle at this size): the step kernel against
    the per-layer launch path. Layer 0's KV is checked tightly (_check_kv);
    after 32 random-init layers the different attention summation order is
    amplified, so logits are held to 5e-2 here -- the 1e-2 oracle bar is
    asserted above on the same head_dim-128 / 4-heads-per-kv-head attention
    (config d128) -- and the greedy token must agree wherever the top-2
    logit margin exceeds the measured difference."""
    cfg = PRESETS["llama3-8b"]
    w = _w8b()
    lens = [(97 * b + 300) % 1100 + 1 for b in range(B)]
    pool, runner, inp, _ = _setup(cfg, w, lens, retired=(1,) if B > 2 else ())
    base = pool.data.clone()
    ids_ref, lg_ref = runner.decode(**inp, want_logits=True)
    torch.cuda.synchronize()
    kv_ref = pool.data.clone()
    pool.data.copy_(base)
    runner.use_step_kernel = True
    ids, lg = runner.decode(**inp, want_logits=True)
    torch.cuda.synchronize()
    _check_kv(pool, kv_ref, cfg)
    for b in range(B):
        if B > 2 and b == 1:
            continue
        assert rel(lg[b], lg_ref[b]) < 5e-2, b
        top = lg_ref[b].float().topk(2).values
        if float(top[0] - top[1]) > 2 * float((lg[b].float() - lg_ref[b].float()).abs().max()):
            assert int(ids[b]) == int(ids_ref[b]), b


_W8B = {}


def _w8b():
    if "w" not in _W8B:
        _W8B["w"] = LlamaWeights(PRESETS["llama3-8b"], seed=0)
    return _W8B["w"]
