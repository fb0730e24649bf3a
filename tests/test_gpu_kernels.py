"""Kernel parity on a B200: every K1-K9 entry point through the C ABI
against the CPU oracle (bit-exact for byte/index work, fp32 reference with
a stated tolerance for floating point)."""

import math

import numpy as np
import pytest
import torch

from conftest import cuda_available
from oracle import attention_ref, kvpool_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a B200")]

from paper_2512_14142_b200.gpu import lib as L  # noqa: E402
from paper_2512_14142_b200.gpu import ops  # noqa: E402

DEV = "cuda"


def rel_err(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def make_pool(nb, Lyr, Hkv, D, seed=0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    pool = torch.randn(nb * Lyr * 2 * Hkv * 16 * D, generator=g, device=DEV).bfloat16()
    return pool, ops.geometry(Lyr, Hkv, D, nb)


# ---------------------------------------------------------------- K1 / K2 swap

@pytest.mark.parametrize("mode", [L.SWAP_KERNEL, L.SWAP_DMA, L.SWAP_STAGED])
@pytest.mark.parametrize("Lyr,Hkv,D,n_tokens", [(4, 2, 64, 1), (4, 2, 64, 17), (4, 2, 64, 300),
                                                (32, 8, 128, 1000), (80, 1, 128, 129)])
def test_swap_out_matches_oracle_and_round_trips_bit_exact(mode, Lyr, Hkv, D, n_tokens):
    nb_total = 160
    pool, geo = make_pool(nb_total, Lyr, Hkv, D, seed=n_tokens)
    nb = (n_tokens + 15) // 16
    rng = np.random.default_rng(n_tokens)
    src = rng.choice(nb_total, nb, replace=False).tolist()
    bpt = Lyr * 2 * Hkv * D * 2
    slot = torch.zeros(n_tokens * bpt, dtype=torch.uint8, pin_memory=True)
    ops.swap_out(geo, pool, src, n_tokens, slot, mode)
    torch.cuda.synchronize()
    pool_np = pool.view(torch.int16).cpu().numpy().view(np.uint16)
    want = kvpool_ref.swap_out_ref(pool_np, src, n_tokens, Lyr, Hkv, D)
    got = slot.numpy().view(np.uint16).reshape(want.shape)
    assert np.array_equal(got, want)
    # scatter into different blocks, gather again: identical bytes
    dst = [b for b in rng.permutation(nb_total).tolist() if b not in src][:nb]
    before = pool.clone()
    ops.swap_in(geo, pool, dst, n_tokens, slot, mode)
    slot2 = torch.zeros(slot.shape, dtype=torch.uint8, pin_memory=True)
    ops.swap_out(geo, pool, dst, n_tokens, slot2, mode)
    torch.cuda.synchronize()
    assert torch.equal(slot, slot2)
    # swap-in wrote only the valid tokens of dst blocks
    want_pool = kvpool_ref.swap_in_ref(before.view(torch.int16).cpu().numpy().view(np.uint16), dst,
                                       n_tokens, want, Lyr, Hkv, D)
    assert np.array_equal(pool.view(torch.int16).cpu().numpy().view(np.uint16), want_pool)


def test_swap_rejects_bad_arguments():
    pool, geo = make_pool(8, 2, 2, 64)
    slot = torch.zeros(100 * 2 * 2 * 2 * 64 * 2, dtype=torch.uint8, pin_memory=True)
    from paper_2512_14142_b200.gpu.lib import DeviceError
    with pytest.raises(DeviceError):
        ops.swap_out(geo, pool, [0, 1], 100, slot)          # 100 tokens need 7 blocks
    with pytest.raises(DeviceError):
        ops.swap_out(geo, pool, [0, 99], 20, slot)          # block id out of range
    with pytest.raises(DeviceError):
        ops.swap_out(geo, pool, [0, 1], 20, torch.zeros(slot.shape, dtype=torch.uint8))  # pageable slot


def test_copy_blocks():
    pool, geo = make_pool(16, 2, 2, 64)
    ref = pool.clone().view(16, -1)
    ops.copy_blocks(geo, pool, [1, 2], [7, 9])
    torch.cuda.synchronize()
    v = pool.view(16, -1)
    assert torch.equal(v[7], ref[1]) and torch.equal(v[9], ref[2]) and torch.equal(v[0], ref[0])


# ---------------------------------------------------------------- K3 table build

def test_block_table_build_matches_oracle():
    ptr = [0, 3, 3, 8, 9]
    ids = [4, 5, 6, 10, 11, 12, 13, 14, 2]
    rows = [3, 0, 2]
    ctx_src = [40, 0, 70, 9]
    d = lambda v: torch.tensor(v, dtype=torch.int32, device=DEV)  # noqa: E731
    table = torch.empty(3, 6, dtype=torch.int32, device=DEV)
    ctx = torch.empty(3, dtype=torch.int32, device=DEV)
    ops.block_table_build(d(ptr), d(ids), d(rows), d(ctx_src), 6, table, ctx)
    t, c = kvpool_ref.table_build_ref(ptr, ids, rows, ctx_src, 6)
    assert table.cpu().numpy().tolist() == t.tolist()
    assert ctx.cpu().numpy().tolist() == c.tolist()


# ---------------------------------------------------------------- K5 rope + append

@pytest.mark.parametrize("Hq,Hkv,D", [(8, 2, 64), (32, 8, 128)])
def test_rope_kv_append(Hq, Hkv, D):
    Lyr, nb, T = 3, 12, 37
    pool, geo = make_pool(nb, Lyr, Hkv, D)
    pool.zero_()
    g = torch.Generator(device=DEV).manual_seed(3)
    qkv = torch.randn(T, (Hq + 2 * Hkv) * D, generator=g, device=DEV).bfloat16()
    orig = qkv.clone()
    positions = torch.arange(100, 100 + T, dtype=torch.int32, device=DEV)
    blocks = [9, 2, 5, 7, 11, 0, 1, 3, 4]
    slots = [blocks[p // 16] * 16 + p % 16 for p in range(100, 100 + T)]
    slots[5] = -1  # skipped row
    ops.rope_kv_append(geo, pool, 1, qkv, Hq, positions, torch.tensor(slots, dtype=torch.int32, device=DEV),
                       500000.0)
    torch.cuda.synchronize()
    q_ref = attention_ref.rope_ref(orig[:, : Hq * D].view(T, Hq, D).float().cpu(), positions.cpu(), 500000.0)
    assert rel_err(qkv[:, : Hq * D].view(T, Hq, D), q_ref) < 4e-3
    k_ref = attention_ref.rope_ref(orig[:, Hq * D:(Hq + Hkv) * D].view(T, Hkv, D).float().cpu(),
                                   positions.cpu(), 500000.0)
    v_ref = orig[:, (Hq + Hkv) * D:].view(T, Hkv, D).cpu()
    p6 = pool.view(nb, Lyr, 2, Hkv, 16, D).cpu()
    for t in range(T):
        if slots[t] < 0:
            continue
        b, o = divmod(slots[t], 16)
        assert torch.equal(p6[b, 1, 1, :, o], v_ref[t])
        assert rel_err(p6[b, 1, 0, :, o], k_ref[t]) < 4e-3
    b, o = divmod(blocks[(100 + 5) // 16] * 16 + (105 % 16), 16)
    assert torch.count_nonzero(p6[b, 1, :, :, o]) == 0


# ---------------------------------------------------------------- K4 decode attention

@pytest.mark.parametrize("Hq,Hkv,D", [(32, 8, 128), (8, 2, 64), (8, 1, 128), (16, 2, 64)])
@pytest.mark.parametrize("ctxs", [[1, 16, 17, 300], [2316, 5, 0, 1000, 64], [8000]])
def test_decode_attention(Hq, Hkv, D, ctxs):
    Lyr = 2
    B = len(ctxs)
    max_blocks = max(1, max((c + 15) // 16 for c in ctxs))
    nb = B * max_blocks + 3
    pool, geo = make_pool(nb, Lyr, Hkv, D, seed=B)
    perm = torch.randperm(nb)[: B * max_blocks].view(B, max_blocks).int()
    table = perm.clone()
    for b, c in enumerate(ctxs):
        table[b, (c + 15) // 16:] = -1
    g = torch.Generator(device=DEV).manual_seed(7)
    stride = (Hq + 2 * Hkv) * D
    qkv = torch.randn(B, stride, generator=g, device=DEV).bfloat16()
    out = torch.empty(B, Hq * D, dtype=torch.bfloat16, device=DEV)
    ws = ops.decode_workspace(B, Hq, D, max_blocks, DEV)
    scale = 1 / math.sqrt(D)
    ctx_d = torch.tensor(ctxs, dtype=torch.int32, device=DEV)
    ops.decode_attention(geo, pool, 1, qkv, stride, B, Hq, table.to(DEV), ctx_d, scale, out, ws)
    torch.cuda.synchronize()
    ref = attention_ref.decode_ref(pool.cpu(), 1, qkv[:, : Hq * D].view(B, Hq, D).cpu(), table, ctxs, scale,
                                   Lyr, Hkv, D)
    got = out.view(B, Hq, D).cpu().float()
    for b, c in enumerate(ctxs):
        if c == 0:
            assert torch.count_nonzero(got[b]) == 0
        else:
            assert rel_err(got[b], ref[b]) < 1e-2, (b, c)


# ---------------------------------------------------------------- K7 prefill attention

@pytest.mark.parametrize("Hq,Hkv,D", [(32, 8, 128), (8, 2, 64), (8, 1, 128), (4, 2, 64)])
@pytest.mark.parametrize("lens_ctx", [[(5, 5)], [(64, 64), (1, 300), (130, 1100)], [(700, 2316)],
                                      [(33, 1000), (17, 17), (100, 2000)], [(2048, 2048)]])
def test_prefill_attention(Hq, Hkv, D, lens_ctx):
    """Varlen paged prefill (tcgen05 kernel; G = 1..8 q heads per kv head as
    the 128 MMA rows) vs the fp32 oracle: fresh prompts, short appends onto
    long resident contexts, a 2048-token causal prompt (16 KV tiles, the
    lazy-rescale path), tiles that end mid-page."""
    Lyr = 2
    S = len(lens_ctx)
    max_blocks = max((c + 15) // 16 for _, c in lens_ctx)
    nb = S * max_blocks + 1
    pool, geo = make_pool(nb, Lyr, Hkv, D, seed=S)
    table = torch.randperm(nb)[: S * max_blocks].view(S, max_blocks).int()
    cu = [0]
    for n, _ in lens_ctx:
        cu.append(cu[-1] + n)
    T = cu[-1]
    stride = (Hq + 2 * Hkv) * D
    g = torch.Generator(device=DEV).manual_seed(11)
    qkv = torch.randn(T, stride, generator=g, device=DEV).bfloat16()
    out = torch.empty(T, Hq * D, dtype=torch.bfloat16, device=DEV)
    ctx = [c for _, c in lens_ctx]
    scale = 1 / math.sqrt(D)
    ops.prefill_attention(geo, pool, 0, qkv, stride, torch.tensor(cu, dtype=torch.int32, device=DEV), S,
                          max(n for n, _ in lens_ctx), Hq, table.to(DEV),
                          torch.tensor(ctx, dtype=torch.int32, device=DEV), scale, out)
    torch.cuda.synchronize()
    ref = attention_ref.prefill_ref(pool.cpu(), 0, qkv[:, : Hq * D].view(T, Hq, D).cpu(), cu, table, ctx, scale,
                                    Lyr, Hkv, D)
    assert rel_err(out.view(T, Hq, D), ref) < 1e-2


# ---------------------------------------------------------------- K6 / K9 GEMM (tcgen05)

@pytest.mark.parametrize("M,N,K", [(1, 4096, 4096), (3, 6144, 4096), (16, 512, 512), (17, 1536, 512),
                                   (32, 28672, 4096), (64, 4096, 14336), (65, 4096, 4096), (128, 256, 64),
                                   (300, 6144, 4096), (513, 1024, 512), (2048, 4096, 4096), (129, 32000, 512),
                                   (7, 128256, 4096), (100, 1000, 512), (90, 4104, 14336), (128, 28672, 4096)])
def test_gemm_matches_fp32(M, N, K):
    g = torch.Generator(device=DEV).manual_seed(M * 7 + N)
    a = (torch.randn(M, K, generator=g, device=DEV)).bfloat16()
    w = (torch.randn(N, K, generator=g, device=DEV) * 0.02).bfloat16()
    ref = a.float() @ w.float().T
    out = ops.gemm(a, w)
    torch.cuda.synchronize()
    assert rel_err(out, ref) < 5e-3


@pytest.mark.parametrize("M", [4, 100, 200])
def test_gemm_residual_in_place(M):
    N, K = 1024, 2048
    g = torch.Generator(device=DEV).manual_seed(5)
    a = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    w = (torch.randn(N, K, generator=g, device=DEV) * 0.02).bfloat16()
    x = torch.randn(M, N, generator=g, device=DEV).bfloat16()
    ref = a.float() @ w.float().T + x.float()
    ops.gemm(a, w, out=x, residual=x)
    torch.cuda.synchronize()
    assert rel_err(x, ref) < 5e-3


def test_gemm_split_k_is_deterministic_and_resets_counters():
    from paper_2512_14142_b200.gpu import lib as L
    need = L.load().astraea_gemm_workspace_bytes(8, 4096, 4096)
    assert need > 0  # this shape uses split-K
    ws = torch.zeros(need // 4 + 1, dtype=torch.float32, device=DEV)
    a = torch.randn(8, 4096, device=DEV).bfloat16()
    w = (torch.randn(4096, 4096, device=DEV) * 0.02).bfloat16()
    outs = [ops.gemm(a, w, workspace=ws) for _ in range(5)]
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    assert torch.count_nonzero(ws[:32]) == 0   # arrival counters (4096/128 = 32 tiles) back to zero


def test_split_k_gemms_of_different_shapes_share_one_workspace():
    """Regression: partials of one shape must not clobber another's counters."""
    from paper_2512_14142_b200.gpu import lib as L
    lib = L.load()
    shapes = [(6144, 4096), (128256, 4096), (4096, 4096), (4096, 14336)]
    need = max(lib.astraea_gemm_workspace_bytes(4, n, k) for n, k in shapes)
    ws = torch.zeros(need // 4 + 1, dtype=torch.float32, device=DEV)
    g = torch.Generator(device=DEV).manual_seed(9)
    for rep in range(2):
        for n, k in shapes:
            a = torch.randn(4, k, generator=g, device=DEV).bfloat16()
            w = (torch.randn(n, k, generator=g, device=DEV) * 0.02).bfloat16()
            out = ops.gemm(a, w, workspace=ws)
            assert rel_err(out, a.float() @ w.float().T) < 5e-3, (rep, n, k)


# ---------------------------------------------------------------- K8 small ops

def test_rmsnorm_silu_embedding_argmax():
    g = torch.Generator(device=DEV).manual_seed(2)
    x = torch.randn(33, 4096, generator=g, device=DEV).bfloat16()
    r = torch.randn(33, 4096, generator=g, device=DEV).bfloat16()
    w = (1 + 0.1 * torch.randn(4096, generator=g, device=DEV)).bfloat16()
    y = torch.empty_like(x)
    ro = torch.empty_like(x)
    ops.rmsnorm(x, w, 1e-5, out=y, residual=r, resid_out=ro)
    s = (x.float() + r.float()).bfloat16().float()
    ref = s * torch.rsqrt(s.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert rel_err(y, ref) < 4e-3
    assert torch.equal(ro, (x.float() + r.float()).bfloat16())
    gu = torch.randn(9, 2 * 1536, generator=g, device=DEV).bfloat16()
    m = ops.silu_mul(gu)
    ref = torch.nn.functional.silu(gu[:, :1536].float()) * gu[:, 1536:].float()
    assert rel_err(m, ref) < 8e-3
    table = torch.randn(1000, 512, generator=g, device=DEV).bfloat16()
    ids = torch.tensor([3, 999, 0, 3], dtype=torch.int32, device=DEV)
    assert torch.equal(ops.embedding(ids, table), table[ids.long()])
    logits = torch.randn(5, 128256, generator=g, device=DEV).bfloat16()
    logits[2, 77] = 100.0
    logits[2, 99] = 100.0  # tie -> lowest index
    am = ops.argmax(logits)
    torch.cuda.synchronize()
    assert am.tolist()[2] == 77
    assert am.tolist() == [int(v) for v in logits.float().argmax(-1).tolist()[:2]] + [77] + \
        [int(v) for v in logits.float().argmax(-1).tolist()[3:]]


def _key(tok):
    # ARGMAX-epilogue key of a token with some positive value (value bits irrelevant here)
    return (0x40000000 << 32) | (0xFFFFFFFF - tok)


def test_decode_advance_drives_rows_and_records_history():
    B = 3
    dev = DEV
    n_gen = torch.tensor([2, 4, 1], dtype=torch.int32, device=dev)
    base = torch.tensor([10, 0, 31], dtype=torch.int32, device=dev)
    first = torch.tensor([7, 8, 9], dtype=torch.int32, device=dev)
    table = torch.tensor([[5, 6, -1], [1, -1, -1], [2, 3, -1]], dtype=torch.int32, device=dev)
    step = torch.zeros(1, dtype=torch.int32, device=dev)
    keys = torch.zeros(B, dtype=torch.int64, device=dev)
    tok, pos, slot, ctx = (torch.empty(B, dtype=torch.int32, device=dev) for _ in range(4))
    hist = torch.zeros(B, 5, dtype=torch.int32, device=dev)
    seen = []
    for s in range(5):
        ops.decode_advance(step, B, n_gen, base, first, keys, table, 16, tok, pos, slot, ctx, hist, 5)
        assert keys.tolist() == [0, 0, 0]            # advance re-zeroes the argmax keys
        seen.append((tok.tolist(), pos.tolist(), slot.tolist(), ctx.tolist()))
        keys.copy_(torch.tensor([_key(t + 100) for t in tok.tolist()], dtype=torch.int64))
    assert seen[0] == ([7, 8, 9], [10, 0, 31], [5 * 16 + 10, 16, 3 * 16 + 15], [11, 1, 32])
    assert seen[1] == ([107, 108, 0], [11, 1, 0], [5 * 16 + 11, 17, -1], [12, 2, 0])
    assert seen[4][2] == [-1, -1, -1]
    h = hist.tolist()
    assert h[0][:3] == [7, 107, 207] and h[2][:2] == [9, 109] and h[1][:5] == [8, 108, 208, 308, 408]


@pytest.mark.parametrize("M", [1, 5, 64, 100])
def test_gemm_argmax_epilogue_matches_torch(M):
    V, K = 32000, 512
    g = torch.Generator(device=DEV).manual_seed(M)
    x = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    w = (torch.randn(V, K, generator=g, device=DEV) * 0.05).bfloat16()
    ssq = _rms_parts(x, K // 128).contiguous()
    keys = torch.zeros(M, dtype=torch.int64, device=DEV)
    logits = torch.empty(M, V, dtype=torch.bfloat16, device=DEV)
    ops.gemm_ex(x, w, logits, kind=L.EPI_ARGMAX, ssq_in=ssq, rms_dim=K, rms_eps=1e-5, argmax_keys=keys)
    torch.cuda.synchronize()
    h = x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-5)
    ref = h @ w.float().T
    ids = ops.keys_to_ids(keys).cpu()
    top2 = ref.topk(2, dim=-1)
    for r in range(M):
        if float(top2.values[r, 0] - top2.values[r, 1]) > 1e-3:   # unambiguous winner
            assert int(ids[r]) == int(top2.indices[r, 0])
    assert rel_err(logits, ref) < 1e-2


# ---------------------------------------------------------------- fused GEMM epilogues

def _rms_parts(x, parts):
    """Per-128-column sums of squares, [parts][M] (what a producer emits)."""
    xf = x.float()
    return torch.stack([xf[:, p * 128:(p + 1) * 128].pow(2).sum(-1) for p in range(parts)])


@pytest.mark.parametrize("M", [3, 17, 64, 100, 200])
def test_gemm_residual_emits_norm_statistics(M):
    N, K = 1024, 512
    g = torch.Generator(device=DEV).manual_seed(M)
    a = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    w = (torch.randn(N, K, generator=g, device=DEV) * 0.05).bfloat16()
    x = torch.randn(M, N, generator=g, device=DEV).bfloat16()
    ref = (a.float() @ w.float().T + x.float()).bfloat16()
    ssq = torch.empty(N // 128, M, dtype=torch.float32, device=DEV)
    ops.gemm_ex(a, w, x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=ssq)
    torch.cuda.synchronize()
    assert rel_err(x, ref) < 5e-3
    assert rel_err(ssq, _rms_parts(x, N // 128)) < 1e-5   # statistics of the stored bf16 output


@pytest.mark.parametrize("M,F", [(1, 1536), (16, 1536), (40, 1536), (100, 1536), (150, 1536), (100, 14336)])
def test_gemm_rms_scaled_silu(M, F):
    K = 512
    g = torch.Generator(device=DEV).manual_seed(7 + M)
    x = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    wgu = (torch.randn(2 * F, K, generator=g, device=DEV) * 0.05).bfloat16()
    from paper_2512_14142_b200.gpu.model import interleave_gate_up
    ssq = _rms_parts(x, K // 128).contiguous()
    out = torch.empty(M, F, dtype=torch.bfloat16, device=DEV)
    ops.gemm_ex(x, interleave_gate_up(wgu, F).contiguous(), out, kind=L.EPI_SILU, ssq_in=ssq, rms_dim=K,
                rms_eps=1e-5)
    torch.cuda.synchronize()
    h = x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-5)
    gu = h @ wgu.float().T
    ref = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    assert rel_err(out, ref) < 1e-2


@pytest.mark.parametrize("M", [2, 33, 100, 130])
@pytest.mark.parametrize("Hq,Hkv,D", [(32, 8, 128), (8, 2, 64)])
def test_gemm_qkv_rope_append(M, Hq, Hkv, D):
    K, Lyr, nb = 512, 2, 40
    pool, geo = make_pool(nb, Lyr, Hkv, D)
    pool.zero_()
    g = torch.Generator(device=DEV).manual_seed(M + D)
    x = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    w = (torch.randn((Hq + 2 * Hkv) * D, K, generator=g, device=DEV) * 0.05).bfloat16()
    positions = torch.arange(50, 50 + M, dtype=torch.int32, device=DEV)
    blocks = list(range(nb))[::-1]
    slots = torch.tensor([blocks[p // 16] * 16 + p % 16 for p in range(50, 50 + M)], dtype=torch.int32,
                         device=DEV)
    slots[0] = -1
    q = torch.empty(M, Hq * D, dtype=torch.bfloat16, device=DEV)
    ssq = _rms_parts(x, K // 128).contiguous()
    ops.gemm_ex(x, w, q, kind=L.EPI_QKV_ROPE, ssq_in=ssq, rms_dim=K, rms_eps=1e-5, pool=pool, geo=geo, layer=1,
                num_q_heads=Hq, positions=positions, slots=slots, rope_theta=500000.0)
    torch.cuda.synchronize()
    h = x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-5)
    qkv = (h @ w.float().T).bfloat16().float().cpu()
    pc = positions.cpu()
    q_ref = attention_ref.rope_ref(qkv[:, : Hq * D].view(M, Hq, D), pc, 500000.0)
    k_ref = attention_ref.rope_ref(qkv[:, Hq * D:(Hq + Hkv) * D].view(M, Hkv, D), pc, 500000.0)
    v_ref = qkv[:, (Hq + Hkv) * D:].view(M, Hkv, D)
    assert rel_err(q.view(M, Hq, D), q_ref) < 1e-2
    p6 = pool.view(nb, Lyr, 2, Hkv, 16, D).cpu().float()
    ks = torch.stack([p6[int(s) // 16, 1, 0, :, int(s) % 16] for s in slots.tolist()[1:]])
    vs = torch.stack([p6[int(s) // 16, 1, 1, :, int(s) % 16] for s in slots.tolist()[1:]])
    assert rel_err(ks, k_ref[1:]) < 1e-2 and rel_err(vs, v_ref[1:]) < 1e-2
    first = blocks[50 // 16] * 16 + 50 % 16
    assert torch.count_nonzero(p6[first // 16, 1, :, :, first % 16]) == 0   # slot -1 skipped


@pytest.mark.parametrize("M", [1, 3, 20, 64])
def test_gemm_chain_equals_separate_gemms(M):
    """O -> gate/up -> down -> lm_head argmax, chained vs one launch each
    (single-phase chains: above 32 rows a lone GEMM takes the one-CTA kernel,
    checked against the chain within bf16 tolerance at the end)."""
    from paper_2512_14142_b200.gpu.model import interleave_gate_up
    d, F, V = 512, 1536, 4096
    g = torch.Generator(device=DEV).manual_seed(M)
    att = torch.randn(M, d, generator=g, device=DEV).bfloat16()
    x0 = torch.randn(M, d, generator=g, device=DEV).bfloat16()
    wo = (torch.randn(d, d, generator=g, device=DEV) * 0.05).bfloat16()
    wgu = interleave_gate_up((torch.randn(2 * F, d, generator=g, device=DEV) * 0.05).bfloat16(), F).contiguous()
    wd = (torch.randn(d, F, generator=g, device=DEV) * 0.05).bfloat16()
    wl = (torch.randn(V, d, generator=g, device=DEV) * 0.05).bfloat16()
    ws = torch.zeros(64 << 20, dtype=torch.float32, device=DEV)
    outs = {}
    for chained in (False, True):
        x = x0.clone()
        h = torch.empty(M, F, dtype=torch.bfloat16, device=DEV)
        s1 = torch.empty(d // 128, M, dtype=torch.float32, device=DEV)
        s2 = torch.empty_like(s1)
        keys = torch.zeros(M, dtype=torch.int64, device=DEV)
        ph = [dict(a=att, w=wo, out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s1),
              dict(a=x, w=wgu, out=h, kind=L.EPI_SILU, ssq_in=s1, rms_dim=d, rms_eps=1e-5),
              dict(a=h, w=wd, out=x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s2),
              dict(a=x, w=wl, out=None, kind=L.EPI_ARGMAX, ssq_in=s2, rms_dim=d, rms_eps=1e-5, argmax_keys=keys)]
        for _ in range(2):   # twice: the phase counters must reset between launches
            x.copy_(x0)
            keys.zero_()
            if chained:
                ops.gemm_chain(ph, ws)
            else:
                for p in ph:
                    if M <= 32:
                        kw = {k: v for k, v in p.items() if k not in ("a", "w", "out")}
                        ops.gemm_ex(p["a"], p["w"], p["out"], workspace=ws, **kw)
                    else:
                        ops.gemm_chain([p], ws)
        torch.cuda.synchronize()
        outs[chained] = (x.clone(), h.clone(), keys.clone())
    assert torch.equal(outs[True][0], outs[False][0])
    assert torch.equal(outs[True][1], outs[False][1])
    assert torch.equal(outs[True][2], outs[False][2])
    if M > 32:   # the lone-GEMM route (one-CTA kernel) agrees within bf16 rounding
        x = x0.clone()
        h = torch.empty(M, F, dtype=torch.bfloat16, device=DEV)
        s1 = torch.empty(d // 128, M, dtype=torch.float32, device=DEV)
        s2 = torch.empty_like(s1)
        keys = torch.zeros(M, dtype=torch.int64, device=DEV)
        ops.gemm_ex(att, wo, x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s1, workspace=ws)
        ops.gemm_ex(x, wgu, h, kind=L.EPI_SILU, ssq_in=s1, rms_dim=d, rms_eps=1e-5, workspace=ws)
        ops.gemm_ex(h, wd, x, kind=L.EPI_RESIDUAL, residual=x, ssq_out=s2, workspace=ws)
        torch.cuda.synchronize()
        assert rel_err(x, outs[True][0]) < 1e-2 and rel_err(h, outs[True][1]) < 1e-2


@pytest.mark.parametrize("M,N,K", [(600, 640, 320), (4096, 2048, 512), (129, 1024, 200), (257, 6144, 4096)])
def test_pair_gemm_shapes_match_fp32(M, N, K):
    """The CTA-pair prefill GEMM (cta_group::2): partial 256-row / 256-column
    tiles, K tails (TMA zero fill), more tiles than pairs (persistent,
    double-buffered TMEM)."""
    g = torch.Generator(device=DEV).manual_seed(M + N + K)
    a = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    w = (torch.randn(N, K, generator=g, device=DEV) * 0.05).bfloat16()
    res = torch.randn(M, N, generator=g, device=DEV).bfloat16()
    out = res.clone()
    ops.gemm(a, w, out, residual=out)
    torch.cuda.synchronize()
    ref = a.float() @ w.float().T + res.float()
    assert rel_err(out, ref) < 1e-2


def test_row_ssq_matches_torch():
    x = torch.randn(37, 4096, device=DEV).bfloat16()
    s = ops.row_ssq(x)
    torch.cuda.synchronize()
    ref = x.float().view(37, 32, 128).pow(2).sum(-1).T
    assert s.shape == (32, 37) and torch.allclose(s, ref, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("Hq,Hkv,D", [(32, 8, 128), (8, 4, 64), (16, 4, 64)])
@pytest.mark.parametrize("ctxs", [[1], [900], [1, 16, 17, 300], [2316, 5, 0, 1000, 64],
                                  [37 * (b % 7) + 1 for b in range(24)], [8000, 3]])
def test_fused_chain_attention_matches_oracle(Hq, Hkv, D, ctxs):
    """The decode attention run as the chain's first phase (aligned split when
    the (row, kv head) sequences fit the grid, contiguous page ranges when
    they do not -- 24 rows x 8 heads) against the fp32 oracle; the chained
    GEMM consumes exactly what the attention wrote; twice on one workspace
    (launch epochs, counter resets)."""
    Lyr = 2
    B = len(ctxs)
    max_blocks = max(1, max((c + 15) // 16 for c in ctxs))
    nb = B * max_blocks + 3
    pool, geo = make_pool(nb, Lyr, Hkv, D, seed=B + D)
    perm = torch.randperm(nb, generator=torch.Generator().manual_seed(B))[: B * max_blocks].view(B, max_blocks).int()
    table = perm.clone()
    for b, c in enumerate(ctxs):
        table[b, (c + 15) // 16:] = -1
    g = torch.Generator(device=DEV).manual_seed(11)
    stride = (Hq + 2 * Hkv) * D
    qkv = torch.randn(B, stride, generator=g, device=DEV).bfloat16()
    N = 256
    wo = (torch.randn(N, Hq * D, generator=g, device=DEV) * 0.05).bfloat16()
    scale = 1 / math.sqrt(D)
    ctx_d = torch.tensor(ctxs, dtype=torch.int32, device=DEV)
    table_d = table.to(DEV)
    ws = torch.zeros(64 << 20, dtype=torch.float32, device=DEV)
    ref = attention_ref.decode_ref(pool.cpu(), 1, qkv[:, : Hq * D].view(B, Hq, D).cpu(), table, ctxs, scale,
                                   Lyr, Hkv, D)
    for rep in range(2):
        att = torch.full((B, Hq * D), float("nan"), dtype=torch.bfloat16, device=DEV)
        y = torch.empty(B, N, dtype=torch.bfloat16, device=DEV)
        attn = dict(pool=pool, geo=geo, layer=1, num_q_heads=Hq, q=qkv, q_stride=stride, table=table_d,
                    ctx=ctx_d, scale=scale, out=att)
        ops.gemm_chain([dict(a=att, w=wo, out=y)], ws, attn=attn)
        torch.cuda.synchronize()
        got = att.view(B, Hq, D).cpu().float()
        for b, c in enumerate(ctxs):
            if c == 0:
                assert torch.count_nonzero(got[b]) == 0, (rep, b)
            else:
                assert rel_err(got[b], ref[b]) < 1e-2, (rep, b, c)
        y_ref = torch.empty_like(y)
        ops.gemm_ex(att, wo, y_ref, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref), rep


@pytest.mark.parametrize("M,N", [(100, 4096), (128, 6144), (200, 4096), (97, 4104)])
def test_short_prefill_split_k_rows(M, N):
    """Short prefills on the one-CTA kernel with split-K (tiles < SMs): fp32
    partials summed in split order by the last split -- matches fp32, is
    bit-reproducible, and leaves the tile counters at zero (a second run on
    the same workspace gives the same bits), in-place residual included."""
    K = 4096
    g = torch.Generator(device=DEV).manual_seed(M + N)
    a = torch.randn(M, K, generator=g, device=DEV).bfloat16()
    w = (torch.randn(N, K, generator=g, device=DEV) * 0.02).bfloat16()
    x0 = torch.randn(M, N, generator=g, device=DEV).bfloat16()
    ref = a.float() @ w.float().T + x0.float()
    from paper_2512_14142_b200.gpu import lib as L
    need = L.load().astraea_gemm_workspace_bytes(M, N, K)
    ws = torch.zeros(need // 4 + 1, dtype=torch.float32, device=DEV)   # one workspace for both runs
    outs = []
    for _ in range(2):
        x = x0.clone()
        ops.gemm(a, w, out=x, residual=x, workspace=ws)
        torch.cuda.synchronize()
        outs.append(x)
    assert rel_err(outs[0], ref) < 5e-3
    assert torch.equal(outs[0], outs[1])
