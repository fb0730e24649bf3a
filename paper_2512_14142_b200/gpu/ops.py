"""Tensor-level wrappers over the C ABI (shape checks + pointer passing).

Every function launches exactly the sm_100a kernels named in
include/astraea_b200.h on the current torch stream (or the given one) and
returns without synchronising. Inputs must already live on the device.
"""

from __future__ import annotations

import ctypes

import torch

from . import lib as L


# Kernels launched through this module (the bench's ``gpu_launches`` claim).
LAUNCHES = [0]


def _s(stream):
    return L.stream_handle(stream)


def _count(n=1):
    LAUNCHES[0] += n




def geometry(num_layers, num_kv_heads, head_dim, num_blocks, block_tokens=16) -> L.KvGeometry:
    return L.KvGeometry(num_layers, num_kv_heads, head_dim, block_tokens, num_blocks)


def gemm(a: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None,
         residual: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
         stream=None) -> torch.Tensor:
    """out[M,N] = a[M,K] @ w[N,K]^T (+ residual), tcgen05 tensor cores."""
    lib = L.require_cuda()
    M, K = a.shape
    N = w.shape[0]
    assert w.shape[1] == K and a.dtype == torch.bfloat16 and w.dtype == torch.bfloat16
    assert a.stride(1) == 1 and w.stride(1) == 1
    if out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=a.device)
    need = lib.astraea_gemm_workspace_bytes(M, N, K)
    if need and (workspace is None or workspace.numel() * workspace.element_size() < need):
        workspace = torch.zeros(need // 4 + 1, dtype=torch.float32, device=a.device)
    L.check(lib.astraea_gemm_bf16(
        L.ptr(a), a.stride(0), L.ptr(w), w.stride(0), L.ptr(out), out.stride(0), M, N, K,
        L.ptr(residual), L.EPI_RESIDUAL if residual is not None else L.EPI_NONE,
        L.ptr(workspace), 0 if workspace is None else workspace.numel() * workspace.element_size(),
        _s(stream)), "gemm_bf16")
    _count()
    return out


def _epilogue(kind=L.EPI_NONE, residual=None, ssq_out=None, ssq_in=None, rms_dim=0, rms_eps=1e-5, pool=None,
              geo=None, layer=0, num_q_heads=0, positions=None, slots=None, rope_theta=0.0, rope_table=None,
              argmax_keys=None, argmax_col_offset=0):
    e = L.Epilogue()
    e.argmax_col_offset = argmax_col_offset
    e.kind = kind
    e.residual_dev = L.ptr(residual)
    e.ssq_out_dev = L.ptr(ssq_out)
    e.ssq_in_dev = L.ptr(ssq_in)
    e.ssq_in_parts = 0 if ssq_in is None else ssq_in.shape[0]
    e.rms_dim = rms_dim
    e.rms_eps = rms_eps
    e.argmax_keys_dev = L.ptr(argmax_keys)
    e.argmax_col_offset = argmax_col_offset
    if kind == L.EPI_QKV_ROPE:
        e.pool_dev = L.ptr(pool)
        e.geo = geo
        e.layer = layer
        e.num_q_heads = num_q_heads
        e.positions_dev = L.ptr(positions)
        e.slots_dev = L.ptr(slots)
        e.rope_theta = rope_theta
        e.rope_table_dev = L.ptr(rope_table)
    return e


def gemm_chain(phases, workspace, stream=None, attn=None):
    """Dependent decode GEMMs in one persistent launch (astraea_gemm_chain).

    ``phases``: list of dicts with a, w, out and the ``gemm_ex`` epilogue
    keywords; every ``a`` has the same number of rows (M <= 64). ``attn``
    (optional dict: pool, geo, layer, num_q_heads, q, q_stride, table, ctx,
    scale, out, and ``before``, default 0; or a list of up to two such
    dicts): a layer's decode attention runs right before GEMM phase
    ``before`` in the same launch (astraea_gemm_chain_attn); its ``out``
    must be that phase's ``a``."""
    lib = L.require_cuda()
    n = len(phases)
    arr = (L.GemmPhase * n)()
    M = phases[0]["a"].shape[0]
    for i, ph in enumerate(phases):
        a, w, out = ph["a"], ph["w"], ph.get("out")
        assert a.shape[0] == M
        q = arr[i]
        q.A, q.lda = L.ptr(a), a.stride(0)
        q.W, q.ldw = L.ptr(w), w.stride(0)
        q.C, q.ldc = L.ptr(out), (out.stride(0) if out is not None else 0)
        q.N, q.K = w.shape[0], a.shape[1]
        q.epi = _epilogue(**{k: v for k, v in ph.items() if k not in ("a", "w", "out")})
    need = lib.astraea_gemm_chain_workspace_bytes(M, n, arr)
    assert workspace.numel() * workspace.element_size() >= need, "chain workspace too small"
    if attn is None:
        L.check(lib.astraea_gemm_chain(M, n, arr, L.ptr(workspace), workspace.numel() * workspace.element_size(),
                                       _s(stream)), "gemm_chain")
    else:
        attns = attn if isinstance(attn, (list, tuple)) else [attn]
        ats = (L.AttnPhase * len(attns))()
        before = (ctypes.c_int32 * len(attns))()
        for k, d in enumerate(attns):
            at = ats[k]
            at.pool_dev, at.geo, at.layer = L.ptr(d["pool"]), d["geo"], d["layer"]
            at.num_q_heads, at.q_dev, at.q_row_stride = d["num_q_heads"], L.ptr(d["q"]), d["q_stride"]
            at.table_dev, at.max_blocks = L.ptr(d["table"]), d["table"].shape[1]
            at.ctx_dev, at.scale, at.out_dev = L.ptr(d["ctx"]), d["scale"], L.ptr(d["out"])
            before[k] = d.get("before", 0)
        L.check(lib.astraea_gemm_chain_attn(M, len(attns), ats, before, n, arr, L.ptr(workspace),
                                            workspace.numel() * workspace.element_size(), _s(stream)),
                "gemm_chain_attn")
    _count()


class StepProgram:
    """A decode step as one persistent launch (astraea_step_program_build /
    astraea_step_launch).

    ``phases``: dicts in program order. GEMM phases: ``kind="gemm"``, ``a``,
    ``w``, ``out``, ``epi`` (the epilogue kind) and the other ``gemm_ex``
    epilogue keywords, plus ``a_from`` /
    ``epi_from`` (indices of the producing phases, -1 for launch inputs).
    ATTN phases: ``kind="attn"``, ``pool``, ``geo``, ``layer``,
    ``num_q_heads``, ``q``, ``q_stride``, ``table``, ``ctx``, ``scale``,
    ``out``, ``qkv_from``. All rows: M <= 64. The tensors must stay alive
    (and at the same addresses) for as long as the program is launched.
    """

    def __init__(self, M, phases, workspace_pool):
        lib = L.require_cuda()
        n = len(phases)
        arr = (L.StepPhase * n)()
        for i, ph in enumerate(phases):
            q = arr[i]
            q.a_from = ph.get("a_from", -1)
            q.epi_from = ph.get("epi_from", -1)
            q.qkv_from = ph.get("qkv_from", -1)
            if ph["kind"] == "gemm":
                q.kind = L.PHASE_GEMM
                a, w, out = ph["a"], ph["w"], ph.get("out")
                g = q.gemm
                g.A, g.lda = L.ptr(a), a.stride(0)
                g.W, g.ldw = L.ptr(w), w.stride(0)
                g.C, g.ldc = L.ptr(out), (out.stride(0) if out is not None else 0)
                g.N, g.K = w.shape[0], a.shape[1]
                g.epi = _epilogue(kind=ph.get("epi", L.EPI_NONE),
                                  **{k: v for k, v in ph.items()
                                     if k not in ("kind", "epi", "a", "w", "out", "a_from", "epi_from", "qkv_from")})
            else:
                q.kind = L.PHASE_ATTN
                q.pool_dev, q.geo, q.layer = L.ptr(ph["pool"]), ph["geo"], ph["layer"]
                q.num_q_heads, q.q_dev, q.q_row_stride = ph["num_q_heads"], L.ptr(ph["q"]), ph["q_stride"]
                q.table_dev, q.max_blocks = L.ptr(ph["table"]), ph["table"].shape[1]
                q.ctx_dev, q.scale, q.out_dev = L.ptr(ph["ctx"]), ph["scale"], L.ptr(ph["out"])
        self.M, self.n = M, n
        dev = phases[0].get("a", phases[0].get("q")).device
        need = lib.astraea_step_workspace_bytes(M, n, arr)
        if need == 0:
            raise L.DeviceError("decode step program rejected (shapes)")
        self.ws = workspace_pool.get(need, dev)
        nb = lib.astraea_step_program_bytes(n)
        self.host = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        L.check(lib.astraea_step_program_build(M, n, arr, L.ptr(self.host), nb, L.ptr(self.ws),
                                               self.ws.numel() * 4), "step_program_build")
        self.prog = torch.empty(nb, dtype=torch.uint8, device=dev)
        self.prog.copy_(self.host, non_blocking=True)   # stream-ordered before the first launch
        self.keep = phases   # tensors referenced by the program

    def launch(self, stream=None, l2_ahead=0):
        lib = L.require_cuda()
        L.check(lib.astraea_step_launch(self.M, self.n, L.ptr(self.prog), L.ptr(self.ws), l2_ahead, _s(stream)),
                "step_launch")
        _count()


class StepWorkspace:
    """Zero-filled step workspace shared by the programs of one stream (it
    holds the launch epoch and the dataflow flags). Grows by replacement;
    programs built on an older buffer keep it alive."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes, device):
        if self.buf is None or self.buf.numel() * 4 < nbytes:
            self.buf = torch.zeros(nbytes // 4 + 64, dtype=torch.float32, device=device)
        return self.buf


def gemm_ex(a, w, out, kind=L.EPI_NONE, residual=None, ssq_out=None, ssq_in=None, rms_dim=0, rms_eps=1e-5,
            pool=None, geo=None, layer=0, num_q_heads=0, positions=None, slots=None, rope_theta=0.0,
            rope_table=None, argmax_keys=None, workspace=None, stream=None, argmax_col_offset=0):
    """GEMM with a fused epilogue program (astraea_gemm_bf16_ex)."""
    lib = L.require_cuda()
    M, K = a.shape
    N = w.shape[0]
    e = L.Epilogue()
    e.kind = kind
    e.residual_dev = L.ptr(residual)
    e.ssq_out_dev = L.ptr(ssq_out)
    e.ssq_in_dev = L.ptr(ssq_in)
    e.ssq_in_parts = 0 if ssq_in is None else ssq_in.shape[0]
    e.rms_dim = rms_dim
    e.rms_eps = rms_eps
    e.argmax_keys_dev = L.ptr(argmax_keys)
    if kind == L.EPI_QKV_ROPE:
        e.pool_dev = L.ptr(pool)
        e.geo = geo
        e.layer = layer
        e.num_q_heads = num_q_heads
        e.positions_dev = L.ptr(positions)
        e.slots_dev = L.ptr(slots)
        e.rope_theta = rope_theta
        e.rope_table_dev = L.ptr(rope_table)
    need = lib.astraea_gemm_workspace_bytes(M, N, K)
    if need and (workspace is None or workspace.numel() * workspace.element_size() < need):
        workspace = torch.zeros(need // 4 + 1, dtype=torch.float32, device=a.device)
    L.check(lib.astraea_gemm_bf16_ex(
        L.ptr(a), a.stride(0), L.ptr(w), w.stride(0), L.ptr(out), out.stride(0) if out is not None else 0, M, N, K,
        ctypes.byref(e),
        L.ptr(workspace), 0 if workspace is None else workspace.numel() * workspace.element_size(),
        _s(stream)), "gemm_bf16_ex")
    _count()
    return out


def row_ssq(x, out=None, stream=None):
    """RMSNorm statistics of x [rows][dim]: [ceil(dim/128)][rows] fp32 (astraea_row_ssq)."""
    lib = L.require_cuda()
    rows, dim = x.shape
    if out is None:
        out = torch.empty(-(-dim // 128), rows, dtype=torch.float32, device=x.device)
    L.check(lib.astraea_row_ssq(L.ptr(x), rows, dim, L.ptr(out), _s(stream)), "row_ssq")
    _count()
    return out


def keys_to_ids(keys):
    """Token ids from ARGMAX-epilogue keys (int64 view of the packed keys)."""
    return (4294967295 - (keys & 4294967295)).to(torch.int32)


def rope_table(positions, head_dim, theta, out=None, stream=None):
    lib = L.require_cuda()
    T = positions.shape[0]
    if out is None:
        out = torch.empty(T, head_dim // 2, 2, dtype=torch.float32, device=positions.device)
    L.check(lib.astraea_rope_table(L.ptr(positions), T, head_dim, theta, L.ptr(out), _s(stream)), "rope_table")
    _count()
    return out


def rmsnorm(x, weight, eps, out=None, residual=None, resid_out=None, stream=None):
    lib = L.require_cuda()
    rows, dim = x.shape
    if out is None:
        out = torch.empty_like(x)
    L.check(lib.astraea_rmsnorm(L.ptr(x), L.ptr(residual), L.ptr(weight), L.ptr(out), L.ptr(resid_out),
                                rows, dim, eps, _s(stream)), "rmsnorm")
    _count()
    return out


def silu_mul(gu, out=None, stream=None):
    lib = L.require_cuda()
    T, F2 = gu.shape
    F = F2 // 2
    if out is None:
        out = torch.empty(T, F, dtype=gu.dtype, device=gu.device)
    L.check(lib.astraea_silu_mul(L.ptr(gu), L.ptr(out), T, F, _s(stream)), "silu_mul")
    _count()
    return out


def embedding(ids, table, out=None, ssq_out=None, stream=None):
    lib = L.require_cuda()
    T = ids.shape[0]
    dim = table.shape[1]
    if out is None:
        out = torch.empty(T, dim, dtype=table.dtype, device=table.device)
    L.check(lib.astraea_embedding(L.ptr(ids), L.ptr(table), L.ptr(out), T, dim, L.ptr(ssq_out), _s(stream)),
            "embedding")
    _count()
    return out


def argmax(logits, out=None, stream=None):
    lib = L.require_cuda()
    rows, vocab = logits.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.int32, device=logits.device)
    L.check(lib.astraea_argmax(L.ptr(logits), rows, vocab, L.ptr(out), _s(stream)), "argmax")
    _count()
    return out


def rope_kv_append(geo, pool, layer, qkv, num_q_heads, positions, slots, theta, stream=None):
    lib = L.require_cuda()
    L.check(lib.astraea_rope_kv_append(ctypes.byref(geo), L.ptr(pool), layer, L.ptr(qkv), qkv.shape[0],
                                       num_q_heads, L.ptr(positions), L.ptr(slots), theta, _s(stream)),
            "rope_kv_append")
    _count()


def decode_attention(geo, pool, layer, q, q_row_stride, B, num_q_heads, table, ctx, scale, out,
                     workspace, stream=None):
    lib = L.require_cuda()
    L.check(lib.astraea_paged_decode_attention(
        ctypes.byref(geo), L.ptr(pool), layer, L.ptr(q), q_row_stride, B, num_q_heads, L.ptr(table),
        table.shape[1], L.ptr(ctx), scale, L.ptr(out), L.ptr(workspace),
        workspace.numel() * workspace.element_size(), _s(stream)), "paged_decode_attention")
    _count()
    return out


def decode_workspace(B, num_q_heads, head_dim, max_blocks, device) -> torch.Tensor:
    lib = L.load()
    n = lib.astraea_decode_workspace_bytes(B, num_q_heads, head_dim, max_blocks)
    return torch.zeros(n // 4 + 1, dtype=torch.float32, device=device)


def prefill_attention(geo, pool, layer, q, q_row_stride, cu_q, S, max_q_len, num_q_heads, table, ctx,
                      scale, out, stream=None):
    lib = L.require_cuda()
    L.check(lib.astraea_paged_prefill_attention(
        ctypes.byref(geo), L.ptr(pool), layer, L.ptr(q), q_row_stride, L.ptr(cu_q), S, max_q_len,
        num_q_heads, L.ptr(table), table.shape[1], L.ptr(ctx), scale, L.ptr(out), _s(stream)),
        "paged_prefill_attention")
    _count()
    return out


def block_table_build(csr_ptr, csr_ids, rows, ctx_src, max_blocks, table, ctx, stream=None):
    lib = L.require_cuda()
    L.check(lib.astraea_block_table_build(L.ptr(csr_ptr), L.ptr(csr_ids), L.ptr(rows), L.ptr(ctx_src),
                                          rows.shape[0], max_blocks, L.ptr(table), L.ptr(ctx), _s(stream)),
            "block_table_build")
    _count()


def decode_advance(step, B, n_gen, base_pos, first_tok, sampled, table, block_tokens, tokens, positions,
                   slots, ctx, hist=None, hist_stride=0, stream=None):
    lib = L.require_cuda()
    L.check(lib.astraea_decode_advance(
        L.ptr(step), B, L.ptr(n_gen), L.ptr(base_pos), L.ptr(first_tok), L.ptr(sampled), L.ptr(table),
        table.shape[1], block_tokens, L.ptr(tokens), L.ptr(positions), L.ptr(slots), L.ptr(ctx),
        L.ptr(hist), hist_stride, _s(stream)), "decode_advance")
    _count()


def swap_out(geo, pool, block_ids, n_tokens, slot, mode=L.SWAP_KERNEL, stream=None):
    lib = L.require_cuda()
    ids = L.i32_array(block_ids)
    L.check(lib.astraea_kv_swap_out(ctypes.byref(geo), L.ptr(pool), ids, len(block_ids), n_tokens,
                                    L.ptr(slot), mode, _s(stream)), "kv_swap_out")
    _count(-(-len(block_ids) // 900) if mode == L.SWAP_KERNEL else 0)


def swap_in(geo, pool, block_ids, n_tokens, slot, mode=L.SWAP_KERNEL, stream=None):
    lib = L.require_cuda()
    ids = L.i32_array(block_ids)
    L.check(lib.astraea_kv_swap_in(ctypes.byref(geo), L.ptr(pool), ids, len(block_ids), n_tokens,
                                   L.ptr(slot), mode, _s(stream)), "kv_swap_in")
    _count(-(-len(block_ids) // 900) if mode == L.SWAP_KERNEL else 0)


def copy_blocks(geo, pool, src_ids, dst_ids, stream=None):
    lib = L.require_cuda()
    L.check(lib.astraea_kv_copy_blocks(ctypes.byref(geo), L.ptr(pool), L.i32_array(src_ids),
                                       L.i32_array(dst_ids), len(src_ids), _s(stream)), "kv_copy_blocks")


class BlockAllocator:
    """Host free list over the pool's blocks (native, LIFO)."""

    def __init__(self, num_blocks: int):
        self._lib = L.load()
        h = ctypes.c_void_p()
        L.check(self._lib.astraea_alloc_create(num_blocks, ctypes.byref(h)), "alloc_create")
        self._h = h
        self.num_blocks = num_blocks

    def take(self, n: int) -> list[int]:
        if n == 0:
            return []
        buf = (ctypes.c_int32 * n)()
        L.check(self._lib.astraea_alloc_take(self._h, n, buf), f"alloc_take({n})")
        return list(buf)

    def give(self, ids) -> None:
        if not ids:
            return
        L.check(self._lib.astraea_alloc_give(self._h, L.i32_array(ids), len(ids)), "alloc_give")

    @property
    def free(self) -> int:
        return self._lib.astraea_alloc_free_count(self._h)

    def __del__(self):
        try:
            self._lib.astraea_alloc_destroy(self._h)
        except Exception:
            pass
