"""KvDataPath: the device side of every KV transition and every batch.

The reference's KV manager, subclassed in ``plugin.py`` (kvcache.py:152-292),
forwards the eight transitions of SURVEY.md Appendix C here; the plugin's
engine hands every admitted batch to :meth:`KvDataPath.launch_batch`.

Streams
  compute  prefill + decode of batches, in admission order;
  swap     K1 gathers and K2 scatters (side stream), overlapping compute.

Ordering rules (all device-side, the host never waits in ``model`` mode)
  * a swap-out waits on the event that finished the request's last KV write;
  * blocks freed by a completed swap-out are fenced: the next compute launch
    waits on the gather's event before anything can overwrite them;
  * a swap-in waits on the compute stream's current tail (its fresh blocks
    may still be read by in-flight work) and the request's next batch waits
    on the scatter's event;
  * host slots are returned to torch's pinned pool only after the event of
    the last copy that touched them has completed.

Token content: each request's fed-token history stays on the device (the
prompt pieces uploaded per batch plus the decode-fed tokens written by the
decode-advance kernel), so a recompute after a discard re-prefills exactly
the original context without any device-to-host round trip.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from ..reference import load as _load_reference
from ..tokens import segment_token_ids
from . import lib as L
from . import ops
from .model import LlamaConfig, LlamaRunner, LlamaWeights

BT = 16
ProtocolError = _load_reference().ProtocolError   # the reference's own (errors.py:25)
RESULTS_SOFT_LIMIT = 256


class KvPool:
    """The paged HBM pool: ``[num_blocks][L][2][Hkv][16][D]`` bf16."""

    def __init__(self, cfg: LlamaConfig, num_blocks: int, device="cuda"):
        self.cfg = cfg
        self.geo = ops.geometry(cfg.num_layers, cfg.num_kv_heads, cfg.head_dim, num_blocks)
        lib = L.load()
        self.block_bytes = lib.astraea_kv_block_bytes(self.geo)
        self.bytes_per_token = lib.astraea_kv_bytes_per_token(self.geo)
        self.data = torch.zeros(num_blocks * self.block_bytes // 2, dtype=torch.bfloat16, device=device)
        self.alloc = ops.BlockAllocator(num_blocks)
        self.num_blocks = num_blocks


@dataclass
class ReqDev:
    blocks: list = field(default_factory=list)
    tokens: int = 0                      # KV rows materialised on the device
    hist: list = field(default_factory=list)   # device int32 pieces, total == context tokens fed
    hist_len: int = 0
    pending: Optional[torch.Tensor] = None     # 0-d device int32: next token to feed
    ready: Optional[torch.cuda.Event] = None   # KV of this request complete after this event
    slot: Optional[torch.Tensor] = None        # pinned host slot
    slot_tokens: int = 0
    swap_ev: Optional[tuple] = None            # (start, end) events of the last swap


def _blocks_for(tokens: int) -> int:
    return (tokens + BT - 1) // BT


def _width_bucket(n: int) -> int:
    return 1 << max(4, (n - 1).bit_length())


def _loc(location) -> str:
    """Cache location by value, so states of the host mirror *and* of the
    unmodified reference package (its own CacheLocation enum) both work."""
    return location.value


class KvDataPath:
    def __init__(self, cfg: LlamaConfig, weights: Optional[LlamaWeights] = None, num_blocks: int = 4096,
                 device="cuda", swap_mode: int = L.SWAP_STAGED, seed: int = 0, measure: bool = False,
                 token_seed: int = 0, runner_factory=None, token_vocab: Optional[int] = None):
        """``runner_factory(weights, pool)``: the model runner (default
        LlamaRunner; a tensor-parallel rank passes a TpLlamaRunner over its
        shard -- every rank then executes the same plans).
        ``token_vocab``: the vocabulary prompt ids are drawn from (default
        cfg.vocab; a TP shard config carries only its lm_head slice)."""
        L.require_cuda()
        self.cfg = cfg
        self.device = torch.device(device)
        self.weights = weights or LlamaWeights(cfg, device=device, seed=seed)
        self.pool = KvPool(cfg, num_blocks, device)
        self.runner = (runner_factory or LlamaRunner)(self.weights, self.pool)
        self.token_vocab = token_vocab or cfg.vocab
        self.compute = torch.cuda.Stream(device=self.device)
        self.swapper = torch.cuda.Stream(device=self.device)
        self.swap_mode = swap_mode
        self.measure = measure
        self.token_seed = token_seed
        self.reqs: dict[str, ReqDev] = {}
        self._fences: list = []
        self._deferred: list = []   # (event, tensor) kept alive until event completes
        self.stats = {"batches": 0, "prefill_tokens": 0, "decode_steps": 0, "decode_row_steps": 0,
                      "swap_out_bytes": 0, "swap_in_bytes": 0, "swap_outs": 0, "swap_ins": 0,
                      "discards": 0, "recompute_tokens": 0, "h2d_bytes": 0, "d2h_bytes": 0,
                      "kernel_launches": 0}
        self.results: list = []     # (event, pinned hist copy) per batch; see drain_results()
        self.use_graphs = True
        self._graphs: dict = {}
        self._graph_pool = None
        self.last_batch_events = None
        self.staged: dict = {}      # (request id, segment) -> device int32 prompt ids

    def prestage(self, workload) -> None:
        """Upload every segment's prompt ids to HBM ahead of time (bench
        ``value`` mode: inputs resident before the timed region)."""
        keys, ids = [], []
        for req in workload:
            for seg in req.segments:
                toks = segment_token_ids(req.id, seg.index, seg.n_in, self.token_vocab, self.token_seed)
                keys.append((req.id, seg.index, len(ids), len(toks)))
                ids.extend(toks)
        buf = torch.tensor(ids or [0], dtype=torch.int32, device=self.device)
        self.staged = {(rid, si): buf[a:a + n] for rid, si, a, n in keys}
        torch.cuda.synchronize(self.device)

    # ------------------------------------------------------------------ helpers

    def _rd(self, state) -> ReqDev:
        rd = self.reqs.get(state.spec.id)
        if rd is None:
            rd = self.reqs[state.spec.id] = ReqDev()
        return rd

    def _free_blocks(self, rd: ReqDev, fence: Optional[torch.cuda.Event] = None) -> None:
        if rd.blocks:
            if fence is not None:
                self._fences.append(fence)
            self.pool.alloc.give(rd.blocks)
        rd.blocks = []
        rd.tokens = 0

    def _defer(self, event, obj) -> None:
        self._deferred.append((event, obj))
        if len(self._deferred) > 64:
            self._deferred = [(e, o) for e, o in self._deferred if not e.query()]

    def _compute_tail(self) -> torch.cuda.Event:
        ev = torch.cuda.Event()
        ev.record(self.compute)
        return ev

    # ------------------------------------------------------------------ KV transitions

    def drop(self, state) -> None:
        """Transitions 2 and 8: discard (estimated or deadlock-evicted)."""
        rd = self._rd(state)
        self._free_blocks(rd)
        self.stats["discards"] += 1

    def swap_out_begin(self, state) -> None:
        """Transition 3: K1 gather of the request's blocks to a pinned slot."""
        rd = self._rd(state)
        n = state.kv_tokens
        if rd.tokens != n or len(rd.blocks) != _blocks_for(n):
            raise ProtocolError(f"{state.spec.id}: device holds {rd.tokens} tokens, host says {n}")
        slot = torch.empty(n * self.pool.bytes_per_token, dtype=torch.uint8, pin_memory=True)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.swapper):
            if rd.ready is not None:
                self.swapper.wait_event(rd.ready)
            s0.record(self.swapper)
            ops.swap_out(self.pool.geo, self.pool.data, rd.blocks, n, slot, self.swap_mode, self.swapper)
            s1.record(self.swapper)
        rd.slot, rd.slot_tokens, rd.swap_ev = slot, n, (s0, s1)
        self.stats["swap_out_bytes"] += n * self.pool.bytes_per_token
        self.stats["swap_outs"] += 1
        self.stats["kernel_launches"] += 0 if self.swap_mode == L.SWAP_DMA else 1

    def swap_out_done(self, state) -> None:
        """Transition 4: blocks return to the pool, fenced on the gather."""
        rd = self._rd(state)
        self._free_blocks(rd, fence=rd.swap_ev[1])

    def swap_in_begin(self, state) -> None:
        """Transition 5: fresh blocks + K2 scatter from the pinned slot."""
        rd = self._rd(state)
        n = state.kv_tokens
        if rd.slot is None or rd.slot_tokens != n:
            raise ProtocolError(f"{state.spec.id}: no host slot of {n} tokens")
        rd.blocks = self.pool.alloc.take(_blocks_for(n))
        tail = self._compute_tail()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.swapper):
            self.swapper.wait_event(tail)
            s0.record(self.swapper)
            ops.swap_in(self.pool.geo, self.pool.data, rd.blocks, n, rd.slot, self.swap_mode, self.swapper)
            s1.record(self.swapper)
        rd.tokens = n
        rd.ready = s1
        rd.swap_ev = (s0, s1)
        self._fences.append(s1)
        self.stats["swap_in_bytes"] += n * self.pool.bytes_per_token
        self.stats["swap_ins"] += 1
        self.stats["kernel_launches"] += 0 if self.swap_mode == L.SWAP_DMA else 1

    def swap_in_done(self, state) -> None:
        """Transition 6: the slot can go once the scatter has read it."""
        rd = self._rd(state)
        self._defer(rd.swap_ev[1], rd.slot)
        rd.slot, rd.slot_tokens = None, 0

    def release(self, state, where) -> None:
        """Transition 7: the request finished."""
        rd = self.reqs.pop(state.spec.id, None)
        if rd is None:
            return
        if _loc(where) == "gpu":
            self._free_blocks(rd)
        if rd.slot is not None:
            self._defer(rd.swap_ev[1], rd.slot)

    def swap_seconds(self, state, direction: str) -> float:
        """Measured duration of the request's last gather/scatter (syncs)."""
        rd = self._rd(state)
        s0, s1 = rd.swap_ev
        s1.synchronize()
        return s0.elapsed_time(s1) / 1000.0

    # ------------------------------------------------------------------ batches

    def launch_batch(self, members) -> Optional[list]:
        """Transition 1 + the batch itself: (re)prefill, then the decode loop.

        ``members`` are ``plugin.AdmittedMember`` (pre-admission cache
        location). Returns per-member seconds when ``measure`` is set.
        """
        cfg = self.cfg
        dev = self.device
        B = len(members)
        # reserve every member's blocks up front: a batch the pool cannot hold
        # fails before any member's device state changes
        grow = 0
        for m in members:
            rd = self.reqs.get(m.state.spec.id)
            held = len(rd.blocks) if rd is not None else 0
            grow += max(0, _blocks_for(m.state.context_after(m.segment_index)) - held)
        if grow > self.pool.alloc.free:
            raise ProtocolError(f"batch needs {grow} KV blocks, only {self.pool.alloc.free} free")
        plan = []
        pieces_meta = []   # per prefill member: list of device pieces or ("new", offset, n)
        new_ids_host = []
        for m in members:
            st = m.state
            rid = st.spec.id
            seg = st.spec.segment(m.segment_index)
            rd = self._rd(st)
            ctx_before = st.context_before_current
            ctx_after = st.context_after(m.segment_index)
            prior = _loc(m.prior_location)
            if prior == "gpu":
                if rd.tokens != ctx_before or rd.hist_len != ctx_before:
                    raise ProtocolError(f"{rid}: resident KV {rd.tokens} != context {ctx_before}")
                start = ctx_before
                recompute = False
            elif prior in ("none", "dropped"):
                if rd.blocks:
                    raise ProtocolError(f"{rid}: {m.prior_location} request still holds blocks")
                start = 0
                recompute = ctx_before > 0
                if rd.hist_len != ctx_before:
                    raise ProtocolError(f"{rid}: history {rd.hist_len} != context {ctx_before}")
            else:
                raise ProtocolError(f"{rid}: cannot run from {m.prior_location}")
            need = _blocks_for(ctx_after) - len(rd.blocks)
            if need > 0:
                rd.blocks = rd.blocks + self.pool.alloc.take(need)
            n_new = seg.n_in
            staged = self.staged.get((rid, m.segment_index))
            off = len(new_ids_host)
            if staged is None:
                new_ids_host.extend(segment_token_ids(rid, m.segment_index, n_new, self.token_vocab, self.token_seed))
            plen = (ctx_before - start) + n_new
            plan.append(dict(rd=rd, start=start, plen=plen, new_off=off, n_new=n_new, n_gen=seg.n_gen,
                             ctx_before=ctx_before, recompute=recompute, staged=staged))
            if recompute:
                self.stats["recompute_tokens"] += ctx_before
        # ---- one H2D upload of every int32 the batch needs
        pre = [i for i, p in enumerate(plan) if p["plen"] > 0]
        S = len(pre)
        csr_ptr = [0]
        csr_ids = []
        for p in plan:
            csr_ids.extend(p["rd"].blocks)
            csr_ptr.append(len(csr_ids))
        # table width bucketed to a power of two (>= 16): the same kernel
        # arguments whether the step runs eagerly or as a graph replay
        max_blocks = _width_bucket(max(1, max(len(p["rd"].blocks) for p in plan)))
        pos_parts, slot_parts, cu_q, pre_ctx = [], [], [0], []
        for i in pre:   # vectorised: a recompute feeds thousands of tokens
            p = plan[i]
            pos = np.arange(p["start"], p["start"] + p["plen"], dtype=np.int64)
            bl = np.asarray(p["rd"].blocks, dtype=np.int64)
            pos_parts.append(pos)
            slot_parts.append(bl[pos // BT] * BT + pos % BT)
            cu_q.append(cu_q[-1] + p["plen"])
            pre_ctx.append(p["start"] + p["plen"])
        positions = np.concatenate(pos_parts) if pos_parts else np.zeros(0, dtype=np.int64)
        slots = np.concatenate(slot_parts) if slot_parts else np.zeros(0, dtype=np.int64)
        T = cu_q[-1]
        max_q = max([plan[i]["plen"] for i in pre], default=0)
        n_gen = [p["n_gen"] for p in plan]
        base_pos = [p["ctx_before"] + p["n_new"] for p in plan]
        all_ctx_src = [p["ctx_before"] + p["n_new"] for p in plan]
        pre_ctx_src = [0] * B
        for j, i in enumerate(pre):
            pre_ctx_src[i] = pre_ctx[j]
        fields = [("csr_ptr", csr_ptr), ("csr_ids", csr_ids), ("pre_rows", pre), ("all_rows", list(range(B))),
                  ("pre_ctx_src", pre_ctx_src), ("positions", positions), ("slots", slots), ("cu_q", cu_q),
                  ("n_gen", n_gen), ("base_pos", base_pos), ("new_ids", new_ids_host), ("all_ctx_src", all_ctx_src)]
        sizes = [len(v) for _, v in fields]
        blob = np.zeros(sum(sizes) + 1, dtype=np.int32)
        o = 0
        offs = {}
        for (name, vals), n in zip(fields, sizes):
            blob[o:o + n] = vals
            offs[name] = (o, n)
            o += n
        host = torch.from_numpy(blob).pin_memory()
        max_ngen = max(n_gen)
        with torch.cuda.stream(self.compute):
            for ev in self._fences:
                self.compute.wait_event(ev)
            self._fences.clear()
            t_start = torch.cuda.Event(enable_timing=True)
            t_start.record(self.compute)
            d = host.to(dev, non_blocking=True)
            self.stats["h2d_bytes"] += blob.nbytes

            def view(name):
                a, n = offs[name]
                return d[a:a + n]

            table = torch.empty(B, max_blocks, dtype=torch.int32, device=dev)
            ctx_all = torch.empty(B, dtype=torch.int32, device=dev)
            ops.block_table_build(view("csr_ptr"), view("csr_ids"), view("all_rows"), view("all_ctx_src"),
                                  max_blocks, table, ctx_all, stream=self.compute)
            first_tok_parts = []
            if S:
                pre_table = torch.empty(S, max_blocks, dtype=torch.int32, device=dev)
                pre_ctx_d = torch.empty(S, dtype=torch.int32, device=dev)
                ops.block_table_build(view("csr_ptr"), view("csr_ids"), view("pre_rows"), view("pre_ctx_src"),
                                      max_blocks, pre_table, pre_ctx_d, stream=self.compute)
                new_ids = view("new_ids")
                pieces = []
                for i in pre:
                    p = plan[i]
                    if p["recompute"]:
                        pieces.extend(p["rd"].hist)
                    a = p["new_off"]
                    pieces.append(p["staged"] if p["staged"] is not None else new_ids[a:a + p["n_new"]])
                ids = torch.cat(pieces) if len(pieces) > 1 else pieces[0]
                cu = view("cu_q")
                last_rows = (cu[1:] - 1).long()
                sampled_pre = self.runner.prefill(ids, view("positions"), view("slots"), cu, pre_table, pre_ctx_d,
                                                  last_rows, max_q, stream=self.compute)
                self.stats["prefill_tokens"] += T
            j = 0
            for i, p in enumerate(plan):
                if p["plen"] > 0:
                    first_tok_parts.append(sampled_pre[j:j + 1])
                    j += 1
                else:
                    pend = p["rd"].pending
                    first_tok_parts.append(pend.view(1) if pend is not None
                                           else torch.zeros(1, dtype=torch.int32, device=dev))
            first_tok = torch.cat(first_tok_parts)
            # ---- decode loop, driven on the device (one CUDA-graph replay per step)
            g = self._decode_graph(B, max_blocks) if (self.use_graphs and max_ngen <= self.HIST_MAX) else None
            if g is not None:
                gb = g["bufs"]
                gb["step"].zero_()
                gb["sampled"].zero_()
                gb["hist"].zero_()      # rows past their n_gen read back as 0, as in the eager path
                gb["n_gen"][:B].copy_(view("n_gen"))
                gb["base_pos"][:B].copy_(view("base_pos"))
                gb["first_tok"][:B].copy_(first_tok)
                gb["table"].fill_(-1)
                gb["table"][:, :max_blocks].copy_(table)
                step, sampled, hist_buf = gb["step"], gb["sampled"], gb["hist"]
                def run_step(_g=g):
                    _g["graph"].replay()
                    ops.LAUNCHES[0] += _g["launches"]   # kernels inside the replayed graph
                adv_args = (gb["n_gen"], gb["base_pos"], gb["first_tok"], sampled, gb["table"], gb["tokens"],
                            gb["pos"], gb["slots"], gb["ctx"], hist_buf, hist_buf.shape[1])
            else:
                step = torch.zeros(1, dtype=torch.int32, device=dev)
                hist_buf = torch.zeros(B, max_ngen + 1, dtype=torch.int32, device=dev)
                tokens = torch.empty(B, dtype=torch.int32, device=dev)
                pos_d = torch.empty(B, dtype=torch.int32, device=dev)
                slot_d = torch.empty(B, dtype=torch.int32, device=dev)
                ctx_d = torch.empty(B, dtype=torch.int32, device=dev)
                sampled = torch.zeros(B, dtype=torch.int64, device=dev)   # argmax keys
                adv_args = (view("n_gen"), view("base_pos"), first_tok, sampled, table, tokens, pos_d, slot_d,
                            ctx_d, hist_buf, max_ngen + 1)

                def run_step():
                    ops.decode_advance(step, B, adv_args[0], adv_args[1], adv_args[2], sampled, table, BT, tokens,
                                       pos_d, slot_d, ctx_d, hist_buf, max_ngen + 1, stream=self.compute)
                    self.runner.decode(tokens, pos_d, slot_d, table, ctx_d, stream=self.compute, keys_out=sampled)
            retire_at = set(n_gen)
            retire_ev = {}
            for s in range(max_ngen):
                run_step()
                if (s + 1) in retire_at:
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(self.compute)
                    retire_ev[s + 1] = ev
            # final advance: records every row's pending (next) token
            n_gen_d, base_d, first_d, keys_d, table_d, tok_d, pos_dd, slot_dd, ctx_dd, hist_d, hstride = adv_args
            ops.decode_advance(step, B, n_gen_d, base_d, first_d, keys_d, table_d, BT, tok_d, pos_dd, slot_dd,
                               ctx_dd, hist_d, hstride, stream=self.compute)
            hist = hist_buf[:B, : max_ngen + 1].clone()
            self.stats["decode_steps"] += max_ngen
            self.stats["decode_row_steps"] += sum(n_gen)
            # pending token recorded by the final advance
            done_ev = torch.cuda.Event(enable_timing=True)
            done_ev.record(self.compute)
            # result readback (the batch's generated tokens) into pinned memory
            hist_host = torch.empty(hist.shape, dtype=torch.int32, pin_memory=True)
            hist_host.copy_(hist, non_blocking=True)
            self.stats["d2h_bytes"] += hist.numel() * 4
            rb = torch.cuda.Event()
            rb.record(self.compute)
            self.results.append((rb, hist_host))
            if len(self.results) > RESULTS_SOFT_LIMIT:   # nobody drains: keep only what is in flight
                self.results = [(e, h) for e, h in self.results if not e.query()]
        # ---- host bookkeeping (no sync)
        for i, (m, p) in enumerate(zip(members, plan)):
            rd = p["rd"]
            if p["n_new"] > 0:
                a = offs["new_ids"][0] + p["new_off"]
                rd.hist.append(p["staged"] if p["staged"] is not None else d[a:a + p["n_new"]])
            rd.hist.append(hist[i, : p["n_gen"]])
            rd.hist_len = p["ctx_before"] + p["n_new"] + p["n_gen"]
            rd.pending = hist[i, p["n_gen"]]
            rd.tokens = rd.hist_len
            rd.ready = retire_ev[p["n_gen"]]
            if len(rd.hist) > 8:
                with torch.cuda.stream(self.compute):
                    rd.hist = [torch.cat(rd.hist)]
        self.stats["batches"] += 1
        self.last_batch_events = (t_start, retire_ev, done_ev)
        if not self.measure:
            return None
        done_ev.synchronize()
        return [t_start.elapsed_time(retire_ev[p["n_gen"]]) / 1000.0 for p in plan]

    HIST_MAX = 1024

    def _decode_graph(self, B: int, max_blocks: int):
        """One decode step (advance + full forward + fused sampling) captured
        as a CUDA graph over persistent buffers, keyed by (B, block-table
        width bucket). Replayed once per step; PDL edges are kept."""
        mb = _width_bucket(max_blocks)
        key = (B, mb)
        g = self._graphs.get(key)
        if g is not None:
            return g
        dev = self.device
        i32 = dict(dtype=torch.int32, device=dev)
        bufs = {
            "step": torch.zeros(1, **i32), "n_gen": torch.zeros(B, **i32), "base_pos": torch.zeros(B, **i32),
            "first_tok": torch.zeros(B, **i32), "sampled": torch.zeros(B, dtype=torch.int64, device=dev),
            "table": torch.full((B, mb), -1, **i32), "tokens": torch.zeros(B, **i32), "pos": torch.zeros(B, **i32),
            "slots": torch.full((B,), -1, **i32), "ctx": torch.zeros(B, **i32),
            "hist": torch.zeros(B, self.HIST_MAX + 1, **i32),
        }

        def step():
            ops.decode_advance(bufs["step"], B, bufs["n_gen"], bufs["base_pos"], bufs["first_tok"], bufs["sampled"],
                               bufs["table"], BT, bufs["tokens"], bufs["pos"], bufs["slots"], bufs["ctx"],
                               bufs["hist"], self.HIST_MAX + 1, stream=self.compute)
            self.runner.decode(bufs["tokens"], bufs["pos"], bufs["slots"], bufs["table"], bufs["ctx"],
                               stream=self.compute, keys_out=bufs["sampled"])

        # warm-up (n_gen = 0: every row retired, nothing is written to the pool)
        with torch.cuda.stream(self.compute):
            step()
        self.compute.synchronize()
        if self._graph_pool is None:
            self._graph_pool = torch.cuda.graph_pool_handle()
        graph = torch.cuda.CUDAGraph()
        n0 = ops.LAUNCHES[0]
        with torch.cuda.graph(graph, pool=self._graph_pool, stream=self.compute):
            step()
        g = {"graph": graph, "bufs": bufs, "launches": ops.LAUNCHES[0] - n0}
        ops.LAUNCHES[0] = n0
        self._graphs[key] = g
        return g

    # ------------------------------------------------------------------ end of run

    def reset(self) -> None:
        """Abandon every request and return all blocks (a replay that was
        stopped part-way, e.g. the bench's e2e window)."""
        self.synchronize()
        for rd in self.reqs.values():
            if rd.blocks:
                self.pool.alloc.give(rd.blocks)
        self.reqs.clear()
        self._fences.clear()
        self.results = []

    def drain_results(self) -> list:
        """Hand over (and forget) every batch's (event, pinned tokens) readback."""
        out, self.results = self.results, []
        return out

    def synchronize(self) -> None:
        self.compute.synchronize()
        self.swapper.synchronize()
        self._deferred.clear()

    def audit(self, states) -> None:
        """Device conservation: blocks held == ceil(kv_tokens / 16) for every
        GPU-located request, none otherwise (mirrors kvcache.py:295-307)."""
        held = 0
        for st in states:
            rd = self.reqs.get(st.spec.id)
            nb = len(rd.blocks) if rd else 0
            want = _blocks_for(st.kv_tokens) if _loc(st.cache_location) == "gpu" else 0
            if nb != want:
                raise ProtocolError(f"device blocks drifted for {st.spec.id}: {nb} held, {want} expected")
            held += nb
        if held + self.pool.alloc.free != self.pool.num_blocks:
            raise ProtocolError(f"block leak: {held} held + {self.pool.alloc.free} free != {self.pool.num_blocks}")

    def summary(self) -> dict:
        out = dict(self.stats)
        out["free_blocks"] = self.pool.alloc.free
        out["num_blocks"] = self.pool.num_blocks
        out["kv_bytes_per_token"] = self.pool.bytes_per_token
        return out
