"""Tensor parallelism (BASELINE C5): the weight sharding
the GPU ranks use, checked on CPU with world_size 2 over gloo -- the
sharded forward (partial sums all-reduced after the O and down projections,
vocabulary-sliced lm_head gathered) equals the unsharded model."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

from paper_2512_14142_b200.gpu.model import PRESETS, LlamaConfig  # noqa: E402
from paper_2512_14142_b200.gpu.tp import shard_config, shard_logical  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_tensor_parallel_forward_equals_unsharded(tmp_path):
    out = tmp_path / "tp.json"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    procs = [subprocess.Popen([sys.executable, str(HERE / "mp_tp_worker.py"), str(r), "2", str(out)], env=env)
             for r in range(2)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = json.loads(out.read_text())
    assert res["rel"] < 1e-2 and res["argmax_equal"], res


def test_llama3_70b_tp8_shard_shape_is_the_preset():
    full = LlamaConfig("llama3-70b", 80, 8192, 64, 8, 128, 28672, 128256)
    sc = shard_config(full, 8)
    preset = PRESETS["llama3-70b-tp8"]
    assert (sc.num_layers, sc.hidden, sc.num_q_heads, sc.num_kv_heads, sc.head_dim, sc.ffn) == \
        (preset.num_layers, preset.hidden, preset.num_q_heads, preset.num_kv_heads, preset.head_dim, preset.ffn)
    assert sc.kv_bytes_per_token == 40960   # per GPU


def test_shards_partition_every_matrix():
    """Concatenating the ranks' slices rebuilds every sharded matrix."""
    import mp_tp_worker
    cfg = mp_tp_worker.CFG
    wd = mp_tp_worker.full_weights()
    world = 2
    shards = [shard_logical(wd, cfg, r, world) for r in range(world)]
    D, Hq, Hkv, F = cfg.head_dim, cfg.num_q_heads, cfg.num_kv_heads, cfg.ffn
    for li, lw in enumerate(wd["layers"]):
        sl = [s["layers"][li] for s in shards]
        q = torch.cat([x["wqkv"][: Hq // world * D] for x in sl])
        k = torch.cat([x["wqkv"][Hq // world * D:(Hq + Hkv) // world * D] for x in sl])
        v = torch.cat([x["wqkv"][(Hq + Hkv) // world * D:] for x in sl])
        assert torch.equal(torch.cat([q, k, v]), lw["wqkv"])
        assert torch.equal(torch.cat([x["wo"] for x in sl], dim=1), lw["wo"])
        assert torch.equal(torch.cat([x["wdown"] for x in sl], dim=1), lw["wdown"])
        gate = torch.cat([x["wgu"][: F // world] for x in sl])
        up = torch.cat([x["wgu"][F // world:] for x in sl])
        assert torch.equal(torch.cat([gate, up]), lw["wgu"])
    assert torch.equal(torch.cat([s["lm_head"] for s in shards]), wd["lm_head"])
