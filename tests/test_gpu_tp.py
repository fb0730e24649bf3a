"""Tensor-parallel ranks on the B200 kernels (BASELINE C5 path): two ranks
(sharing cuda:0, partial sums exchanged over gloo) run prefill + decode of
the small model with TpLlamaRunner; logits on every rank match the fp32
oracle of the unsharded model, and the greedy tokens agree across ranks."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a B200")]

HERE = Path(__file__).resolve().parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2])
def test_tensor_parallel_ranks_match_oracle(world, tmp_path):
    out = tmp_path / "tp.json"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    procs = [subprocess.Popen([sys.executable, str(HERE / "mp_gpu_tp_worker.py"), str(r), str(world), str(out)],
                              env=env) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    ranks = json.loads(out.read_text())
    for res in ranks:
        for step in res:
            assert step["rel"] < 1e-2, step
    assert all(r == ranks[0] for r in ranks) or all(
        [s["token"] for s in r] == [s["token"] for s in ranks[0]] for r in ranks)


def test_tensor_parallel_engine(tmp_path, golden):
    """C5's deployment shape on the B200 kernels: two tensor-parallel ranks
    (each holding half the heads, FFN and vocabulary, and only its kv-head
    shard of the KV pool) execute every plan of the same reference schedule
    -- prefill, decode, swaps, discards. Both ranks' reports equal the
    reference's golden bytes, they generate identical tokens, and each
    rank's pool holds half a token's KV."""
    name = "c1b200/3600"
    out = tmp_path / "tp_engine.json"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    procs = [subprocess.Popen([sys.executable, str(HERE / "mp_gpu_tp_engine_worker.py"), str(r), "2", name,
                               str(out)], env=env) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=900) == 0
    r0, r1 = json.loads(out.read_text())
    assert r0["sha"] == r1["sha"] == golden[name]["sha256"]
    assert r0["tokens"] == r1["tokens"]
    assert r0["free"] and r1["free"] and r0["swap_outs"] > 0
    from paper_2512_14142_b200.gpu.model import PRESETS
    assert r0["kv_bytes_per_token"] * 2 == PRESETS["small"].kv_bytes_per_token
