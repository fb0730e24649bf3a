"""Replica sharding over ranks: world_size 2 over gloo on
CPU. Each rank takes the round-robin shard of the (arrival, id)-ordered
trace that bench.py uses and runs the engine on it; the shards are disjoint,
cover the trace, and reproduce a single-process run of each shard byte for
byte (no data-path collective is involved)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import mp_shard_worker

HERE = Path(__file__).resolve().parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_sharding_is_disjoint_and_reproducible(tmp_path):
    out = tmp_path / "gathered.json"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    procs = [subprocess.Popen([sys.executable, str(HERE / "mp_shard_worker.py"), str(r), "2", "6", str(out)],
                              env=env) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=180) == 0
    (ids0, js0), (ids1, js1) = json.loads(out.read_text())
    assert not set(ids0) & set(ids1)
    assert len(ids0) == len(ids1) == 6
    for rank, js in ((0, js0), (1, js1)):
        assert mp_shard_worker.shard_report(rank, 2, 6)[1] == js
