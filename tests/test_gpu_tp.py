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
