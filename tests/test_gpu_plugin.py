"""The unmodified reference engine (baseline/_ref, travels to the GPU box)
with the B200 data path attached through paper_2512_14142_b200.plugin:
report bytes equal the golden ones, every device transition executes, and
the device pool is fully returned."""

import hashlib
import sys
from pathlib import Path

import pytest

import scenarios
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a B200")]

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.mark.skipif(not (REF / "agentsched").exists(), reason="reference install (baseline/_ref) absent")
@pytest.mark.parametrize("name", ["c1b200/6000", "hetero/0/stateful-mlfq"])
def test_unmodified_reference_drives_the_b200_path(name, golden):
    sys.path.insert(0, str(REF))
    import agentsched
    from gpu_util import datapath_for
    from paper_2512_14142_b200.plugin import run_reference_on_gpu
    wl, pol, pred, mem, cfg = scenarios.build(agentsched, name)
    dp = datapath_for(mem.capacity_tokens)
    rep = run_reference_on_gpu(agentsched, dp, wl, pol, pred, mem, cfg)
    assert hashlib.sha256(rep.to_json().encode()).hexdigest() == golden[name]["sha256"]
    s = dp.summary()
    assert s["free_blocks"] == s["num_blocks"]
    assert s["batches"] > 0 and s["decode_steps"] > 0
    assert s["swap_outs"] == golden[name]["kv_decisions"].get("swap:estimated", 0)
