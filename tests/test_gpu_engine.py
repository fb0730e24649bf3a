"""GPU engine parity: with the data path executing every plan on the B200
(prefill, decode, swaps, discards), the model-clock RunReport is
byte-identical to the reference's golden report, and the device pool's
block accounting mirrors the host token accounting at every batch."""

import hashlib

import pytest

import scenarios
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a B200")]

from gpu_util import datapath_for  # noqa: E402
from paper_2512_14142_b200 import plugin, reference  # noqa: E402
from paper_2512_14142_b200.gpu.engine import GpuEngine  # noqa: E402

host = reference.load()   # the unmodified reference package

SCENARIOS = ["fig2/fcfs", "c1/stateful-mlfq/12000/adaptive", "c1b200/6000", "hetero/0/stateful-mlfq",
             "c1/fcfs/3600/adaptive", "aging/5.0", "c1cal/6000"]


@pytest.mark.parametrize("name", SCENARIOS)
@pytest.mark.parametrize("swap_mode", [2])   # the default: staged
def test_model_clock_report_matches_reference(name, swap_mode, golden):
    wl, pol, pred, mem, cfg = scenarios.build(host, name)
    dp = datapath_for(mem.capacity_tokens, swap_mode=swap_mode)
    rep = GpuEngine(wl, pol, pred, mem, cfg, dp, clock="model").run()
    assert hashlib.sha256(rep.to_json().encode()).hexdigest() == golden[name]["sha256"]
    dev = rep.device
    assert dev["free_blocks"] == dev["num_blocks"]
    decisions = golden[name]["kv_decisions"]
    assert dev["swap_outs"] == decisions.get("swap:estimated", 0)
    assert dev["discards"] == decisions.get("discard:estimated", 0) + decisions.get("discard:deadlock-evicted", 0)


@pytest.mark.parametrize("swap_mode", [0, 1])   # zero-copy SM kernel, per-block 2-D DMA
def test_other_swap_modes_engine(swap_mode):
    name = "c1b200/3600"
    wl, pol, pred, mem, cfg = scenarios.build(host, name)
    dp = datapath_for(mem.capacity_tokens, swap_mode=swap_mode)
    rep = GpuEngine(wl, pol, pred, mem, cfg, dp).run()
    assert rep.device["swap_ins"] > 100 and rep.device["free_blocks"] == rep.device["num_blocks"]


def test_measured_clock_produces_valid_report():
    wl, pol, pred, mem, cfg = scenarios.build(host, "c1b200/6000")
    dp = datapath_for(mem.capacity_tokens)
    rep = GpuEngine(wl, pol, pred, mem, cfg, dp, clock="measured").run()
    assert host.audit_time_decomposition(rep) <= 1e-9
    host.audit_waste_log(rep)
    assert all(r.total_compute > 0 for r in rep.per_request)
    assert plugin.requests_per_second(rep) > 0


def test_graph_and_eager_decode_paths_agree():
    """CUDA-graph decode steps produce exactly the tokens of eager launches."""
    name = "c1b200/6000"
    toks = {}
    for graphs in (True, False):
        wl, pol, pred, mem, cfg = scenarios.build(host, name)
        dp = datapath_for(mem.capacity_tokens)
        dp.use_graphs = graphs
        GpuEngine(wl, pol, pred, mem, cfg, dp).run()
        toks[graphs] = [h.cpu().tolist() for _, h in dp.drain_results()]
    assert toks[True] == toks[False]


@pytest.fixture(scope="module")
def w8b():
    from paper_2512_14142_b200.gpu.model import PRESETS, LlamaWeights
    return LlamaWeights(PRESETS["llama3-8b"], seed=0)


@pytest.mark.parametrize("name", ["c2/12000", "c2/40000"])
def test_8b_engine_c2_report_matches_reference(name, golden, w8b):
    """The bench's model (Llama-3-8B shape) executing every plan of the C2
    trace (64 requests, the reference's default tables, 131,072 B/token):
    the report is byte-identical to the reference's golden, the device saw
    the golden's swap and discard decisions, and every block came back."""
    from paper_2512_14142_b200.gpu.model import PRESETS
    wl, pol, pred, mem, cfg = scenarios.build(host, name)
    dp = datapath_for(mem.capacity_tokens, model="llama3-8b", weights=w8b)
    assert dp.pool.bytes_per_token == 131072
    rep = GpuEngine(wl, pol, pred, mem, cfg, dp, clock="model").run()
    assert hashlib.sha256(rep.to_json().encode()).hexdigest() == golden[name]["sha256"]
    dev = rep.device
    assert dev["free_blocks"] == dev["num_blocks"] and dev["decode_steps"] > 1000
    decisions = golden[name]["kv_decisions"]
    assert dev["swap_outs"] == decisions.get("swap:estimated", 0)
    assert dev["discards"] == decisions.get("discard:estimated", 0) + decisions.get("discard:deadlock-evicted", 0)
    assert PRESETS["llama3-8b"].kv_bytes_per_token == 131072


def test_calibration_tables_load_into_the_reference_predictor():
    """gpu/calibrate.py on the tiny model: every table entry is a positive
    device time, decode is timed from a CUDA graph replay, and the tables load
    into the reference's ServiceTimePredictor (predictor.py:47-66)."""
    from paper_2512_14142_b200.gpu import calibrate
    dp = datapath_for(4096, model="tiny")
    cal = calibrate.calibrate(dp, prefill_points=(32, 64), decode_batches=(1, 2), decode_ctx=48, swap_tokens=64)
    prof = cal["predictor"]["prefill_profile"]
    assert all(t > 0 for _, t in prof) and all(a[1] <= b[1] for a, b in zip(prof, prof[1:]))
    assert set(cal["decode_step_seconds_by_batch"]) == {"1", "2"}
    assert all(v > 0 for v in cal["decode_step_seconds_by_batch"].values())
    assert cal["swap_bandwidth_tokens_per_s"] > 0 and cal["swap"]["mode"] == "staged"
    pred = calibrate.predictor_from_calibration(host, cal)
    assert pred.to_config()["prefill_profile"][0][0] == 32
