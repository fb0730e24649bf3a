"""The global multi-replica scheduler (paper_2512_14142_b200/cluster.py) on
CPU: with one replica it IS the reference's run() (report bytes equal the
reference goldens); with N replicas every replica's report equals the
reference run on the requests placed there, placement by free tokens is
deterministic and differs from round-robin, the plugin path (recorder
devices) leaves every replica's bytes unchanged, and two gloo ranks that
each execute only their own replica compute the same placement."""

import hashlib
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

import scenarios
from recorder import Recorder
from paper_2512_14142_b200 import reference
from paper_2512_14142_b200.cluster import ClusterScheduler

ns = reference.load()
HERE = Path(__file__).resolve().parent

ONE_REPLICA = ["fig2/fcfs", "c1/stateful-mlfq/12000/adaptive", "c1b200/6000", "hetero/0/stateful-mlfq",
               "aging/5.0", "c2/12000", "c1/las/3600/adaptive", "noise/0"]


def factory(name):
    """make_replica for scenario ``name``: each replica gets fresh reference
    objects of the scenario's configuration."""
    def make(i):
        _, pol, pred, mem, cfg = scenarios.build(ns, name)
        return pol, pred, mem, cfg
    return make


@pytest.mark.parametrize("name", ONE_REPLICA)
def test_one_replica_is_the_reference_run(name, golden):
    wl = scenarios.build(ns, name)[0]
    rep = ClusterScheduler(ns, wl, 1, factory(name)).run()
    js = rep.replicas[0].to_json()
    assert js == scenarios.run_scenario(ns, name).to_json()
    if name in golden:
        assert hashlib.sha256(js.encode()).hexdigest() == golden[name]["sha256"]


def sub_trace_report(name, wl, placement, k):
    sub = [r for r in wl if placement[r.id] == k]
    _, pol, pred, mem, cfg = scenarios.build(ns, name)
    return ns.run(sub, pol, pred, mem, cfg)


@pytest.mark.parametrize("name,n", [("c2/12000", 2), ("c2/12000", 4), ("c1/stateful-mlfq/12000/adaptive", 3),
                                    ("c1b200/6000", 2)])
@pytest.mark.parametrize("placement", ["free-tokens", "round-robin"])
def test_replicas_equal_reference_runs_of_their_requests(name, n, placement):
    wl = scenarios.build(ns, name)[0]
    rep = ClusterScheduler(ns, wl, n, factory(name), placement=placement).run()
    assert sorted(rep.placement) == sorted(r.id for r in wl)
    assert sum(rep.per_replica_requests) == len(wl)
    for k in range(n):
        if rep.replicas[k] is None:
            assert rep.per_replica_requests[k] == 0
            continue
        assert rep.replicas[k].to_json() == sub_trace_report(name, wl, rep.placement, k).to_json()
    agg = rep.aggregates()
    assert agg["count"] == len(wl) and agg["p99_jct"] >= agg["avg_jct"] > 0


def test_free_token_placement_is_deterministic_and_balances_memory():
    name = "c2/12000"
    wl = scenarios.build(ns, name)[0]
    a = ClusterScheduler(ns, wl, 4, factory(name)).run()
    b = ClusterScheduler(ns, wl, 4, factory(name)).run()
    rr = ClusterScheduler(ns, wl, 4, factory(name), placement="round-robin").run()
    assert a.placement == b.placement
    assert a.placement != rr.placement
    assert all(c > 0 for c in a.per_replica_requests)
    # the first arrivals, with every replica empty, go 0, 1, 2, 3 (ties: fewer requests, lower index)
    first = sorted(wl, key=lambda r: (r.arrival_time, r.id))[:4]
    assert [a.placement[r.id] for r in first] == [0, 1, 2, 3]


def test_recorder_devices_leave_replica_bytes_unchanged():
    name = "c1b200/6000"
    wl = scenarios.build(ns, name)[0]
    host = ClusterScheduler(ns, wl, 2, factory(name)).run()
    recs = [Recorder(), Recorder()]
    dev = ClusterScheduler(ns, wl, 2, factory(name), device_for=lambda i: recs[i]).run()
    assert dev.placement == host.placement
    for k in range(2):
        assert dev.replicas[k].to_json() == host.replicas[k].to_json()
        assert dev.replicas[k].device["batches"] > 0
        launched = {rid for e in recs[k].log if e[0] == "batch" for rid, *_ in e[1:]}
        assert launched == {rid for rid, r in host.placement.items() if r == k}


def test_configuration_errors():
    name = "c2/12000"
    wl = scenarios.build(ns, name)[0]
    with pytest.raises(ns.ConfigError):
        ClusterScheduler(ns, wl, 0, factory(name))
    with pytest.raises(ns.ConfigError):
        ClusterScheduler(ns, wl, 2, factory(name), placement="random")
    with pytest.raises(ns.ConfigError):
        ClusterScheduler(ns, wl, 2, factory(name), clock="measured")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_gloo_ranks_run_one_cluster_schedule(tmp_path):
    """Each rank runs the whole cluster schedule on the host and attaches a
    device (recorder) to its own replica only: the placements agree across
    ranks and each rank's replica report equals the host-only cluster's."""
    out = tmp_path / "gathered.json"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    procs = [subprocess.Popen([sys.executable, str(HERE / "mp_cluster_worker.py"), str(r), "2", str(out)], env=env)
             for r in range(2)]
    for p in procs:
        assert p.wait(timeout=180) == 0
    g = json.loads(out.read_text())
    name = "c2/12000"
    wl = scenarios.build(ns, name)[0]
    host = ClusterScheduler(ns, wl, 2, factory(name)).run()
    digest = hashlib.sha256(json.dumps(sorted(host.placement.items())).encode()).hexdigest()
    for rank in range(2):
        assert g[rank]["placement"] == digest
        assert g[rank]["report"] == host.replicas[rank].to_json()
        assert g[rank]["batches"] > 0
