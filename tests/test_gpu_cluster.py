"""The global multi-replica scheduler with real data paths: two replicas,
each with its own KvDataPath (pool, weights, streams) on the one B200 of the
test box, placed by free tokens. Every replica's report equals the
reference run on the requests placed on it, the device executed every batch
and swap of its replica, and every block came back."""

import pytest

import scenarios
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a B200")]

from gpu_util import datapath_for  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402
from paper_2512_14142_b200.cluster import ClusterScheduler  # noqa: E402

ns = reference.load()


@pytest.mark.parametrize("name", ["c1b200/6000", "c2/12000"])
def test_two_replicas_on_device(name):
    wl = scenarios.build(ns, name)[0]
    mem0 = scenarios.build(ns, name)[3]
    dps = [datapath_for(mem0.capacity_tokens, seed=i) for i in range(2)]

    def make(i):
        _, pol, pred, mem, cfg = scenarios.build(ns, name)
        return pol, pred, mem, cfg

    rep = ClusterScheduler(ns, wl, 2, make, device_for=lambda i: dps[i]).run()
    assert all(n > 0 for n in rep.per_replica_requests)
    for k in range(2):
        sub = [r for r in wl if rep.placement[r.id] == k]
        _, pol, pred, mem, cfg = scenarios.build(ns, name)
        assert rep.replicas[k].to_json() == ns.run(sub, pol, pred, mem, cfg).to_json()
        dev = rep.replicas[k].device
        assert dev["free_blocks"] == dev["num_blocks"] and dev["batches"] > 0
        decisions = rep.replicas[k].audits["waste_log"]
        swaps = sum(1 for e in decisions if e["chosen"] == "swap")
        assert dev["swap_outs"] == swaps
