"""Worker for tests/test_cluster.py: one gloo rank running the whole cluster
schedule with a device (recorder) on its own replica only."""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch.distributed as dist  # noqa: E402

import scenarios  # noqa: E402
from recorder import Recorder  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402
from paper_2512_14142_b200.cluster import ClusterScheduler  # noqa: E402

if __name__ == "__main__":
    rank, world, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ns = reference.load()
    name = "c2/12000"
    wl = scenarios.build(ns, name)[0]

    def make(i):
        _, pol, pred, mem, cfg = scenarios.build(ns, name)
        return pol, pred, mem, cfg

    rec = Recorder()
    rep = ClusterScheduler(ns, wl, world, make, device_for=lambda i: rec if i == rank else None).run()
    mine = {"placement": hashlib.sha256(json.dumps(sorted(rep.placement.items())).encode()).hexdigest(),
            "report": rep.replicas[rank].to_json(), "batches": rep.replicas[rank].device["batches"]}
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        Path(out).write_text(json.dumps(gathered))
    dist.barrier()
    dist.destroy_process_group()
