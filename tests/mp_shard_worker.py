"""Worker for tests/test_multiprocess.py: one gloo rank replaying its shard."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch.distributed as dist  # noqa: E402


def shard_report(rank, world, n_per_rank):
    import argparse
    import bench
    from paper_2512_14142_b200 import reference
    host = reference.load()
    args = argparse.Namespace(qps=4.0, requests=n_per_rank, capacity=6000)
    shard, pred = bench.build_workload(args, rank, world)
    pol, mem, cfg = bench.make_run(host, shard, pred, args, 131072)
    rep = host.Engine(shard, pol, pred, mem, cfg).run()
    return [r.id for r in shard], rep.to_json()


if __name__ == "__main__":
    rank, world, n, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids, js = shard_report(rank, world, n)
    gathered = [None] * world
    dist.all_gather_object(gathered, (ids, js))
    if rank == 0:
        Path(out).write_text(json.dumps(gathered))
    dist.barrier()
    dist.destroy_process_group()
