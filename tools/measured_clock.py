"""Run the bench workload under the measured clock N times (B200 durations,
virtual API waits) and print JCT aggregates and the device counters of each
run: shows how the measured-clock schedule varies run to run."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2512_14142_b200 import reference
host = reference.load()   # the unmodified reference package
from paper_2512_14142_b200.gpu import lib as L
from paper_2512_14142_b200.gpu.datapath import KvDataPath
from paper_2512_14142_b200 import plugin
from paper_2512_14142_b200.gpu.engine import GpuEngine
from paper_2512_14142_b200.gpu.model import PRESETS

sys.argv = [sys.argv[0]] + sys.argv[1:]
args = bench.parse()
cfg = PRESETS[args.model]
shard, pred = bench.build_workload(args, 0, 1)
blocks = math.ceil(args.capacity / 16) + 2 * len(shard) + 64
dp = KvDataPath(cfg, num_blocks=blocks, swap_mode=L.SWAP_KERNEL)
for i in range(3):
    pol, mem, scfg = bench.make_run(host, shard, pred, args, cfg.kv_bytes_per_token)
    rep = GpuEngine(shard, pol, pred, mem, scfg, dp, clock="measured").run()
    agg = rep.aggregates()
    print(json.dumps({"run": i, "avg_jct": agg["avg_jct"], "p99_jct": agg["p99_jct"],
                      "req_per_s": plugin.requests_per_second(rep),
                      "device": {k: rep.device[k] for k in ("batches", "prefill_tokens", "decode_steps", "swap_outs",
                                                            "swap_ins", "discards", "recompute_tokens")}}), flush=True)
