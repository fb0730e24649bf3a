"""Worker for tests/test_gpu_tp.py::test_tensor_parallel_engine: one
tensor-parallel rank of the data path (a KvDataPath over its weight and KV
shard with a TpLlamaRunner) executing every plan of a reference schedule; the
ranks share cuda:0 and exchange partial sums over gloo."""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import scenarios  # noqa: E402
from paper_2512_14142_b200 import reference  # noqa: E402
from paper_2512_14142_b200.gpu.datapath import KvDataPath  # noqa: E402
from paper_2512_14142_b200.gpu.engine import GpuEngine  # noqa: E402
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaWeights  # noqa: E402
from paper_2512_14142_b200.gpu.tp import TpLlamaRunner, shard_config, shard_logical  # noqa: E402

if __name__ == "__main__":
    rank, world, name, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ns = reference.load()
    cfg = PRESETS["small"]
    wd = LlamaWeights(cfg, device="cpu", seed=5).to_cpu_dict()
    sc = shard_config(cfg, world)
    w = LlamaWeights.from_logical(sc, shard_logical(wd, cfg, rank, world), device="cuda")
    wl, pol, pred, mem, scfg = scenarios.build(ns, name)
    blocks = -(-mem.capacity_tokens // 16) + len(wl) + 16
    dp = KvDataPath(sc, weights=w, num_blocks=blocks, token_vocab=cfg.vocab,
                    runner_factory=lambda ww, pool: TpLlamaRunner(ww, pool, rank, world))
    dp.use_graphs = False   # gloo collectives cannot be captured (NCCL ones can)
    rep = GpuEngine(wl, pol, pred, mem, scfg, dp).run()
    toks = [h.cpu().tolist() for _, h in dp.drain_results()]
    res = {"sha": hashlib.sha256(rep.to_json().encode()).hexdigest(),
           "tokens": hashlib.sha256(json.dumps(toks).encode()).hexdigest(), "batches": rep.device["batches"],
           "swap_outs": rep.device["swap_outs"], "kv_bytes_per_token": dp.pool.bytes_per_token,
           "free": rep.device["free_blocks"] == rep.device["num_blocks"]}
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    if rank == 0:
        Path(out).write_text(json.dumps(gathered))
    dist.barrier()
    dist.destroy_process_group()
