"""Worker for tests/test_tp.py: one gloo rank of a tensor-parallel forward
(CPU, fp32 restatement) of the shard that paper_2512_14142_b200.gpu.tp
assigns it."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import llama_ref  # noqa: E402
from paper_2512_14142_b200.gpu.model import LlamaConfig, LlamaWeights  # noqa: E402
from paper_2512_14142_b200.gpu.tp import shard_config, shard_logical  # noqa: E402

CFG = LlamaConfig("tp-test", 2, 256, 4, 2, 64, 512, 1024)


def full_weights():
    return LlamaWeights(CFG, device="cpu", seed=11).to_cpu_dict()


if __name__ == "__main__":
    rank, world, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wd = full_weights()
    shard = shard_logical(wd, CFG, rank, world)
    sc = shard_config(CFG, world)
    assert shard["layers"][0]["wqkv"].shape[0] == sc.qkv_dim and shard["lm_head"].shape[0] == sc.vocab
    ids = [(7 * i + 3) % CFG.vocab for i in range(19)]
    logits = llama_ref.forward_tp(shard, CFG, ids, rank, world, dist.all_reduce, dist.all_gather)
    if rank == 0:
        ref = llama_ref.forward(wd, CFG, ids)
        err = float((logits - ref).norm() / ref.norm())
        Path(out).write_text(json.dumps({"rel": err, "argmax_equal": bool((logits.argmax(-1) == ref.argmax(-1)).all())}))
    dist.barrier()
    dist.destroy_process_group()
