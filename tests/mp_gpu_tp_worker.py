"""Worker for tests/test_gpu_tp.py: one tensor-parallel rank running the
sm_100a kernels (TpLlamaRunner) on cuda:0; the ranks share the one GPU and
exchange partial sums over gloo (NCCL needs one GPU per rank)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import llama_ref  # noqa: E402
from paper_2512_14142_b200.gpu.datapath import KvPool  # noqa: E402
from paper_2512_14142_b200.gpu.model import PRESETS, LlamaWeights  # noqa: E402
from paper_2512_14142_b200.gpu.tp import TpLlamaRunner, shard_config, shard_logical  # noqa: E402
from paper_2512_14142_b200.tokens import segment_token_ids  # noqa: E402


def run(rank, world, model="small"):
    cfg = PRESETS[model]
    wd = LlamaWeights(cfg, device="cpu", seed=21).to_cpu_dict()
    sc = shard_config(cfg, world)
    w = LlamaWeights.from_logical(sc, shard_logical(wd, cfg, rank, world), device="cuda")
    pool = KvPool(sc, 32)
    runner = TpLlamaRunner(w, pool, rank, world)
    d = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
    ids = segment_token_ids("tp", 1, 37, cfg.vocab)
    blocks = [5, 9, 2, 30]
    T = len(ids)
    tok, lg = runner.prefill(d(ids), d(list(range(T))), d([blocks[p // 16] * 16 + p % 16 for p in range(T)]),
                             d([0, T]), d([blocks]).view(1, -1), d([T]), torch.tensor([T - 1], device="cuda"), T,
                             want_logits=True)
    out = [(int(tok[0]), lg[0].float().cpu())]
    seq = list(ids) + [int(tok[0])]
    for _ in range(3):
        p = len(seq) - 1
        nt, lg = runner.decode(d([seq[-1]]), d([p]), d([blocks[p // 16] * 16 + p % 16]), d([blocks]).view(1, -1),
                               d([p + 1]), want_logits=True)
        out.append((int(nt[0]), lg[0].float().cpu()))
        seq.append(int(nt[0]))
    torch.cuda.synchronize()
    res = []
    for i, (t, l) in enumerate(out):
        ref = llama_ref.forward(wd, cfg, seq[: T + i])[-1]
        res.append({"rel": float((l - ref).norm() / ref.norm()), "token": t, "ref_token": int(ref.argmax())})
    return res


if __name__ == "__main__":
    rank, world, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    res = run(rank, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    if rank == 0:
        Path(out).write_text(json.dumps(gathered))
    dist.barrier()
    dist.destroy_process_group()
