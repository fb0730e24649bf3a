"""8B-shape (2 layers) prefill logits vs the oracle for a few prompts: the
noise floor of the 1e-2 bar (run once per ASTRAEA_PREFILL_ATTN value)."""
import os
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
from test_gpu_8b import CFG, KvPool, LlamaRunner, LlamaWeights, llama_ref, prefill, rel, segment_token_ids
torch.backends.cuda.matmul.allow_tf32 = False
w = LlamaWeights(CFG, seed=11)
logical = w.to_cpu_dict(device="cuda")
out = []
for name, T in [("p512", 512), ("q512", 512), ("r300", 300), ("s1000", 1000)]:
    pool = KvPool(CFG, 80)
    runner = LlamaRunner(w, pool)
    ids = segment_token_ids(name, 1, T, CFG.vocab)
    tok, logits = prefill(runner, [ids], [list(range(3, 3 + (T + 15) // 16))])
    with torch.no_grad():
        ref = llama_ref.forward(logical, CFG, ids, last_only=True)[0]
        ref32 = llama_ref.forward(logical, CFG, ids, last_only=True, bf16_points=False)[0]
    out.append((name, T, round(rel(logits[0], ref), 5), round(rel(logits[0], ref32), 5), round(rel(ref, ref32), 5)))
print(os.environ.get("ASTRAEA_PREFILL_ATTN", "t"), out)
