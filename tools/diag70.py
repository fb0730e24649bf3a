import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import torch
from test_gpu_8b import *
torch.backends.cuda.matmul.allow_tf32 = False
B=8
w = LlamaWeights(CFG70, seed=12)
logical = w.to_cpu_dict(device=DEV)
per = 24
for mode in ["fused", "unchained"]:
    pool = KvPool(CFG70, B * per + 8)
    runner = LlamaRunner(w, pool)
    if mode == "unchained": runner.fuse_attention = False
    lens = [30 + (330 * b) // max(1, B - 1) for b in range(B)]
    seqs = [segment_token_ids(f"s{b}", 1, lens[b], CFG70.vocab) for b in range(B)]
    tables = [list(range(b * per, (b + 1) * per))[::-1] for b in range(B)]
    tok, plog = prefill(runner, seqs, tables)
    pre = []
    for b in range(B):
        with torch.no_grad(): ref = llama_ref.forward(logical, CFG70, seqs[b], last_only=True)[0]
        pre.append(round(rel(plog[b], ref), 5))
    pos = [len(s) for s in seqs]
    for b in range(B): seqs[b] = seqs[b] + [int(tok[b])]
    out, logits = runner.decode(d([s[-1] for s in seqs]), d(pos), d([tables[b][p // 16] * 16 + p % 16 for b, p in enumerate(pos)]), d(tables), d([p + 1 for p in pos]), want_logits=True)
    torch.cuda.synchronize()
    dec=[]; dec32=[]
    for b in range(B):
        with torch.no_grad():
            ref = llama_ref.forward(logical, CFG70, seqs[b], last_only=True)[0]
            ref32 = llama_ref.forward(logical, CFG70, seqs[b], last_only=True, bf16_points=False)[0]
        dec.append(round(rel(logits[b], ref), 5)); dec32.append(round(rel(logits[b], ref32),5))
    print(mode, "prefill", pre, "decode", dec, "decode_vs_fp32", dec32, flush=True)
