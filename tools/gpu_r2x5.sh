fmt='
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print(d["tokens"], "qkv %.1f o %.1f gu %.1f down %.1f attn %.1f | fwd %.2f ms"%(d["qkv_us"],d["o_us"],d["gu_us"],d["down_us"],d["attn_us"],d["forward_ms"]))
'
timeout 1500 python -m pytest -x -q -m gpu tests 2>&1 | tail -3
timeout 300 python tools/rows_trace.py --tokens 128 2>&1 | tail -4
timeout 600 python tools/prefill_ops.py --tokens 128 256 512 2048 --reps 10 2>&1 | python -c "$fmt"
timeout 600 python tools/attn_ab.py --batch 1 16 32 --ctx 673 --no-step-standalone 2>&1 | tail -3
