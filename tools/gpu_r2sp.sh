fmt='
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print(d["tokens"], "qkv %.1f o %.1f gu %.1f down %.1f attn %.1f | fwd %.2f ms"%(d["qkv_us"],d["o_us"],d["gu_us"],d["down_us"],d["attn_us"],d["forward_ms"]))
'
for cfg in "ASTRAEA_ROWS_SPLITS=2" "ASTRAEA_ROWS_SPLITS=3" "ASTRAEA_ROWS_SPLITS=4" "ASTRAEA_ROWS_SPLITS=2"; do
  echo "== $cfg"; env $cfg timeout 600 python tools/prefill_ops.py --tokens 64 96 128 --reps 10 2>&1 | python -c "$fmt"
done
