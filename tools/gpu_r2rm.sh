fmt='
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print(d["tokens"], "qkv %.1f o %.1f gu %.1f down %.1f attn %.1f | fwd %.2f ms"%(d["qkv_us"],d["o_us"],d["gu_us"],d["down_us"],d["attn_us"],d["forward_ms"]))
'
for cfg in "ASTRAEA_X=0" "ASTRAEA_ROWS_M=512" "ASTRAEA_ROWS_M=512 ASTRAEA_ROWS_LONGK_M=512" "ASTRAEA_ROWS_M=384 ASTRAEA_ROWS_LONGK_M=384" "ASTRAEA_X=0"; do
  echo "== $cfg"; env $cfg timeout 600 python tools/prefill_ops.py --tokens 320 384 512 --reps 10 2>&1 | python -c "$fmt"
done
ASTRAEA_ROWS_M=512 ASTRAEA_ROWS_LONGK_M=512 timeout 600 python -m pytest -x -q tests/test_gpu_kernels.py -k "gemm or rows" 2>&1 | tail -1
