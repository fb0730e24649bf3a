# staged rows epilogue: parity + trace + prefill op timings
fmt='
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print(d["tokens"], "qkv %.1f o %.1f gu %.1f down %.1f attn %.1f | fwd %.2f ms"%(d["qkv_us"],d["o_us"],d["gu_us"],d["down_us"],d["attn_us"],d["forward_ms"]))
'
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_8b.py 2>&1 | tail -3
timeout 300 python tools/rows_trace.py --tokens 128 2>&1 | tail -4
for cfg in "ASTRAEA_X=0" "ASTRAEA_ROWS_BN=128" "ASTRAEA_ROWS_LONGK=0"; do
  echo "== $cfg"; env $cfg timeout 600 python tools/prefill_ops.py --tokens 128 256 512 --reps 10 2>&1 | python -c "$fmt"
done
