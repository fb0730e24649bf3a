fmt='
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print(d["tokens"], "qkv %.1f o %.1f gu %.1f down %.1f attn %.1f | fwd %.2f ms"%(d["qkv_us"],d["o_us"],d["gu_us"],d["down_us"],d["attn_us"],d["forward_ms"]))
'
for cfg in "ASTRAEA_GEMM_CHAIN_MAX_M=64" "ASTRAEA_GEMM_CHAIN_MAX_M=32" "ASTRAEA_GEMM_CHAIN_MAX_M=16" "ASTRAEA_GEMM_CHAIN_MAX_M=8" "ASTRAEA_GEMM_CHAIN_MAX_M=64"; do
  echo "== $cfg"; env $cfg timeout 600 python tools/prefill_ops.py --tokens 8 16 24 32 48 64 --reps 10 2>&1 | python -c "$fmt"
done
ASTRAEA_GEMM_CHAIN_MAX_M=16 timeout 600 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_model.py 2>&1 | tail -1
