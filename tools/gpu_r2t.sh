timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_8b.py -x -q 2>&1 | tail -2
timeout 600 python tools/prefill_ops.py --tokens 128 256 512 2048 --reps 10 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['tokens'], 'qkv %.1f o %.1f gu %.1f down %.1f attn %.1f | fwd %.2f ms'%(d['qkv_us'],d['o_us'],d['gu_us'],d['down_us'],d['attn_us'],d['forward_ms']))
"
timeout 600 python tools/prefill_ops.py --tokens 32 128 512 --ctx-before 1000 --reps 10 2>&1 | grep "^{" > gpurun_out/prefill_ops_r2.log
