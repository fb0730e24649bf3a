timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill" > gpurun_out/pytest_ptc.log 2>&1; tail -15 gpurun_out/pytest_ptc.log
timeout 600 python tools/prefill_ops.py --tokens 128 512 2048 > gpurun_out/prefill_ops_tc.log 2>&1
timeout 600 python tools/prefill_ops.py --tokens 32 128 512 --ctx-before 1000 >> gpurun_out/prefill_ops_tc.log 2>&1
ASTRAEA_PREFILL_ATTN=m timeout 600 python tools/prefill_ops.py --tokens 2048 >> gpurun_out/prefill_ops_tc.log 2>&1
python -c "
import json
for l in open('gpurun_out/prefill_ops_tc.log'):
  if l.startswith('{'):
    d=json.loads(l); print(d['tokens'], d['ctx_before'], 'attn %.1f us %.0f TF/s'%(d['attn_us'], d['attn_tflops']), 'fwd %.2f ms'%d['forward_ms'])
  else: print(l[:300])
"
