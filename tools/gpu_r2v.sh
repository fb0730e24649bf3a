TRACE_FINISHERS=1 ASTRAEA_TRACE_PHASE=0 timeout 300 python tools/chain_trace.py --batch 16 --ctx 673 --layers 16 2>&1 | grep "finishers_by_done" | cut -c1-500
timeout 600 python tools/attn_ab.py --batch 1 8 16 32 --no-step-standalone 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_8b.py -x -q 2>&1 | tail -2
