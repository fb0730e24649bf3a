timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/attn_ab.py --batch 1 4 16 32 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']), 'standalone %.3f ms'%d['step_ms_standalone'], 'attn %.1f us'%d['attn_us'])
"
timeout 300 python tools/chain_trace.py --batch 16 --ctx 673 --layers 16 2>&1 | tail -1
timeout 300 python tools/chain_trace.py --batch 1 --ctx 673 --layers 16 2>&1 | tail -1
