timeout 900 python -m pytest tests/test_gpu_8b.py tests/test_gpu_model.py tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_as3.log 2>&1; tail -3 gpurun_out/pytest_as3.log
for v in main as2 as1; do
  if [ $v = main ]; then unset ASTRAEA_LIB; else export ASTRAEA_LIB=$PWD/paper_2512_14142_b200/lib/variants/$v/libastraea_b200.so; fi
  echo "== $v"; timeout 600 python tools/attn_ab.py --batch 1 4 8 16 32 64 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']), 'standalone %.3f ms'%d['step_ms_standalone'], 'attn %.1f us'%d['attn_us'])
  else: print(l.strip()[:200])
"
done
