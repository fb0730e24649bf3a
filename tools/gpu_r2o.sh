timeout 900 python -m pytest tests/test_gpu_8b.py tests/test_gpu_model.py tests/test_gpu_kernels.py tests/test_gpu_step.py -x -q > gpurun_out/pytest_df.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_df.log; tail -3 gpurun_out/pytest_df.log
for v in main noflow; do
  if [ $v = main ]; then unset ASTRAEA_LIB; else export ASTRAEA_LIB=$PWD/paper_2512_14142_b200/lib/variants/$v/libastraea_b200.so; fi
  echo "== $v"; timeout 600 python tools/attn_ab.py --batch 1 2 4 16 32 --no-step-standalone 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"
done
unset ASTRAEA_LIB
timeout 300 python tools/chain_trace.py --batch 1 --ctx 673 --layers 16 2>&1 | tail -3 | head -1
timeout 300 python tools/chain_trace.py --batch 16 --ctx 673 --layers 16 2>&1 | tail -3 | head -1
