timeout 900 python -m pytest tests/test_gpu_8b.py tests/test_gpu_model.py tests/test_gpu_step.py -x -q 2>&1 | tail -2
for v in main wbefore main wbefore; do
  if [ $v = main ]; then unset ASTRAEA_LIB; else export ASTRAEA_LIB=$PWD/paper_2512_14142_b200/lib/variants/$v/libastraea_b200.so; fi
  echo "== $v"; timeout 600 python tools/attn_ab.py --batch 1 2 4 8 16 --ctx 540 --no-step-standalone 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"
done
unset ASTRAEA_LIB
timeout 300 python tools/chain_trace.py --batch 1 --ctx 540 --layers 16 2>&1 | grep '"layer": 16' | head -2
