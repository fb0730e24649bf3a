timeout 900 python -m pytest tests/test_gpu_8b.py tests/test_gpu_model.py -x -q 2>&1 | tail -2
export ASTRAEA_LIB=$PWD/paper_2512_14142_b200/lib/variants/small2/libastraea_b200.so
timeout 900 python -m pytest tests/test_gpu_8b.py tests/test_gpu_model.py -x -q 2>&1 | tail -2
for v in main small2 small3 main small2; do
  if [ $v = main ]; then unset ASTRAEA_LIB; else export ASTRAEA_LIB=$PWD/paper_2512_14142_b200/lib/variants/$v/libastraea_b200.so; fi
  echo "== $v"; timeout 600 python tools/attn_ab.py --batch 1 2 4 8 16 --no-step-standalone 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"
done
