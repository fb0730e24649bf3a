fmt='
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print(d["tokens"], "qkv %.1f o %.1f gu %.1f down %.1f attn %.1f | fwd %.2f ms"%(d["qkv_us"],d["o_us"],d["gu_us"],d["down_us"],d["attn_us"],d["forward_ms"]))
'
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_8b.py tests/test_gpu_engine.py 2>&1 | tail -2
timeout 300 python tools/rows_trace.py --tokens 128 --op qkv 2>&1 | tail -1
timeout 600 python tools/prefill_ops.py --tokens 128 256 512 2048 --reps 10 2>&1 | python -c "$fmt"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf2048.csv python tools/prefill_launches.py --tokens 2048 > /dev/null 2>&1
python tools/prefill_launches.py --summarise gpurun_out/pf2048.csv | head -20
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf128.csv python tools/prefill_launches.py --tokens 128 > /dev/null 2>&1
python tools/prefill_launches.py --summarise gpurun_out/pf128.csv | head -20
