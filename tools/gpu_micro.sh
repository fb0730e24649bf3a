rm -f gpurun_out/micro.log
timeout 600 python -m pytest tests/test_gpu_step.py -x -q 2>&1 | grep -E "Error|assert|passed|failed" | head -20 >> gpurun_out/micro.log
timeout 300 python tools/step_micro.py 1 16 2>&1 | grep -v slowest >> gpurun_out/micro.log
timeout 300 python tools/step_timing.py --batch 1 4 16 --l2 0 >> gpurun_out/micro.log 2>&1
cat gpurun_out/micro.log
