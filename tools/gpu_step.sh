timeout 600 python -m pytest tests/test_gpu_step.py -x -q > gpurun_out/step_tests.log 2>&1; echo "rc=$?" >> gpurun_out/step_tests.log
timeout 300 python tools/step_timing.py > gpurun_out/step_timing.log 2>&1; echo "rc=$?" >> gpurun_out/step_timing.log
tail -n 30 gpurun_out/step_tests.log; cat gpurun_out/step_timing.log
