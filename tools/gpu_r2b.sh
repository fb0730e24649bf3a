timeout 1500 python -m pytest tests/test_gpu_8b.py tests/test_gpu_engine.py tests/test_gpu_model.py -x -q -rs > gpurun_out/pytest_8b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_8b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -n 30 gpurun_out/pytest_8b.log; tail -3 gpurun_out/smoke.log
