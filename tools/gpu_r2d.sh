timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k swap > gpurun_out/pytest_swap.log 2>&1; tail -3 gpurun_out/pytest_swap.log
timeout 600 python tools/swap_load.py --batch 4 --ctas 32 > gpurun_out/swap_load_b4.log 2>&1
timeout 600 python tools/swap_load.py --batch 16 --ctas 32 > gpurun_out/swap_load_b16.log 2>&1
timeout 600 python tools/swap_load.py --batch 4 --ctas 32 --tokens 2300 --ctx 2000 > gpurun_out/swap_load_b4_2300.log 2>&1
grep -v modes gpurun_out/swap_load_b*.log
