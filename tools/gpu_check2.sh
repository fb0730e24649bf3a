timeout 600 ncu --set full --import-source on --clock-control none -k regex:swap -c 2 -o gpurun_out/ncu_swap python tools/prof_kernels.py swap --ctx 2048 > gpurun_out/ncu_swap.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -c 2500 gpurun_out/bench.log
