nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:gemm_chain -s 2 -c 1 -o gpurun_out/r2_ncu_chain_b1 python tools/prof_kernels.py chain --batch 1 --ctx 673 > gpurun_out/ncu1.log 2>&1
timeout 600 $NCU -k regex:gemm_chain -s 2 -c 1 -o gpurun_out/r2_ncu_chain_b16 python tools/prof_kernels.py chain --batch 16 --ctx 673 > gpurun_out/ncu2.log 2>&1
timeout 600 $NCU -k regex:prefill_tc -s 8 -c 1 -o gpurun_out/r2_ncu_prefill_tc python tools/prof_kernels.py prefill --tokens 2048 > gpurun_out/ncu3.log 2>&1
timeout 600 $NCU -k regex:swap_kernel -c 2 -o gpurun_out/r2_ncu_swap python tools/prof_kernels.py swap --ctx 2048 > gpurun_out/ncu4.log 2>&1
timeout 2400 python tools/sweep.py pressure --out gpurun_out/r2_sweep_pressure_c3.json > gpurun_out/sweep_pressure.log 2>&1
timeout 1200 python tools/sweep.py rate --out gpurun_out/r2_sweep_rate_c4.json > gpurun_out/sweep_rate.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench.log; tail -3 gpurun_out/sweep_pressure.log gpurun_out/sweep_rate.log
