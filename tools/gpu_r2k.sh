nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:gemm_chain -s 2 -c 1 -o gpurun_out/r2_ncu_chain_b1 python tools/prof_kernels.py chain --batch 1 --ctx 673 > /dev/null 2>&1
timeout 600 $NCU -k regex:gemm_chain -s 2 -c 1 -o gpurun_out/r2_ncu_chain_b16 python tools/prof_kernels.py chain --batch 16 --ctx 673 > /dev/null 2>&1
timeout 600 $NCU -k regex:prefill_tc -s 32 -c 1 -o gpurun_out/r2_ncu_prefill_tc python tools/prof_kernels.py prefill --tokens 2048 > /dev/null 2>&1
timeout 600 $NCU -k regex:decode_tma -s 2 -c 1 -o gpurun_out/r2_ncu_decode_tma_b16 python tools/prof_kernels.py attn --batch 16 --ctx 673 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-extras --measured-runs 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ls -la gpurun_out/*.ncu-rep
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 2500 gpurun_out/bench.log; tail -c 600 gpurun_out/bench_ref.log
