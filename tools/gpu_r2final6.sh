nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/calibrate.py --out gpurun_out/r2_b200_cost_tables_v7.json > gpurun_out/calib_v7.log 2>&1; tail -c 800 gpurun_out/calib_v7.log
cp gpurun_out/r2_b200_cost_tables_v7.json profiles/r2_b200_cost_tables.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_v10.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_v10.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_v10.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_v10.log
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log; tail -c 400 gpurun_out/bench_v10.log; tail -c 300 gpurun_out/bench_ref_v10.log
