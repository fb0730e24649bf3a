nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python tools/calibrate.py --out gpurun_out/r2_b200_cost_tables_v5.json > gpurun_out/calib_v5.log 2>&1; tail -c 800 gpurun_out/calib_v5.log
cp gpurun_out/r2_b200_cost_tables_v5.json profiles/r2_b200_cost_tables.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_v8.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_v8.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_v8.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_v8.log
timeout 900 python -m pytest -x -q tests/test_gpu_engine.py -k calibration 2>&1 | tail -1
