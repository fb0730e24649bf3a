timeout 2400 python tools/sweep.py pressure --out gpurun_out/r2_sweep_pressure_c3_final.json > gpurun_out/sweep_pressure_final.log 2>&1
timeout 1500 python tools/sweep.py rate --out gpurun_out/r2_sweep_rate_c4_final.json > gpurun_out/sweep_rate_final.log 2>&1
tail -n 3 gpurun_out/sweep_pressure_final.log gpurun_out/sweep_rate_final.log
