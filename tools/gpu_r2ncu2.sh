NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:gemm_rows -s 4 -c 4 -o gpurun_out/r2_ncu_rows_staged_t128 python tools/prof_kernels.py prefill --tokens 128 > gpurun_out/ncu_rows2.log 2>&1
ls -la gpurun_out/r2_ncu_rows_staged_t128.ncu-rep
