NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:gemm_rows -s 3 -c 3 -o gpurun_out/r2_ncu_rows_t128 python tools/prof_kernels.py prefill --tokens 128 > gpurun_out/ncu_rows.log 2>&1
ls -la gpurun_out/r2_ncu_rows_t128.ncu-rep
