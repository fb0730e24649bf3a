# ncu captures of the main kernels (one GPU). Outputs under gpurun_out/.
set -x
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:gemm_chain -s 2 -c 1 -o gpurun_out/ncu_chain_b1 python tools/prof_kernels.py chain --batch 1 > gpurun_out/ncu_chain_b1.log 2>&1
timeout 600 $NCU -k regex:gemm_chain -s 2 -c 1 -o gpurun_out/ncu_chain_b16 python tools/prof_kernels.py chain --batch 16 > gpurun_out/ncu_chain_b16.log 2>&1
timeout 600 $NCU -k regex:decode_mma -s 2 -c 1 -o gpurun_out/ncu_attn_b16 python tools/prof_kernels.py attn --batch 16 > gpurun_out/ncu_attn.log 2>&1
timeout 600 $NCU -k regex:gemm_rows -s 4 -c 2 -o gpurun_out/ncu_prefill python tools/prof_kernels.py prefill --tokens 2048 > gpurun_out/ncu_prefill.log 2>&1
timeout 600 $NCU -k regex:swap -c 2 -o gpurun_out/ncu_swap python tools/prof_kernels.py swap --ctx 2048 > gpurun_out/ncu_swap.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_step_b1.csv python tools/prof_step.py --layers-path --steps 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
