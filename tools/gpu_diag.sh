timeout 600 python tools/diag_determinism.py > gpurun_out/diag_pdl1.log 2>&1
ASTRAEA_PDL=0 timeout 600 python tools/diag_determinism.py > gpurun_out/diag_pdl0.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_b1.csv python tools/profile_step.py --batch 1 --ctx 900 --steps 2 --prefill 512 > gpurun_out/ncu_b1.log 2>&1
python tools/launches.py gpurun_out/launch_b1.csv > gpurun_out/launch_b1_summary.txt 2>&1
cat gpurun_out/diag_pdl1.log gpurun_out/diag_pdl0.log | tail -30
