timeout 600 python tools/prefill_ops.py --tokens 128 512 2048 > gpurun_out/prefill_ops.log 2>&1
timeout 600 python tools/prefill_ops.py --tokens 32 128 512 --ctx-before 1000 >> gpurun_out/prefill_ops.log 2>&1
timeout 600 python tools/prefill_ops.py --tokens 512 2048 --seqs 4 >> gpurun_out/prefill_ops.log 2>&1
cat gpurun_out/prefill_ops.log
