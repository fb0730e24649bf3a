timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill" 2>&1 | tail -2
timeout 300 python tools/prefill_trace.py --tokens 2048
timeout 300 python tools/prefill_trace.py --tokens 512 --ctx-before 1000
