timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "decode_attention" > gpurun_out/pytest_attn.log 2>&1; tail -3 gpurun_out/pytest_attn.log
ASTRAEA_DECODE_ATTN=t timeout 600 python tools/attn_ab.py > gpurun_out/attn_ab_t.log 2>&1
ASTRAEA_DECODE_ATTN=m timeout 600 python tools/attn_ab.py --no-step > gpurun_out/attn_ab_m.log 2>&1
cat gpurun_out/attn_ab_t.log gpurun_out/attn_ab_m.log
