export ASTRAEA_BENCH_SHARE_GPU=1 ASTRAEA_BENCH_TRACEBACK_S=240
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --measured-runs 1 --no-cpu-baseline --model small > gpurun_out/bench_n2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2.log
grep -v "^\s*$" gpurun_out/bench_n2.log | grep -E "File|Thread|rc=|^\{" | head -60 | cut -c1-200
