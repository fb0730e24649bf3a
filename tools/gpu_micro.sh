rm -f gpurun_out/micro.log
for v in "0 1" "0 2"; do
set -- $v
echo "kvprefetch=$1 minpages=$2" >> gpurun_out/micro.log
ASTRAEA_CHAIN_KV_PREFETCH=$1 ASTRAEA_CHAIN_ATTN_MIN_PAGES=$2 timeout 300 python tools/step_timing.py --batch 1 4 16 --l2 0 2>&1 | grep layers >> gpurun_out/micro.log
done
ASTRAEA_CHAIN_KV_PREFETCH=0 timeout 300 python tools/chain_trace.py --layers 16 >> gpurun_out/micro.log 2>&1
cat gpurun_out/micro.log
