export ASTRAEA_LIB=$PWD/paper_2512_14142_b200/lib/variants/skipkv/libastraea_b200.so
TRACE_FINISHERS=1 ASTRAEA_TRACE_PHASE=3 timeout 300 python tools/chain_trace.py --batch 16 --ctx 673 --layers 16 2>&1 | grep "finishers_by_done" | cut -c1-900
