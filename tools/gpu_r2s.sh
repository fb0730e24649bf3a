for B in 16 1; do ASTRAEA_TRACE_PHASE=0 timeout 300 python tools/chain_trace.py --batch $B --ctx 673 --layers 16 2>&1 | grep epilogue_us; done
