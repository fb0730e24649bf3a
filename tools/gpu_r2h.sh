timeout 300 python tools/chain_trace.py --batch 16 --ctx 673 --layers 16 --per-cta 2>&1 | tail -4
