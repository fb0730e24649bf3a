for n in 0 8 16 32 48; do echo "== L2PRE $n"; ASTRAEA_CHAIN_L2PRE=$n timeout 300 python tools/attn_ab.py --batch 1 4 16 32 --ctx 540 --no-step-standalone 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['batch'], '%.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"; done
for n in 0 16; do echo "== L2PRE $n (repeat)"; ASTRAEA_CHAIN_L2PRE=$n timeout 300 python tools/attn_ab.py --batch 1 16 --ctx 540 --no-step-standalone 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['batch'], '%.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"; done
