for n in 2 1 3 4 2; do echo "== MIN_PAGES $n"; ASTRAEA_CHAIN_ATTN_MIN_PAGES=$n timeout 300 python tools/attn_ab.py --batch 1 8 16 32 --ctx 540 --no-step-standalone 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['batch'], '%.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"; done
