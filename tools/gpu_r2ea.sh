for cfg in "ASTRAEA_X=0" "ASTRAEA_CHAIN_ATTN_EARLY=0" "ASTRAEA_CHAIN_KV_PREFETCH=1" "ASTRAEA_X=0"; do echo "== $cfg"; env $cfg timeout 300 python tools/attn_ab.py --batch 1 2 16 --ctx 540 --no-step-standalone 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['batch'], '%.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"; done
