for mp in 1 2 3 4; do echo "== min_pages $mp"; ASTRAEA_CHAIN_ATTN_MIN_PAGES=$mp timeout 600 python tools/attn_ab.py --batch 1 2 4 --no-step-standalone 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"; done
for e in 0 1; do echo "== attn_early $e"; ASTRAEA_CHAIN_ATTN_EARLY=$e timeout 600 python tools/attn_ab.py --batch 1 --no-step-standalone 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['batch'], 'fused %.3f ms (%.3f)'%(d['step_ms_fused'], d['step_frac_fused']))
"; done
