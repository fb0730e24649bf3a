timeout 300 python tools/diag_prefill8b.py
ASTRAEA_PREFILL_ATTN=m timeout 300 python tools/diag_prefill8b.py
