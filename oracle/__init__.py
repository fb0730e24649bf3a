"""CPU oracle for the B200 data path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only
as the checker or the timed CPU baseline -- never as the product path.

What is pinned and how:

* Scheduling order and KV-policy decisions: pinned to the reference itself
  (pkg/src/agentsched, run unmodified in the build container by
  tests/golden/make_golden.py; 79 scenarios, SHA-256 of RunReport.to_json).
* KV block bytes (swap gather/scatter, table build, append slots): integer /
  byte work restated in numpy here (``kvpool_ref``); exact equality required.
* Attention, GEMM, RMSNorm, RoPE, SiLU, the Llama forward: fp32 torch on CPU
  (``attention_ref``, ``llama_ref``). The reference has no model (SURVEY.md
  section 0), so these restate Llama-3; the restatement is **pinned to
  Hugging Face transformers' ``LlamaForCausalLM``** (5.5.0, in the image) on
  identical weights -- logits, greedy continuation, the paged decode over
  HF's cached K/V and the TP restatement agree to fp32 rounding
  (tests/test_oracle_pin.py). Device tolerance: north star's 1e-2 relative.
"""
