"""CPU oracle for the B200 data path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only
as the checker or the timed CPU baseline -- never as the product path.

What is pinned and how:

* Scheduling order and KV-policy decisions: pinned to the reference itself
  (pkg/src/agentsched, run unmodified in the build container by
  tests/golden/make_golden.py; 76 scenarios, SHA-256 of RunReport.to_json).
* KV block bytes (swap gather/scatter, table build, append slots): integer /
  byte work restated in numpy here (``kvpool_ref``); exact equality required.
* Attention, GEMM, RMSNorm, RoPE, SiLU, the Llama forward: fp32 torch on CPU
  (``attention_ref``, ``llama_ref``). **Parity unpinned**: the reference has
  no model, no tensors and no dependency implementing one (SURVEY.md
  section 0, pyproject dependencies = []), so these restate the standard
  Llama-3 architecture; the tolerance is the north star's 1e-2 relative.
"""
