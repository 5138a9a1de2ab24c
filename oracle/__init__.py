"""CPU oracle for the B200 image path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (paper_2502_00937_b200/) imports this package.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg use it, and
only as the checker or the timed CPU baseline, never as the thing measured or shipped.

* tiling.py / tile_plan.c : integer tile plan (reference core.py:58-120) — PINNED against the
  reference's own outputs (tests/golden/tiling.json, generator.json, policies.json).
* preprocess.py           : numpy fp32 op-for-op restatement of K1 (builder-defined geometry;
  the reference has no pixel arithmetic) — parity unpinned by the reference.
* encoders.py             : torch fp32 CPU CLIP-ViT and Mllama-vision forward — parity unpinned
  by the reference (it has no encoder); cross-checked layer-by-layer against the independent
  HuggingFace transformers modules in tests/test_oracle_hf.py.
"""
