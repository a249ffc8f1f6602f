"""CPU oracle for the DuetServe mixed-iteration hot path (arXiv 2511.04791).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_2511_04791_b200``,
``libduet.so``) imports, links or executes this package; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may.  It shares no code with ``csrc/``: inputs come from
``synth`` (numbers only), everything else here is written from the paper.

Modules
  ``oracle.layer``    — the transformer-layer forward with a paged KV cache
                        (§2) under the readings of DESIGN.md,
                        float64 throughout; per-row causal attention.
  ``oracle.roofline`` — the attention-aware roofline predictor (§4.1)
                        and the partition optimizer (§4.2, Alg. 1),
                        step by step, plus a brute-force exhaustive search.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to
something other than itself: brute-force loops, library special cases
(torch SDPA / rms_norm / silu in float64), closed forms, invariants and the
SPEC.md worked examples.  Functions without such a pin say "parity unpinned".
"""
