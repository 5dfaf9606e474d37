"""CPU oracle for the block-diffusion decode hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/inferix/{attention,kvcache,engine,parallel}.py`).
Every function cites the reference file:line it follows.

Rules (enforced by review):
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs
    (`cpu_baseline`, `--impl reference`) may import anything under `oracle/`.
  * It is the checker, never the thing measured or shipped: the product package
    `paper_2511_20714_b200` never imports it and has no CPU fallback.

Pinning: the restatement is checked against golden vectors produced by running
the *live* reference in the build container (`tests/golden/make_golden.py`,
fixtures committed under `tests/golden/`). 3D RoPE is not part of the reference
(`attention.py:6`, `SPEC.md:90`), so `oracle.rope` is "parity unpinned".
"""
