"""CPU ORACLE FOR THE SMASH H^2 / HSS HOT PATH -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy (+ a tiny C helper for exact FMA), the
reference algorithm of arXiv 1705.05443's Python package (mounted read-only at
/root/reference during development; NOT present on the GPU box):

  * adaptive cluster tree .............. smash/cluster.py:247-353
  * admissibility / pair lists ......... smash/cluster.py:64-85, 374-447
  * Chebyshev/Lagrange basis ........... smash/lowrank.py:103-144 (+ a 3-D extension)
  * strong RRQR / interpolative compr .. smash/lowrank.py:163-255
  * truncated SVD ...................... smash/lowrank.py:265-276
  * H^2 / HSS builders ................. smash/h2.py:25-54, smash/hss.py:219-303
  * node-wise matvec ................... smash/apply.py:26-80
  * kernels log|x-y|, 1/|x-y|, exp(-|x-y|), 1/(x-y)  (the BASELINE kernels; the
    first three are an extension the reference lacks)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg / ``--impl reference`` arm may import this package, and only as the
checker or the timed CPU baseline.  The product package
``paper_1705_05443_b200`` never imports it and has no CPU fallback.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference (with the
SURVEY.md 8(c) monkeypatch extension) in the development container and stores
its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
oracle against them.
"""

from .smash_oracle import *  # noqa: F401,F403
