"""ORACLE — plain, slow, fp64 CPU implementation of gamma-EigenGame
(arxiv 2206.04993, PAPER.md).  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import, call or execute anything in this package.
The product path (`paper_2206_04993_b200/`) never imports it and shares no
code, header, helper or constant generator with it; the only common module is
`synth/` (seeded input draws, none of the method's arithmetic).

Every function cites the PAPER.md passage it follows ("PAPER.md:<line>",
section / equation / algorithm).  Numerics are float64 numpy; library
primitives (matmul, triangular solve, numpy.linalg.eigh where stated) serve
as steps, with no blocking, fusion or reordering beyond the paper's own
definitions.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): every public function is
pinned to something other than itself — the paper's printed numbers
(Appendix B 2x2 example, Fig. 1 caption), closed forms (2x2 quadratic,
1-D CCA correlation), the Appendix B "Equivalence to EigenGame Unloaded"
formula, the fixed-point lemma, finite differences of the utility,
library eigensolvers, brute force / power iteration at d <= 16, Monte-Carlo
unbiasedness (Appendix C) and Theorem 1 convergence.  No function is
"parity unpinned" (see DESIGN.md §Oracle pins for the table).
"""
from . import linalg, game, estimators, metrics  # noqa: F401
