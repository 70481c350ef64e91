"""CPU oracle for the 3DGS-LM inner-solver path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference algorithm
(`/root/reference/pkg/src/splatlm/*.py` plus the SPEC-only PCG / Eq. 7
combine).  It exists to CHECK the CUDA product path; it is never the thing
measured or shipped.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.

Pinning: every function is checked against the reference itself (imported
from /root/reference when present, see tests/test_oracle_vs_reference.py) and
against committed golden fixtures generated from the reference
(tests/golden/, script tests/golden/make_golden.py).  PCG / Eq. 7 have no code
in the reference; their restatement is pinned by the SPEC's known-answer
examples and by a dense linear solve.
"""

from .lm_oracle import *  # noqa: F401,F403
