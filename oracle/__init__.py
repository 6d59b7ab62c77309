"""CPU oracle for the Ozaki scheme on integer matrix units (arXiv 2306.11975).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product (``paper_2306_11975_b200``) never imports it and shares
no code with it.

Parity status per function:
  slice_width / split / int_gemm / level_sums / dgemm(mode L, mode P) /
  dd_gemm -- all pinned by tests/test_oracle_*.py against paper/SPEC worked
  examples, exact rational (fractions.Fraction) arithmetic, big-integer brute
  force, closed forms and invariants.  No function is "parity unpinned".
"""
from .oracle import *  # noqa: F401,F403
