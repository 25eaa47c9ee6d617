"""CPU oracle for the RSF + peeling GP likelihood path (TEST INFRASTRUCTURE).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import anything under `oracle/`.  The product
path (`paper_1603_08057_b200`) never imports it and shares no code with it.

Parts (each function cites the PAPER.md passage it follows; "P:n" is
/root/reference/PAPER.md line n):
  kernels.py  covariance entries K, dK/dtheta
  dense.py    O1: the plain definition via dense Cholesky (exact up to
              rounding): l(theta), g(theta)
  tree.py     adaptive quadtree
  rsf.py      O2: recursive skeletonization factorization, step by step
              (ID, proxy trick, elimination, apply/solve/sqrt/logdet)
                                                      P:201-283, P:299-308, P:381-389
  peel.py     O2: weak-admissibility matrix peeling
  mle.py      O2: Alg. 1 (l-hat and g-hat)
  hutch.py    Hutchinson estimator (next row f2)
  profile.py  profile likelihood, kriging mean (f3)

Pins (tests/test_oracle_pins.py) tie these to closed forms, brute force and
special cases; see DESIGN.md §3 for the list and for the one part that is
"parity unpinned".
"""
