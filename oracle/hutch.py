"""Hutchinson trace estimator (oracle; test infrastructure).

The plain definition of Eq. hutch:
    Tr(G) ~ (1/q) sum_{i=1..q} u_i^T G u_i,   u_i with i.i.d. Rademacher entries,
which is unbiased for any square G (u^T G u = u^T ((G + G^T)/2) u).  The probes are an
INPUT (`probe(rows, p)` -> the +-1 entries of probe p at original point indices `rows`),
so the oracle and the CUDA path can be compared on identical probes.  Returns the
estimate and its standard error (sample standard deviation / sqrt(q)).
Reading R-Q: the sample count is q ("M" in P:804 is a notation slip).
"""
from __future__ import annotations

import numpy as np


def hutch_trace(apply_G, n: int, q: int, probe):
    """(estimate, standard error) of Tr(G) from q Rademacher probes; apply_G maps n x k -> n x k."""
    rows = np.arange(n)
    U = np.stack([probe(rows, p) for p in range(q)], axis=1)     # n x q
    GU = apply_G(U)
    s = np.einsum("ij,ij->j", U, GU)                             # u_p^T G u_p
    est = float(np.mean(s))
    se = float(np.std(s, ddof=1) / np.sqrt(q)) if q > 1 else float("inf")
    return est, se
