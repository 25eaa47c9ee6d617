"""Log profile likelihood and kriging mean (next row f3; oracle, test infrastructure).

Plain definitions with dense matrices:
  Eq. prof: z ~ N(mu 1, s2 Sigma(theta)), mu and s2 profiled out,
      l~(theta) = -1/2 log|Sigma| - n/2 log(z^T (Sigma + 1 1^T)^-1 z) + n/2 (log n - 1 - log 2pi)
      g~_i      = -1/2 Tr(Sigma^-1 Sigma_i) + n/2 v^T Sigma_i v / (z^T v),   v = (Sigma + 1 1^T)^-1 z
  reading R-Prof: the paper prints "(log n - 1 - 2 pi)"; maximizing over s2 gives log 2 pi there.
  Remark conditional: E[z' | z] = Sigma_12 Sigma_22^-1 z.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .dense import dense_sigma
from .kernels import Kernel


def dense_profile_eval(kern: Kernel, xy: np.ndarray, z: np.ndarray) -> dict:
    n = len(xy)
    S = dense_sigma(kern, xy)
    c, low = sla.cho_factor(S, lower=True)
    logdet = 2.0 * float(np.sum(np.log(np.diag(c))))
    St = S + np.ones((n, n))                      # Sigma + 1 1^T, formed explicitly
    v = np.linalg.solve(St, z)
    Q = float(z @ v)
    ell = -0.5 * logdet - 0.5 * n * np.log(Q) + 0.5 * n * (np.log(n) - 1.0 - np.log(2.0 * np.pi))
    Sinv = sla.cho_solve((c, low), np.eye(n))
    idx = np.arange(n)
    grad, qs, ts = [], [], []
    for name in kern.theta:
        if name == "sigma2":
            raise ValueError("sigma2 is profiled out")
        Si = kern.dsigma_block(name, xy, idx, idx)
        q = float(v @ (Si @ v))
        t = float(np.sum(Sinv * Si))
        qs.append(q)
        ts.append(t)
        grad.append(-0.5 * t + 0.5 * n * q / Q)
    return dict(ell=float(ell), grad=np.array(grad), Q=Q, q=np.array(qs), trace=np.array(ts), logdet=logdet)


def dense_cond_mean(kern: Kernel, xy: np.ndarray, z: np.ndarray, xy_new: np.ndarray) -> np.ndarray:
    """Sigma_12 Sigma_22^-1 z; Sigma_12 = sigma2 k(x', x) (distinct observations: no nugget)."""
    S = dense_sigma(kern, xy)
    return kern.sigma_points(xy_new, xy) @ np.linalg.solve(S, z)


def dense_cond_cov(kern: Kernel, xy: np.ndarray, xy_new: np.ndarray) -> np.ndarray:
    """Sigma_11 - Sigma_12 Sigma_22^-1 Sigma_12^T (Remark conditional): the covariance of
    z' | z, where [z'; z] follows the GP with the new points first (nugget on every observation's
    own diagonal, reading R-I), plain definition with a dense solve."""
    joint = np.vstack([xy_new, xy])
    S = dense_sigma(kern, joint)
    m = len(xy_new)
    S11, S12, S22 = S[:m, :m], S[:m, m:], S[m:, m:]
    return S11 - S12 @ np.linalg.solve(S22, S12.T)
