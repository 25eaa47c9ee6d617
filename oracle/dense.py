"""O1 - the plain definition of l(theta) and g(theta) by dense linear algebra.

Oracle / test infrastructure only.  Follows:
  Eq. loglikelihood  P:37-39   l = -1/2 z^T Sigma^-1 z - 1/2 log|Sigma| - n/2 log 2 pi
  Eq. gradient       P:43-47   g_i = 1/2 z^T Sigma^-1 Sigma_i Sigma^-1 z - 1/2 Tr(Sigma^-1 Sigma_i)
  dense Cholesky     P:50      (the O(n^3) approach the paper avoids)

Steps: assemble Sigma; Cholesky L L^T (LAPACK, a library
primitive); logdet = 2 sum log L_jj; alpha = L^-1 z, q0 = alpha^T alpha;
Sigma^-1 formed explicitly; u = Sigma^-1 z; for each theta_i: q_i = u^T Sigma_i u,
t_i = sum_jk (Sigma^-1)_jk (Sigma_i)_jk (= Tr(Sigma^-1 Sigma_i) since both are
symmetric), g_i = q_i/2 - t_i/2.  Feasible for n <= 16384.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla

from .kernels import Kernel


def dense_sigma(kern: Kernel, xy: np.ndarray) -> np.ndarray:
    n = len(xy)
    idx = np.arange(n)
    return kern.sigma_block(xy, idx, idx)


def dense_eval(kern: Kernel, xy: np.ndarray, z: np.ndarray, *, fisher: bool = False,
               block: int = 2048) -> dict:
    """Exact (up to rounding) l, g and their ingredients."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    n = len(xy)
    S = dense_sigma(kern, xy)
    L = sla.cholesky(S, lower=True, overwrite_a=True, check_finite=False)
    logdet = 2.0 * float(np.sum(np.log(np.diag(L))))
    a = sla.solve_triangular(L, z, lower=True, check_finite=False)
    q0 = float(a @ a)
    ell = -0.5 * q0 - 0.5 * logdet - 0.5 * n * math.log(2.0 * math.pi)
    # explicit inverse: Sigma^-1 = L^-T L^-1
    Linv = sla.solve_triangular(L, np.eye(n), lower=True, check_finite=False)
    del L, S
    Sinv = Linv.T @ Linv
    del Linv
    u = Sinv @ z
    idx = np.arange(n)
    qs, ts, fis = [], [], []
    for name in kern.theta:
        q = 0.0
        t = 0.0
        f = 0.0
        for r0 in range(0, n, block):
            rows = idx[r0:r0 + block]
            Si = kern.dsigma_block(name, xy, rows, idx)
            q += float(u[rows] @ (Si @ u))
            t += float(np.sum(Sinv[rows] * Si))
        if fisher:
            # Tr((Sigma^-1 Sigma_i)^2) = sum_jk P_jk P_kj with P = Sigma^-1 Sigma_i
            SiF = kern.dsigma_block(name, xy, idx, idx)
            P = Sinv @ SiF
            f = 0.5 * float(np.sum(P * P.T))
            del SiF, P
        qs.append(q)
        ts.append(t)
        fis.append(f)
    grad = [0.5 * q - 0.5 * t for q, t in zip(qs, ts)]
    out = dict(ell=ell, grad=np.array(grad), logdet=logdet, quad=q0,
               q=np.array(qs), trace=np.array(ts), u=u, trace_inv=float(np.trace(Sinv)),
               utu=float(u @ u))
    if fisher:
        out["fisher_sd"] = np.sqrt(np.array(fis))
    return out


def dense_sample(kern: Kernel, xy: np.ndarray, w: np.ndarray) -> np.ndarray:
    """z = L w with L the dense Cholesky factor of Sigma (configs 1-2 input recipe)."""
    S = dense_sigma(kern, np.ascontiguousarray(xy, dtype=np.float64))
    L = sla.cholesky(S, lower=True, overwrite_a=True, check_finite=False)
    return L @ w


def dense_matvec(kern: Kernel, xy: np.ndarray, x: np.ndarray, block: int = 1024) -> np.ndarray:
    """Sigma @ x by on-the-fly blocks, O(n^2) time, O(n*block) memory (pin P11)."""
    n = len(xy)
    idx = np.arange(n)
    x = np.asarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    for r0 in range(0, n, block):
        rows = idx[r0:r0 + block]
        y[rows] = kern.sigma_block(xy, rows, idx) @ x
    return y
