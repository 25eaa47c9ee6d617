"""P7 - closed forms for a separable covariance (oracle; test infrastructure only).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline leg may use this
module; the product path never imports it.

On a tensor grid x_(i,j) = (a_i, b_j) (point index i * m_b + j) the squared-exponential
kernel -- the alpha -> infinity limit of the rational quadratic, P:24 -- factors,
exp(-r^2 / (2 rho^2)) = exp(-(dx)^2 / (2 rho^2)) exp(-(dy)^2 / (2 rho^2)), so

    Sigma = sigma2 K_a (x) K_b + tau I        (Eq. normaldist's Sigma, reading R-H)

and with K_a = Q_a diag(lam) Q_a^T, K_b = Q_b diag(mu) Q_b^T every quantity of
Eq. loglikelihood and Eq. gradient has a closed form through two
sqrt(n)-sized eigenproblems:

    log|Sigma|              = sum_ij log(sigma2 lam_i mu_j + tau)
    Sigma^-1 z              = (Q_a (x) Q_b) diag(1 / ev) (Q_a (x) Q_b)^T z,  ev_ij = sigma2 lam_i mu_j + tau
    Tr(Sigma^-1 Sigma_rho)  = sum_ij sigma2 (lam'_i mu_j + lam_i mu'_j) / ev_ij,
                              lam'_i = q_i^T (dK_a/drho) q_i  (Hellmann-Feynman; the diagonal of
                              Q^T K' Q is all the trace needs)
    Tr(Sigma^-1)            = sum_ij 1 / ev_ij
    Tr(Sigma^-1 Sigma_sigma2) = sum_ij lam_i mu_j / ev_ij
    u^T Sigma_rho u         = sigma2 <U, K'_a U K_b + K_a U K'_b>,  U = reshape(u, m_a x m_b)

Library primitives: numpy.linalg.eigh (symmetric eigendecomposition) and matrix products.
Pinned against the dense oracle O1 (tests/test_oracle_pins.py::test_P7_*).  A sample
z ~ N(0, Sigma) is (Q_a (x) Q_b) diag(sqrt(ev)) w.
"""
from __future__ import annotations

import math

import numpy as np


class SeparableSE:
    """Sigma(theta) = sigma2 K_a (x) K_b + tau I for the squared-exponential kernel."""

    def __init__(self, a: np.ndarray, b: np.ndarray, rho: float, sigma2: float, tau: float):
        self.a = np.asarray(a, dtype=np.float64)
        self.b = np.asarray(b, dtype=np.float64)
        self.rho, self.sigma2, self.tau = float(rho), float(sigma2), float(tau)
        self.n = self.a.size * self.b.size

        def k1(x):
            d2 = (x[:, None] - x[None, :]) ** 2
            K = np.exp(-d2 / (2.0 * self.rho ** 2))
            return K, K * d2 / self.rho ** 3           # k and dk/drho of one axis factor

        Ka, Kap = k1(self.a)
        Kb, Kbp = k1(self.b)
        self.Ka, self.Kb, self.Kap, self.Kbp = Ka, Kb, Kap, Kbp
        self.lam, self.Qa = np.linalg.eigh(Ka)
        self.mu, self.Qb = np.linalg.eigh(Kb)
        self.lamp = np.einsum("ki,kl,li->i", self.Qa, Kap, self.Qa)
        self.mup = np.einsum("ki,kl,li->i", self.Qb, Kbp, self.Qb)
        self.ev = self.sigma2 * np.outer(self.lam, self.mu) + self.tau

    # Z (m_a x m_b) <-> vectors in point order i * m_b + j
    def _mat(self, v):
        return np.asarray(v, dtype=np.float64).reshape(self.a.size, self.b.size)

    def points(self) -> np.ndarray:
        return np.stack([np.repeat(self.a, self.b.size), np.tile(self.b, self.a.size)], axis=1)

    def logdet(self) -> float:
        return float(np.sum(np.log(self.ev)))

    def matvec(self, x) -> np.ndarray:
        X = self._mat(x)
        return (self.sigma2 * self.Ka @ X @ self.Kb + self.tau * X).ravel()

    def solve(self, z) -> np.ndarray:
        Zh = self.Qa.T @ self._mat(z) @ self.Qb
        return (self.Qa @ (Zh / self.ev) @ self.Qb.T).ravel()

    def sample(self, w) -> np.ndarray:
        """z = (Q_a (x) Q_b) diag(sqrt(ev)) w, so that Cov(z) = Sigma for w ~ N(0, I)."""
        return (self.Qa @ (np.sqrt(self.ev) * self._mat(w)) @ self.Qb.T).ravel()

    def dsigma_matvec(self, name: str, x) -> np.ndarray:
        X = self._mat(x)
        if name == "rho":
            Y = self.sigma2 * (self.Kap @ X @ self.Kb + self.Ka @ X @ self.Kbp)
        elif name == "sigma2":
            Y = self.Ka @ X @ self.Kb
        elif name == "nugget":
            Y = X
        else:
            raise ValueError(f"separable closed form has no parameter {name!r}")
        return Y.ravel()

    def trace(self, name: str) -> float:
        """Tr(Sigma^-1 Sigma_name)."""
        if name == "rho":
            return float(np.sum(self.sigma2 * (np.outer(self.lamp, self.mu) + np.outer(self.lam, self.mup))
                                / self.ev))
        if name == "sigma2":
            return float(np.sum(np.outer(self.lam, self.mu) / self.ev))
        if name == "nugget":
            return float(np.sum(1.0 / self.ev))
        raise ValueError(name)

    def eval(self, z, theta) -> dict:
        """ell, g (Eq. loglikelihood, Eq. gradient) and their parts."""
        z = np.asarray(z, dtype=np.float64)
        u = self.solve(z)
        quad = float(z @ u)
        logdet = self.logdet()
        ell = -0.5 * quad - 0.5 * logdet - 0.5 * self.n * math.log(2.0 * math.pi)
        q = np.array([float(u @ self.dsigma_matvec(t, u)) for t in theta])
        tr = np.array([self.trace(t) for t in theta])
        return dict(ell=ell, grad=0.5 * q - 0.5 * tr, logdet=logdet, quad=quad, q=q, trace=tr,
                    trace_inv=self.trace("nugget"), utu=float(u @ u))
