"""Covariance kernel entries and their theta-derivatives (oracle; test infrastructure).

Sigma_jk = sigma2 * k(r_jk) + nugget * [j == k]   (reading R-H: nugget not scaled
by sigma2; R-I: delta by observation INDEX, not by location).

Families (r = ||x - y||):
  rq        k = (1 + r^2/(2 alpha rho^2))^(-alpha)
  matern12  k = exp(-s),                 s = r/rho                 P:912-917 (nu=1/2)
  matern32  k = (1+s) exp(-s),           s = sqrt(3) r/rho         P:912-917 (nu=3/2)
  matern52  k = (1+s+s^2/3) exp(-s),     s = sqrt(5) r/rho         P:912-917 (nu=5/2)
  sqexp     k = exp(-r^2/(2 rho^2))      the alpha -> inf RQ limit, P:24 (test-only)

Derivatives are written out from those definitions by the chain rule (the
paper assumes Sigma_i available); tests pin them to central finite
differences (pin P2).

Anisotropic kernels (next row f1): with rho2 > 0 the distance is the
scaled ||x - y||_theta = sqrt(dx^2/rho^2 + dy^2/rho2^2) and the family is evaluated
at unit length, k(||x - y||_theta); theta_1 = rho, theta_2 = rho2.  With alpha = 1/2
(RQ) and the Matern 3/2 family these are Eqs. specrq and specmatern.
"""
from __future__ import annotations

import numpy as np

FAMILIES = ("rq", "matern12", "matern32", "matern52", "sqexp")
PARAMS = ("rho", "sigma2", "nugget", "alpha", "rho2")


def pairwise_r(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Euclidean distances ||x_a - y_b|| for rows of X (m x 2) and Y (p x 2)."""
    dx = X[:, None, 0] - Y[None, :, 0]
    dy = X[:, None, 1] - Y[None, :, 1]
    return np.sqrt(dx * dx + dy * dy)


def k_of_r(family: str, r, rho: float, alpha: float = 1.0):
    """Unit-variance correlation k(r) (no nugget)."""
    r = np.asarray(r, dtype=np.float64)
    if family == "rq":
        u = r * r / (2.0 * rho * rho)
        return np.exp(-alpha * np.log1p(u / alpha))
    if family == "matern12":
        s = r / rho
        return np.exp(-s)
    if family == "matern32":
        s = np.sqrt(3.0) * r / rho
        return (1.0 + s) * np.exp(-s)
    if family == "matern52":
        s = np.sqrt(5.0) * r / rho
        return (1.0 + s + s * s / 3.0) * np.exp(-s)
    if family == "sqexp":
        return np.exp(-r * r / (2.0 * rho * rho))
    raise ValueError(family)


def dk_drho(family: str, r, rho: float, alpha: float = 1.0):
    """d k / d rho (chain rule on the definitions above)."""
    r = np.asarray(r, dtype=np.float64)
    if family == "rq":
        u = r * r / (2.0 * rho * rho)
        # dk/du = -(1+u/alpha)^(-alpha-1), du/drho = -2u/rho = -r^2/rho^3
        return (r * r / rho ** 3) * np.exp((-alpha - 1.0) * np.log1p(u / alpha))
    if family == "matern12":
        s = r / rho
        return (s / rho) * np.exp(-s)
    if family == "matern32":
        s = np.sqrt(3.0) * r / rho
        return (s * s / rho) * np.exp(-s)
    if family == "matern52":
        s = np.sqrt(5.0) * r / rho
        return s * s * (1.0 + s) * np.exp(-s) / (3.0 * rho)
    if family == "sqexp":
        return (r * r / rho ** 3) * np.exp(-r * r / (2.0 * rho * rho))
    raise ValueError(family)


def dk_dalpha(family: str, r, rho: float, alpha: float = 1.0):
    """d k / d alpha (RQ only): k * [u/(alpha+u) - log1p(u/alpha)]."""
    if family != "rq":
        raise ValueError("alpha is a parameter of the rational-quadratic family only")
    r = np.asarray(r, dtype=np.float64)
    u = r * r / (2.0 * rho * rho)
    x = u / alpha
    k = np.exp(-alpha * np.log1p(x))
    # the bracket u/(alpha+u) - log1p(u/alpha) = x/(1+x) - log1p(x) cancels for small x; its
    # Taylor series is  sum_{j>=2} (-1)^(j+1) (j-1)/j x^j
    #   = -x^2/2 + 2x^3/3 - 3x^4/4 + ...,  used for x < 1e-3 (5 terms: truncation < 1e-18 x^2)
    series = x * x * (-0.5 + x * (2.0 / 3.0 + x * (-0.75 + x * (0.8 + x * (-5.0 / 6.0)))))
    with np.errstate(invalid="ignore"):
        direct = x / (1.0 + x) - np.log1p(x)
    return k * np.where(x < 1e-3, series, direct)


class Kernel:
    """theta-parameterised covariance Sigma(theta) = sigma2*k + nugget*I."""

    def __init__(self, family: str, rho: float, sigma2: float = 1.0,
                 nugget: float = 0.0, alpha: float = 1.0, theta=("rho",), rho2: float = 0.0):
        if family not in FAMILIES:
            raise ValueError(family)
        if not (rho > 0 and sigma2 > 0 and alpha > 0 and nugget >= 0 and rho2 >= 0):
            raise ValueError("rho, sigma2, alpha must be > 0, nugget and rho2 >= 0")
        for t in theta:
            if t not in PARAMS:
                raise ValueError(t)
            if t == "alpha" and family != "rq":
                raise ValueError("alpha only for rq")
            if t == "rho2" and not rho2 > 0:
                raise ValueError("rho2 only for anisotropic kernels")
        self.family, self.rho, self.sigma2 = family, float(rho), float(sigma2)
        self.nugget, self.alpha, self.theta = float(nugget), float(alpha), tuple(theta)
        self.rho2 = float(rho2)

    def with_param(self, name: str, value: float) -> "Kernel":
        d = dict(family=self.family, rho=self.rho, sigma2=self.sigma2,
                 nugget=self.nugget, alpha=self.alpha, theta=self.theta, rho2=self.rho2)
        d[name] = value
        return Kernel(**d)

    def value(self, name: str) -> float:
        return getattr(self, name)

    # --- blocks -------------------------------------------------------------
    # --- geometry: isotropic r, or the anisotropic scaled distance q and dx^2, dy^2
    def _k(self, P, Q):
        if self.rho2 > 0:
            q, _, _ = self._q(P, Q)
            return k_of_r(self.family, q, 1.0, self.alpha)
        return k_of_r(self.family, pairwise_r(P, Q), self.rho, self.alpha)

    def _q(self, P, Q):
        dx = P[:, None, 0] - Q[None, :, 0]
        dy = P[:, None, 1] - Q[None, :, 1]
        return np.sqrt((dx / self.rho) ** 2 + (dy / self.rho2) ** 2), dx * dx, dy * dy

    def sigma_block(self, xy, rows, cols):
        """Sigma(rows, cols) with the nugget on equal indices (R-I)."""
        rows = np.asarray(rows)
        cols = np.asarray(cols)
        B = self.sigma2 * self._k(xy[rows], xy[cols])
        if self.nugget != 0.0:
            B = B + self.nugget * (rows[:, None] == cols[None, :])
        return B

    def sigma_points(self, P, Q):
        """sigma2 * k between two coordinate sets (no nugget; proxy rows)."""
        return self.sigma2 * self._k(P, Q)

    def dsigma_block(self, name: str, xy, rows, cols):
        """Sigma_i(rows, cols) = d Sigma / d theta_i."""
        rows = np.asarray(rows)
        cols = np.asarray(cols)
        if name == "nugget":
            return (rows[:, None] == cols[None, :]).astype(np.float64)
        return self.dsigma_points(name, xy[rows], xy[cols])

    def dsigma_points(self, name: str, P, Q):
        if name == "nugget":
            return np.zeros((len(P), len(Q)))
        if self.rho2 > 0:
            return self._dsig_aniso(name, P, Q)
        return self._dsig_r(name, pairwise_r(P, Q))

    def _dsig_aniso(self, name, P, Q):
        """Chain rule through q: dk/dtheta_1 = k'(q) dq/dtheta_1, dq/dtheta_1 = -dx^2/(theta_1^3 q),
        k'(q) = -(dk/drho at unit length)/q."""
        q, dx2, dy2 = self._q(P, Q)
        if name == "sigma2":
            return k_of_r(self.family, q, 1.0, self.alpha)
        if name == "alpha":
            return self.sigma2 * dk_dalpha(self.family, q, 1.0, self.alpha)
        if name in ("rho", "rho2"):
            with np.errstate(divide="ignore", invalid="ignore"):
                g = np.where(q > 0, dk_drho(self.family, q, 1.0, self.alpha) / (q * q), 0.0)
            if name == "rho":
                return self.sigma2 * g * dx2 / self.rho ** 3
            return self.sigma2 * g * dy2 / self.rho2 ** 3
        raise ValueError(name)

    def _dsig_r(self, name, r):
        if name == "rho":
            return self.sigma2 * dk_drho(self.family, r, self.rho, self.alpha)
        if name == "alpha":
            return self.sigma2 * dk_dalpha(self.family, r, self.rho, self.alpha)
        if name == "sigma2":
            return k_of_r(self.family, r, self.rho, self.alpha)
        raise ValueError(name)
