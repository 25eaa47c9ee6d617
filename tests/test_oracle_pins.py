"""Pins for the oracle (CPU only): each ties an oracle function to something
other than itself -- closed forms, brute force, library special cases,
invariants (pins P1-P14)."""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg as sla

from oracle.dense import dense_eval, dense_matvec, dense_sample, dense_sigma
from oracle.kernels import Kernel, k_of_r
from oracle.mle import rsf_mle_eval
from oracle.peel import peel_trace
from oracle.rsf import RSF, interp_decomp, proxy_points
from oracle.separable import SeparableSE
from oracle.tree import QuadTree
from workloads import config, philox4x32, philox_normal, points_for, separable_axes, w_for

GOLD = os.path.join(os.path.dirname(__file__), "golden")
LOG2PI = math.log(2 * math.pi)


def _rng(seed=0):
    return np.random.default_rng(seed)


def _uniform(n, seed=0):
    return _rng(seed).random((n, 2))


# ------------------------------------------------------------------ inputs
def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox_kat.json)."""
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for case in kat["cases"]:
        c = [int(v, 16) if isinstance(v, str) else v for v in case["ctr"]]
        k = [int(v, 16) if isinstance(v, str) else v for v in case["key"]]
        out = philox4x32(np.array([c[0]], dtype=np.uint64), c[1], c[2], c[3], k[0], k[1])
        assert [int(o[0]) for o in out] == [int(v, 16) for v in case["out"]]


def test_config_points_in_unit_square_and_deterministic():
    for cid, n in [(1, 1024), (3, 4096), (4, 20000)]:
        c = config(cid)
        p = points_for(c, n)
        assert p.shape == (n, 2)
        assert p.min() >= 0.0 and p.max() < 1.0
        assert np.array_equal(p, points_for(c, n))
    w = w_for(config(2), 200001)
    assert abs(w.mean()) < 0.01 and abs(w.std() - 1) < 0.01


# ------------------------------------------------------------------ P1, P2 kernels
def test_P1_kernel_hand_values():
    g = json.load(open(os.path.join(GOLD, "kernel_values.json")))
    for c in g["cases"]:
        v = k_of_r(c["family"], math.sqrt(c["r2"]), c["rho"], c.get("alpha", 1.0))
        assert abs(float(v) - c["k"]) <= 4e-16 * abs(c["k"]) + 1e-300, c


@pytest.mark.parametrize("family", ["rq", "matern12", "matern32", "matern52", "sqexp"])
def test_P1_sigma_diagonal_and_symmetry(family):
    xy = _uniform(40, 1)
    K = Kernel(family, 0.3, sigma2=1.7, nugget=0.01, alpha=1.3)
    S = dense_sigma(K, xy)
    assert np.allclose(np.diag(S), 1.7 + 0.01, rtol=0, atol=1e-15)
    assert np.array_equal(S, S.T)
    # duplicates: nugget by index (R-I)
    xy2 = np.vstack([xy[:3], xy[:1]])
    S2 = dense_sigma(K, xy2)
    assert S2[0, 3] == pytest.approx(1.7, abs=1e-15)


def _richardson(f, x, h):
    d1 = (f(x + h) - f(x - h)) / (2 * h)
    d2 = (f(x + h / 2) - f(x - h / 2)) / h
    return (4 * d2 - d1) / 3


@pytest.mark.parametrize("family,param", [
    ("rq", "rho"), ("rq", "alpha"), ("rq", "sigma2"), ("rq", "nugget"),
    ("matern12", "rho"), ("matern32", "rho"), ("matern52", "rho"), ("sqexp", "rho"),
    ("matern32", "sigma2"), ("matern52", "nugget")])
def test_P2_derivative_entries_vs_finite_differences(family, param):
    xy = _uniform(30, 2) * 0.6
    base = Kernel(family, 0.21, sigma2=1.3, nugget=0.02, alpha=1.5, theta=(param,))
    idx = np.arange(len(xy))
    an = base.dsigma_block(param, xy, idx, idx)
    v0 = base.value(param)

    def f(v):
        return base.with_param(param, v).sigma_block(xy, idx, idx)
    fd = _richardson(f, v0, 1e-3 * v0)
    scale = np.max(np.abs(an)) + 1e-300
    assert np.max(np.abs(an - fd)) <= 1e-9 * scale
    if param in ("rho", "alpha"):
        assert np.all(np.diag(an) == 0.0)


# ------------------------------------------------------------------ P3, P4, P5 small n
def test_P3_n1_closed_form():
    K = Kernel("matern32", 0.2, sigma2=1.4, nugget=0.3, theta=("rho", "sigma2", "nugget"))
    xy = np.array([[0.3, 0.6]])
    z = np.array([0.77])
    d = dense_eval(K, xy, z)
    a = 1.4 + 0.3
    assert d["ell"] == pytest.approx(-z[0] ** 2 / (2 * a) - 0.5 * math.log(a) - 0.5 * LOG2PI, rel=1e-14)
    gs = 0.5 * z[0] ** 2 / a ** 2 - 0.5 / a
    assert d["grad"][0] == 0.0
    assert d["grad"][1] == pytest.approx(gs, rel=1e-13)
    assert d["grad"][2] == pytest.approx(gs, rel=1e-13)


@pytest.mark.parametrize("family", ["rq", "matern12", "matern52"])
def test_P4_n2_closed_form(family):
    K = Kernel(family, 0.35, sigma2=1.1, nugget=0.05, alpha=0.8, theta=("rho",))
    xy = np.array([[0.1, 0.2], [0.4, 0.6]])
    z = np.array([0.9, -0.4])
    r = 0.5
    from oracle.kernels import dk_drho
    a = 1.1 + 0.05
    b = 1.1 * float(k_of_r(family, r, 0.35, 0.8))
    bp = 1.1 * float(dk_drho(family, r, 0.35, 0.8))
    det = a * a - b * b
    quad = (a * (z @ z) - 2 * b * z[0] * z[1]) / det
    tr = -2 * b * bp / det
    u = np.array([a * z[0] - b * z[1], a * z[1] - b * z[0]]) / det
    q = 2 * bp * u[0] * u[1]
    d = dense_eval(K, xy, z)
    assert d["logdet"] == pytest.approx(math.log(det), rel=1e-13)
    assert d["quad"] == pytest.approx(quad, rel=1e-13)
    assert d["trace"][0] == pytest.approx(tr, rel=1e-12)
    assert d["grad"][0] == pytest.approx(0.5 * q - 0.5 * tr, rel=1e-12)


def _leibniz_det(M):
    n = len(M)
    tot = Fraction(0)
    for p in itertools.permutations(range(n)):
        inv = sum(1 for i in range(n) for j in range(i + 1, n) if p[i] > p[j])
        prod = Fraction(1)
        for i in range(n):
            prod *= M[i][p[i]]
        tot += -prod if inv % 2 else prod
    return tot


def test_P5_small_n_exact_rational_arithmetic():
    """n = 6: determinant by the Leibniz formula and inverse by the adjugate, in
    exact rational arithmetic on the float entries -- independent of Cholesky."""
    n = 6
    K = Kernel("rq", 0.4, sigma2=1.0, nugget=0.02, alpha=1.0, theta=("rho",))
    xy = _uniform(n, 5)
    z = _rng(6).standard_normal(n)
    S = dense_sigma(K, xy)
    Si = K.dsigma_block("rho", xy, np.arange(n), np.arange(n))
    M = [[Fraction(float(S[i, j])) for j in range(n)] for i in range(n)]
    det = _leibniz_det(M)
    adj = [[None] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            minor = [[M[r][c] for c in range(n) if c != j] for r in range(n) if r != i]
            adj[j][i] = (-1) ** (i + j) * _leibniz_det(minor)
    inv = np.array([[float(adj[i][j] / det) for j in range(n)] for i in range(n)])
    quad = float(z @ inv @ z)
    tr = float(np.sum(inv * Si))
    q = float(z @ inv @ Si @ inv @ z)
    ell = -0.5 * quad - 0.5 * math.log(float(det)) - 0.5 * n * LOG2PI
    d = dense_eval(K, xy, z)
    assert d["ell"] == pytest.approx(ell, rel=1e-13)
    assert d["grad"][0] == pytest.approx(0.5 * q - 0.5 * tr, rel=1e-11)


# ------------------------------------------------------------------ P6 diagonal
def test_P6_diagonal_sigma_underflow():
    m = 32
    d = 1.0 / m
    g = (np.arange(m) + 0.5) * d
    xy = np.array([(a, b) for a in g for b in g])
    K = Kernel("matern12", d / 750.0, sigma2=1.3, nugget=0.2, theta=("rho",))
    assert float(k_of_r("matern12", d, d / 750.0)) == 0.0
    z = _rng(7).standard_normal(len(xy))
    n = len(xy)
    out = dense_eval(K, xy, z)
    assert out["logdet"] == pytest.approx(n * math.log(1.5), rel=1e-14)
    assert out["trace"][0] == 0.0
    F = RSF(K, xy, 1e-8, 64)
    assert F.logdet == pytest.approx(n * math.log(1.5), rel=1e-13)
    assert all(len(b.S) == 0 for b in F.levels[F.tree.L])      # k = 0 ID path (R-BB)
    assert np.allclose(F.solve(z), z / 1.5, rtol=1e-14)


# ------------------------------------------------------------------ P7 separable
def _separable_case(ma=24, mb=20, rho=0.15, sigma2=1.2, tau=0.05, seed=8):
    r = _rng(seed)
    a = np.sort(r.random(ma))
    b = np.sort(r.random(mb))
    S = SeparableSE(a, b, rho, sigma2, tau)
    K = Kernel("sqexp", rho, sigma2=sigma2, nugget=tau, theta=("rho", "sigma2", "nugget"))
    z = r.standard_normal(ma * mb)
    return S, K, S.points(), z


def test_P7_separable_closed_form_dense():
    """oracle/separable.py (Kronecker eigen closed forms) against O1 (dense Cholesky, explicit
    inverse): every part of l and g for rho, sigma2 and the nugget."""
    S, K, xy, z = _separable_case()
    d = dense_eval(K, xy, z)
    c = S.eval(z, K.theta)
    assert c["logdet"] == pytest.approx(d["logdet"], rel=1e-12)
    assert c["quad"] == pytest.approx(d["quad"], rel=1e-10)
    assert c["ell"] == pytest.approx(d["ell"], rel=1e-11)
    np.testing.assert_allclose(c["trace"], d["trace"], rtol=1e-10)
    np.testing.assert_allclose(c["q"], d["q"], rtol=1e-10)
    np.testing.assert_allclose(c["grad"], d["grad"], rtol=1e-9)
    assert c["trace_inv"] == pytest.approx(d["trace_inv"], rel=1e-10)
    # Sigma from the closed form's matvec equals the dense matrix
    sig = dense_sigma(K, xy)
    x = _rng(3).standard_normal(len(xy))
    np.testing.assert_allclose(S.matvec(x), sig @ x, rtol=1e-12, atol=1e-12)


def test_P7_separable_sample_has_covariance_sigma():
    """sample(w) = A w with A A^T = Sigma: A^T Sigma^-1 A = I tested on random w, and
    the sample's dense quadratic form z^T Sigma^-1 z = w^T w (O1 Cholesky)."""
    S, K, xy, _ = _separable_case(ma=12, mb=10)
    w = _rng(5).standard_normal(S.n)
    z = S.sample(w)
    d = dense_eval(K, xy, z)
    assert d["quad"] == pytest.approx(float(w @ w), rel=1e-10)
    A = np.stack([S.sample(e) for e in np.eye(S.n)], axis=1)
    np.testing.assert_allclose(A @ A.T, dense_sigma(K, xy), rtol=1e-10, atol=1e-12)


def test_P7_separable_closed_form_rsf_and_peel():
    S, K, xy, z = _separable_case(ma=40, mb=36)
    K = Kernel("sqexp", S.rho, sigma2=S.sigma2, nugget=S.tau, theta=("rho",))
    F = RSF(K, xy, 1e-11, 32)
    assert F.tree.L >= 2
    assert F.logdet == pytest.approx(S.logdet(), rel=1e-9)
    assert float(z @ F.solve(z)) == pytest.approx(float(z @ S.solve(z)), rel=1e-6)
    Fi = RSF(K, xy, 1e-11, 32, which="rho")

    def G(X):
        return 0.5 * (F.solve(Fi.apply(X)) + Fi.apply(F.solve(X)))
    from oracle.mle import make_probe
    t = peel_trace(G, F.tree, 1e-8, make_probe(11, 0, philox_normal), block=16)
    assert t == pytest.approx(S.trace("rho"), rel=1e-6)


def test_separable_axes_recipe():
    a, b = separable_axes(64)
    g = (np.arange(64) + 0.5) / 64
    assert np.all(np.abs(a - g) <= 0.4 / 64 + 1e-15) and np.all(np.abs(b - g) <= 0.4 / 64 + 1e-15)
    assert np.all(np.diff(a) > 0) and np.all(np.diff(b) > 0) and not np.allclose(a, b)
    a2, _ = separable_axes(64)
    np.testing.assert_array_equal(a, a2)


# ------------------------------------------------------------------ P8, P9, P10
def test_P8_trace_is_derivative_of_logdet():
    xy = _uniform(150, 9)
    K = Kernel("matern32", 0.2, sigma2=1.0, nugget=0.01, theta=("rho",))
    z = np.ones(150)
    t = dense_eval(K, xy, z)["trace"][0]
    fd = _richardson(lambda v: dense_eval(K.with_param("rho", v), xy, z)["logdet"], 0.2, 2e-4)
    assert t == pytest.approx(fd, rel=1e-8)


def test_P9_sigma2_nugget_identities():
    xy = _uniform(200, 10)
    K = Kernel("rq", 0.15, sigma2=1.7, nugget=0.03, alpha=1.2, theta=("sigma2", "nugget"))
    z = _rng(11).standard_normal(200)
    d = dense_eval(K, xy, z)
    n = 200
    assert d["trace"][0] == pytest.approx((n - 0.03 * d["trace_inv"]) / 1.7, rel=1e-11)
    assert d["trace"][1] == pytest.approx(d["trace_inv"], rel=1e-12)
    assert d["q"][0] == pytest.approx((d["quad"] - 0.03 * d["utu"]) / 1.7, rel=1e-10)
    assert 1.7 * d["grad"][0] + 0.03 * d["grad"][1] == pytest.approx(0.5 * d["quad"] - n / 2, rel=1e-10)


@pytest.mark.parametrize("family,theta", [
    ("rq", ("rho", "alpha", "sigma2", "nugget")), ("matern12", ("rho", "sigma2")),
    ("matern32", ("rho", "nugget")), ("matern52", ("rho", "sigma2", "nugget"))])
def test_P10_gradient_vs_finite_differences_of_ell(family, theta):
    xy = _uniform(120, 12)
    K = Kernel(family, 0.25, sigma2=1.2, nugget=0.05, alpha=1.4, theta=theta)
    z = _rng(13).standard_normal(120)
    d = dense_eval(K, xy, z)
    for i, name in enumerate(theta):
        v = K.value(name)
        fd = _richardson(lambda x: dense_eval(K.with_param(name, x), xy, z)["ell"], v, 1e-3 * v)
        assert d["grad"][i] == pytest.approx(fd, rel=1e-7, abs=1e-9)


# ------------------------------------------------------------------ P11, P12 RSF
@pytest.fixture(scope="module")
def cfg1_case():
    c = config(1)
    xy = points_for(c)
    K = Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    z = dense_sample(K, xy, w_for(c))
    F = RSF(K, xy, c.eps_fact, c.leaf)
    return c, xy, K, z, F


def test_P11_rsf_solve_residual_bruteforce(cfg1_case):
    c, xy, K, z, F = cfg1_case
    x = F.solve(z)
    res = np.linalg.norm(dense_matvec(K, xy, x) - z) / np.linalg.norm(z)
    assert res <= 10 * c.eps


def test_P11_apply_solve_sqrt_identities(cfg1_case):
    c, xy, K, z, F = cfg1_case
    v = _rng(14).standard_normal(len(xy))
    assert np.linalg.norm(F.apply(F.solve(v)) - v) <= 1e-11 * np.linalg.norm(v)
    n = 300
    xs = _uniform(n, 15)
    Fs = RSF(K, xs, 1e-8, 32)
    Sq = Fs.sqrt(np.eye(n))
    Fa = Fs.apply(np.eye(n))
    assert np.max(np.abs(Sq @ Sq.T - Fa)) <= 1e-12 * np.max(np.abs(Fa))
    # apply approximates Sigma itself
    Sd = dense_sigma(K, xs)
    assert np.linalg.norm(Fa - Sd) <= 1e-6 * np.linalg.norm(Sd)


def test_P11_apply_only_compression_matches_sigma_i(cfg1_case):
    c, xy, K, z, F = cfg1_case
    Fi = RSF(K, xy, c.eps_fact, c.leaf, which="rho")
    idx = np.arange(len(xy))
    Si = K.dsigma_block("rho", xy, idx, idx)
    v = _rng(16).standard_normal(len(xy))
    assert np.linalg.norm(Fi.apply(v) - Si @ v) <= 1e-6 * np.linalg.norm(Si @ v)
    V = Fi.apply(np.eye(len(xy)))
    assert np.max(np.abs(V - V.T)) <= 1e-12 * np.max(np.abs(V))


def test_P12_rsf_limits():
    K = Kernel("matern32", 0.2, sigma2=1.0, nugget=0.01)
    xy = _uniform(50, 17)
    S = dense_sigma(K, xy)
    F = RSF(K, xy, 1e-6, 64)                 # n <= leaf: dense Cholesky
    assert F.tree.L == 0
    assert F.logdet == pytest.approx(np.linalg.slogdet(S)[1], rel=1e-13)
    xy = _uniform(600, 18)
    S = dense_sigma(K, xy)
    F = RSF(K, xy, 1e-14, 32)                # eps -> round-off: RSF == dense
    assert F.logdet == pytest.approx(np.linalg.slogdet(S)[1], rel=1e-12)
    b = _rng(19).standard_normal(600)
    assert np.linalg.norm(S @ F.solve(b) - b) <= 1e-10 * np.linalg.norm(b)


def test_interp_decomp_exact_rank():
    r = _rng(20)
    A = r.standard_normal((40, 5)) @ r.standard_normal((5, 12))
    piv, k, T = interp_decomp(A, 1e-10)
    assert k == 5
    assert np.linalg.norm(A[:, piv[k:]] - A[:, piv[:k]] @ T) <= 1e-12 * np.linalg.norm(A)
    piv, k, T = interp_decomp(np.zeros((10, 4)), 1e-8)
    assert k == 0


def test_tree_invariants_and_proxies():
    xy = points_for(config(4), 5000)
    t = QuadTree(xy, 64)
    for lev in t.levels:
        for b in lev:
            p = xy[b.idx]
            assert np.all(p[:, 0] >= b.cx - b.h) and np.all(p[:, 0] < b.cx + b.h)
            assert np.all(p[:, 1] >= b.cy - b.h) and np.all(p[:, 1] < b.cy + b.h)
            if b.children:
                assert np.array_equal(np.sort(np.concatenate([c.idx for c in b.children])), b.idx)
            else:
                assert len(b.idx) <= 64
    assert np.array_equal(np.sort(np.concatenate([b.idx for b in t.leaves()])), np.arange(5000))
    G = proxy_points(0.3, 0.4, 0.1)
    rr = np.hypot(G[:, 0] - 0.3, G[:, 1] - 0.4)
    assert len(G) == 256 and rr.min() > 0.175 and rr.max() < 0.245
    # 100 coincident points: degenerate leaf at max depth, no infinite recursion
    t2 = QuadTree(np.full((100, 2), 0.3), 64)
    assert t2.L == 30 and len(t2.leaves()) == 1


# ------------------------------------------------------------------ P13 peeling
def _tree(n=700, leaf=32, seed=21):
    return QuadTree(_uniform(n, seed), leaf)


def _probe(seed=3):
    from oracle.mle import make_probe
    return make_probe(seed, 0, philox_normal)


def test_P13_peel_identity_and_block_diagonal():
    t = _tree()
    n = len(t.xy)
    assert peel_trace(lambda X: X.copy(), t, 1e-6, _probe()) == pytest.approx(n, abs=1e-9)
    D = np.zeros((n, n))
    r = _rng(22)
    for b in t.leaves():
        B = r.standard_normal((len(b.idx), len(b.idx)))
        D[np.ix_(b.idx, b.idx)] = B + B.T
    assert peel_trace(lambda X: D @ X, t, 1e-6, _probe()) == pytest.approx(np.trace(D), abs=1e-9)


def test_P13_peel_recovers_exact_low_rank_off_diagonal():
    t = _tree()
    n = len(t.xy)
    r = _rng(23)
    U = r.standard_normal((n, 3))
    G = U @ U.T + np.diag(r.random(n))
    d = {}
    tr = peel_trace(lambda X: G @ X, t, 1e-10, _probe(), diag=d)
    assert tr == pytest.approx(np.trace(G), rel=1e-10)
    assert max(max(rk) for rk in d["ranks"]) == 3


def test_P13_peel_duplicate_parameter_gives_n(cfg1_case):
    c, xy, K, z, F = cfg1_case
    G = lambda X: 0.5 * (F.solve(F.apply(X)) + F.apply(F.solve(X)))  # noqa: E731
    assert peel_trace(G, F.tree, 1e-6, _probe(), block=64) == pytest.approx(len(xy), rel=1e-9)


def test_P13_peel_smooth_operator_vs_dense_trace():
    t = _tree(900, 32, 24)
    K = Kernel("matern32", 0.3, sigma2=1.0, nugget=0.1)
    S = dense_sigma(K, t.xy)
    Sinv = np.linalg.inv(S)
    d = {}
    tr = peel_trace(lambda X: Sinv @ X, t, 1e-7, _probe(), diag=d)
    assert tr == pytest.approx(np.trace(Sinv), rel=1e-6)
    assert d["cancellation"] == pytest.approx(1.0)


# ------------------------------------------------------------------ P14 statistics
def test_P14_score_has_mean_zero_and_fisher_variance():
    n = 128
    xy = _uniform(n, 25)
    K = Kernel("matern32", 0.2, sigma2=1.0, nugget=0.05, theta=("rho",))
    S = dense_sigma(K, xy)
    L = np.linalg.cholesky(S)
    r = _rng(26)
    gs = []
    for _ in range(200):
        z = L @ r.standard_normal(n)
        gs.append(dense_eval(K, xy, z)["grad"][0])
    gs = np.array(gs)
    sd = dense_eval(K, xy, np.zeros(n), fisher=True)["fisher_sd"][0]
    assert abs(gs.mean()) < 3 * sd / math.sqrt(len(gs))
    assert 0.75 < gs.std() / sd < 1.25


def test_dk_dalpha_small_u_series_matches_exact_bracket():
    """The small-u branch of d k / d alpha (series) against the bracket evaluated in exact
    rational arithmetic: x/(1+x) - log1p(x) from 40 terms of the alternating series with
    Fraction, at points on both sides of the x = 1e-3 switch."""
    from oracle.kernels import dk_dalpha
    rho, alpha = 0.1, 1.5
    for x in (1e-9, 3e-6, 2e-4, 9.9e-4, 1.1e-3, 5e-3):
        u = x * alpha
        r = math.sqrt(2.0 * rho * rho * u)
        xf = Fraction(r * r) / Fraction(2.0 * rho * rho) / Fraction(alpha)
        br = sum(Fraction((-1) ** (j + 1) * (j - 1), j) * xf ** j for j in range(2, 40))
        exact = float(br) * float(k_of_r("rq", r, rho, alpha))
        assert float(dk_dalpha("rq", r, rho, alpha)) == pytest.approx(exact, rel=1e-10, abs=1e-300)


def test_O2_sigma2_nugget_branch_matches_O1():
    """O2's reading-R-G branch (oracle/mle.py: t_sigma2 = (n - tau Tr F^-1)/sigma2,
    q_sigma2 = (q0 - tau u^T u)/sigma2, nugget: G = F^-1, q = u^T u) against O1, which forms
    Sigma_sigma2 = k and Sigma_tau = I explicitly."""
    xy = _uniform(400, 31)
    K = Kernel("matern32", 0.15, sigma2=1.3, nugget=0.02, theta=("rho", "sigma2", "nugget"))
    z = dense_sample(K, xy, _rng(32).standard_normal(400))
    d = dense_eval(K, xy, z)
    o = rsf_mle_eval(K, xy, z, 1e-12, 1e-9, 32, 77, philox_normal, block=16)
    np.testing.assert_allclose(o["trace"], d["trace"], rtol=1e-7)
    np.testing.assert_allclose(o["q"], d["q"], rtol=1e-8)
    np.testing.assert_allclose(o["grad"], d["grad"], rtol=1e-5)


# ------------------------------------------------------------------ O2 vs O1 (config 1)
def test_O2_matches_O1_config1_gates(cfg1_case):
    c, xy, K, z, F = cfg1_case
    d = dense_eval(K, xy, z)
    o = rsf_mle_eval(K, xy, z, c.eps_fact, c.eps_peel, c.leaf, c.seed, philox_normal, block=16)
    assert abs(o["logdet"] - d["logdet"]) <= 10 * c.eps * abs(d["logdet"])
    assert abs(o["quad"] - d["quad"]) <= 10 * c.eps * abs(d["quad"])
    assert np.all(np.abs(o["grad"] - d["grad"]) <= 1e-3 * np.abs(d["grad"]))
