"""Anisotropic kernels and the paper's own grid workload (next row f1; PAPER P:704-727,
Eqs. specrq / specmatern P:710-716).  CPU: oracle pins (finite differences, isotropic limit,
hand values of the paper's forms, dense g vs finite differences of l).  GPU: the CUDA path
against the dense oracle on a 48 x 48 grid with theta = [10, 7] on [0, 100]^2 (= [0.1, 0.07]
on the unit square, reading R-f1)."""
import math

import numpy as np
import pytest

from oracle.dense import dense_eval, dense_sample
from oracle.kernels import FAMILIES, Kernel
from workloads import paper_grid_points, w_for, config

TH = (0.1, 0.07)


def _pts(n=60, seed=0):
    return np.random.default_rng(seed).random((n, 2))


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("name", ["rho", "rho2"])
def test_aniso_derivatives_vs_finite_differences(family, name):
    xy = _pts()
    k = Kernel(family, TH[0], 1.3, 1e-4, 0.5, ("rho", "rho2"), rho2=TH[1])
    idx = np.arange(len(xy))
    D = k.dsigma_block(name, xy, idx, idx)
    v = k.value(name)
    h = 1e-4 * v
    f = lambda t: k.with_param(name, t).sigma_block(xy, idx, idx)
    fd = (8 * (f(v + h) - f(v - h)) - (f(v + 2 * h) - f(v - 2 * h))) / (12 * h)   # Richardson
    assert np.max(np.abs(fd - D)) <= 1e-8 * np.max(np.abs(D))
    assert np.all(np.diag(D) == 0.0)


@pytest.mark.parametrize("family", FAMILIES)
def test_isotropic_limit(family):
    """rho2 = rho: the anisotropic kernel is the isotropic one, and d/drho_1 + d/drho_2 = d/drho."""
    xy = _pts(40, 1)
    idx = np.arange(len(xy))
    ka = Kernel(family, 0.08, 1.0, 1e-3, 0.7, ("rho", "rho2"), rho2=0.08)
    ki = Kernel(family, 0.08, 1.0, 1e-3, 0.7, ("rho",))
    assert np.allclose(ka.sigma_block(xy, idx, idx), ki.sigma_block(xy, idx, idx), rtol=1e-14, atol=1e-15)
    s = ka.dsigma_block("rho", xy, idx, idx) + ka.dsigma_block("rho2", xy, idx, idx)
    assert np.allclose(s, ki.dsigma_block("rho", xy, idx, idx), rtol=1e-12, atol=1e-14)


def test_paper_kernel_hand_values():
    """Eq. specrq with alpha = 1/2 at ||x-y||_theta^2 = 3 is 1/2; Eq. specmatern at
    ||x-y||_theta = 1/sqrt(3) is 2/e."""
    th1, th2 = TH
    # dx^2/th1^2 + dy^2/th2^2 = 3 with dx/th1 = 1, dy/th2 = sqrt(2)
    P = np.array([[0.0, 0.0]])
    Q = np.array([[th1, math.sqrt(2.0) * th2]])
    rq = Kernel("rq", th1, 1.0, 0.0, 0.5, ("rho",), rho2=th2)
    assert rq.sigma_points(P, Q)[0, 0] == pytest.approx(0.5, rel=1e-15)
    Q = np.array([[th1 / math.sqrt(6.0), th2 / math.sqrt(6.0)]])   # q^2 = 1/6 + 1/6 = 1/3
    m = Kernel("matern32", th1, 1.0, 0.0, 1.0, ("rho",), rho2=th2)
    assert m.sigma_points(P, Q)[0, 0] == pytest.approx(2.0 / math.e, rel=1e-15)


def test_dense_gradient_vs_finite_differences_of_ell():
    xy = paper_grid_points(16)
    k = Kernel("matern32", TH[0], 1.0, 1e-4, 1.0, ("rho", "rho2"), rho2=TH[1])
    z = np.random.default_rng(3).standard_normal(len(xy))
    d = dense_eval(k, xy, z)
    for i, name in enumerate(("rho", "rho2")):
        v = k.value(name)
        h = 1e-5 * v
        lp = dense_eval(k.with_param(name, v + h), xy, z)["ell"]
        lm = dense_eval(k.with_param(name, v - h), xy, z)["ell"]
        assert d["grad"][i] == pytest.approx((lp - lm) / (2 * h), rel=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("family,alpha", [("matern32", 1.0), ("rq", 0.5)])
def test_gpu_aniso_paper_grid_vs_dense(family, alpha):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1603_08057_b200 as R
    m = 48
    xy = paper_grid_points(m)
    ok = Kernel(family, TH[0], 1.0, 1e-4, alpha, ("rho", "rho2"), rho2=TH[1])
    rk = R.Kernel(family, TH[0], 1.0, 1e-4, alpha, ("rho", "rho2"), rho2=TH[1])
    c = config(2)
    z = dense_sample(ok, xy, w_for(c, len(xy)))
    d = dense_eval(ok, xy, z)
    dev = torch.device("cuda:0")
    ctx = R.Context(0)
    eps, eps_fact = 1e-6, 1e-10      # paper: eps_fact = eps_peel / 1000, tightened for kappa ~ 1e6
    F = R.Factor(ctx, torch.from_numpy(xy).to(dev), rk, eps_fact, 64)
    assert abs(F.logdet() - d["logdet"]) <= 10 * eps * abs(d["logdet"])
    r = R.gp_mle_eval(ctx, torch.from_numpy(xy).to(dev), torch.from_numpy(z).to(dev), rk, eps_fact, 64,
                      R.Opts(eps_peel=eps))
    assert abs(r.diag.quad - d["quad"]) <= 10 * eps * abs(d["quad"])
    g = np.array(r.grad)
    assert np.all(np.abs(g - d["grad"]) <= 1e-3 * np.abs(d["grad"])), (g, d["grad"])
