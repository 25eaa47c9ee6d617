"""Hutchinson estimator (next row f2): oracle pins on CPU and the CUDA
estimator against the oracle on identical Rademacher probes (GPU)."""
import math

import numpy as np
import pytest

from oracle.hutch import hutch_trace
from workloads import philox_rademacher

SEED = 1603080570


def _probe(rows, p):
    return philox_rademacher(SEED, rows.astype(np.uint64), p)


def test_rademacher_entries():
    v = philox_rademacher(SEED, np.arange(20000, dtype=np.uint64), 3)
    assert set(np.unique(v)) == {-1.0, 1.0}
    assert abs(v.mean()) < 0.03     # 4.2 standard deviations of a fair +-1 mean at n = 20000


def test_identity_and_diagonal_exact():
    """u^T D u = sum_i d_i u_i^2 = Tr(D) for every Rademacher u: exact for any q."""
    n = 300
    est, se = hutch_trace(lambda X: X, n, 8, _probe)
    assert est == n and se == 0.0
    d = np.random.default_rng(1).random(n) * 5 - 1
    est, se = hutch_trace(lambda X: d[:, None] * X, n, 5, _probe)
    assert est == pytest.approx(d.sum(), rel=1e-14) and se < 1e-12


def test_unbiased_random_symmetric():
    """E[u^T G u] = Tr(G): 4000 probes of a random symmetric 40 x 40 within 5 standard errors."""
    G = np.random.default_rng(2).standard_normal((40, 40))
    G = G + G.T
    est, se = hutch_trace(lambda X: G @ X, 40, 4000, _probe)
    assert abs(est - np.trace(G)) <= 5 * se


@pytest.mark.gpu
def test_gpu_hutch_matches_oracle_on_identical_probes():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1603_08057_b200 as R
    from oracle.dense import dense_sample, dense_sigma
    from oracle.kernels import Kernel as OK
    from workloads import config, points_for, w_for
    dev = torch.device("cuda:0")
    ctx = R.Context(0)
    # P6 diagonal Sigma (kernel underflows between grid neighbours): Tr(F^-1) = n / (s2 + tau) exactly
    m = 32
    g = (np.arange(m) + 0.5) / m
    xy = np.array([(a, b) for a in g for b in g])
    rk = R.Kernel("matern12", (1.0 / m) / 750.0, 1.3, 0.2, 1.0, ("rho",))
    F = R.Factor(ctx, torch.from_numpy(xy).to(dev), rk, 1e-8, 64)
    t, se = R.hutch_trace(F, None, 40, SEED)
    assert t == pytest.approx(len(xy) / 1.5, rel=1e-13) and se < 1e-9
    # config 1: same probes through the dense oracle
    c = config(1)
    xy = points_for(c)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    rk = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    S = dense_sigma(ok, xy)
    Si = ok.dsigma_block("rho", xy, np.arange(len(xy)), np.arange(len(xy)))
    F = R.Factor(ctx, torch.from_numpy(xy).to(dev), rk, c.eps_fact, c.leaf)
    Fi = R.Factor(ctx, torch.from_numpy(xy).to(dev), rk, c.eps_fact, c.leaf, which=0)
    q = 96
    t_gpu, se_gpu = R.hutch_trace(F, Fi, q, SEED)
    t_or, se_or = hutch_trace(lambda X: np.linalg.solve(S, Si @ X), len(xy), q, _probe)
    assert abs(t_gpu - t_or) <= 1e-6 * abs(t_or)
    assert se_gpu == pytest.approx(se_or, rel=1e-4)
    ti_gpu, _ = R.hutch_trace(F, None, q, SEED)
    ti_or, _ = hutch_trace(lambda X: np.linalg.solve(S, X), len(xy), q, _probe)
    assert abs(ti_gpu - ti_or) <= 1e-6 * abs(ti_or)


@pytest.mark.gpu
def test_gpu_peel_vs_hutch_full_size_config3():
    """Full BASELINE size (config 3, n = 262,144; no dense reference): the peeled Tr(F^-1 F_rho)
    agrees with an independent Hutchinson estimate (256 probes) within 5 standard errors."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1603_08057_b200 as R
    from workloads import config, points_for
    c = config(3)
    dev = torch.device("cuda:0")
    ctx = R.Context(0)
    rk = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    xy = torch.from_numpy(points_for(c)).to(dev)
    F = R.Factor(ctx, xy, rk, c.eps_fact, c.leaf)
    Fi = R.Factor(ctx, xy, rk, c.eps_fact, c.leaf, which=0)
    tp, pd = R.peel_trace(F, Fi, c.eps_peel)
    th, se = R.hutch_trace(F, Fi, 256, SEED)
    assert math.isfinite(tp) and se > 0
    assert abs(tp - th) <= 5 * se, (tp, th, se)
