"""Profile likelihood and kriging mean (next row f3): oracle pins
(CPU) and the CUDA path against the dense oracle (GPU)."""
import numpy as np
import pytest

from oracle.kernels import Kernel
from oracle.profile import dense_cond_mean, dense_profile_eval
from workloads import config, points_for, w_for


def _case(n=200, seed=0):
    xy = np.random.default_rng(seed).random((n, 2))
    k = Kernel("matern32", 0.12, 1.0, 1e-2, 1.0, ("rho", "nugget"))
    z = 0.7 + 1.9 * np.random.default_rng(seed + 1).standard_normal(n)
    return xy, k, z


def test_profile_gradient_vs_finite_differences():
    xy, k, z = _case()
    d = dense_profile_eval(k, xy, z)
    for i, name in enumerate(k.theta):
        v = k.value(name)
        h = 1e-5 * v
        lp = dense_profile_eval(k.with_param(name, v + h), xy, z)["ell"]
        lm = dense_profile_eval(k.with_param(name, v - h), xy, z)["ell"]
        assert d["grad"][i] == pytest.approx((lp - lm) / (2 * h), rel=1e-6)


def test_profile_scaling_identity():
    """Q(s z) = s^2 Q(z)  =>  l~(s z) = l~(z) - n log s  (the profiled variance absorbs the scale)."""
    xy, k, z = _case(150, 3)
    a = dense_profile_eval(k, xy, z)["ell"]
    b = dense_profile_eval(k, xy, 3.7 * z)["ell"]
    assert b == pytest.approx(a - len(z) * np.log(3.7), rel=1e-12)


def test_profile_is_maximum_over_scale():
    """With Sigma + 1 1^T as the covariance model of z, maximizing the Gaussian log-likelihood of
    z ~ N(0, s2 (Sigma + 1 1^T)) over s2 gives l~ + 1/2 log(1 + 1^T Sigma^-1 1) (matrix determinant lemma)."""
    xy, k, z = _case(120, 5)
    n = len(z)
    d = dense_profile_eval(k, xy, z)
    S = np.array(k.sigma_block(xy, np.arange(n), np.arange(n))) + np.ones((n, n))
    s2 = d["Q"] / n
    sign, ld = np.linalg.slogdet(s2 * S)
    full = -0.5 * n - 0.5 * ld - 0.5 * n * np.log(2 * np.pi)
    Sig = np.array(k.sigma_block(xy, np.arange(n), np.arange(n)))
    corr = 0.5 * np.log(1.0 + np.ones(n) @ np.linalg.solve(Sig, np.ones(n)))
    assert full == pytest.approx(d["ell"] - corr, rel=1e-12)


def test_cond_mean_interpolates_without_nugget():
    """nugget = 0: Sigma_12 = Sigma_22 rows at the data locations, so the mean reproduces z."""
    xy = np.random.default_rng(7).random((80, 2))
    k = Kernel("matern12", 0.1, 1.3, 0.0, 1.0, ("rho",))
    z = np.random.default_rng(8).standard_normal(80)
    m = dense_cond_mean(k, xy, z, xy[:10])
    assert np.allclose(m, z[:10], rtol=1e-9, atol=1e-9)


@pytest.mark.gpu
def test_gpu_profile_and_cond_mean_vs_dense():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1603_08057_b200 as R
    c = config(2)
    n = 4096
    xy = points_for(c, n)
    ok = Kernel("matern32", c.rho, 1.0, c.nugget, 1.0, ("rho", "nugget"))
    rk = R.Kernel("matern32", c.rho, 1.0, c.nugget, 1.0, ("rho", "nugget"))
    z = 0.5 + 2.0 * w_for(c, n)
    d = dense_profile_eval(ok, xy, z)
    dev = torch.device("cuda:0")
    ctx = R.Context(0)
    r = R.gp_profile_eval(ctx, torch.from_numpy(xy).to(dev), torch.from_numpy(z).to(dev), rk, c.eps_fact, c.leaf,
                          R.Opts(eps_peel=c.eps_peel))
    assert abs(r.ell - d["ell"]) <= 1e-5 * abs(d["ell"])
    assert abs(r.diag.quad - d["Q"]) <= 10 * c.eps * d["Q"]
    g = np.array(r.grad)
    assert np.all(np.abs(g - d["grad"]) <= 1e-3 * np.abs(d["grad"])), (g, d["grad"])
    with pytest.raises(R.RsfError):
        R.gp_profile_eval(ctx, torch.from_numpy(xy).to(dev), torch.from_numpy(z).to(dev),
                          R.Kernel("matern32", c.rho, 1.0, c.nugget, 1.0, ("sigma2",)), c.eps_fact, c.leaf)
    # kriging mean at 300 new locations
    F = R.Factor(ctx, torch.from_numpy(xy).to(dev), rk, c.eps_fact, c.leaf)
    xn = np.random.default_rng(9).random((300, 2))
    want = dense_cond_mean(ok, xy, z, xn)
    got = R.gp_cond_mean(F, torch.from_numpy(z).to(dev), torch.from_numpy(xn).to(dev)).cpu().numpy()
    # Tolerance derived, not fitted: m_hat - m = Sigma_12 (F^-1 z - Sigma^-1 z) and
    # F^-1 z - Sigma^-1 z = Sigma^-1 (Sigma x - z) with x = F^-1 z, so
    #   ||m_hat - m|| <= ||Sigma_12||_2 ||Sigma^-1||_2 ||Sigma x - z||,
    # and the north star's solve gate bounds ||Sigma x - z|| <= 10 eps ||z|| (asserted here too).
    from oracle.dense import dense_sigma
    S = dense_sigma(ok, xy)
    x = F.solve(torch.from_numpy(z).to(dev)).cpu().numpy()
    res = np.linalg.norm(S @ x - z)
    assert res <= 10 * c.eps * np.linalg.norm(z)
    S12 = ok.sigma_points(xn, xy)
    bound = np.linalg.norm(S12, 2) / np.linalg.eigvalsh(S)[0] * res
    assert np.linalg.norm(got - want) <= bound, (np.linalg.norm(got - want), bound)
    got_h = R.gp_cond_mean(F, np.ascontiguousarray(z), np.ascontiguousarray(xn), np.empty(300))
    assert np.array_equal(got_h, got)


def test_cond_cov_closed_forms():
    """dense_cond_cov against (a) one data point at the new location: sigma2 + tau -
    sigma2^2 / (sigma2 + tau); (b) the Schur-complement identity S^-1 = [(Sigma_joint)^-1]_11."""
    from oracle.profile import dense_cond_cov
    from oracle.dense import dense_sigma
    k = Kernel("matern32", 0.2, 1.3, 0.05, 1.0, ("rho",))
    x = np.array([[0.3, 0.4]])
    S = dense_cond_cov(k, x, x.copy())
    assert S[0, 0] == pytest.approx(1.3 + 0.05 - 1.3 ** 2 / 1.35, rel=1e-12)
    r = np.random.default_rng(12)
    xd, xn = r.random((60, 2)), r.random((7, 2))
    S = dense_cond_cov(k, xd, xn)
    J = np.linalg.inv(dense_sigma(k, np.vstack([xn, xd])))
    np.testing.assert_allclose(np.linalg.inv(S), J[:7, :7], rtol=1e-9)


@pytest.mark.gpu
def test_gpu_cond_sample_mean_and_covariance():
    """gp_cond_sample (Remark conditional): with w = 0 it returns the conditional mean;
    its linear map B (columns: out(w = e_j) - out(0) over all m + n2 joint coordinates) satisfies
    B B^T = Sigma_11 - Sigma_12 Sigma_22^-1 Sigma_12^T (dense oracle)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1603_08057_b200 as R
    from oracle.profile import dense_cond_cov
    dev = torch.device("cuda:0")
    r = np.random.default_rng(13)
    n2, m = 1500, 120
    xd, xn = r.random((n2, 2)), r.random((m, 2))
    ok = Kernel("matern32", 0.1, 1.0, 1e-2, 1.0, ("rho",))
    rk = R.Kernel("matern32", 0.1, 1.0, 1e-2, 1.0, ("rho",))
    z = r.standard_normal(n2)
    ctx = R.Context(0)
    F = R.Factor(ctx, torch.from_numpy(np.vstack([xn, xd])).to(dev), rk, 1e-11, 64)
    F22 = R.Factor(ctx, torch.from_numpy(xd).to(dev), rk, 1e-11, 64)
    N = n2 + m
    W = torch.zeros((N + 1, N), dtype=torch.float64, device=dev)
    W[1:] = torch.eye(N, dtype=torch.float64, device=dev)
    out = R.gp_cond_sample(F, F22, torch.from_numpy(z).to(dev), W).cpu().numpy()
    mu = dense_cond_mean(ok, xd, z, xn)
    assert np.linalg.norm(out[0] - mu) <= 1e-6 * np.linalg.norm(mu)
    B = (out[1:] - out[0]).T            # m x N
    S = dense_cond_cov(ok, xd, xn)
    assert np.linalg.norm(B @ B.T - S) <= 1e-6 * np.linalg.norm(S)
    # host buffers give the same result
    oh = R.gp_cond_sample(F, F22, z.copy(), np.ascontiguousarray(W[:3].cpu().numpy()))
    np.testing.assert_allclose(oh, out[:3], rtol=1e-12, atol=1e-14)
