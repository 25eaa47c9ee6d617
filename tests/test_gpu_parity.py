"""Parity of the CUDA path (through the C ABI) against the oracle.

Gates (BASELINE.json north_star): relative error of log|Sigma| and of
z^T Sigma^-1 z <= 10 eps, solve residual ||Sigma x - z|| / ||z|| <= 10 eps, relative
error of each g_i <= 1e-3, at the configured eps = 1e-6 (ID tolerance eps_fact = eps/100,
reading R-A).  Small configurations compare element by element with the dense oracle
O1; full-size configurations use sampled rows the oracle computes one by one.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.dense import dense_eval, dense_sample, dense_sigma  # noqa: E402
from oracle.kernels import Kernel as OK  # noqa: E402
from workloads import config, points_for, w_for  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_08057_b200 as R  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx():
    return R.Context(0)


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV)


def _kern(c, theta=None):
    th = c.theta if theta is None else theta
    return (OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, th),
            R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, th))


def _case(cid, n=None, **over):
    c = config(cid, **over) if over else config(cid)
    n = n or c.n
    xy = points_for(c, n)
    ok, rk = _kern(c)
    z = dense_sample(ok, xy, w_for(c, n))
    return c, xy, ok, rk, z


def _gates(c, d, F, x, z, S):
    eps = c.eps
    ld = F.logdet()
    assert abs(ld - d["logdet"]) <= 10 * eps * abs(d["logdet"])
    assert abs(z @ x - d["quad"]) <= 10 * eps * abs(d["quad"])
    assert np.linalg.norm(S @ x - z) <= 10 * eps * np.linalg.norm(z)


@pytest.fixture(scope="module")
def cfg1(ctx):
    c, xy, ok, rk, z = _case(1)
    d = dense_eval(ok, xy, z, fisher=True)
    F = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf)
    return c, xy, ok, rk, z, d, F, dense_sigma(ok, xy)


def test_cfg1_logdet_quad_residual(cfg1):
    c, xy, ok, rk, z, d, F, S = cfg1
    x = F.solve(_d(z)).cpu().numpy()
    _gates(c, d, F, x, z, S)


def test_cfg1_apply_solve_sample_identities(cfg1, ctx):
    c, xy, ok, rk, z, d, F, S = cfg1
    v = np.random.default_rng(0).standard_normal(len(xy))
    av = F.apply(_d(v)).cpu().numpy()
    assert np.linalg.norm(av - S @ v) <= 1e-6 * np.linalg.norm(S @ v)
    back = F.apply(F.solve(_d(v))).cpu().numpy()
    assert np.linalg.norm(back - v) <= 1e-11 * np.linalg.norm(v)
    # F^{1/2} (F^{1/2})^T = F on a small problem (columns of the identity as a block)
    n = 300
    xs = np.random.default_rng(1).random((n, 2))
    Fs = R.Factor(ctx, _d(xs), rk, 1e-8, 32)
    eye = torch.eye(n, dtype=torch.float64, device=DEV)
    Sq = Fs.sample(eye.clone()).cpu().numpy().T
    Fa = Fs.apply(eye.clone()).cpu().numpy().T
    assert np.max(np.abs(Sq @ Sq.T - Fa)) <= 1e-12 * np.max(np.abs(Fa))


def test_cfg1_sigma_i_compression(cfg1, ctx):
    c, xy, ok, rk, z, d, F, S = cfg1
    n = len(xy)
    Fi = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf, which=0)
    eye = torch.eye(n, dtype=torch.float64, device=DEV)
    V = Fi.apply(eye).cpu().numpy().T
    Si = ok.dsigma_block("rho", xy, np.arange(n), np.arange(n))
    assert np.max(np.abs(V - V.T)) <= 1e-12 * np.max(np.abs(V))
    assert np.linalg.norm(V - Si) <= 1e-6 * np.linalg.norm(Si)
    with pytest.raises(R.RsfError):
        Fi.logdet()


def test_cfg1_peel_trace(cfg1, ctx):
    c, xy, ok, rk, z, d, F, S = cfg1
    Fi = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf, which=0)
    tr, pd = R.peel_trace(F, Fi, c.eps_peel)
    assert abs(tr - d["trace"][0]) <= 1e-5 * abs(d["trace"][0])
    assert 1.0 <= pd.cancellation < 1.1
    tinv, _ = R.peel_trace(F, None, c.eps_peel)
    assert abs(tinv - d["trace_inv"]) <= 1e-5 * d["trace_inv"]


def test_cfg1_gp_mle_eval_gates(cfg1, ctx):
    c, xy, ok, rk, z, d, F, S = cfg1
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
    assert abs(r.diag.logdet - d["logdet"]) <= 10 * c.eps * abs(d["logdet"])
    assert abs(r.diag.quad - d["quad"]) <= 10 * c.eps * d["quad"]
    n = len(xy)
    assert r.ell == pytest.approx(-0.5 * r.diag.quad - 0.5 * r.diag.logdet - 0.5 * n * math.log(2 * math.pi), rel=1e-14)
    g = np.array(r.grad)
    assert np.all(np.abs(g - d["grad"]) <= 1e-3 * np.abs(d["grad"]))
    # Fisher-scaled error (R-J): far below one standard deviation of the score
    assert np.all(np.abs(g - d["grad"]) <= 1e-3 * d["fisher_sd"])


@pytest.mark.parametrize("cid,n,extra", [
    (3, 4096, {}),                      # jittered 64 x 64 grid, RQ, theta = (rho, alpha)
    (4, 8192, {}),                      # clustered, adaptive tree, Matern 1/2, theta = (rho, sigma2)
    (5, 4096, {}),                      # Matern 5/2, leaf 128, eps_fact 1e-9, theta = (rho, sigma2, nugget)
])
def test_small_configs_vs_dense(ctx, cid, n, extra):
    c, xy, ok, rk, z = _case(cid, n, **extra)
    d = dense_eval(ok, xy, z)
    S = dense_sigma(ok, xy)
    F = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf)
    x = F.solve(_d(z)).cpu().numpy()
    _gates(c, d, F, x, z, S)
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
    g = np.array(r.grad)
    assert np.all(np.abs(g - d["grad"]) <= 1e-3 * np.abs(d["grad"])), (g, d["grad"])


def test_cfg2_full_vs_dense(ctx):
    c, xy, ok, rk, z = _case(2)
    d = dense_eval(ok, xy, z)
    S = dense_sigma(ok, xy)
    F = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf)
    x = F.solve(_d(z)).cpu().numpy()
    _gates(c, d, F, x, z, S)
    del S
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
    g = np.array(r.grad)
    assert np.all(np.abs(g - d["grad"]) <= 1e-3 * np.abs(d["grad"])), (g, d["grad"])


def _sampled_residual(ok, xy, x, z, rows):
    res = np.array([ok.sigma_block(xy, np.array([i]), np.arange(len(xy)))[0] @ x - z[i] for i in rows])
    return math.sqrt(len(xy) / len(rows) * float(res @ res)) / np.linalg.norm(z)


@pytest.mark.parametrize("cid", [3, 4])
def test_full_size_factor_solve_sampled_rows(ctx, cid):
    """Full BASELINE sizes (262,144 and 1,048,576 points): the solve residual on 48 rows
    the oracle evaluates one by one, plus apply(solve(b)) = b."""
    c = config(cid)
    xy = points_for(c)
    ok, rk = _kern(c)
    F = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf)
    w = _d(w_for(c))
    z = F.sample(w)
    x = F.solve(z)
    back = F.apply(x)
    zn, xn, bn = z.cpu().numpy(), x.cpu().numpy(), back.cpu().numpy()
    assert np.linalg.norm(bn - zn) <= 1e-10 * np.linalg.norm(zn)
    rows = np.random.default_rng(cid).choice(len(xy), 48, replace=False)
    assert _sampled_residual(ok, xy, xn, zn, rows) <= 10 * c.eps
    assert math.isfinite(F.logdet())


def test_separable_closed_form(ctx):
    """P7: squared-exponential kernel on a tensor grid; log|Sigma|, z^T Sigma^-1 z and
    Tr(Sigma^-1 Sigma_rho) in closed form from two 1-D eigenproblems."""
    r = np.random.default_rng(8)
    ma, mb, rho, s2, tau = 96, 80, 0.05, 1.2, 0.05
    a = np.sort(r.random(ma))
    b = np.sort(r.random(mb))
    xy = np.array([(x, y) for x in a for y in b])
    Ka = np.exp(-(a[:, None] - a[None]) ** 2 / (2 * rho ** 2))
    Kb = np.exp(-(b[:, None] - b[None]) ** 2 / (2 * rho ** 2))
    Kap = Ka * (a[:, None] - a[None]) ** 2 / rho ** 3
    Kbp = Kb * (b[:, None] - b[None]) ** 2 / rho ** 3
    la, Qa = np.linalg.eigh(Ka)
    lb, Qb = np.linalg.eigh(Kb)
    lap = np.einsum("ij,ik,kj->j", Qa, Kap, Qa)
    lbp = np.einsum("ij,ik,kj->j", Qb, Kbp, Qb)
    ev = s2 * np.outer(la, lb) + tau
    logdet = float(np.sum(np.log(ev)))
    tr = float(np.sum(s2 * (np.outer(lap, lb) + np.outer(la, lbp)) / ev))
    z = r.standard_normal(ma * mb)
    zh = Qa.T @ z.reshape(ma, mb) @ Qb
    quad = float(np.sum(zh ** 2 / ev))
    rk = R.Kernel("sqexp", rho, s2, tau, 1.0, ("rho",))
    F = R.Factor(ctx, _d(xy), rk, 1e-10, 64)
    Fi = R.Factor(ctx, _d(xy), rk, 1e-10, 64, which=0)
    assert F.logdet() == pytest.approx(logdet, rel=1e-8)
    assert float(z @ F.solve(_d(z)).cpu().numpy()) == pytest.approx(quad, rel=1e-6)
    t, _ = R.peel_trace(F, Fi, 1e-8)
    assert t == pytest.approx(tr, rel=1e-6)


def test_diagonal_sigma_underflow(ctx):
    """P6: kernel underflows to exactly 0 between grid neighbours -> Sigma = (s2 + tau) I."""
    m = 32
    d = 1.0 / m
    g = (np.arange(m) + 0.5) * d
    xy = np.array([(a, b) for a in g for b in g])
    rk = R.Kernel("matern12", d / 750.0, 1.3, 0.2, 1.0, ("rho",))
    F = R.Factor(ctx, _d(xy), rk, 1e-8, 64)
    assert F.logdet() == pytest.approx(len(xy) * math.log(1.5), rel=1e-13)
    z = np.random.default_rng(3).standard_normal(len(xy))
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, 1e-8, 64)
    assert r.grad[0] == pytest.approx(0.0, abs=1e-12)


def test_edge_cases_small_n(ctx):
    rk = R.Kernel("matern32", 0.2, 1.4, 0.3, 1.0, ("rho", "sigma2", "nugget"))
    xy = np.array([[0.3, 0.6]])
    z = np.array([0.77])
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, 1e-8, 64)
    a = 1.7
    assert r.ell == pytest.approx(-z[0] ** 2 / (2 * a) - 0.5 * math.log(a) - 0.5 * math.log(2 * math.pi), rel=1e-14)
    gs = 0.5 * z[0] ** 2 / a ** 2 - 0.5 / a
    assert r.grad[0] == pytest.approx(0.0, abs=1e-15)
    assert r.grad[1] == pytest.approx(gs, rel=1e-12) and r.grad[2] == pytest.approx(gs, rel=1e-12)
    # n <= leaf: the RSF is the dense Cholesky
    xy = np.random.default_rng(4).random((50, 2))
    ok = OK("matern32", 0.2, 1.4, 0.3, 1.0, ("rho", "sigma2", "nugget"))
    z = np.random.default_rng(5).standard_normal(50)
    d = dense_eval(ok, xy, z)
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, 1e-8, 64)
    assert r.ell == pytest.approx(d["ell"], rel=1e-12)
    assert np.allclose(r.grad, d["grad"], rtol=1e-9)


def test_duplicates_and_degenerate_leaf(ctx):
    """100 coincident points (a depth-30 degenerate leaf) among random ones."""
    r = np.random.default_rng(6)
    xy = np.vstack([np.full((100, 2), 0.3), r.random((900, 2))])
    ok = OK("rq", 0.1, 1.0, 0.05, 1.0, ("rho",))
    rk = R.Kernel("rq", 0.1, 1.0, 0.05, 1.0, ("rho",))
    z = r.standard_normal(1000)
    d = dense_eval(ok, xy, z)
    F = R.Factor(ctx, _d(xy), rk, 1e-8, 64)
    assert F.info().levels == 30
    assert F.logdet() == pytest.approx(d["logdet"], rel=1e-5)
    rr = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, 1e-8, 64)
    assert abs(rr.grad[0] - d["grad"][0]) <= 1e-3 * abs(d["grad"][0])


def test_invalid_inputs_fail_loudly(ctx):
    rk = R.Kernel("rq", 0.1, 1.0, 0.01)
    ok_pts = np.random.default_rng(7).random((100, 2))
    for bad in (ok_pts * 2.0, np.where(np.arange(200).reshape(100, 2) == 5, np.nan, ok_pts)):
        with pytest.raises(R.RsfError) as e:
            R.Factor(ctx, _d(bad), rk, 1e-8, 64)
        assert e.value.code == 1
    with pytest.raises(R.RsfError):
        R.Factor(ctx, _d(ok_pts), rk, 0.0, 64)
    with pytest.raises(R.RsfError):
        R.Factor(ctx, _d(ok_pts), rk, 1e-8, 0)
    with pytest.raises(R.RsfError):
        R.Factor(ctx, _d(ok_pts), R.Kernel("rq", -0.1), 1e-8, 64)
    # numerical failure: exact duplicates and no nugget -> singular Sigma -> RSF_ENUMERIC
    dup = np.vstack([ok_pts, ok_pts[:10]])
    with pytest.raises(R.RsfError) as e:
        R.Factor(ctx, _d(dup), R.Kernel("matern12", 0.1, 1.0, 0.0), 1e-8, 16)
    assert e.value.code == 2


def test_determinism_and_host_buffers(ctx):
    c, xy, ok, rk, z = _case(1)
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed)
    a = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, c.eps_fact, c.leaf, o)
    b = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, c.eps_fact, c.leaf, o)
    h = R.gp_mle_eval(ctx, np.ascontiguousarray(xy), np.ascontiguousarray(z), rk, c.eps_fact, c.leaf, o)
    assert a.ell == b.ell == h.ell
    assert a.grad == b.grad == h.grad


def test_kernel_launches_are_counted(ctx):
    c, xy, ok, rk, z = _case(1)
    l0 = R.kernel_launches()
    R.gp_mle_eval(ctx, _d(xy), _d(z), rk, c.eps_fact, c.leaf)
    assert R.kernel_launches() - l0 > 100


_FUSED_PROBE = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1603_08057_b200 as R
from workloads import config, points_for
c = config(2)
n = 4096
xy = points_for(c, n)
dev = torch.device("cuda:0")
ctx = R.Context(0)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
F = R.Factor(ctx, torch.from_numpy(xy).to(dev), K, 1e-8, 32)
Fi = R.Factor(ctx, torch.from_numpy(xy).to(dev), K, 1e-8, 32, which=0)
B = torch.from_numpy(np.random.default_rng(11).standard_normal((40, n))).to(dev)
np.save(sys.argv[2], np.concatenate([F.solve(B.clone()).cpu().numpy(), Fi.apply(B.clone()).cpu().numpy()], axis=0))
"""


def test_fused_sweeps_match_batched_gemm_path(tmp_path):
    """The fused small-box level sweeps (sweep.cu, every level of a leaf-32 tree; FMA kernel and
    the DMMA kernel of RSF_SWEEP_MMA=1) against the batched-GEMM level steps (RSF_FUSED=0):
    F^-1 B and F_i B on 40 right-hand sides agree to round-off."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "probe.py"
    script.write_text(_FUSED_PROBE)
    out = {}
    for flag, mma in (("1", "0"), ("0", "0"), ("1", "1")):
        f = tmp_path / f"out{flag}{mma}.npy"
        env = dict(os.environ, RSF_FUSED=flag, RSF_SWEEP_MMA=mma)
        subprocess.run([sys.executable, str(script), root, str(f)], env=env, check=True, timeout=600)
        out[flag + mma] = np.load(f)
    b = out["00"]
    for key in ("10", "11"):   # FMA fused kernel (|I| <= 128), DMMA fused kernel (|I| <= 256)
        assert np.linalg.norm(out[key] - b) <= 1e-10 * np.linalg.norm(b), key


@pytest.fixture(scope="module")
def cfg2_4096(ctx):
    """Config 2's recipe (Matern 3/2, theta = (rho, sigma2)) at n = 4096: dense oracle O1."""
    c, xy, ok, rk, z = _case(2, 4096)
    d = dense_eval(ok, xy, z)
    return c, xy, ok, rk, z, d


def test_cfg2_sigma_rho_compression_and_traces(ctx, cfg2_4096):
    """Sigma_rho compression (apply-only, R-F) against the dense derivative matrix on 24 random
    vectors; peeled Tr(F^-1 F_rho) and Tr(F^-1) (G = F^-1, R-G) against the dense traces."""
    c, xy, ok, rk, z, d = cfg2_4096
    n = len(xy)
    F = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf)
    Fi = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf, which=0)
    V = np.random.default_rng(21).standard_normal((24, n))
    Si = ok.dsigma_block("rho", xy, np.arange(n), np.arange(n))
    got = Fi.apply(_d(V)).cpu().numpy()
    want = V @ Si
    assert np.linalg.norm(got - want) <= 1e-6 * np.linalg.norm(want)
    tr, pd = R.peel_trace(F, Fi, c.eps_peel)
    assert abs(tr - d["trace"][0]) <= 1e-5 * abs(d["trace"][0])
    tinv, _ = R.peel_trace(F, None, c.eps_peel)
    assert abs(tinv - d["trace_inv"]) <= 1e-5 * d["trace_inv"]


def test_abi_strided_and_host_blocks(ctx, cfg2_4096):
    """rsf_solve on a strided (ld > n) host block equals the device result; nrhs = 0 is a no-op;
    ld < n is rejected (RSF_EINVAL)."""
    import ctypes as C
    from paper_1603_08057_b200 import _lib
    c, xy, ok, rk, z, d = cfg2_4096
    n = len(xy)
    F = R.Factor(ctx, _d(xy), rk, c.eps_fact, c.leaf)
    B = np.random.default_rng(22).standard_normal((3, n))
    ref = F.solve(_d(B)).cpu().numpy()
    ld = n + 5
    H = np.zeros((3, ld))
    H[:, :n] = B
    out = np.zeros_like(H)
    st = R.lib.rsf_solve(F.h, H.ctypes.data, out.ctypes.data, 3, ld)
    assert st == 0
    assert np.array_equal(out[:, :n], ref)
    assert R.lib.rsf_solve(F.h, H.ctypes.data, out.ctypes.data, 0, ld) == 0
    assert R.lib.rsf_solve(F.h, H.ctypes.data, out.ctypes.data, 3, n - 1) == _lib.RSF_EINVAL


_PAR_PROBE = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1603_08057_b200 as R
from workloads import config, points_for, w_for
c = config(3)
n = 4096
xy = torch.from_numpy(points_for(c, n)).cuda()
z = torch.from_numpy(w_for(c, n)).cuda()
ctx = R.Context(0)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, ("rho", "alpha", "nugget"))
r = R.gp_mle_eval(ctx, xy, z, K, 1e-9, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
r2 = R.gp_mle_eval(ctx, xy, z, K, 1e-9, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
json.dump({"ell": r.ell, "grad": list(r.grad), "trace": list(r.diag.trace)[:3],
           "same2": r2.ell == r.ell and list(r2.grad) == list(r.grad),
           "flags": [[x.diag.jobs, x.diag.concurrent, x.diag.serial_fallback] for x in (r, r2)]},
          open(sys.argv[2], "w"))
"""


def test_concurrent_trace_jobs_equal_serial_order(tmp_path):
    """gp_mle_eval with theta = (rho, alpha, nugget): three trace jobs (two compressions + peelings
    and the Tr(F^-1) peeling) run concurrently on their own streams; the result must be
    bit-identical to the serial order (RSF_PAR_TRACES=0), also when a concurrent job runs out of
    memory and the evaluation falls back to the serial order (RSF_TEST_PAR_OOM=1)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "par.py"
    script.write_text(_PAR_PROBE)
    out = {}
    for flag, oom in (("1", "0"), ("0", "0"), ("1", "1")):
        f = tmp_path / f"par{flag}{oom}.json"
        env = dict(os.environ, RSF_PAR_TRACES=flag, RSF_TEST_PAR_OOM=oom)
        subprocess.run([sys.executable, str(script), root, str(f)], env=env, check=True, timeout=600)
        out[flag + oom] = json.load(open(f))
    res = {k: {kk: v[kk] for kk in ("ell", "grad", "trace")} for k, v in out.items()}
    assert res["10"] == res["00"]
    # out of memory in a concurrent job: everything is redone in the serial order, and the
    # context's memory plan runs the next evaluation of the same shape serially from the start
    assert res["11"] == res["00"]
    assert all(np.isfinite(out["10"]["grad"]))
    assert all(v["same2"] for v in out.values())
    assert out["10"]["flags"] == [[3, 1, 0], [3, 1, 0]]
    assert out["00"]["flags"] == [[3, 0, 0], [3, 0, 0]]
    assert out["11"]["flags"] == [[3, 1, 1], [3, 0, 0]]


@pytest.mark.parametrize("cid,n", [(1, 1024), (2, 2304)])
def test_cuda_vs_O2_same_algorithm(ctx, cid, n):
    """The two independent implementations of the same algorithm -- the CUDA path and the serial
    oracle O2 (oracle/rsf.py, oracle/peel.py, oracle/mle.py) -- on the same inputs and the same
    Philox probe counters: log|F| and z^T F^-1 z agree to the factorizations'
    accuracy (both approximate Sigma at eps_fact), the peeled traces to eps_peel scale, g to 1e-3;
    and both meet the gates against the dense O1."""
    from threadpoolctl import threadpool_limits
    from oracle.mle import rsf_mle_eval
    from workloads import philox_normal
    c = config(cid)
    xy = points_for(c, n)
    ok, rk = _kern(c)
    z = dense_sample(ok, xy, w_for(c, n))
    d = dense_eval(ok, xy, z)
    with threadpool_limits(1):
        o2 = rsf_mle_eval(ok, xy, z, c.eps_fact, c.eps_peel, c.leaf, c.seed, philox_normal, block=8)
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), rk, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
    p = len(c.theta)
    assert abs(r.diag.logdet - o2["logdet"]) <= 10 * c.eps * abs(d["logdet"])
    assert abs(r.diag.quad - o2["quad"]) <= 10 * c.eps * abs(d["quad"])
    tr = np.array([r.diag.trace[i] for i in range(p)])
    np.testing.assert_allclose(tr, o2["trace"], rtol=1e-5)
    np.testing.assert_allclose(np.array(r.grad), o2["grad"], rtol=1e-3)
    assert np.all(np.abs(o2["grad"] - d["grad"]) <= 1e-3 * np.abs(d["grad"]))
