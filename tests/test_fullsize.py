"""Parity at the benchmarked sizes (n = 2^18 and 2^20) through the C ABI.

* P7 separable surrogate: a jittered tensor grid of config 3's size
  (512 x 512) and of the metric's size (1024 x 1024), squared-exponential kernel (the
  alpha -> infinity RQ limit), theta = (rho, sigma2, nugget).  gp_mle_eval's log|Sigma|,
  z^T Sigma^-1 z, every q_i, every Tr(Sigma^-1 Sigma_i) and every g_i are compared with the
  Kronecker closed forms of oracle/separable.py (pinned against O1 in test_oracle_pins.py).
  z ~ N(0, Sigma(0.8 rho)) is drawn by the closed form and the likelihood is evaluated at rho
  (reading R-J: |g| >> its standard deviation there, so the relative gate is meaningful).
* Config 3 itself (n = 262,144, RQ, theta = (rho, alpha)) on the frozen z (reading R-V,
  workloads/data/MANIFEST.json): bitwise reproducibility of l and g, and g against central
  differences (Richardson) of l(theta) = -1/2 z^T F^-1 z - 1/2 log|F| - n/2 log 2 pi
  (Eq. gradient) from RSFs at perturbed theta.
* Multi-chunk / batch-split peeling against O1 at config 2's recipe (n = 4096): probe_block 64
  and 1 MB batch budgets force the c0 > 0 chunk path, V_i growth across chunks, the split
  batches and regenerated W_i^T blocks.
"""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.dense import dense_eval, dense_sample  # noqa: E402
from oracle.kernels import Kernel as OK  # noqa: E402
from oracle.separable import SeparableSE  # noqa: E402
from workloads import SEED_SEPARABLE, STREAM_W, config, frozen_z, philox_normal_pair, points_for, separable_axes, w_for  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_08057_b200 as R  # noqa: E402

DEV = torch.device("cuda:0")
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
EPS = 1e-6            # the configured tolerance (BASELINE.json)


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV)


def _record(name, d):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "fullsize_parity.jsonl"), "a") as f:
        f.write(json.dumps({"case": name, **d}) + "\n")


@pytest.fixture(scope="module")
def ctx():
    return R.Context(0)


def _w(n, seed):
    m = (n + 1) // 2
    c = np.arange(m, dtype=np.uint64)
    a, b = philox_normal_pair(c, 0, 0, 0, seed, STREAM_W)
    w = np.empty(2 * m)
    w[0::2], w[1::2] = a, b
    return w[:n]


# surrogate parameters: config 3's length scale, nugget and eps_fact
RHO, TAU, EPS_FACT = 0.02, 1e-4, 1e-11


@pytest.mark.parametrize("m", [512, 1024])
def test_P7_separable_surrogate_fullsize(ctx, m):
    a, b = separable_axes(m)
    z = SeparableSE(a, b, 0.8 * RHO, 1.0, TAU).sample(_w(m * m, SEED_SEPARABLE))
    S = SeparableSE(a, b, RHO, 1.0, TAU)
    theta = ("rho", "sigma2", "nugget")
    ref = S.eval(z, theta)
    K = R.Kernel("sqexp", RHO, 1.0, TAU, theta=theta)
    r = R.gp_mle_eval(ctx, _d(S.points()), _d(z), K, EPS_FACT, 64, R.Opts(eps_peel=EPS))
    d = r.diag
    err = {"logdet": abs(d.logdet - ref["logdet"]) / abs(ref["logdet"]),
           "quad": abs(d.quad - ref["quad"]) / abs(ref["quad"]),
           "q": [abs(d.q[i] - ref["q"][i]) / abs(ref["q"][i]) for i in range(3)],
           "trace": [abs(d.trace[i] - ref["trace"][i]) / abs(ref["trace"][i]) for i in range(3)],
           "grad": [abs(r.grad[i] - ref["grad"][i]) / abs(ref["grad"][i]) for i in range(3)]}
    _record(f"P7_separable_m{m}", {"n": m * m, "err": err, "grad": list(r.grad), "grad_ref": list(ref["grad"]),
                                    "t_total": d.t_total})
    assert err["logdet"] <= 10 * EPS
    assert err["quad"] <= 10 * EPS
    assert max(err["grad"]) <= 1e-3, err


@pytest.fixture(scope="module")
def cfg3(ctx):
    c = config(3)
    xy = points_for(c)
    z = frozen_z(3)
    return c, _d(xy), _d(z), z


def _ell_at(ctx, c, xy, z, n, logdet_only=False, **kw):
    """l(theta) from the Sigma factor alone: log|F| and z^T F^-1 z."""
    K = R.Kernel(c.family, kw.get("rho", c.rho), kw.get("sigma2", c.sigma2), kw.get("nugget", c.nugget),
                 kw.get("alpha", c.alpha), theta=())
    # the evaluation's own seed: the RRQR sketches (and through them the skeletons) of the
    # standalone factor are then those of the factor inside gp_mle_eval
    F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, opts=R.Opts(eps_peel=c.eps_peel, seed=c.seed))
    ld = F.logdet()
    if logdet_only:
        F.close()
        return ld
    u = F.solve(z)
    quad = float(torch.dot(z, u))
    F.close()
    return -0.5 * quad - 0.5 * ld - 0.5 * n * math.log(2 * math.pi)


def _richardson(f, v, rel=1e-2):
    h = rel * v
    d1 = (f(v + h) - f(v - h)) / (2 * h)
    d2 = (f(v + 2 * h) - f(v - 2 * h)) / (4 * h)
    return (4 * d1 - d2) / 3


def test_cfg3_frozen_z_reproducible_and_gradient_vs_fd(ctx, cfg3):
    c, xy, z, zh = cfg3
    n = c.n
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed)
    r1 = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
    r2 = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
    assert r1.ell == r2.ell and r1.grad == r2.grad           # bitwise, fixed (input, seed, build, GPU)
    # against O2 (reading R-V: z = F_O2^{1/2} w, so z^T F_O2^-1 z = w^T w exactly; O2's log|F|
    # is in the manifest) -- the SURVEY §8(c).5 gates "vs O2" at config 3
    import json as _j
    from workloads import DATA_DIR
    man = _j.load(open(os.path.join(DATA_DIR, "MANIFEST.json")))["3"]
    w = w_for(c)
    err_ld = abs(r1.diag.logdet - man["logdet_O2"]) / abs(man["logdet_O2"])
    err_q = abs(r1.diag.quad - float(w @ w)) / float(w @ w)
    _record("cfg3_vs_O2", {"logdet": r1.diag.logdet, "logdet_O2": man["logdet_O2"], "rel_logdet": err_ld,
                           "quad": r1.diag.quad, "wTw": float(w @ w), "rel_quad": err_q})
    assert err_ld <= 10 * EPS and err_q <= 10 * EPS
    ell0 = _ell_at(ctx, c, xy, z, n)
    assert abs(ell0 - r1.ell) <= 1e-9 * abs(r1.ell)
    fd = []
    for name, v in (("rho", c.rho), ("alpha", c.alpha)):
        h = 1e-2 * v

        def ell(x):
            return _ell_at(ctx, c, xy, z, n, **{name: x})
        d1 = (ell(v + h) - ell(v - h)) / (2 * h)
        d2 = (ell(v + 2 * h) - ell(v - 2 * h)) / (4 * h)
        fd.append((4 * d1 - d2) / 3)                            # Richardson: O(h^4)
    err = [abs(r1.grad[i] - fd[i]) / abs(fd[i]) for i in range(2)]
    # P8 at full size: the peeled traces alone against d log|Sigma| / d theta_i
    tfd = [_richardson(lambda x, nm=nm: _ell_at(ctx, c, xy, z, n, logdet_only=True, **{nm: x}), v)
           for nm, v in (("rho", c.rho), ("alpha", c.alpha))]
    terr = [abs(r1.diag.trace[i] - tfd[i]) / abs(tfd[i]) for i in range(2)]
    _record("cfg3_frozen_z", {"n": n, "ell": r1.ell, "grad": list(r1.grad), "grad_fd": fd, "rel_err": err,
                              "q": [r1.diag.q[i] for i in range(2)], "trace": [r1.diag.trace[i] for i in range(2)],
                              "trace_fd_logdet": tfd, "trace_rel_err": terr, "t_total": r1.diag.t_total})
    assert max(err) <= 1e-3, (r1.grad, fd, err)
    assert max(terr) <= 1e-5, (terr,)


def test_cfg5_recipe_quarter_million_vs_finite_differences(ctx):
    """Config 5's recipe (Matern 5/2, theta = (rho, sigma2, nugget), leaf 128, eps_fact 1e-9) at
    n = 2^18 (the full n = 2^22 exceeds one GPU): every g_i against Richardson differences of l,
    every trace against differences of log|Sigma| (P8), and the sigma2 / nugget identities (P9)."""
    c = config(5)
    n = 1 << 18
    xy = _d(points_for(c, n))
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf)
    z = F.sample(_d(w_for(c, n)))
    F.close()
    r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
    names = list(c.theta)
    vals = {"rho": c.rho, "sigma2": c.sigma2, "nugget": c.nugget}
    gfd = [_richardson(lambda x, nm=nm: _ell_at(ctx, c, xy, z, n, **{nm: x}), vals[nm]) for nm in names]
    tfd = [_richardson(lambda x, nm=nm: _ell_at(ctx, c, xy, z, n, logdet_only=True, **{nm: x}), vals[nm])
           for nm in names]
    gerr = [abs(r.grad[i] - gfd[i]) / abs(gfd[i]) for i in range(3)]
    terr = [abs(r.diag.trace[i] - tfd[i]) / abs(tfd[i]) for i in range(3)]
    _record("cfg5_recipe_n262144", {"grad": list(r.grad), "grad_fd": gfd, "rel_err": gerr,
                                     "trace": [r.diag.trace[i] for i in range(3)], "trace_fd_logdet": tfd,
                                     "trace_rel_err": terr, "t_total": r.diag.t_total})
    # P9: sigma2 g_sigma2 + tau g_tau = 1/2 z^T Sigma^-1 z - n/2 (exact identity of the model)
    lhs = c.sigma2 * r.grad[1] + c.nugget * r.grad[2]
    assert abs(lhs - (0.5 * r.diag.quad - 0.5 * n)) <= 1e-8 * (0.5 * n)
    assert max(terr) <= 1e-5, terr
    assert max(gerr) <= 1e-3, (r.grad, gfd, gerr)


def test_cfg4_full_2pow20_memory_saving_vs_finite_differences(ctx):
    """Config 4 itself -- n = 2^20 clustered points, Matern 1/2, theta = (rho, sigma2): the metric's
    workload, on one B200 in the memory-saving mode (FP32-stored peeled levels, FP64 arithmetic;
    DESIGN.md §7g).  No dense reference exists at this size: g against Richardson differences of l
    (P10) and the peeled traces against differences of log|F| (P8), z = F^{1/2} w (R-V)."""
    torch.cuda.empty_cache()                        # the memory of earlier tests back to the driver
    c = config(4)
    n = c.n
    xy = _d(points_for(c))
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed, peel_f32=1)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, opts=o)
    z = F.sample(_d(w_for(c)))
    F.close()
    r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
    assert r.ell == _ell_at(ctx, c, xy, z, n)       # the evaluation's factor, solve and l
    vals = {"rho": c.rho, "sigma2": c.sigma2}
    names = list(c.theta)
    gfd = [_richardson(lambda x, nm=nm: _ell_at(ctx, c, xy, z, n, **{nm: x}), vals[nm]) for nm in names]
    tfd = [_richardson(lambda x, nm=nm: _ell_at(ctx, c, xy, z, n, logdet_only=True, **{nm: x}), vals[nm])
           for nm in names]
    gerr = [abs(r.grad[i] - gfd[i]) / abs(gfd[i]) for i in range(2)]
    terr = [abs(r.diag.trace[i] - tfd[i]) / abs(tfd[i]) for i in range(2)]
    _record("cfg4_n1048576_memory_saving", {"grad": list(r.grad), "grad_fd": gfd, "rel_err": gerr,
                                            "trace": [r.diag.trace[i] for i in range(2)], "trace_fd_logdet": tfd,
                                            "trace_rel_err": terr, "t_total": r.diag.t_total})
    assert max(terr) <= 1e-5, terr
    assert max(gerr) <= 1e-3, (r.grad, gfd, gerr)


def test_multichunk_batch_split_peeling_vs_O1(ctx, monkeypatch):
    c = config(2)
    n = 4096
    xy = points_for(c, n)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    z = dense_sample(ok, xy, w_for(c, n))
    d = dense_eval(ok, xy, z)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    monkeypatch.setenv("RSF_PEEL_BUDGET_MB", "1")
    monkeypatch.setenv("RSF_PEEL_WCACHE_MB", "0")
    r = R.gp_mle_eval(ctx, _d(xy), _d(z), K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed,
                                                                         probe_block=64))
    cols = [r.diag.peel[0].cols[lv] for lv in range(1, r.diag.peel[0].levels + 1)]
    assert max(cols) > 64, cols                     # several chunks per probe group
    assert abs(r.diag.logdet - d["logdet"]) <= 10 * c.eps * abs(d["logdet"])
    assert abs(r.diag.quad - d["quad"]) <= 10 * c.eps * abs(d["quad"])
    g = np.array(r.grad)
    _record("multichunk_cfg2_n4096", {"grad": list(g), "grad_ref": list(d["grad"]), "cols": cols})
    assert np.all(np.abs(g - d["grad"]) <= 1e-3 * np.abs(d["grad"])), (g, d["grad"])
    np.testing.assert_allclose([r.diag.trace[i] for i in range(2)], d["trace"], rtol=1e-5)
