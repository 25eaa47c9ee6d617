"""Strong-admissibility peeling (next row f4).

CPU pins of the oracle oracle/peel_strong.py (against exact traces, block structures and the
separable closed form) and GPU parity of the CUDA path (rsf_opts.strong = 1) against the dense
oracle O1 and the separable closed form.  Perfect quadtrees only (jittered / tensor grids)."""
import numpy as np
import pytest

from oracle.dense import dense_eval, dense_sample, dense_sigma
from oracle.kernels import Kernel
from oracle.mle import make_probe
from oracle.peel_strong import box_coords, check_perfect, interaction_lists, peel_trace_strong
from oracle.separable import SeparableSE
from oracle.tree import QuadTree
from workloads import config, philox_normal, points_for, separable_axes, w_for


def _grid_tree(m, leaf=64):
    xy = points_for(config(3), m * m)
    return xy, QuadTree(xy, leaf)


def _probe():
    return make_probe(17, 0, philox_normal)


def test_interaction_lists_cover_every_pair_once():
    """Admissible blocks (IL at levels 2..L) plus the leaf near field cover every ordered pair of
    leaves exactly once (the partition strong peeling relies on)."""
    xy, t = _grid_tree(64)       # L = 3
    leaves = t.levels[t.L]
    cover = {}
    for lev in range(2, t.L + 1):
        il = interaction_lists(t, lev)
        for b in t.levels[lev]:
            for c in il[b.id]:
                for lb in leaves:
                    if not _desc(lb, b):
                        continue
                    for lc in leaves:
                        if _desc(lc, c):
                            cover[(lb.id, lc.id)] = cover.get((lb.id, lc.id), 0) + 1
    for lb in leaves:
        xb, yb = box_coords(lb)
        for lc in leaves:
            xc, yc = box_coords(lc)
            near = max(abs(xb - xc), abs(yb - yc)) <= 1
            assert cover.get((lb.id, lc.id), 0) == (0 if near else 1), (box_coords(lb), box_coords(lc))
    # 36 classes: at most one box per class in every parent-neighbourhood window
    for lev in range(2, t.L + 1):
        il = interaction_lists(t, lev)
        for b in t.levels[lev]:
            cls = [(box_coords(c)[0] % 6, box_coords(c)[1] % 6) for c in il[b.id]]
            assert len(cls) == len(set(cls)) and (box_coords(b)[0] % 6, box_coords(b)[1] % 6) not in cls


def _desc(a, b):
    while a is not None and a.level > b.level:
        a = a.parent
    return a is b


def test_perfect_tree_required():
    xy = points_for(config(4), 2000)          # clustered: leaves at several depths
    t = QuadTree(xy, 16)
    with pytest.raises(ValueError):
        check_perfect(t)


def test_strong_peel_identity_and_block_diagonal():
    xy, t = _grid_tree(32)
    n = len(xy)
    assert peel_trace_strong(lambda X: X.copy(), t, 1e-6, _probe()) == pytest.approx(n, abs=1e-9)
    D = np.zeros((n, n))
    r = np.random.default_rng(3)
    for b in t.levels[t.L]:
        B = r.standard_normal((len(b.idx), len(b.idx)))
        D[np.ix_(b.idx, b.idx)] = B + B.T
    assert peel_trace_strong(lambda X: D @ X, t, 1e-6, _probe()) == pytest.approx(np.trace(D), abs=1e-9)


def test_strong_peel_near_field_only_operator_is_exact():
    """An operator with only leaf near-field blocks (all admissible blocks zero): the 9-class
    extraction must return its exact trace (a single class would mix neighbours in)."""
    xy, t = _grid_tree(32)
    n = len(xy)
    r = np.random.default_rng(4)
    G = np.zeros((n, n))
    leaves = t.levels[t.L]
    for b in leaves:
        for c in leaves:
            if max(abs(box_coords(b)[0] - box_coords(c)[0]), abs(box_coords(b)[1] - box_coords(c)[1])) <= 1 \
                    and b.id <= c.id:
                B = r.standard_normal((len(b.idx), len(c.idx)))
                G[np.ix_(b.idx, c.idx)] = B
                G[np.ix_(c.idx, b.idx)] = B.T
    assert peel_trace_strong(lambda X: G @ X, t, 1e-6, _probe()) == pytest.approx(np.trace(G), rel=1e-12)


@pytest.mark.slow
def test_strong_peel_separable_inverse_closed_form():
    """G = Sigma^-1 of the P7 separable surrogate on a 128 x 128 tensor grid (L = 4) applied by
    the Kronecker closed form; Tr(Sigma^-1) also closed form."""
    a, b = separable_axes(128)
    S = SeparableSE(a, b, 0.05, 1.0, 1e-2)
    t = QuadTree(S.points(), 64)
    assert t.L == 4
    check_perfect(t)
    d = {}
    tr = peel_trace_strong(lambda X: np.stack([S.solve(X[:, j]) for j in range(X.shape[1])], axis=1),
                           t, 1e-9, _probe(), diag=d, block=32)
    assert tr == pytest.approx(S.trace("nugget"), rel=1e-7)
    # genuinely low-rank admissible blocks above the leaves: ranks well below the box sizes
    for lev, rk in zip(range(2, t.L), d["ranks"]):
        assert max(rk) < len(t.levels[lev][0].idx) / 2, (lev, max(rk))


# ------------------------------------------------------------------ GPU parity
torch = pytest.importorskip("torch")


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1603_08057_b200 as R
    return R, torch.device("cuda:0")


@pytest.mark.gpu
@pytest.mark.parametrize("m", [32, 64])
def test_gpu_strong_peel_vs_dense(m):
    R, dev = _cuda()
    c = config(3)
    xy = points_for(c, m * m)
    ok = Kernel("matern32", 0.1, 1.0, 1e-2, 1.0, ("rho",))
    rk = R.Kernel("matern32", 0.1, 1.0, 1e-2, 1.0, ("rho",))
    z = dense_sample(ok, xy, w_for(c, m * m))
    d = dense_eval(ok, xy, z)
    ctx = R.Context(0)
    X = torch.from_numpy(xy).to(dev)
    F = R.Factor(ctx, X, rk, 1e-10, 64)
    Fi = R.Factor(ctx, X, rk, 1e-10, 64, which=0)
    tr, pd = R.peel_trace(F, Fi, 1e-7, R.Opts(strong=1, probe_block=64))
    assert abs(tr - d["trace"][0]) <= 1e-5 * abs(d["trace"][0])
    tinv, _ = R.peel_trace(F, None, 1e-7, R.Opts(strong=1))
    assert abs(tinv - d["trace_inv"]) <= 1e-5 * d["trace_inv"]
    # non-perfect tree: fails loudly
    xr = torch.from_numpy(np.random.default_rng(1).random((700, 2))).to(dev)
    Fr = R.Factor(ctx, xr, rk, 1e-8, 16)
    with pytest.raises(R.RsfError):
        R.peel_trace(Fr, None, 1e-6, R.Opts(strong=1))


@pytest.mark.gpu
def test_gpu_strong_gp_mle_eval_separable_closed_form():
    """l and every g_i of the P7 surrogate on a 256 x 256 tensor grid (n = 65,536, L = 5)
    through gp_mle_eval with strong-admissibility peeling, against the closed forms."""
    R, dev = _cuda()
    m = 256
    a, b = separable_axes(m)
    from workloads import SEED_SEPARABLE, STREAM_W, philox_normal_pair
    n = m * m
    cc = np.arange((n + 1) // 2, dtype=np.uint64)
    w0, w1 = philox_normal_pair(cc, 0, 0, 0, SEED_SEPARABLE, STREAM_W)
    w = np.empty(n)
    w[0::2], w[1::2] = w0, w1
    z = SeparableSE(a, b, 0.032, 1.0, 1e-3).sample(w)
    S = SeparableSE(a, b, 0.04, 1.0, 1e-3)
    th = ("rho", "sigma2", "nugget")
    ref = S.eval(z, th)
    K = R.Kernel("sqexp", 0.04, 1.0, 1e-3, theta=th)
    r = R.gp_mle_eval(R.Context(0), torch.from_numpy(S.points()).to(dev), torch.from_numpy(z).to(dev), K, 1e-10, 64,
                      R.Opts(eps_peel=1e-7, strong=1))
    assert abs(r.diag.logdet - ref["logdet"]) <= 1e-5 * abs(ref["logdet"])
    g = np.array(r.grad)
    assert np.all(np.abs(g - ref["grad"]) <= 1e-3 * np.abs(ref["grad"])), (g, ref["grad"])
