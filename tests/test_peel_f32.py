"""FP32 storage of the peeled levels (rsf_opts.peel_f32): the row bases V_i and the
cores Brow_i of every finished level G^(m) are kept in FP32 and the subtraction
Y' -= sum_m G^(m) W runs on the FP64 DMMA kernel with an FP32-stored op(B) widened in shared memory.
The traces must still meet the gates against the dense oracle O1 (exact traces), and the
stored bytes of the peeled representation halve."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.dense import dense_eval, dense_sample  # noqa: E402
from oracle.kernels import Kernel as OK  # noqa: E402
from workloads import config, points_for, w_for  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1603_08057_b200 as R  # noqa: E402

DEV = torch.device("cuda:0")


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV)


@pytest.mark.parametrize("cid,n,pb", [(1, 1024, 512), (2, 4096, 512), (2, 4096, 64)])
def test_peel_f32_matches_oracle(cid, n, pb):
    c = config(cid)
    xy = points_for(c, n)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    z = dense_sample(ok, xy, w_for(c, n))
    d = dense_eval(ok, xy, z)
    ctx = R.Context(0)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    r64 = R.gp_mle_eval(ctx, _d(xy), _d(z), K, c.eps_fact, c.leaf,
                        R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=pb))
    r32 = R.gp_mle_eval(ctx, _d(xy), _d(z), K, c.eps_fact, c.leaf,
                        R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=pb, peel_f32=1))
    assert r32.ell == r64.ell                       # the factor, the solve and l do not change
    p = len(c.theta)
    g32 = np.array(r32.grad)
    assert np.all(np.abs(g32 - d["grad"]) <= 1e-3 * np.abs(d["grad"])), (g32, d["grad"])
    tr32 = np.array([r32.diag.trace[i] for i in range(p)])
    np.testing.assert_allclose(tr32, d["trace"], rtol=1e-5)
    for i in range(p):
        b64, b32 = r64.diag.peel[i].stored_bytes, r32.diag.peel[i].stored_bytes
        if b64 > 0:
            assert b32 <= 0.55 * b64, (b32, b64)
