"""Sharded evaluation on ONE GPU: RSF_EMU_WORLD=P emulates a
group of P ranks in one process -- every emulated rank's probe-column slice is generated,
pushed through G and the peeled levels, written into its slot of the gather buffer (the
layout ncclAllGather produces), merged, and the extraction columns are split the same way
(comm.cuh).  Checked against the dense oracle O1 with the BASELINE gates and against the
unsharded evaluation.  (Ranks that wait on one another are never run as separate launches
on one GPU; the NCCL transport itself needs >= 2 GPUs.)"""
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


@pytest.mark.parametrize("cid,n,P,f32", [(1, 1024, 2, 0), (1, 1024, 3, 0), (2, 4096, 4, 0), (2, 4096, 2, 1)])
def test_emulated_group_matches_oracle_and_unsharded(cid, n, P, f32, monkeypatch):
    c = config(cid)
    xy = points_for(c, n)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    z = dense_sample(ok, xy, w_for(c, n))
    d = dense_eval(ok, xy, z)
    ctx = R.Context(0)
    assert ctx.group() == (0, 1)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    # (f32: the memory-saving mode of DESIGN.md §7g through the same emulated group)
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=64, peel_f32=f32)
    r1 = R.gp_mle_eval(ctx, _d(xy), _d(z), K, c.eps_fact, c.leaf, o)
    monkeypatch.setenv("RSF_EMU_WORLD", str(P))
    rP = R.gp_mle_eval(ctx, _d(xy), _d(z), K, c.eps_fact, c.leaf, o)
    g1, gP = np.array(r1.grad), np.array(rP.grad)
    assert rP.ell == r1.ell                        # factor, solve and l are not split
    assert np.all(np.abs(gP - d["grad"]) <= 1e-3 * np.abs(d["grad"])), (gP, d["grad"])
    tr1 = np.array([r1.diag.trace[i] for i in range(len(c.theta))])
    trP = np.array([rP.diag.trace[i] for i in range(len(c.theta))])
    np.testing.assert_allclose(trP, d["trace"], rtol=1e-5)
    np.testing.assert_allclose(trP, tr1, rtol=1e-6)


def test_job_result_exchange_round_trip(monkeypatch):
    """The fixed-size job-result records of a rank group (one all-gather after the trace jobs,
    DESIGN.md §7) carry every q_i, trace and peeling diagnostic unchanged: a single-GPU
    evaluation routed through the same pack / gather / unpack path is bit-identical."""
    c = config(2)
    n = 4096
    xy = points_for(c, n)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    z = dense_sample(ok, xy, w_for(c, n))
    ctx = R.Context(0)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed)
    r1 = R.gp_mle_eval(ctx, _d(xy), _d(z), K, c.eps_fact, c.leaf, o)
    monkeypatch.setenv("RSF_EMU_EXCHANGE", "1")
    r2 = R.gp_mle_eval(ctx, _d(xy), _d(z), K, c.eps_fact, c.leaf, o)
    assert r2.ell == r1.ell and list(r2.grad) == list(r1.grad)
    for i in range(2):
        a, b = r1.diag.peel[i], r2.diag.peel[i]
        assert list(a.cols) == list(b.cols) and list(a.rank_max) == list(b.rank_max)
        assert list(a.rank_min) == list(b.rank_min) and list(a.rank_med) == list(b.rank_med)
        assert a.stored_bytes == b.stored_bytes and a.nL == b.nL and a.applies == b.applies
        assert r1.diag.q[i] == r2.diag.q[i] and r1.diag.trace[i] == r2.diag.trace[i]


@pytest.mark.parametrize("cid,n,P,f32", [(1, 1024, 2, 0), (2, 4096, 3, 0), (2, 4096, 2, 1)])
def test_nccl_transport_one_rank_group(cid, n, P, f32, monkeypatch):
    """The NCCL transport on ONE GPU: RSF_NCCL_FORCE=1 makes a world = 1 group keep its one-rank
    communicator (ncclCommInitRank through the dlopen'd entry points, one ncclCommSplit per trace
    job) and issue every collective of the sharded path through it -- the in-place all-gather of
    each probe chunk's slot buffer, the trace partial sums, the job-result records -- while the
    column slices of the P emulated parts fill the slots.  One rank waits on no other, so nothing
    here can hang; the results must equal the emulated group's without NCCL bit for bit."""
    c = config(cid)
    xy = points_for(c, n)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    z = dense_sample(ok, xy, w_for(c, n))
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    # (f32: the memory-saving mode also agrees on the free memory across the group, one more
    # host-staged all-gather per probe group)
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=64, peel_f32=f32)
    monkeypatch.setenv("RSF_EMU_WORLD", str(P))
    ctx0 = R.Context(0)
    n0 = R.nccl_calls()
    r0 = R.gp_mle_eval(ctx0, _d(xy), _d(z), K, c.eps_fact, c.leaf, o)
    assert R.nccl_calls() == n0                    # a single-GPU context issues no collective
    monkeypatch.setenv("RSF_NCCL_FORCE", "1")
    ctx1 = R.Context(0, group=(R.nccl_unique_id(), 0, 1))
    assert ctx1.group() == (0, 1)
    r1 = R.gp_mle_eval(ctx1, _d(xy), _d(z), K, c.eps_fact, c.leaf, o)
    calls = R.nccl_calls() - n0
    # at least one all-gather per peeled level and trace job, plus the result exchange
    assert calls >= len(c.theta) * 2 + 1, calls
    assert r1.ell == r0.ell and list(r1.grad) == list(r0.grad)
    for i in range(len(c.theta)):
        assert r1.diag.trace[i] == r0.diag.trace[i] and r1.diag.q[i] == r0.diag.q[i]
        assert list(r1.diag.peel[i].cols) == list(r0.diag.peel[i].cols)
    # a second evaluation reuses the per-job communicators
    r2 = R.gp_mle_eval(ctx1, _d(xy), _d(z), K, c.eps_fact, c.leaf, o)
    assert list(r2.grad) == list(r0.grad)
    ctx1.close()
    ctx0.close()
