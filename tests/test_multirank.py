"""N > 1 host logic on CPU: world_size-2 gloo process groups for the bench's max-over-ranks
aggregation (replicas and the sharded strong-scaling form) and the NCCL-id bootstrap of a
sharded group; the probe-column partition of include/rsf.h."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    t_local = 2.0 + rank          # rank 1 is the slow one
    t_all, value = bench.aggregate(t_local, steps=3, world=world)
    _, vs = bench.aggregate(t_local, steps=3, world=world, strong=True)
    q.put((rank, t_all, value, vs))
    dist.destroy_process_group()


def test_aggregate_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for rank, t_all, value, vs in res:
        assert t_all == pytest.approx(3.0)
        assert value == pytest.approx(world * 3 / 3.0)
        assert vs == pytest.approx(3 / 3.0)       # one shared evaluation per step


def test_aggregate_single_rank():
    import bench
    t, v = bench.aggregate(4.0, steps=2, world=1)
    assert t == 4.0 and v == 0.5


def _id_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1603_08057_b200 as R
    uid, r, w = R.group_id_from_process_group()
    q.put((rank, r, w, uid))
    dist.destroy_process_group()


def test_nccl_id_bootstrap_gloo():
    """rank 0's 128-byte NCCL id reaches every rank unchanged (the bytes rsf_ctx_create_group
    needs); ncclGetUniqueId itself needs no GPU."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_id_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    assert [x[1] for x in res] == [0, 1] and all(x[2] == world for x in res)
    assert len(res[0][3]) == 128 and res[0][3] == res[1][3]


def test_column_slices_partition_every_block():
    """include/rsf.h rsf_debug_col_slice: contiguous, disjoint, covering, balanced to one
    column, larger slices first -- for every block width the peeling uses."""
    import paper_1603_08057_b200 as R
    for P in (1, 2, 3, 4, 7, 8):
        for k in list(range(0, 70)) + [512, 1000, 4096, 4103]:
            sl = [R.col_slice(k, P, r) for r in range(P)]
            assert sl[0][0] == 0 and sl[-1][1] == k
            for (a, b), (c, d) in zip(sl, sl[1:]):
                assert b == c
            sizes = [b - a for a, b in sl]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)


def test_trace_jobs_dealt_to_rank_groups():
    """include/rsf.h rsf_debug_job_runs: with J jobs on W ranks there are G = min(J, W) groups;
    every job runs on at least one rank, the groups partition the ranks (sizes differ by at most
    one), and every rank of a group runs the same jobs."""
    import paper_1603_08057_b200 as R
    for J in (1, 2, 3, 4):
        for W in (1, 2, 3, 4, 5, 8):
            runs = [[R.lib.rsf_debug_job_runs(J, W, r, j) for j in range(J)] for r in range(W)]
            assert all(v in (0, 1) for row in runs for v in row)
            for j in range(J):
                assert sum(runs[r][j] for r in range(W)) >= 1
            G = min(J, W)
            groups = {}
            for r in range(W):
                groups.setdefault(tuple(runs[r]), []).append(r)
            assert len(groups) == G
            sizes = [len(v) for v in groups.values()]
            assert max(sizes) - min(sizes) <= 1
            if W >= J:
                assert all(sum(row) == 1 for row in runs)   # one job per rank group
    assert R.lib.rsf_debug_job_runs(0, 2, 0, 0) == -1


def test_weighted_job_groups():
    """include/rsf.h rsf_debug_job_group: ranks per trace-job group by estimated work (config 4:
    the rho job weighs 3, the Tr(F^-1) job 1).  Every group gets a rank, equal weights give
    r mod G, and the work per rank is balanced as well as whole ranks allow (no move of one rank
    to another group lowers the largest work per rank)."""
    import ctypes as C
    import paper_1603_08057_b200 as R

    def groups(gw, W):
        a = (C.c_double * len(gw))(*gw)
        return [R.lib.rsf_debug_job_group(len(gw), a, W, r) for r in range(W)]

    for G in (1, 2, 3):
        for W in range(G, 9):
            assert groups([1.0] * G, W) == [r % G for r in range(W)]
    assert groups([3.0, 1.0], 4) == [0, 1, 0, 0]
    assert groups([3.0, 1.0], 8) == [0, 1, 0, 0, 0, 1, 0, 0]   # 6 ranks : 2 ranks
    for gw in ([3.0, 1.0], [3.0, 3.0, 1.0], [5.0, 1.0, 2.0]):
        for W in range(len(gw), 9):
            g = groups(gw, W)
            cnt = [g.count(i) for i in range(len(gw))]
            assert min(cnt) >= 1 and sum(cnt) == W
            worst = max(gw[i] / cnt[i] for i in range(len(gw)))
            for a in range(len(gw)):          # moving one rank from a to b never helps
                for b in range(len(gw)):
                    if a == b or cnt[a] == 1:
                        continue
                    c2 = list(cnt); c2[a] -= 1; c2[b] += 1
                    assert max(gw[i] / c2[i] for i in range(len(gw))) >= worst - 1e-12
    a = (C.c_double * 2)(3.0, 1.0)
    assert R.lib.rsf_debug_job_group(2, a, 1, 0) == -1
