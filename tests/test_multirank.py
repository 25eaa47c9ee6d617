"""N > 1 host logic on CPU: world_size-2 gloo process group, the bench's
max-over-ranks aggregation and the per-rank replica seeds."""
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
    q.put((rank, t_all, value))
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
    for rank, t_all, value in res:
        assert t_all == pytest.approx(3.0)
        assert value == pytest.approx(world * 3 / 3.0)


def test_aggregate_single_rank():
    import bench
    t, v = bench.aggregate(4.0, steps=2, world=1)
    assert t == 4.0 and v == 0.5
