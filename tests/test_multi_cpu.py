"""N > 1 host logic on CPU (gloo, world_size 2): every rank processes its own
pairs (no data-path collective); timing is max-over-ranks and the aggregate
value counts all ranks' pairs (bench.py's weak-scaling contract)."""
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
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    # each rank "registers" its own shard; rank 1 is slower
    local = 0.5 + rank
    t = bench.max_over_ranks(local, dist, torch.device("cpu"))
    bench.barrier(dist, torch.device("cpu"))
    steps = 4
    value = world * steps / t
    q.put((rank, t, value))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_weak_scaling_aggregation_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(90)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    assert all(abs(t - 1.5) < 1e-12 for _, t, _ in res)   # max over ranks
    assert all(abs(v - 2 * 4 / 1.5) < 1e-9 for _, _, v in res)
