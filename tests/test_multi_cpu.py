"""N > 1 host logic on CPU (gloo, world_size 2): every rank processes its own
pairs (no data-path collective); timing is max-over-ranks and the aggregate
value counts all ranks' pairs (bench.py's weak-scaling contract)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def _uid_worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_1807_02587_b200 import treereg as tr
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    uid = tr.share_unique_id(dist, lambda: bytes(range(128)))
    q.put((rank, uid))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_sharded_comm_id_exchange_gloo():
    """The communicator id made on rank 0 reaches every rank (the path
    Comm.from_torch_distributed takes before ncclCommInitRank)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert got[0] == got[1] == bytes(range(128))


def test_shard_bounds_partition():
    sys.path.insert(0, ROOT)
    from paper_1807_02587_b200 import treereg as tr
    for n in (1, 7, 76800, 1_000_000):
        for w in (1, 2, 3, 8):
            b = [tr.shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
