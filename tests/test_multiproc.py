"""N>1 path of bench.py on CPU with gloo (world size 2): independent replicas (one seed per
rank), max-over-ranks timing and whole-job aggregation. No GPU needed."""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import bench
    import paper_1105_5331_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = dict(dims=(6, 5, 4), rank=2, c=0.5, l1=1.0, l2=1.0)
    T, u0 = bench.make_problem(P, cfg, bench.rank_seed(rank))
    ms = 10.0 * (rank + 1)
    ms_max = bench.reduce_max(ms, dist, "cpu")
    q.put((rank, float(T.sum()), float(u0.sum()), ms_max, bench.aggregate(20, world, ms_max)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, t0, u0, m0, v0), (r1, t1, u1, m1, v1) = out
    assert (r0, r1) == (0, 1)
    assert t0 != t1 and u0 != u1          # different seeds -> independent problems
    assert m0 == m1 == 20.0               # max over ranks seen by every rank
    assert v0 == v1 == pytest.approx(2 * 20 / 0.020)
