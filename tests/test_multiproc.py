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


def _solver_worker(rank, world, port, q):
    """Each rank runs its own replica solve (the oracle's N-GMRES on the problem of seed = rank, the
    reference's only parallelism: independent seeds, bench.cpp:88-120), times it, and the job
    reports max-over-ranks time and whole-job iterations/s, as bench.py does on GPUs."""
    import sys
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import bench
    from oracle import pyoracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = bench.CONFIGS["c0"]
    T, u0 = bench.make_problem(O, cfg, bench.rank_seed(rank))
    o = O.Tensor.dense(cfg["dims"], T)
    dist.barrier()
    t0 = time.perf_counter()
    res = o.ngmres(u0, window=20, max_iters=30, tol_grad=1e-10, gradient_scale=float(sum(cfg["dims"]) * cfg["rank"]))
    ms = (time.perf_counter() - t0) * 1e3
    ms_max = bench.reduce_max(ms, dist, "cpu")
    iters = len(res["trace"]) - 1
    tot = bench.reduce_max(float(iters), dist, "cpu")  # every replica runs the same budget
    q.put((rank, res["f"], iters, ms, ms_max, bench.aggregate(iters, world, ms_max), tot))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replica_solves_gloo():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.multiprocessing as mp

    import bench
    from oracle import pyoracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solver_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = bench.CONFIGS["c0"]
    for rank, f, iters, ms, ms_max, value, _ in out:
        # the replica equals the same solve run alone (deterministic, independent of the other rank)
        T, u0 = bench.make_problem(O, cfg, rank)
        ref = O.Tensor.dense(cfg["dims"], T).ngmres(u0, window=20, max_iters=30, tol_grad=1e-10,
                                                     gradient_scale=float(sum(cfg["dims"]) * cfg["rank"]))
        assert f == ref["f"] and iters == len(ref["trace"]) - 1
        assert ms_max >= ms
    assert out[0][4] == out[1][4]
    assert out[0][5] == pytest.approx(2 * out[0][2] / (out[0][4] * 1e-3))


def test_reference_arm_under_torchrun_prints_one_line():
    """bench.py --impl reference launched like the driver's N>1 runs (torchrun, 2 ranks, CPU):
    rank 0 alone runs and prints one JSON line, the other rank exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--config", "c0", "--steps", "4", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["timed"]["iterations"] == 4
