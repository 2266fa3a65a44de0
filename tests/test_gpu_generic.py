"""Dense shapes outside the fibre-tile passes: order 1 (tensor.cpp:214-216) and mode-0 fibres longer
than a shared-memory tile (I_0 > 416) run the generic per-mode kernels (csrc/generic.cu). The
reference accepts every shape (tensor.cpp:206-240), so the drop-in must too: per-call MTTKRP /
gradient / f within 1e-12 of the oracle, ALS sweeps, and whole N-GMRES solves. The same kernels
are also forced (CPFIT_FORCE_GENERIC=1 at tensor creation) onto shapes the fibre path takes, so
both implementations are checked against the oracle on the same inputs."""
import os

import numpy as np
import pytest

from conftest import random_factors, rel

pytestmark = pytest.mark.gpu

LONG = [((1000, 30, 20), 8), ((500, 100, 100), 16), ((600, 7), 5), ((450, 6, 5, 4), 3), ((2000, 3, 3), 32)]
FORCED = [((20, 20, 20), 3), ((5, 5, 5, 5), 3), ((33, 6, 5), 16), ((12, 10, 8, 6), 4), ((7, 1, 9), 4),
          ((40, 30), 17), ((8, 3, 4, 2, 3), 5), ((100, 30, 20), 32)]
ORDER1 = [((7,), 2), ((300,), 5), ((1000,), 1)]


def _tensor(P, O, dims, seed, force=False):
    rng = np.random.default_rng(seed)
    flat = rng.random(int(np.prod(dims))) * 2 - 1
    old = os.environ.get("CPFIT_FORCE_GENERIC")
    if force:
        os.environ["CPFIT_FORCE_GENERIC"] = "1"
    try:
        t = P.DataTensor.dense(flat, dims)
    finally:
        if force:
            if old is None:
                os.environ.pop("CPFIT_FORCE_GENERIC", None)
            else:
                os.environ["CPFIT_FORCE_GENERIC"] = old
    return t, O.Tensor.dense(dims, flat), rng


@pytest.mark.parametrize("dims,rank,force", [(d, r, False) for d, r in LONG + ORDER1] +
                         [(d, r, True) for d, r in FORCED])
def test_generic_per_call(gpu, O, dims, rank, force):
    P = gpu
    t, o, rng = _tensor(P, O, dims, sum(dims) + rank, force)
    u = random_factors(rng, dims, rank)
    for mode in range(len(dims)):
        e = rel(t.mttkrp(u, mode), o.mttkrp(u, mode))
        assert e <= 1e-12, (dims, rank, mode, e)
    f, g = P.objective_and_gradient(t, u)
    fo, go = o.eval(u)
    assert abs(f - fo) <= 1e-12 * abs(fo), (f, fo)
    assert rel(g, go) <= 1e-12
    assert abs(P.objective(t, u) - fo) <= 1e-12 * abs(fo)


@pytest.mark.parametrize("dims,rank,force", [((1000, 30, 20), 8, False), ((600, 7), 5, False),
                                             ((450, 6, 5, 4), 3, False), ((300,), 1, False),
                                             ((20, 20, 20), 3, True), ((12, 10, 8, 6), 4, True)])
def test_generic_als_sweep(gpu, O, dims, rank, force):
    P = gpu
    t, o, rng = _tensor(P, O, dims, 7, force)
    u = random_factors(rng, dims, rank)
    assert rel(P.als_sweep(t, u), o.als_sweep(u)) <= 1e-9


@pytest.mark.parametrize("dims,rank,c,force", [((520, 30, 20), 4, 0.5, False), ((20, 20, 20), 3, 0.5, True),
                                               ((450, 10, 8, 6), 3, 0.5, False)])
def test_generic_ngmres_solve_matches_oracle(gpu, O, dims, rank, c, force):
    """Whole device solves of BASELINE-generator problems on generic shapes: first 20 trace rows
    (f <= 1e-8, restart flags), stop reason, final f <= 1e-8 and iterations +-2 %."""
    P = gpu
    T, _, _ = P.dense_test_problem(dims, rank, c, 1.0, 1.0, 0, noise_mode=1)
    old = os.environ.get("CPFIT_FORCE_GENERIC")
    if force:
        os.environ["CPFIT_FORCE_GENERIC"] = "1"
    try:
        t = P.DataTensor.dense(T, dims)
    finally:
        if force:
            os.environ.pop("CPFIT_FORCE_GENERIC", None) if old is None else os.environ.__setitem__(
                "CPFIT_FORCE_GENERIC", old)
    o = O.Tensor.dense(dims, T)
    u0 = P.uniform_initial_guess(dims, rank, 0)
    nu = float(sum(dims) * rank)
    ref = o.ngmres(u0, window=20, max_iters=500, tol_grad=1e-10, gradient_scale=nu)
    res = P.ngmres_solve(t, u0, P.NgmresOptions(window=20, max_iters=500, tol_grad=1e-10, gradient_scale=nu))
    for a, b in list(zip(res.trace, ref["trace"]))[:20]:
        assert a["restart"] == b["restart"], (a, b)
        assert abs(a["f"] - b["f"]) <= 1e-8 * abs(b["f"]), (a, b)
    n, nr = len(res.trace) - 1, len(ref["trace"]) - 1
    print(f"{dims} R={rank}: device {n} iterations, oracle {nr}")
    assert res.stop_reason == ref["stop"]
    assert abs(n - nr) <= max(1, int(0.02 * nr))
    assert abs(res.f - ref["f"]) <= 1e-8 * abs(ref["f"])


def test_order1_known_answer(gpu):
    # tensor.cpp:214-216: the unfolding of a 1-way tensor is a column, MTTKRP = T 1^T
    P = gpu
    t = P.DataTensor.dense(np.arange(1.0, 8.0), (7,))
    out = t.mttkrp(np.ones(14), 0)
    assert np.array_equal(out, np.outer(np.arange(1.0, 8.0), np.ones(2)))
