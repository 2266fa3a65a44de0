"""Batched solves (the reference's seed sweeps, bench.cpp:80-158): every solve
of a concurrent batch must equal the same solve run alone through the single-solve API (the
device code path is deterministic, so the results are bitwise equal), for N-GMRES, ALS and N-CG."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(P):
    dims, rank = (20, 20, 20), 3
    T, _, _ = P.dense_test_problem(dims, rank, 0.5, 1.0, 1.0, 0, noise_mode=1)
    t = P.DataTensor.dense(T, dims)
    starts = np.stack([P.uniform_initial_guess(dims, rank, s) for s in range(7)])
    return t, dims, rank, starts


@pytest.mark.parametrize("concurrency", [1, 3, 16])
def test_batch_ngmres_equals_single_solves(gpu, concurrency):
    P = gpu
    t, dims, rank, starts = _problem(P)
    nu = float(sum(dims) * rank)
    o = P.NgmresOptions(window=20, max_iters=2000, tol_grad=1e-10, gradient_scale=nu)
    b = P.solve_batch(t, starts, o, method=0, concurrency=concurrency)
    for i, u0 in enumerate(starts):
        r = P.ngmres_solve(t, u0, o)
        assert b.iters[i] == len(r.trace) - 1
        assert b.stop_reason[i] == r.stop_reason == P.GRAD_TOL
        assert b.f[i] == r.f
        assert np.array_equal(b.solutions[i], r.solution)


def test_batch_als_and_ncg_equal_single_solves(gpu):
    P = gpu
    t, dims, rank, starts = _problem(P)
    o = P.NgmresOptions(max_iters=300, tol_grad=1e-9)
    ba = P.solve_batch(t, starts[:4], o, method=1, concurrency=4)
    bn = P.solve_batch(t, starts[:4], o, method=2, concurrency=4)
    for i, u0 in enumerate(starts[:4]):
        ra = P.als_solve(t, u0, tol_grad=1e-9, max_iters=300)
        assert ba.iters[i] == len(ra.trace) - 1 and ba.f[i] == ra.f
        assert np.array_equal(ba.solutions[i], ra.solution)
        rn = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-9, max_iters=300))
        assert bn.f[i] == rn.f and bn.stop_reason[i] == rn.stop_reason
        assert np.array_equal(bn.solutions[i], rn.solution)


def test_batch_argument_errors(gpu):
    P = gpu
    t, dims, rank, starts = _problem(P)
    with pytest.raises(ValueError):
        P.solve_batch(t, starts, P.NgmresOptions(), method=3)
    bad = starts.copy()
    bad[2, 5] = np.nan
    with pytest.raises(ValueError):
        P.solve_batch(t, bad, P.NgmresOptions())


def test_batch_sparse_equals_single_solves(gpu):
    """Sparse order 3 (exact line polynomial from the nonzeros): concurrent solves equal single ones."""
    P = gpu
    dims, R = (30, 25, 20), 3
    coords, vals, _ = P.random_sparse_problem(dims, 2000, R, 0.01, 4)
    t = P.DataTensor.coo(dims, coords, vals)
    starts = np.stack([P.uniform_initial_guess(dims, R, 40 + s) for s in range(4)])
    o = P.NgmresOptions(window=10, max_iters=200, tol_grad=1e-9, gradient_scale=float(sum(dims) * R))
    b = P.solve_batch(t, starts, o, method=0, concurrency=4)
    for i, u0 in enumerate(starts):
        r = P.ngmres_solve(t, u0, o)
        assert b.iters[i] == len(r.trace) - 1 and b.f[i] == r.f
        assert np.array_equal(b.solutions[i], r.solution)
