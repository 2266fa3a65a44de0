"""GPU parity of the device-resident N-CG solve (ncg.cpp:9-122) against the CPU oracle's
restatement (oracle/oracle_solvers.cpp ncg_minimize): same seeded inputs, trace rows (iteration
numbers including the ones skipped by stalled iterations, resets, counters), f per row within
1e-8 relative over the first 20 rows, and the final f / stop reason / iteration count."""
import numpy as np
import pytest

from conftest import random_factors, random_sparse, rel

pytestmark = pytest.mark.gpu


def _rows_match(res, ref, n_f=20, tol=1e-8):
    assert len(res.trace) >= 1 and len(ref["trace"]) >= 1
    for a, b in list(zip(res.trace, ref["trace"]))[:n_f]:
        assert a["iter"] == b["iter"]
        assert a["restart"] == b["restart"]
        assert a["fevals"] == b["fevals"] and a["gevals"] == b["gevals"]
        assert abs(a["f"] - b["f"]) <= tol * abs(b["f"]), (a, b)
        assert abs(a["beta"] - b["beta"]) <= 1e-6 * max(abs(b["beta"]), 1e-300) or a["iter"] == 0


def test_ncg_first_iterations_match_oracle(gpu, O):
    """Config-0 problem (20^3 R=3): the first 40 N-CG iterations row by row."""
    P = gpu
    dims, rank = (20, 20, 20), 3
    T, _, _ = P.dense_test_problem(dims, rank, 0.5, 1.0, 1.0, 0, noise_mode=1)
    u0 = P.uniform_initial_guess(dims, rank, 0)
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    ref = o.ncg(u0, tol_grad=1e-12, max_iters=40)
    res = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-12, max_iters=40))
    assert len(res.trace) == len(ref["trace"])
    _rows_match(res, ref)
    assert res.stop_reason == ref["stop"]


@pytest.mark.parametrize("dims,rank,seed", [((20, 20, 20), 3, 0), ((12, 9, 7), 4, 3), ((8, 7, 6, 5), 3, 1)])
def test_ncg_full_solve_matches_oracle(gpu, O, dims, rank, seed):
    """Solve to ||g||/||T|| <= 1e-9: stop reason, final f (1e-8 relative), iteration count +-2 %."""
    P = gpu
    T, _, _ = P.dense_test_problem(dims, rank, 0.5, 1.0, 1.0, seed, noise_mode=1)
    u0 = P.uniform_initial_guess(dims, rank, seed)
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    ref = o.ncg(u0, tol_grad=1e-9, max_iters=3000)
    res = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-9, max_iters=3000))
    assert res.stop_reason == ref["stop"]
    n_ref, n = ref["trace"][-1]["iter"], res.trace[-1]["iter"]
    assert abs(n - n_ref) <= max(2, 0.02 * n_ref), (n, n_ref)
    f_ref = ref["trace"][-1]["f"]
    assert abs(res.trace[-1]["f"] - f_ref) <= 1e-8 * abs(f_ref)
    _rows_match(res, ref)
    # best iterate, normalised once (ncg.cpp:122): the model it represents matches
    fo, _ = o.eval(res.solution)
    assert abs(fo - res.f) <= 1e-8 * abs(res.f)
    assert abs(res.f - min(r["f"] for r in ref["trace"])) <= 1e-8 * abs(res.f)


def test_ncg_sparse_matches_oracle(gpu, O):
    P = gpu
    rng = np.random.default_rng(11)
    dims = (15, 12, 10)
    coords, vals = random_sparse(rng, dims, 0.2)
    t = P.DataTensor.coo(dims, coords, vals)
    o = O.Tensor.coo(dims, coords, vals)
    u0 = P.uniform_initial_guess(dims, 3, 2)
    ref = o.ncg(u0, tol_grad=1e-12, max_iters=30)
    res = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-12, max_iters=30))
    assert len(res.trace) == len(ref["trace"])
    _rows_match(res, ref)


def test_ncg_stationary_start_and_errors(gpu):
    """Exact rank-1 data from its own factors: g = 0 at the start -> GradTol with one row
    (ncg.cpp:34-37); tol_grad <= 0 -> ValueError (ncg.cpp:12)."""
    P = gpu
    dims = (3, 4, 2)
    a, b, c = np.ones(3), np.ones(4), np.ones(2)
    T = np.einsum("i,j,k->ijk", a, b, c).reshape(-1, order="F")
    t = P.DataTensor.dense(T, dims)
    u0 = np.concatenate([a, b, c])
    res = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-9, max_iters=10))
    assert res.stop_reason == P.GRAD_TOL and len(res.trace) == 1
    with pytest.raises(ValueError):
        P.ncg_solve(t, u0, P.NcgOptions(tol_grad=0.0))


def test_ncg_iterate_and_solution_layout(gpu, O):
    P = gpu
    dims, rank = (10, 8, 6), 2
    rng = np.random.default_rng(5)
    T = rng.random(int(np.prod(dims)))
    u0 = random_factors(rng, dims, rank)
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    ref = o.ncg(u0, tol_grad=1e-12, max_iters=15)
    res = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-12, max_iters=15))
    assert rel(res.solution, ref["u"]) <= 1e-6


@pytest.mark.parametrize("dims,rank", [((40, 24, 22, 21), 20), ((50, 30, 26), 24)])
def test_ncg_rank_above_16_matches_oracle(gpu, O, dims, rank):
    """RP = 32 (line polynomial of order 3 and 4 with 16 < R <= 32): the first 15 rows."""
    P = gpu
    T, _, _ = P.dense_test_problem(dims, rank, 0.5, 1.0, 1.0, 2, noise_mode=1)
    u0 = P.uniform_initial_guess(dims, rank, 2)
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    ref = o.ncg(u0, tol_grad=1e-12, max_iters=15)
    res = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-12, max_iters=15))
    assert len(res.trace) == len(ref["trace"])
    _rows_match(res, ref, n_f=15)
