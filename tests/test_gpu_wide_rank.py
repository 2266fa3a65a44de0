"""Ranks 33..64 (RP = 64): every tensor kind takes the per-mode path (a dense tensor through the
generic kernels), with the block-level Cholesky / substitution and the shared-memory lambda
sort. Per-call values and N-GMRES / N-CG / ALS traces against the oracle (the reference accepts
any rank, kruskal.hpp / tensor.cpp)."""
import numpy as np
import pytest

from conftest import random_factors, random_sparse, rel

pytestmark = pytest.mark.gpu

DENSE = [((12, 10, 9), 36), ((30, 20, 25), 64), ((6, 5, 7, 4), 50), ((40, 3), 33)]


def _dense(P, O, dims, seed):
    rng = np.random.default_rng(seed)
    flat = rng.random(int(np.prod(dims))) * 2 - 1
    return P.DataTensor.dense(flat, dims), O.Tensor.dense(dims, flat), rng


@pytest.mark.parametrize("dims,rank", DENSE)
def test_wide_rank_dense_per_call(gpu, O, dims, rank):
    P = gpu
    t, o, rng = _dense(P, O, dims, 41)
    u = random_factors(rng, dims, rank)
    for m in range(len(dims)):
        assert rel(t.mttkrp(u, m), o.mttkrp(u, m)) <= 1e-12, m
    f, g = P.objective_and_gradient(t, u)
    fo, go = o.eval(u)
    assert abs(f - fo) <= 1e-12 * abs(fo) and rel(g, go) <= 1e-12
    assert rel(P.gram_hadamard(dims, rank, u), O.gram_hadamard(dims, rank, u)) <= 1e-13
    assert rel(P.normalize_and_reorder(dims, rank, u), O.normalize(dims, rank, u)) <= 1e-13
    # ALS where every Gamma_n is nonsingular (R <= prod of the other sizes; otherwise the ridge
    # retry makes the update rounding-sensitive, as at any rank)
    if all(rank <= int(np.prod(dims)) // d for d in dims):
        assert rel(P.als_sweep(t, u), o.als_sweep(u)) <= 1e-9


@pytest.mark.parametrize("dims,rank,density", [((20, 15, 12), 40, 0.2), ((9, 8, 7, 6), 64, 0.1)])
def test_wide_rank_sparse_per_call(gpu, O, dims, rank, density):
    P = gpu
    rng = np.random.default_rng(43)
    coords, vals = random_sparse(rng, dims, density)
    t, o = P.DataTensor.coo(dims, coords, vals), O.Tensor.coo(dims, coords, vals)
    u = random_factors(rng, dims, rank)
    for m in range(len(dims)):
        assert rel(t.mttkrp(u, m), o.mttkrp(u, m)) <= 1e-12, m
    f, g = P.objective_and_gradient(t, u)
    fo, go = o.eval(u)
    assert abs(f - fo) <= 1e-12 * max(abs(fo), 1.0) and rel(g, go) <= 1e-12
    assert rel(P.als_sweep(t, u), o.als_sweep(u)) <= 1e-9


@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_wide_rank_ngmres_matches_oracle(gpu, O, kind):
    P = gpu
    rng = np.random.default_rng(47)
    dims, rank = (14, 12, 10), 40
    if kind == "dense":
        flat = rng.random(int(np.prod(dims)))
        t, o = P.DataTensor.dense(flat, dims), O.Tensor.dense(dims, flat)
    else:
        coords, vals = random_sparse(rng, dims, 0.3)
        t, o = P.DataTensor.coo(dims, coords, vals), O.Tensor.coo(dims, coords, vals)
    u0 = P.uniform_initial_guess(dims, rank, 5)
    nu = float(sum(dims) * rank)
    k = 15
    ref = o.ngmres(u0, window=10, max_iters=k, tol_grad=1e-300, gradient_scale=nu)
    res = P.ngmres_solve(t, u0, P.NgmresOptions(window=10, max_iters=k, tol_grad=1e-300, gradient_scale=nu))
    n = min(len(ref["trace"]), len(res.trace), 11)
    for it in range(1, n):
        assert res.trace[it]["restart"] == ref["trace"][it]["restart"], it
        assert abs(res.trace[it]["f"] - ref["trace"][it]["f"]) <= 1e-8 * ref["trace"][it]["f"], it


def test_wide_rank_ncg_and_als_match_oracle(gpu, O):
    P = gpu
    t, o, _ = _dense(P, O, (11, 9, 8), 53)
    dims, rank = (11, 9, 8), 35
    u0 = P.uniform_initial_guess(dims, rank, 2)
    ref = o.ncg(u0, tol_grad=1e-300, max_iters=10)
    res = P.ncg_solve(t, u0, P.NcgOptions(tol_grad=1e-300, max_iters=10))
    n = min(len(ref["trace"]), len(res.trace), 8)
    for it in range(1, n):
        assert abs(res.trace[it]["f"] - ref["trace"][it]["f"]) <= 1e-8 * ref["trace"][it]["f"], it
    a_ref = o.als_solve(u0, tol_grad=1e-300, max_iters=10)
    a_res = P.als_solve(t, u0, tol_grad=1e-300, max_iters=10)
    for it in range(1, min(len(a_ref["trace"]), len(a_res.trace))):
        assert abs(a_res.trace[it]["f"] - a_ref["trace"][it]["f"]) <= 1e-8 * a_ref["trace"][it]["f"], it


def test_rank_above_64_rejected(gpu):
    P = gpu
    t = P.DataTensor.dense(np.ones(24), (2, 3, 4))
    with pytest.raises(ValueError):
        P.objective(t, np.ones(9 * 65))
