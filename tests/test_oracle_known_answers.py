"""Pins the CPU oracle (oracle/, a restatement of proj/core/src) to the reference's own
known-answer tests and properties. CPU only."""
import math

import numpy as np
import pytest

from conftest import random_factors, random_sparse, rel


def _t(O, dims, flat):
    return O.Tensor.dense(dims, np.asarray(flat, dtype=float))


def _matricize(T, dims, mode):
    A = np.asarray(T).reshape(dims, order="F")
    return np.moveaxis(A, mode, 0).reshape(dims[mode], -1, order="F")


def _khatri_rao(mats):
    out = mats[0]
    for m in mats[1:]:
        out = np.einsum("ir,jr->jir", out, m).reshape(-1, out.shape[1])
    return out


# ---- tensor.cpp --------------------------------------------------------------------------

def test_mttkrp_ones_example(O):
    # test_tensor.cpp:122-127
    t = _t(O, (2, 2, 2), np.ones(8))
    assert np.allclose(t.mttkrp(np.ones(6), 0), [[4.0], [4.0]], atol=1e-14)


def test_mttkrp_matches_definition_all_modes(O):
    # test_tensor.cpp:129-143: matricize(t, n) * khatri_rao(others)
    rng = np.random.default_rng(17)
    dims = (3, 4, 2)
    flat = rng.random(24) * 2 - 1
    t = _t(O, dims, flat)
    u = random_factors(rng, dims, 3)
    fac = [u[sum(dims[:n]) * 3:sum(dims[:n + 1]) * 3].reshape(dims[n], 3, order="F") for n in range(3)]
    for n in range(3):
        others = [fac[m] for m in range(3) if m != n]
        expect = _matricize(flat, dims, n) @ _khatri_rao(others)
        got = t.mttkrp(u, n)
        assert np.linalg.norm(got - expect) <= 1e-12 * max(1.0, np.linalg.norm(expect))


def test_sparse_laplacian_row_sums(O):
    # test_tensor.cpp:145-154
    coords = np.array([0, 0, 0, 1, 1, 0, 1, 1, 1, 2, 2, 1, 2, 2]).reshape(-1, 2)
    t = O.Tensor.coo((3, 3), coords, [2, -1, -1, 2, -1, -1, 2])
    assert np.allclose(t.mttkrp(np.ones(6), 0)[:, 0], [1, 0, 1], atol=1e-14)


def test_sparse_equals_dense(O):
    rng = np.random.default_rng(23)
    dims = (4, 4, 4)
    coords, vals = random_sparse(rng, dims, 0.3)
    dense = np.zeros(dims, order="F")
    dense[tuple(coords.T)] = vals
    ts = O.Tensor.coo(dims, coords, vals)
    td = O.Tensor.dense(dims, dense.reshape(-1, order="F"))
    u = random_factors(rng, dims, 3)
    for n in range(3):
        b = td.mttkrp(u, n)
        assert np.linalg.norm(ts.mttkrp(u, n) - b) <= 1e-12 * max(1.0, np.linalg.norm(b))


def test_sparse_canonicalization(O):
    # test_tensor.cpp:199-211: duplicates summed, zeros dropped, sorted
    t = O.Tensor.coo((2, 2), np.array([1, 1, 0, 0, 1, 1, 0, 1]).reshape(-1, 2), [2.0, 5.0, -2.0, 1.0])
    c, v = t.sparse_contents()
    assert c.tolist() == [[0, 0], [0, 1]] and v.tolist() == [5.0, 1.0]
    with pytest.raises(ValueError):
        O.Tensor.coo((2, 2), np.array([[2, 0]]), [1.0])


def test_gram_hadamard_examples(O):
    # test_tensor.cpp:176-186
    q = np.array([[1, 0], [0, 1], [0, 0]], dtype=float)
    u = np.concatenate([q.reshape(-1, order="F")] * 3)
    assert np.allclose(O.gram_hadamard((3, 3, 3), 2, u), np.eye(2), atol=1e-14)
    ones = np.ones(6)
    assert abs(O.gram_hadamard((2, 2, 2), 1, ones, 2)[0, 0] - 4.0) <= 1e-14
    assert abs(O.gram_hadamard((2, 2, 2), 1, ones)[0, 0] - 8.0) <= 1e-14


def test_gram_symmetric_psd(O):
    rng = np.random.default_rng(31)
    u = random_factors(rng, (4, 5, 3), 3)
    g = O.gram_hadamard((4, 5, 3), 3, u)
    assert np.array_equal(g, g.T)
    assert np.linalg.eigvalsh(g).min() >= -1e-10 * np.linalg.eigvalsh(g).max()


def test_shape_errors(O):
    with pytest.raises(ValueError):
        O.Tensor.dense((2, 2), [1.0, 2.0, 3.0])
    with pytest.raises(ValueError):
        O.Tensor.dense((2,), [1.0, float("nan")])


# ---- kruskal.cpp -------------------------------------------------------------------------

def test_objective_examples(O):
    # test_kruskal.cpp:61-71
    rng = np.random.default_rng(13)
    dims = (3, 3, 3)
    u = random_factors(rng, dims, 2)
    T = O.full(dims, 2, u)
    t = _t(O, dims, T)
    assert abs(t.objective(u)) <= 1e-10 * t.norm() ** 2
    assert abs(_t(O, (2, 2, 2), np.zeros(8)).objective(np.ones(6)) - 4.0) <= 1e-12
    assert abs(_t(O, (1, 1, 1), [2.0]).objective(np.ones(3)) - 0.5) <= 1e-14


def test_objective_routes_vs_brute_force(O):
    # test_kruskal.cpp:73-93
    rng = np.random.default_rng(19)
    dims = (4, 3, 5)
    for _ in range(5):
        u = random_factors(rng, dims, 3)
        flat = rng.random(60) * 2 - 1
        direct = 0.5 * np.sum((flat - O.full(dims, 3, u)) ** 2)
        assert abs(_t(O, dims, flat).objective(u) - direct) <= 1e-10 * max(1.0, direct)
        coords, vals = random_sparse(rng, dims, 0.35)
        dense = np.zeros(dims, order="F")
        dense[tuple(coords.T)] = vals
        sd = 0.5 * np.sum((dense.reshape(-1, order="F") - O.full(dims, 3, u)) ** 2)
        assert abs(O.Tensor.coo(dims, coords, vals).objective(u) - sd) <= 1e-10 * max(1.0, sd)


def test_gradient_scalar_and_exact_fit(O):
    # test_kruskal.cpp:95-107
    _, g = _t(O, (1, 1, 1), [2.0]).eval(np.ones(3))
    assert np.allclose(g, -1.0, atol=1e-14)
    rng = np.random.default_rng(29)
    dims = (3, 4, 2)
    u = random_factors(rng, dims, 2)
    _, g = _t(O, dims, O.full(dims, 2, u)).eval(u)
    assert np.linalg.norm(g) <= 1e-10 * (1 + np.linalg.norm(u))


@pytest.mark.parametrize("trial", range(4))
def test_gradient_finite_difference(O, trial):
    # test_kruskal.cpp:109-133 / acceptance criterion 1
    rng = np.random.default_rng(37 + trial)
    order = 3 if trial % 2 == 0 else 4
    dims = (5,) * order
    u = random_factors(rng, dims, 3)
    if trial < 2:
        t = _t(O, dims, rng.random(5 ** order) * 2 - 1)
    else:
        coords, vals = random_sparse(rng, dims, 0.3)
        t = O.Tensor.coo(dims, coords, vals)
    _, g = t.eval(u)
    fd = np.empty_like(u)
    for i in range(u.size):
        h = 1e-6 * (1 + abs(u[i]))
        up, dn = u.copy(), u.copy()
        up[i] += h
        dn[i] -= h
        fd[i] = (t.objective(up) - t.objective(dn)) / (2 * h)
    assert np.linalg.norm(fd - g) / max(np.linalg.norm(g), 1e-30) <= 1e-6


def test_normalize_examples(O):
    # test_kruskal.cpp:170-220
    u = np.array([3, 0, 0, 2, 1, 0], dtype=float)
    out = O.normalize((2, 2, 2), 1, u)
    e = 6.0 ** (1 / 3)
    for n in range(3):
        assert abs(np.linalg.norm(out[2 * n:2 * n + 2]) - e) <= 1e-12
    assert abs(out[0] - e) <= 1e-12 and abs(out[1]) <= 1e-12
    rng = np.random.default_rng(53)
    dims = (3, 4, 2)
    k = random_factors(rng, dims, 3)
    once = O.normalize(dims, 3, k)
    assert rel(O.full(dims, 3, once), O.full(dims, 3, k)) <= 1e-12
    assert np.linalg.norm(O.normalize(dims, 3, once) - once) <= 1e-13 * (1 + np.linalg.norm(once))
    # sort by decreasing weight
    a = np.array([[1, 5], [0, 0]], float)
    b = np.array([[1, 1], [0, 0]], float)
    u = np.concatenate([a.reshape(-1, order="F"), b.reshape(-1, order="F"), b.reshape(-1, order="F")])
    out = O.normalize((2, 2, 2), 2, u)
    lam0 = np.prod([np.linalg.norm(out[4 * n:4 * n + 2]) for n in range(3)])
    assert abs(lam0 - 5.0) <= 1e-12
    # zero column term untouched and last
    a = np.array([[0.5, 2], [0.25, 0]])
    b = np.array([[0, 1], [0, 0]], float)
    c = np.array([[1, 1], [1, 0]], float)
    u = np.concatenate([m.reshape(-1, order="F") for m in (a, b, c)])
    out = O.normalize((2, 2, 2), 2, u)
    assert out[2] == 0.5 and out[3] == 0.25 and out[4 + 2] == 0.0


# ---- als.cpp -----------------------------------------------------------------------------

def test_als_scalar_gauss_seidel(O):
    # test_als.cpp:25-32
    t = _t(O, (1, 1, 1), [8.0])
    out = t.als_sweep(np.ones(3))
    assert np.allclose(out, 2.0, atol=1e-12)
    assert abs(t.objective(out)) <= 1e-12


def test_als_fixed_point_and_monotone(O):
    # test_als.cpp:16-49
    rng = np.random.default_rng(101)
    dims = (4, 3, 5)
    k = O.normalize(dims, 2, random_factors(rng, dims, 2))
    t = _t(O, dims, O.full(dims, 2, k))
    assert np.linalg.norm(t.als_sweep(k) - k) <= 1e-10 * (1 + np.linalg.norm(k))
    dims = (5, 4, 6)
    t = _t(O, dims, rng.random(120) * 2 - 1)
    u = random_factors(rng, dims, 3)
    prev = t.objective(u)
    for _ in range(10):
        u = t.als_sweep(u)
        f = t.objective(u)
        assert f <= prev + 1e-12 * (1 + abs(prev))
        prev = f


def test_als_singular_raises(O):
    t = _t(O, (2, 2, 2), np.arange(1, 9))
    with pytest.raises(O.OracleNumericalError):
        t.als_sweep(np.zeros(12))


# ---- ngmres.cpp --------------------------------------------------------------------------

def test_accelerate_known_answers(O):
    u = np.linspace(1, 4, 4)
    g = np.full(4, 0.5)
    uh, al, _ = O.accelerate([u], [g], u, g)
    assert al[0] == 0.0 and np.array_equal(uh, u)
    uh, al, _ = O.accelerate([[0.0]], [[-4.0]], [1.0], [-2.0])
    assert abs(al[0] - 1.0) <= 1e-9 and abs(uh[0] - 2.0) <= 1e-9


def test_accelerate_least_squares_oracle(O):
    # test_ngmres.cpp:47-73
    rng = np.random.default_rng(211)
    a = rng.random((5, 5)) * 2 - 1
    a = a.T @ a + 0.5 * np.eye(5)
    b = rng.random(5) * 2 - 1
    its = [rng.random(5) * 2 - 1 for _ in range(4)]
    ub = rng.random(5) * 2 - 1
    gb = a @ ub - b
    uh, al, rr = O.accelerate(its, [a @ x - b for x in its], ub, gb)
    p = np.stack([gb - (a @ x - b) for x in its], axis=1)
    alpha, *_ = np.linalg.lstsq(p, -gb, rcond=None)
    oracle = np.linalg.norm(gb + p @ alpha)
    assert abs(np.linalg.norm(a @ uh - b) - oracle) <= 1e-10 * max(1.0, oracle)
    assert rr <= 1e-8


def test_linear_gmres_equivalence(O):
    # test_ngmres.cpp:106-141 / acceptance criterion 8
    rng = np.random.default_rng(227)
    a = rng.random((5, 5)) * 2 - 1
    a = a.T @ a + np.eye(5)
    b = rng.random(5) * 2 - 1
    u0 = rng.random(5) * 2 - 1
    u, obs = O.ngmres_linear(a, b, 1.0 / np.trace(a), u0, 64, 12, 0.0, 1e-13, False, fixed_step=1.0)
    assert np.linalg.norm(a @ u - b) <= 1e-9


# ---- line_search.cpp ---------------------------------------------------------------------

def test_more_thuente_known_answers(O):
    r = O.more_thuente(lambda s: ((s - 1) ** 2, 2 * (s - 1)), 1.0, -2.0)
    assert r["status"] == 0 and r["evals"] == 1 and r["step"] == 1.0
    r = O.more_thuente(lambda s: (s, 1.0), 0.0, 1.0)
    assert r["status"] == 2 and r["evals"] == 0
    r = O.more_thuente(lambda s: (0.5 * s * s - s, s - 1), 0.0, -1.0)
    assert r["status"] == 0 and r["evals"] == 1 and abs(r["f"] + 0.5) <= 1e-15
    with pytest.raises(ValueError):
        O.more_thuente(lambda s: (s * s, 2 * s), 0.0, -1.0, ftol=0.5, gtol=0.1)
    r = O.more_thuente(lambda s: (-math.atan(s), -1 / (1 + s * s)), 0.0, -1.0, max_evals=3, gtol=1e-8, ftol=1e-9)
    assert r["status"] == 1 and r["evals"] == 3 and r["step"] > 0 and r["f"] < 0


def test_more_thuente_quadratics(O, P):
    # test_line_search.cpp:70-86 — the same 25 draws as the reference (Rng(71) uniforms)
    _, uni, _ = P.rng_draws(71, 50)
    for k in range(25):
        m = 2 + 48 * uni[2 * k]
        a = 0.1 + 5 * uni[2 * k + 1]
        r = O.more_thuente(lambda s: (a * (s - m) ** 2, 2 * a * (s - m)), a * m * m, -2 * a * m)
        assert r["status"] == 0
        assert abs(r["step"] - m) <= 1e-8 * max(1.0, m)
