"""CPU tests of the product library (no GPU needed): the C-ABI loads and exports every symbol
include/*.h declares; the host-side pieces behind it (the Moré–Thuente state machine the device
loop also runs, the input generators) match the reference's known answers and the oracle; and
the device entry points fail loudly (no CPU fallback) when no GPU is present."""
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", h)).read()
            names |= set(re.findall(r"\b(cpfit_[a-z0-9_]+)\s*\(", txt))
    return names - {"cpfit_phi_fn"}


def test_library_exports_every_declared_symbol(P):
    declared = _declared()
    assert len(declared) >= 30
    for name in sorted(declared):
        assert hasattr(P.api.lib, name), name
    assert set(P.EXPORTED_SYMBOLS) <= declared


def test_device_entry_points_fail_loudly_without_gpu(P):
    if P.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(P.CudaError):
        P.DataTensor.dense(np.ones(8), (2, 2, 2))


# ---- line search: product host state machine vs oracle -----------------------------------

def _phis():
    yield (lambda s: ((s - 1) ** 2, 2 * (s - 1))), 1.0, -2.0
    yield (lambda s: (0.5 * s * s - s, s - 1)), 0.0, -1.0
    yield (lambda s: (-math.atan(s), -1 / (1 + s * s))), 0.0, -1.0


def test_more_thuente_known_answers(P):
    # test_line_search.cpp:33-68
    r = P.more_thuente(lambda s: ((s - 1) ** 2, 2 * (s - 1)), 1.0, -2.0)
    assert r.status == P.CONVERGED and r.evals == 1 and r.step == 1.0
    r = P.more_thuente(lambda s: (s, 1.0), 0.0, 1.0)
    assert r.status == P.NOT_DESCENT and r.evals == 0
    r = P.more_thuente(lambda s: (0.5 * s * s - s, s - 1), 0.0, -1.0)
    assert r.status == P.CONVERGED and r.evals == 1 and abs(r.f + 0.5) <= 1e-15
    with pytest.raises(ValueError):
        P.more_thuente(lambda s: (s * s, 2 * s), 0.0, -1.0, P.LineSearchParams(ftol=0.5, gtol=0.1))
    r = P.more_thuente(lambda s: (-math.atan(s), -1 / (1 + s * s)), 0.0, -1.0,
                       P.LineSearchParams(max_evals=3, gtol=1e-8, ftol=1e-9))
    assert r.status == P.MAX_EVALS and r.evals == 3 and r.step > 0 and r.f < 0


def test_more_thuente_quadratics_land_on_minimiser(P):
    # test_line_search.cpp:70-86 with the reference's own Rng(71) draws
    _, uni, _ = P.rng_draws(71, 50)
    for k in range(25):
        m = 2 + 48 * uni[2 * k]
        a = 0.1 + 5 * uni[2 * k + 1]
        r = P.more_thuente(lambda s: (a * (s - m) ** 2, 2 * a * (s - m)), a * m * m, -2 * a * m)
        assert r.status == P.CONVERGED
        assert abs(r.step - m) <= 1e-8 * max(1.0, m)


def test_more_thuente_randomized_against_oracle_and_wolfe(P, O):
    # test_line_search.cpp:88-119 / acceptance criterion 9: every Converged result satisfies
    # both strong-Wolfe inequalities; evals <= 20; identical decisions to the oracle.
    _, uni, _ = P.rng_draws(73, 400)
    conv = 0
    for k in range(100):
        m = 0.2 + 10 * uni[4 * k]
        a = 0.2 + 4 * uni[4 * k + 1]
        amp = 0.2 * a * uni[4 * k + 2]
        fr = 1 + 4 * uni[4 * k + 3]

        def phi(b):
            return a * (b - m) ** 2 + amp * math.sin(fr * b), 2 * a * (b - m) + amp * fr * math.cos(fr * b)

        f0, g0 = phi(0.0)
        if g0 >= 0:
            continue
        r = P.more_thuente(phi, f0, g0)
        o = O.more_thuente(phi, f0, g0)
        assert (r.status, r.evals, r.step, r.f) == (o["status"], o["evals"], o["step"], o["f"])
        assert r.evals <= 20
        if r.status == P.CONVERGED:
            conv += 1
            fs, gs = phi(r.step)
            assert fs <= f0 + 1e-4 * r.step * g0 and abs(gs) <= 1e-2 * (-g0)
    assert conv >= 90


# ---- generators (problems.cpp / rng.hpp) ---------------------------------------------------

def test_rng_pins(P):
    # test_problems.cpp:17-27: mt19937_64(5489) first draw
    u64, uni, nor = P.rng_draws(5489, 1000)
    assert int(u64[0]) == 14514284786278117030
    assert np.all((uni >= 0) & (uni < 1))
    _, _, z = P.rng_draws(1, 20000)
    assert abs(z.mean()) < 0.05 and abs((z * z).mean() - 1) < 0.05
    # splitmix64 finaliser
    assert P.rng_mix(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("c", [0.0, 0.5, 0.9])
def test_collinear_factors_gram(P, c):
    # test_problems.cpp:42-65 / acceptance criterion 10
    u = P.collinear_factors((12, 12, 12), 3, c, 7)
    for n in range(3):
        a = u[36 * n:36 * (n + 1)].reshape(12, 3, order="F")
        g = a.T @ a
        k = np.full((3, 3), c)
        np.fill_diagonal(k, 1.0)
        assert np.abs(g - k).max() <= 1e-12
    with pytest.raises(ValueError):
        P.collinear_factors((2, 2, 2), 3, 0.5, 9)
    with pytest.raises(ValueError):
        P.collinear_factors((5, 5, 5), 3, 1.0, 9)


def test_noise_magnitudes(P):
    # test_problems.cpp:77-84: reference scaling at l1 = 1 gives 99^(-1/2)
    T, _, T0 = P.dense_test_problem((10, 10, 10), 3, 0.5, 1.0, 0.0, 13, noise_mode=0, want_noise_free=True)
    assert abs(np.linalg.norm(T - T0) / np.linalg.norm(T0) - 99 ** -0.5) <= 1e-12
    # BASELINE scaling: l/100
    T, _, T0 = P.dense_test_problem((10, 10, 10), 3, 0.5, 1.0, 0.0, 13, noise_mode=1, want_noise_free=True)
    assert abs(np.linalg.norm(T - T0) / np.linalg.norm(T0) - 0.01) <= 1e-12
    # noise-free problem is exact
    T, truth, T0 = P.dense_test_problem((8, 8, 8), 3, 0.5, 0.0, 0.0, 11, want_truth=True, want_noise_free=True)
    assert np.array_equal(T, T0)
    assert np.linalg.norm(P.full((8, 8, 8), 3, truth) - T) <= 1e-13 * np.linalg.norm(T)


def test_generator_deterministic(P):
    a = P.dense_test_problem((6, 6, 6), 2, 0.9, 5.0, 2.0, 99)[0]
    b = P.dense_test_problem((6, 6, 6), 2, 0.9, 5.0, 2.0, 99)[0]
    c = P.dense_test_problem((6, 6, 6), 2, 0.9, 5.0, 2.0, 100)[0]
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    g = P.uniform_initial_guess((4, 4, 4), 3, 21)
    assert np.array_equal(g, P.uniform_initial_guess((4, 4, 4), 3, 21))
    assert g.min() >= 0 and g.max() < 1
    assert not np.array_equal(g, P.uniform_initial_guess((4, 4, 4), 3, 22))


def test_laplacian(P):
    # test_problems.cpp:102-174 / acceptance criterion 10
    dims, c, v = P.laplacian_tensor(1, 3)
    assert len(v) == 7
    dense = np.zeros((3, 3))
    dense[c[:, 0], c[:, 1]] = v
    assert np.array_equal(dense, [[2, -1, 0], [-1, 2, -1], [0, -1, 2]])
    for d in range(1, 5):
        for s in range(2, 9 if d <= 2 else 6):
            _, c, v = P.laplacian_tensor(d, s)
            assert len(v) == s ** d + 2 * d * s ** (d - 1) * (s - 1)
            ent = {tuple(x) for x in c.tolist()}
            assert all(tuple(x[d:] + x[:d]) in ent for x in c.tolist())
    # interior row sums vanish
    _, c, v = P.laplacian_tensor(2, 4)
    rows = {}
    for x, val in zip(c.tolist(), v):
        rows[tuple(x[:2])] = rows.get(tuple(x[:2]), 0.0) + val
    for x, s in rows.items():
        if all(0 < k < 3 for k in x):
            assert s == 0.0


def test_random_sparse_problem(P):
    coords, vals, truth = P.random_sparse_problem((50, 40, 30), 5000, 4, 0.01, 3, want_truth=True)
    assert coords.shape == (5000, 3)
    keys = [tuple(x) for x in coords.tolist()]
    assert keys == sorted(keys) and len(set(keys)) == 5000
    assert (coords >= 0).all() and (coords < np.array([50, 40, 30])).all()
    fac = [truth[:200].reshape(50, 4, order="F"), truth[200:360].reshape(40, 4, order="F"),
           truth[360:].reshape(30, 4, order="F")]
    for a in fac:
        assert np.allclose(np.linalg.norm(a, axis=0), 1.0)
    m = np.einsum("ir,ir,ir->i", fac[0][coords[:, 0]], fac[1][coords[:, 1]], fac[2][coords[:, 2]])
    assert abs(np.linalg.norm(vals - m) / np.linalg.norm(m) - 0.01) <= 1e-12
