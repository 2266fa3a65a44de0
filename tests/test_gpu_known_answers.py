"""The reference's own unit-test known answers (proj/tests/test_tensor.cpp, test_kruskal.cpp,
test_als.cpp, test_ngmres.cpp) through the device C-ABI, plus the degenerate shapes they touch:
all-zero and 1x1x1 tensors, unit modes, rank 1, empty sparse tensors, exact fits. The CPU oracle
is pinned to the same answers in tests/test_oracle_known_answers.py."""
import numpy as np
import pytest

from conftest import random_factors, rel

pytestmark = pytest.mark.gpu


def test_mttkrp_ones_example(gpu):
    # test_tensor.cpp:122-127: 2x2x2 ones, all-ones rank-1 factors -> every mode [[4], [4]]
    P = gpu
    t = P.DataTensor.dense(np.ones(8), (2, 2, 2))
    for mode in range(3):
        assert np.array_equal(t.mttkrp(np.ones(6), mode), [[4.0], [4.0]])


def test_sparse_laplacian_row_sums(gpu):
    # test_tensor.cpp:145-154: Laplacian d=1 s=3 (3x3 COO), mode-0 MTTKRP with ones -> [1, 0, 1]
    P = gpu
    dims, coords, vals = P.laplacian_tensor(1, 3)
    t = P.DataTensor.coo(dims, coords, vals)
    out = t.mttkrp(np.ones(6), 0)
    assert np.allclose(out[:, 0], [1.0, 0.0, 1.0], atol=1e-15)


def test_objective_examples(gpu):
    # test_kruskal.cpp:61-71: exact fit -> ~0, zero tensor with ones rank 1 -> 4.0, scalar -> 0.5
    P = gpu
    rng = np.random.default_rng(13)
    dims = (3, 3, 3)
    u = random_factors(rng, dims, 2)
    T = P.full(dims, 2, u)
    exact = P.DataTensor.dense(T, dims)
    assert abs(P.objective(exact, u)) <= 1e-10 * float(T @ T)
    zero = P.DataTensor.dense(np.zeros(8), (2, 2, 2))
    assert abs(P.objective(zero, np.ones(6)) - 4.0) <= 1e-12
    scalar = P.DataTensor.dense(np.array([2.0]), (1, 1, 1))
    assert abs(P.objective(scalar, np.ones(3)) - 0.5) <= 1e-14


def test_gradient_examples(gpu):
    # test_kruskal.cpp:95-107: zero at an exact fit; scalar example -> [-1, -1, -1]
    P = gpu
    rng = np.random.default_rng(29)
    dims = (3, 4, 2)
    u = random_factors(rng, dims, 2)
    t = P.DataTensor.dense(P.full(dims, 2, u), dims)
    _, g = P.objective_and_gradient(t, u)
    assert np.linalg.norm(g) <= 1e-10 * (1.0 + np.linalg.norm(u))
    _, g = P.objective_and_gradient(P.DataTensor.dense(np.array([2.0]), (1, 1, 1)), np.ones(3))
    assert np.allclose(g, [-1.0, -1.0, -1.0], atol=1e-14)


def test_gradient_central_differences(gpu):
    # test_kruskal.cpp:109-133 (acceptance criterion 1): orders 3 and 4, dense and sparse
    P = gpu
    rng = np.random.default_rng(37)
    for dims in [(5, 5, 5), (5, 4, 3, 5)]:
        u = random_factors(rng, dims, 3)
        flat = rng.random(int(np.prod(dims))) * 2 - 1
        mask = rng.random(flat.size) < 0.35
        idx = np.nonzero(mask)[0]
        coords = np.stack(np.unravel_index(idx, dims, order="F"), axis=1).astype(np.int64)
        for t in (P.DataTensor.dense(flat, dims), P.DataTensor.coo(dims, coords, flat[idx])):
            _, g = P.objective_and_gradient(t, u)
            h = 1e-6
            fd = np.empty_like(u)
            for e in range(u.size):
                up, um = u.copy(), u.copy()
                up[e] += h
                um[e] -= h
                fd[e] = (P.objective(t, up) - P.objective(t, um)) / (2 * h)
            assert np.linalg.norm(g - fd) <= 1e-6 * max(1.0, np.linalg.norm(fd))


def test_normalize_examples(gpu):
    P = gpu
    # test_kruskal.cpp:170-181: rank-one (3,0) (0,2) (1,0) -> every column norm 6^(1/3), directions kept
    out = P.normalize_and_reorder((2, 2, 2), 1, np.array([3.0, 0.0, 0.0, 2.0, 1.0, 0.0]))
    e = 6.0 ** (1.0 / 3.0)
    for n in range(3):
        assert abs(np.linalg.norm(out[2 * n:2 * n + 2]) - e) <= 1e-12
    assert abs(out[0] - e) <= 1e-12 and abs(out[1]) <= 1e-12
    # :196-207: lambda_1 = 1, lambda_2 = 5 -> terms swap
    a = np.array([[1, 5], [0, 0]], float)
    b = np.array([[1, 1], [0, 0]], float)
    u = np.concatenate([a.reshape(-1, order="F"), b.reshape(-1, order="F"), b.reshape(-1, order="F")])
    out = P.normalize_and_reorder((2, 2, 2), 2, u)
    lam = [np.prod([np.linalg.norm(out[4 * n + 2 * r:4 * n + 2 * r + 2]) for n in range(3)]) for r in range(2)]
    assert abs(lam[0] - 5.0) <= 1e-12 and abs(lam[1] - 1.0) <= 1e-12
    # :209-220: a zero-column term keeps its columns and goes last
    a = np.array([[0.5, 2], [0.25, 0]])
    b = np.array([[0, 1], [0, 0]], float)
    c = np.array([[1, 1], [1, 0]], float)
    u = np.concatenate([m.reshape(-1, order="F") for m in (a, b, c)])
    out = P.normalize_and_reorder((2, 2, 2), 2, u)
    assert out[2] == 0.5 and out[3] == 0.25 and out[4 + 2] == 0.0
    # idempotent (:183-194)
    rng = np.random.default_rng(53)
    u = random_factors(rng, (3, 4, 2), 3)
    once = P.normalize_and_reorder((3, 4, 2), 3, u)
    twice = P.normalize_and_reorder((3, 4, 2), 3, once)
    assert np.linalg.norm(twice - once) <= 1e-13 * (1 + np.linalg.norm(once))


def test_als_known_answers(gpu):
    P = gpu
    # test_als.cpp:25-32: scalar Gauss-Seidel pass T = [8] from ones -> a = b = c = 2
    out = P.als_sweep(P.DataTensor.dense(np.array([8.0]), (1, 1, 1)), np.ones(3))
    assert np.allclose(out, [2.0, 2.0, 2.0], atol=1e-12)
    # :16-23: an exact rank-R tensor is a fixed point (canonical factors)
    rng = np.random.default_rng(17)
    dims = (6, 5, 4)
    u = P.normalize_and_reorder(dims, 2, random_factors(rng, dims, 2) + 2.0)
    t = P.DataTensor.dense(P.full(dims, 2, u), dims)
    assert rel(P.als_sweep(t, u), u) <= 1e-10
    # :34-49: f is monotone over ALS sweeps (dense)
    T = rng.random(int(np.prod(dims)))
    t = P.DataTensor.dense(T, dims)
    x = random_factors(rng, dims, 3)
    f_prev = P.objective(t, x)
    for _ in range(10):
        x = P.als_sweep(t, x)
        f = P.objective(t, x)
        assert f <= f_prev * (1 + 1e-12)
        f_prev = f


def test_degenerate_shapes_match_oracle(gpu, O):
    """Unit modes, rank 1, rank above the smallest mode, an all-zero dense tensor and an empty
    sparse tensor: per-call values against the oracle."""
    P = gpu
    rng = np.random.default_rng(61)
    for dims, R in [((1, 7, 5), 3), ((6, 1, 1), 2), ((4, 5, 6), 1), ((3, 2, 2), 5), ((1, 1, 1), 2)]:
        flat = rng.random(int(np.prod(dims))) * 2 - 1
        t, o = P.DataTensor.dense(flat, dims), O.Tensor.dense(dims, flat)
        u = random_factors(rng, dims, R)
        for m in range(3):
            assert rel(t.mttkrp(u, m), o.mttkrp(u, m)) <= 1e-12
        f, g = P.objective_and_gradient(t, u)
        fo, go = o.eval(u)
        assert abs(f - fo) <= 1e-12 * max(abs(fo), 1e-300) and rel(g, go) <= 1e-12
    dims = (4, 3, 5)
    zt = P.DataTensor.dense(np.zeros(60), dims)
    assert zt.norm() == 0.0
    u = random_factors(rng, dims, 2)
    fo, go = O.Tensor.dense(dims, np.zeros(60)).eval(u)
    f, g = P.objective_and_gradient(zt, u)
    assert abs(f - fo) <= 1e-12 * fo and rel(g, go) <= 1e-12
    with pytest.raises(ValueError):  # fit_h on a zero tensor (test_kruskal.cpp:155-168)
        P.fit_h(zt, u)
    e = P.DataTensor.coo(dims, np.zeros((0, 3), dtype=np.int64), np.zeros(0))
    assert e.nnz() == 0 and e.norm() == 0.0
    f, g = P.objective_and_gradient(e, u)
    fo, go = O.Tensor.coo(dims, np.zeros((0, 3), dtype=np.int64), np.zeros(0)).eval(u)
    assert abs(f - fo) <= 1e-12 * fo and rel(g, go) <= 1e-12
    for m in range(3):
        assert np.array_equal(e.mttkrp(u, m), np.zeros((dims[m], 2)))


def test_shape_and_rank_errors(gpu):
    # test_tensor.cpp:170-174 and the device limits: invalid_argument -> ValueError
    P = gpu
    t = P.DataTensor.dense(np.ones(24), (2, 3, 4))
    with pytest.raises(ValueError):
        t.mttkrp(np.ones(9 * 2 + 1), 0)  # length does not match the shape
    with pytest.raises(ValueError):
        t.mttkrp(np.ones(9 * 2), 3)  # mode out of range
    with pytest.raises(ValueError):
        P.objective(t, np.ones(9 * 65))  # rank above the device limit (64)
    with pytest.raises(ValueError):
        P.DataTensor.dense(np.ones(5), (2, 3))  # value count
    with pytest.raises(ValueError):
        P.ngmres_solve(t, np.ones(9 * 2), P.NgmresOptions(window=113))  # window above the device limit


def test_coo_canonicalisation_and_rejections(gpu, O):
    """COO input through the C-ABI (tensor.cpp:56-103; test_tensor.cpp:170-211): duplicates are
    summed, explicit zeros and cancelled duplicates dropped, out-of-range coordinates and
    non-finite values rejected (invalid_argument -> ValueError), like the reference."""
    P = gpu
    # the reference's own example: (1,1) = 2 and -2 cancel and are dropped; (0,0) = 5, (0,1) = 1 remain
    coords = np.array([1, 1, 0, 0, 1, 1, 0, 1]).reshape(-1, 2)
    t = P.DataTensor.coo((2, 2), coords, np.array([2.0, 5.0, -2.0, 1.0]))
    o = O.Tensor.coo((2, 2), coords, [2.0, 5.0, -2.0, 1.0])
    assert t.nnz() == 2 and abs(t.norm() - o.norm()) <= 1e-15 * o.norm()
    # duplicates, explicit zeros and a duplicate pair that cancels, order 3, against the oracle
    rng = np.random.default_rng(17)
    dims = (6, 5, 4)
    base = np.stack([rng.integers(0, d, 60) for d in dims], axis=1)
    coords = np.concatenate([base, base[:20], base[40:45]])
    vals = np.concatenate([rng.standard_normal(60), rng.standard_normal(20), np.zeros(5)])
    vals[:3] = 0.0  # explicit zeros
    vals[60:63] = 0.0
    vals[10], vals[70] = 1.5, -1.5  # this duplicate pair cancels
    t, o = P.DataTensor.coo(dims, coords, vals), O.Tensor.coo(dims, coords, vals)
    oc, ov = o.sparse_contents()
    assert t.nnz() == len(ov) and abs(t.norm() - o.norm()) <= 1e-14 * o.norm()
    u = random_factors(rng, dims, 3)
    for m in range(3):
        assert rel(t.mttkrp(u, m), o.mttkrp(u, m)) <= 1e-12
    f, g = P.objective_and_gradient(t, u)
    fo, go = o.eval(u)
    assert abs(f - fo) <= 1e-12 * abs(fo) and rel(g, go) <= 1e-12
    with pytest.raises(ValueError):  # coordinate out of range
        P.DataTensor.coo((2, 2), np.array([[2, 0]]), np.array([1.0]))
    with pytest.raises(ValueError):
        P.DataTensor.coo((2, 2), np.array([[0, -1]]), np.array([1.0]))
    for bad in (np.nan, np.inf, -np.inf):  # non-finite values
        with pytest.raises(ValueError):
            P.DataTensor.coo((2, 2), np.array([[0, 0], [1, 1]]), np.array([1.0, bad]))
        x = np.ones(24)
        x[7] = bad
        with pytest.raises(ValueError):
            P.DataTensor.dense(x, (2, 3, 4))
