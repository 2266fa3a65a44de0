"""Small cases that launch every kernel family of libcpfit_gpu.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; tools/sanitize.sh): dense fibre passes for long
(I0 = 100, 3-stage ring) and short (I0 = 20, deep ring + TMA box) fibres at RP = 8 / 16 / 32, the
S-only passes, level kernels (orders 3 and 4), Grams, ALS solves and normalisation, accelerate,
the exact line polynomials (dense orders 3 and 4, sparse order 3), the solver control kernels
(N-GMRES with polynomial and trial-evaluation line searches, ALS, N-CG), sparse MTTKRP, and the
generic dense kernels. Exits 0 when every call returns."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P

rng = np.random.default_rng(0)


def dense_case(dims, R, iters=3, resid=False):
    T, _, _ = P.dense_test_problem(dims, R, 0.5, 1.0, 1.0, 1, noise_mode=1)
    t = P.DataTensor.dense(T, dims)
    u = P.uniform_initial_guess(dims, R, 2)
    for m in range(len(dims)):
        t.mttkrp(u, m)
    P.objective_and_gradient(t, u)
    P.objective_and_gradient_form(t, u, 1)
    P.als_sweep(t, u)
    nu = float(sum(dims) * R)
    P.ngmres_solve(t, u, P.NgmresOptions(max_iters=iters, tol_grad=1e-12, gradient_scale=nu,
                                         residual_objective=resid, reeval_accepted=resid))
    P.als_solve(t, u, tol_grad=1e-12, max_iters=2)
    P.ncg_solve(t, u, P.NcgOptions(tol_grad=1e-12, max_iters=2))
    if len(dims) in (3, 4):
        P.line_polynomial(t, u, 0.1 * rng.standard_normal(u.size), np.array([0.0, 0.5, 1.0]))
    for kind in (3, 4, 5):
        P.bench_kernel(t, u, kind=kind, reps=1, flush_l2=False)
    t.close()


for dims, R in [((20, 20, 20), 3), ((100, 30, 20), 16), ((20, 7, 3, 5), 9), ((36, 40, 7), 5), ((128, 9, 11), 20),
                ((40, 30), 6)]:
    dense_case(dims, R)
    print("dense", dims, R, flush=True)
dense_case((30, 20, 10), 4, iters=2, resid=True)
print("dense residual / trial evaluations", flush=True)
# generic dense (order 1, long fibres)
dense_case((500, 6, 5), 3, iters=2)
dense_case((50,), 2, iters=2)
print("generic dense", flush=True)
# sparse
dims = (40, 30, 25)
coords, vals, _ = P.random_sparse_problem(dims, 3000, 4, 0.01, 3)
t = P.DataTensor.coo(dims, coords, vals)
u = P.uniform_initial_guess(dims, 4, 3)
for m in range(3):
    t.mttkrp(u, m)
P.objective_and_gradient(t, u)
P.ngmres_solve(t, u, P.NgmresOptions(max_iters=3, tol_grad=1e-12, gradient_scale=float(sum(dims) * 4)))
P.line_polynomial(t, u, 0.1 * rng.standard_normal(u.size), np.array([0.0, 1.0]))
print("sparse", flush=True)
# accelerate (window of 5, n = 1000) and batched solves
wu, wg = rng.standard_normal((5, 1000)), rng.standard_normal((5, 1000))
P.accelerate(wu, wg, rng.standard_normal(1000), rng.standard_normal(1000))
T, _, _ = P.dense_test_problem((20, 20, 20), 3, 0.5, 1.0, 1.0, 0, noise_mode=1)
t = P.DataTensor.dense(T, (20, 20, 20))
P.solve_batch(t, np.stack([P.uniform_initial_guess((20, 20, 20), 3, s) for s in range(3)]),
              P.NgmresOptions(max_iters=3, tol_grad=1e-12, gradient_scale=180.0), 0, 2)
print("accelerate / batch", flush=True)
print("SANITIZE_CASES_OK")
