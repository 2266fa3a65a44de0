"""C4 (10M nnz, R = 10): graph-mode solve time for the first k iterations, k = 5..100, and the
trace's per-iteration evaluation counts / restart flags. usage: python tools/c4_phases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1105_5331_b200 as P

dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
t = P.DataTensor.coo(dims, coords, vals)
u0 = P.uniform_initial_guess(dims, R, 0)
opts = P.NgmresOptions(window=20, max_iters=100, tol_grad=1e-300, gradient_scale=float(sum(dims) * R))
s = P.Solver(t, R, opts, 0)
s.restart(u0, 100)
prev = 0.0
for k in (1, 2, 5, 10, 20, 40, 70, 100):
    ms = min(s.restart(u0, k) for _ in range(3))
    print(f"iters {k:4d}: {ms:8.2f} ms  (+{ms - prev:7.2f} ms since the previous line)", flush=True)
    prev = ms
tr = s.trace(101)
for row in tr[:100:5]:
    print(row)
