import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1105_5331_b200 as P
dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
t = P.DataTensor.coo(dims, coords, vals)
u0 = P.uniform_initial_guess(dims, R, 0)
print("mttkrp ms", [round(P.bench_kernel(t, u0, 0, m, 10, True), 4) for m in range(3)])
print("eval ms", P.bench_kernel(t, u0, 1, 0, 5, True))
