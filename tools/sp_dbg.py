import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1105_5331_b200 as P
from oracle import pyoracle as O
sys.path.insert(0, "tests")
from conftest import random_sparse, random_factors, rel  # noqa
for dims, rank, dens in [((4, 4, 4), 3, 0.3), ((5, 5, 5, 5), 3, 0.3), ((30, 20, 10), 7, 0.05), ((4, 4, 4, 4, 4, 4), 2, 0.02)]:
    rng = np.random.default_rng(3)
    coords, vals = random_sparse(rng, dims, dens)
    t = P.DataTensor.coo(dims, coords, vals)
    o = O.Tensor.coo(dims, coords, vals)
    u = random_factors(rng, dims, rank)
    for mode in range(len(dims)):
        try:
            print(dims, mode, rel(t.mttkrp(u, mode), o.mttkrp(u, mode)), flush=True)
        except Exception as e:
            print(dims, mode, "ERR", e, flush=True); sys.exit(1)
# blocked layout (other-mode sizes > kSpBlockRows), ranks across RP classes
for dims, R in [((3000, 2500, 2100), 10), ((2100, 1500, 1030), 16), ((1500, 1200, 1100), 5), ((1200, 1100, 40, 30), 7)]:
    coords, vals, _ = P.random_sparse_problem(dims, 150_000, R, 0.01, 1)
    t = P.DataTensor.coo(dims, coords, vals)
    o = O.Tensor.coo(dims, coords, vals)
    u = P.uniform_initial_guess(dims, R, 2)
    for mode in range(len(dims)):
        print(dims, R, mode, rel(t.mttkrp(u, mode), o.mttkrp(u, mode)), flush=True)
    f, g = P.objective_and_gradient(t, u)
    fo, go = o.eval(u)
    print(dims, R, "f", abs(f - fo) / abs(fo), "g", rel(g, go), flush=True)
