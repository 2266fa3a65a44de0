import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import paper_1105_5331_b200 as P
cfg = bench.CONFIGS["c2"]
dims, R = cfg["dims"], cfg["rank"]
T, u0 = bench.make_problem(P, cfg, 0)
t = P.DataTensor.dense(T, dims)
nu = float(sum(dims) * R)
o = P.NgmresOptions(window=20, max_iters=50, tol_grad=1e-10, gradient_scale=nu)
starts = np.stack([P.uniform_initial_guess(dims, R, 100 + i) for i in range(8)])
for conc in (1, 2, 4):
    P.solve_batch(t, starts[:conc], o, 0, conc)
    t0 = time.perf_counter()
    b = P.solve_batch(t, starts, o, 0, conc)
    dt = time.perf_counter() - t0
    print(conc, int(b.iters.sum()), round(dt, 4), round(b.iters.sum() / dt, 1))
