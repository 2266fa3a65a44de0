"""Where the end-to-end (C-ABI, host buffers) time goes at C2: tensor upload, solver
construction (graph capture + instantiate), init, loop."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1105_5331_b200 as P

dims, R = (400, 400, 400), 16
T, _, _ = P.dense_test_problem(dims, R, 0.5, 1.0, 1.0, 1, noise_mode=1)
u0 = P.uniform_initial_guess(dims, R, 1)
gs = float(sum(dims) * R)
for rep in range(3):
    t0 = time.perf_counter()
    t = P.DataTensor.dense(T, dims)
    t.norm()
    t1 = time.perf_counter()
    s = P.Solver(t, R, P.NgmresOptions(tol_grad=1e-10, gradient_scale=gs, max_iters=60))
    t2 = time.perf_counter()
    s.set_initial(u0)
    s.init()
    s.state()
    t3 = time.perf_counter()
    s.run(60)
    st = s.state()
    t4 = time.perf_counter()
    res = P.ngmres_solve(t, u0, P.NgmresOptions(tol_grad=1e-10, gradient_scale=gs, max_iters=60))
    t5 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  solver build {1e3*(t2-t1):.1f} ms  init {1e3*(t3-t2):.1f} ms  "
          f"loop {1e3*(t4-t3):.1f} ms ({st['iters']} it)  ngmres_solve {1e3*(t5-t4):.1f} ms ({len(res.trace)-1} it)")
    s.close()
    t.close()
