"""Launch-list driver: one C2 (400^3, R=16) N-GMRES solve for ITERS iterations, for
`ncu --metrics gpu__time_duration.sum` (per-kernel share of an iteration). Run it once
without ncu first; summarise the CSV with tools/launch_summary.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1105_5331_b200 as P

cfg = dict(dims=(400, 400, 400), rank=16, c=0.5, l1=1.0, l2=1.0)
iters = int(os.environ.get("ITERS", "20"))
T, _, _ = P.dense_test_problem(cfg["dims"], cfg["rank"], cfg["c"], cfg["l1"], cfg["l2"], 1, noise_mode=1)
u0 = P.uniform_initial_guess(cfg["dims"], cfg["rank"], 1)
t = P.DataTensor.dense(T, cfg["dims"])
s = P.Solver(t, cfg["rank"], P.NgmresOptions(tol_grad=1e-10, gradient_scale=float(sum(cfg["dims"]) * 16)))
s.set_initial(u0)
s.init()
s.run(iters)
st = s.state()
print("state", st, "launches", s.launches())
