"""Per-phase device time of N-GMRES iterations at C2 (400^3, R=16), from globaltimer stamps
inside the loop graph (CPFIT_PHASE_PROFILE=1; the stamps add ~8 tiny kernels per
iteration, so compare shares, not the absolute total, with bench.py)."""
import os
import sys
import time

os.environ["CPFIT_PHASE_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1105_5331_b200 as P

cfg = dict(dims=(400, 400, 400), rank=16, c=0.5, l1=1.0, l2=1.0)
iters = int(os.environ.get("ITERS", "200"))
# TSEED: tensor seed (bench.py uses rank_seed(0)); USEEDS: comma-separated start seeds, one solve
# each on the same solver (bench.py's consecutive solves use 1, 2, 3, ...)
tseed = int(os.environ.get("TSEED", "1"))
useeds = [int(x) for x in os.environ.get("USEEDS", "1").split(",")]
T, _, _ = P.dense_test_problem(cfg["dims"], cfg["rank"], cfg["c"], cfg["l1"], cfg["l2"], tseed, noise_mode=1)
u0 = P.uniform_initial_guess(cfg["dims"], cfg["rank"], useeds[0])
t = P.DataTensor.dense(T, cfg["dims"])
s = P.Solver(t, cfg["rank"], P.NgmresOptions(tol_grad=1e-10, gradient_scale=float(sum(cfg["dims"]) * 16),
                                             max_iters=iters))
n = 0
fevals = 0
wall = 0.0
for us in useeds:
    s.set_initial(P.uniform_initial_guess(cfg["dims"], cfg["rank"], us))
    s.init()
    s.state()
    t0 = time.perf_counter()
    s.run(iters)
    st = s.state()
    wall += time.perf_counter() - t0
    n += st["iters"]
    fevals += st["fevals"]
ph = s.phase_times()
tot = sum(v for v, _ in ph.values())
print(f"iters {n} fevals {fevals} stop {st['stop']}  wall {1e3 * wall / n:.3f} ms/iter, "
      f"stamped {tot / n:.1f} us/iter")
for k, (us, c) in ph.items():
    print(f"{k:16s} visits {c:6d}  {us / n:8.1f} us/iter  {us / max(c, 1):8.1f} us/visit  {100 * us / tot:5.1f}%")
