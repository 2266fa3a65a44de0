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
T, _, _ = P.dense_test_problem(cfg["dims"], cfg["rank"], cfg["c"], cfg["l1"], cfg["l2"], 1, noise_mode=1)
u0 = P.uniform_initial_guess(cfg["dims"], cfg["rank"], 1)
t = P.DataTensor.dense(T, cfg["dims"])
s = P.Solver(t, cfg["rank"], P.NgmresOptions(tol_grad=1e-10, gradient_scale=float(sum(cfg["dims"]) * 16),
                                             max_iters=iters))
s.set_initial(u0)
s.init()
s.state()
t0 = time.perf_counter()
s.run(iters)
st = s.state()
wall = time.perf_counter() - t0
ph = s.phase_times()
n = st["iters"]
tot = sum(v for v, _ in ph.values())
print(f"iters {n} fevals {st['fevals']} stop {st['stop']}  wall {1e3 * wall / n:.3f} ms/iter, "
      f"stamped {tot / n:.1f} us/iter")
for k, (us, c) in ph.items():
    print(f"{k:16s} visits {c:6d}  {us / n:8.1f} us/iter  {us / max(c, 1):8.1f} us/visit  {100 * us / tot:5.1f}%")
