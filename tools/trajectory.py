"""Prints the device N-GMRES trajectory (trace rows) for a BASELINE config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1105_5331_b200 as P

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reeval = int(os.environ.get("REEVAL", "0"))
T, u0 = bench.make_problem(P, cfg, 0)
dims, R = cfg["dims"], cfg["rank"]
t = P.DataTensor.dense(T, dims)
nu = sum(dims) * R
opts = P.NgmresOptions(window=20, max_iters=iters, tol_grad=1e-300, gradient_scale=float(nu), reeval_accepted=bool(reeval))
s = P.Solver(t, R, opts, 0)
s.set_initial(u0)
s.init()
t0 = time.time()
ms = s.run(iters)
st = s.state()
tr = s.trace(st["iters"] + 1)
prev = None
for r in tr:
    dt = (r["time_s"] - prev) * 1e3 if prev is not None else 0.0
    prev = r["time_s"]
    print(f"{r['iter']:4d} f={r['f']:.15e} h={r['h']:.6e} g={r['gnorm_rel']:.3e} fe={r['fevals']:4d} "
          f"rs={int(r['restart'])} beta={r['beta']:.4g} dt_ms={dt:.3f}")
print("state", st, "ms", ms)
