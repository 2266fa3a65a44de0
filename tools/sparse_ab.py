"""C4 (10M nnz, R=10) sparse MTTKRP / evaluation / N-GMRES rate: blocked kernel vs the row-gather
kernel (CPFIT_SP_UNBLOCKED=1 in a second process), plus parity of the blocked result against the
oracle at full size. usage: python tools/sparse_ab.py [--unblocked]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P

dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
t0 = time.time()
t = P.DataTensor.coo(dims, coords, vals)
up = time.time() - t0
u0 = P.uniform_initial_guess(dims, R, 0)
out = {"unblocked": os.environ.get("CPFIT_SP_UNBLOCKED") == "1", "upload_s": round(up, 3)}
out["mttkrp_ms"] = [round(P.bench_kernel(t, u0, 0, m, 10, True), 4) for m in range(3)]
out["eval_ms"] = round(P.bench_kernel(t, u0, 1, 0, 5, True), 4)
opts = P.NgmresOptions(window=20, max_iters=100, tol_grad=1e-300, gradient_scale=float(sum(dims) * R))
s = P.Solver(t, R, opts, 0)
s.restart(u0, 100)
ms = s.restart(u0, 100)
st = s.state()
out["iters_per_s"] = round(st["iters"] / (ms * 1e-3), 1)
out["f"] = st["best_f"]
if "--oracle" in sys.argv:
    from oracle import pyoracle as O
    o = O.Tensor.coo(dims, coords, vals)
    out["mttkrp_rel"] = [float(np.linalg.norm(t.mttkrp(u0, m) - o.mttkrp(u0, m)) / np.linalg.norm(o.mttkrp(u0, m)))
                         for m in range(3)]
print(json.dumps(out), flush=True)
