"""Kernel time per N-GMRES iteration at BASELINE config 4 (sparse 10000^3, 10M nnz, R = 10), from a
CUPTI capture of the loop run with CPFIT_EAGER=1 (CUPTI does not see into graph conditional bodies):
CUPTI capture of the graph-launched loop (torch.profiler): total device time by kernel."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1105_5331_b200 as P

dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
t = P.DataTensor.coo(dims, coords, vals)
s = P.Solver(t, R, P.NgmresOptions(window=20, max_iters=200, tol_grad=1e-300, gradient_scale=float(sum(dims) * R)))
s.set_initial(P.uniform_initial_guess(dims, R, 0))
s.init()
s.run(10)
s.state()
torch.cuda.init()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.run(30)
    st = s.state()
it = st["iters"] - 10
tot = defaultdict(float)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        nm = e.name.replace("(anonymous namespace)::", "").replace("cpfit_gpu::", "").split("(")[0]
        tot[nm[-48:]] += e.time_range.end - e.time_range.start
print(f"{it} iterations")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
    print(f"  {k:48s} {v / it:8.1f} us/it")
