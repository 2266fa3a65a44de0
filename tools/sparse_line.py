"""C4 (10M nnz, R = 10): the sparse line-search contractions (sp_line8_kernel) timed through the
polynomial builder, plus the whole 100-iteration rate. usage: python tools/sparse_line.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P
from oracle import pyoracle as O

dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
t = P.DataTensor.coo(dims, coords, vals)
rng = np.random.default_rng(5)
u = P.uniform_initial_guess(dims, R, 0)
d = rng.standard_normal(u.size) * 0.01
al = np.array([0.0, 0.5, 1.0])
phi, dphi = P.line_polynomial(t, u, d, al)
o = O.Tensor.coo(dims, coords, vals)
for a, fp in zip(al, phi):
    fo = o.eval(u + a * d)[0]
    print(f"alpha {a}: poly {fp:.15e} oracle {fo:.15e} rel {abs(fp - fo) / abs(fo):.2e}", flush=True)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

torch.cuda.init()
for _ in range(3):
    P.line_polynomial(t, u, d, al)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        P.line_polynomial(t, u, d, al)
ks = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "sp_line8" in e.name]
us = [e.time_range.end - e.time_range.start for e in ks]
print(f"sp_line8_kernel: {len(us)} launches, mean {sum(us) / max(1, len(us)):.1f} us", flush=True)
