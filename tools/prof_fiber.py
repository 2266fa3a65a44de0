"""Profiling driver: the fiber-pass kernels at BASELINE config 2 shape (400^3, R=16) on random
data (kernel time does not depend on values). Used under ncu; prints plain timings otherwise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P

dims, R = (400, 400, 400), 16
rng = np.random.default_rng(0)
T = rng.random(int(np.prod(dims)))
u = rng.random(sum(dims) * R)
t = P.DataTensor.dense(T, dims)
reps = int(os.environ.get("REPS", "3"))
for kind, name in ((3, "fused"), (4, "m0"), (5, "s"), (0, "mttkrp0"), (1, "eval")):
    ms = P.bench_kernel(t, u, kind=kind, mode=0, reps=reps, flush_l2=False)
    print(f"{name}: {ms:.4f} ms")
