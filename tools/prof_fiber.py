"""Profiling driver: the fiber-pass kernels at BASELINE config 2 shape (400^3, R=16) on random
data (kernel time does not depend on values). KINDS selects cpfit_bench_kernel kinds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P

dims = tuple(int(x) for x in os.environ.get("DIMS", "400,400,400").split(","))
R = int(os.environ.get("RANK", "16"))
rng = np.random.default_rng(0)
T = rng.random(int(np.prod(dims)))
u = rng.random(sum(dims) * R)
t = P.DataTensor.dense(T, dims)
reps = int(os.environ.get("REPS", "3"))
names = {8: "mttkrp3_last_only", 2: "als_sweep", 3: "fused", 4: "m0", 5: "s", 0: "mttkrp0", 1: "eval_resid", 6: "fused_resid", 7: "eval_perfiber"}
kinds = [int(k) for k in os.environ.get("KINDS", "3,4,5,6,0,7,1").split(",")]
for kind in kinds:
    ms = P.bench_kernel(t, u, kind=kind, mode=0, reps=reps, flush_l2=False)
    print(f"{names[kind]}: {ms:.4f} ms")
