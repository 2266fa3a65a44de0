"""Warm-cache per-kernel timeline of eagerly launched passes at C2 shape (400^3, R=16) through
CUPTI (torch.profiler): KINDS as in tools/prof_fiber.py (2 = ALS sweep, 7 = evaluation).
Prints each kernel of the last repetition with its duration and the gap before it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1105_5331_b200 as P

dims, R = (400, 400, 400), 16
rng = np.random.default_rng(0)
T = rng.random(int(np.prod(dims)))
u = rng.random(sum(dims) * R)
t = P.DataTensor.dense(T, dims)
kinds = [int(k) for k in os.environ.get("KINDS", "2,7").split(",")]
mode = int(os.environ.get("MODE", "0"))
torch.cuda.init()
for kind in kinds:
    P.bench_kernel(t, u, kind=kind, mode=mode, reps=2, flush_l2=False)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.bench_kernel(t, u, kind=kind, mode=mode, reps=3, flush_l2=False)
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    # bench_kernel runs 3 warm-up calls + reps (3) calls: the last call is the last sixth
    ev = [e for e in ev if "emcpy" not in e.name and "emset" not in e.name]
    n = len(ev) // 6
    last = ev[-n:]
    t0 = last[0].time_range.start
    print(f"kind {kind}: {n} kernels, span {last[-1].time_range.end - t0:.1f} us")
    prev = None
    for e in last:
        gap = e.time_range.start - prev if prev is not None else 0.0
        name = e.name.replace("cpfit_gpu::", "").replace("(anonymous namespace)::", "")[:60]
        print(f"  {e.time_range.start - t0:8.1f} +{gap:5.1f}  {e.time_range.end - e.time_range.start:7.1f} us  {name}")
        prev = e.time_range.end
