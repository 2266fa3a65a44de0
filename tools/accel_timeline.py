"""Warm per-kernel timeline of one device accelerate (N-GMRES step II) at C2 size
(n_u = 19200, window 20) through CUPTI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1105_5331_b200 as P

n, m = 19200, 20
rng = np.random.default_rng(0)
wu = rng.standard_normal((m, n))
wg = rng.standard_normal((m, n))
ub = rng.standard_normal(n)
gb = rng.standard_normal(n)
torch.cuda.init()
for _ in range(3):
    P.accelerate(wu, wg, ub, gb)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    P.accelerate(wu, wg, ub, gb)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = None
for e in ev:
    gap = e.time_range.start - prev if prev is not None else 0.0
    print(f"  {e.time_range.start - t0:8.1f} +{gap:5.1f}  {e.time_range.end - e.time_range.start:7.1f} us  {e.name[:70]}")
    prev = e.time_range.end
