"""Kernel timeline of N-GMRES iterations at C2 (400^3, R=16) through CUPTI (torch.profiler
sees every kernel the process launches, graph bodies included).  Prints per-kernel totals
and the idle gap between consecutive kernels (graph launch/dependency latency)."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1105_5331_b200 as P

cfg = dict(dims=(400, 400, 400), rank=16, c=0.5, l1=1.0, l2=1.0)
warm = int(os.environ.get("WARM", "10"))
iters = int(os.environ.get("ITERS", "20"))
T, _, _ = P.dense_test_problem(cfg["dims"], cfg["rank"], cfg["c"], cfg["l1"], cfg["l2"], 1, noise_mode=1)
u0 = P.uniform_initial_guess(cfg["dims"], cfg["rank"], 1)
t = P.DataTensor.dense(T, cfg["dims"])
s = P.Solver(t, cfg["rank"], P.NgmresOptions(tol_grad=1e-10, gradient_scale=float(sum(cfg["dims"]) * 16)))
s.set_initial(u0)
s.init()
s.run(warm)
s.state()
torch.cuda.init()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.run(warm + iters)
    st = s.state()
print("state", st)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
agg = defaultdict(lambda: [0, 0.0])
busy = 0.0
gaps = []
for i, e in enumerate(ev):
    d = e.time_range.end - e.time_range.start
    agg[e.name.split("(")[0][:80]][0] += 1
    agg[e.name.split("(")[0][:80]][1] += d
    busy += d
    if i:
        gaps.append(e.time_range.start - ev[i - 1].time_range.end)
span = ev[-1].time_range.end - ev[0].time_range.start
n_it = st["iters"] - warm
print(f"span {span:.1f} us over {n_it} iterations = {span / max(n_it, 1):.1f} us/iter; busy {busy:.1f} us "
      f"({100 * busy / span:.1f}%); {len(ev)} kernels ({len(ev) / max(n_it, 1):.1f}/iter); "
      f"median gap {sorted(gaps)[len(gaps) // 2]:.2f} us")
print(f"{'kernel':80s} {'n':>6s} {'us/iter':>9s} {'us/launch':>9s} {'share':>6s}")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:80s} {n:6d} {us / n_it:9.1f} {us / n:9.2f} {100 * us / span:5.1f}%")
