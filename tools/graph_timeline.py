"""Device timeline of the N-GMRES loop as the solver runs it (CUDA graph, not eager) at C2
(400^3, R=16) through CUPTI: per-kernel busy time, the idle time between consecutive kernels
(launch gaps inside the graph), and one iteration's kernel sequence with start offsets.
usage: python tools/graph_timeline.py  [CFG=c2|c3 ITERS=20 WARM=10 SHOW=1]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1105_5331_b200 as P

import bench  # noqa: E402

if os.environ.get("CFG") == "c4":  # the sparse config: 10000^3, 10M nnz, R = 10
    dims, R = (10000, 10000, 10000), 10
    coords, vals, _ = P.random_sparse_problem(dims, 10_000_000, R, 0.01, 0)
    t = P.DataTensor.coo(dims, coords, vals)
    u0 = P.uniform_initial_guess(dims, R, 1)
else:
    cfg = bench.CONFIGS[os.environ.get("CFG", "c2")]  # CFG=c3: the order-4 config
    dims, R = cfg["dims"], cfg["rank"]
    T, u0 = bench.make_problem(P, cfg, 1)
    t = P.DataTensor.dense(T, dims)
s = P.Solver(t, R, P.NgmresOptions(tol_grad=1e-300, gradient_scale=float(sum(dims) * R), max_iters=400))
s.set_initial(u0)
s.init()
w0 = int(os.environ.get("WARM", "10"))
n = int(os.environ.get("ITERS", "20"))
s.run(w0)
s.state()
torch.cuda.init()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.run(w0 + n)
    st = s.state()
it = st["iters"] - w0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev = [e for e in ev if "emcpy" not in e.name and "emset" not in e.name]
ev.sort(key=lambda e: e.time_range.start)


def short(name):
    return name.replace("cpfit_gpu::", "").replace("(anonymous namespace)::", "").split("(")[0][:44]


# busy = union of kernel intervals (the side stream overlaps), idle = the rest of the span
busy, idle, end = 0.0, 0.0, None
gap_after = defaultdict(float)
prev = None
for e in ev:
    a, b = e.time_range.start, e.time_range.end
    if end is None:
        busy += b - a
        end = b
    elif a >= end:
        idle += a - end
        gap_after[short(prev.name)] += a - end
        busy += b - a
        end = b
    elif b > end:
        busy += b - end
        end = b
    prev = e
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"{it} iterations (graph mode), span {span / it:.1f} us/iter: busy {busy / it:.1f}, idle {idle / it:.1f}, "
      f"{len(ev) / it:.1f} kernels/iter")
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    agg[short(e.name)][0] += 1
    agg[short(e.name)][1] += e.time_range.end - e.time_range.start
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:44s} {c / it:5.2f}/it {us / it:7.1f} us/it {us / c:7.1f} us/launch   idle after {gap_after[k] / it:5.1f} us/it")
if os.environ.get("SHOW", "1") == "1":
    # one iteration: from the second-to-last normalize_kernel... print the last ~60 kernels
    k0 = max(0, len(ev) - int(os.environ.get("SHOWN", "70")))
    t0 = ev[k0].time_range.start
    last_end = t0
    for e in ev[k0:]:
        a, b = e.time_range.start, e.time_range.end
        print(f"  {a - t0:8.1f} +{b - a:7.1f}  gap {a - last_end:6.1f}  {short(e.name)}")
        last_end = max(last_end, b)
