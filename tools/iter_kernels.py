"""Per-iteration kernel time by kernel at C2 (400^3, R=16) with the loop issued eagerly
(CPFIT_EAGER=1) so CUPTI sees every kernel; warm caches, real data (bench problem seeds).
Host round trips between kernels make the wall time meaningless here: only the kernel
durations are reported."""
import os
import sys
from collections import defaultdict

os.environ["CPFIT_EAGER"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1105_5331_b200 as P

dims, R = (400, 400, 400), 16
T, _, _ = P.dense_test_problem(dims, R, 0.5, 1.0, 1.0, 0, noise_mode=1)
t = P.DataTensor.dense(T, dims)
s = P.Solver(t, R, P.NgmresOptions(tol_grad=1e-10, gradient_scale=float(sum(dims) * R), max_iters=400))
s.set_initial(P.uniform_initial_guess(dims, R, 1))
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
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    name = e.name.replace("cpfit_gpu::", "").replace("(anonymous namespace)::", "").split("(")[0][:60]
    agg[name][0] += 1
    agg[name][1] += e.time_range.end - e.time_range.start
tot = sum(v for _, v in agg.values())
print(f"{it} iterations, kernel time {tot / it:.1f} us/iter")
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:60s} {c / it:6.2f}/it {us / it:8.1f} us/it {us / c:8.1f} us/launch")
