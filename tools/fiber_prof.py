"""Where the fiber-pass warps wait: barrier-wait cycles per role from the diagnostic build.

  make -C paper_1105_5331_b200/csrc prof
  CPFIT_GPU_LIB=paper_1105_5331_b200/lib/libcpfit_gpu_prof.so KINDS=3,4,5 python tools/fiber_prof.py

Counters (summed over CTAs and warps of the role, cycles): the producers wait on a free T stage
(tempty) and a free W buffer (wempty); S warps on T data (tfull) and the W tile (wfull, for the
per-fiber objective); M0 warps on T data and the W tile. Printed as a share of that role's
summed warp lifetime."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P
from paper_1105_5331_b200.api import lib

dims = tuple(int(x) for x in os.environ.get("DIMS", "400,400,400").split(","))
R = int(os.environ.get("RANK", "16"))
rng = np.random.default_rng(0)
T = rng.random(int(np.prod(dims)))
u = rng.random(sum(dims) * R)
t = P.DataTensor.dense(T, dims)
lib.cpfit_fiber_prof.argtypes = [C.POINTER(C.c_uint64), C.c_int]
names = {3: "fused", 4: "m0", 5: "s", 6: "fused_resid"}
for kind in [int(k) for k in os.environ.get("KINDS", "3,4,5").split(",")]:
    P.bench_kernel(t, u, kind=kind, mode=0, reps=1, flush_l2=False)
    buf = (C.c_uint64 * 12)()
    lib.cpfit_fiber_prof(buf, 1)
    ms = P.bench_kernel(t, u, kind=kind, mode=0, reps=5, flush_l2=False)
    lib.cpfit_fiber_prof(buf, 1)
    v = [float(x) for x in buf]
    prod, sw, mw = v[7], v[8], v[9]
    print(f"{names.get(kind, kind)}: {ms:.4f} ms  (lifetimes: producers {prod:.3g} S-warps {sw:.3g} "
          f"M0-warps {mw:.3g} cycles)")
    def sh(x, tot):
        return f"{100 * x / tot:5.1f}%" if tot else "  -  "
    print(f"  producers tempty {sh(v[0], prod)}  wempty {sh(v[1], prod)}")
    print(f"  S warps   tfull  {sh(v[2], sw)}  wfull  {sh(v[6], sw)}")
    print(f"  M0 warps  tfull  {sh(v[3], mw)}  wfull  {sh(v[4], mw)}")

