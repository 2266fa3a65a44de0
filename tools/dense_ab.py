"""Dense fibre-pass A/B: the fused / M0 / S pass times and the N-GMRES rate of one config for each
library given (one process per library, run twice in alternation so box drift shows).
usage: python tools/dense_ab.py c3 lib_a.so lib_b.so ...   (default: the in-tree library)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import bench
import paper_1105_5331_b200 as P
cfg = bench.CONFIGS[sys.argv[1]]
dims, R = cfg["dims"], cfg["rank"]
T, u0 = bench.make_problem(P, cfg, 0)
t = P.DataTensor.dense(T, dims)
out = {k: round(min(P.bench_kernel(t, u0, kind, 0, 20, True) for _ in range(3)), 5)
       for k, kind in (("fused_ms", 3), ("m0_ms", 4), ("s_ms", 5))}
nu = float(sum(dims) * R)
s = P.Solver(t, R, P.NgmresOptions(window=20, max_iters=2000, tol_grad=bench.stop_tol(sys.argv[1]), gradient_scale=nu), 0)
s.restart(u0, 2000)
ms = min(s.restart(u0, 2000) for _ in range(3))
st = s.state()
out["iters"] = st["iters"]
out["iters_per_s"] = round(st["iters"] / (ms * 1e-3), 1)
print(json.dumps(out))
"""

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
libs = sys.argv[2:] or [""]
for rnd in range(2):
    for lib in libs:
        env = dict(os.environ, ROOT=ROOT)
        if lib:
            env["CPFIT_GPU_LIB"] = lib
        r = subprocess.run([sys.executable, "-c", CHILD, name], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else "ERROR " + r.stderr[-400:]
        print(f"round {rnd} {os.path.basename(lib) or 'in-tree'}: {line}", flush=True)
