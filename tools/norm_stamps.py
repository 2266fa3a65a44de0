"""Phase timing (globaltimer) inside normalize_kernel from the -DCPFIT_NORM_STAMPS build
(lib/libcpfit_gpu_stamps.so): the loop runs eagerly; stamps of the last launch (block 0, the
last block index, and the last block to arrive)."""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["CPFIT_GPU_LIB"] = os.path.join(HERE, "paper_1105_5331_b200", "lib", "libcpfit_gpu_stamps.so")
os.environ["CPFIT_EAGER"] = "1"
sys.path.insert(0, HERE)
import paper_1105_5331_b200 as P
from paper_1105_5331_b200 import api

dims, R = (400, 400, 400), 16
T, _, _ = P.dense_test_problem(dims, R, 0.5, 1.0, 1.0, 0, noise_mode=1)
t = P.DataTensor.dense(T, dims)
s = P.Solver(t, R, P.NgmresOptions(tol_grad=1e-10, gradient_scale=float(sum(dims) * R), max_iters=400))
s.set_initial(P.uniform_initial_guess(dims, R, 1))
s.init()
s.run(int(os.environ.get("ITERS", "6")))
s.state()
buf = (ctypes.c_ulonglong * 32)()
api.lib.cpfit_debug_norm_stamps(buf)
b = list(buf)
for base, name in ((0, "block 0"), (16, "block G-1")):
    t0 = b[base]
    print(name, " ".join(f"{k}:{(b[base + k] - t0) / 1e3:.2f}" for k in (1, 2, 3, 4, 5, 10, 12) if b[base + k] >= t0))
t0 = b[0]
print("last block", " ".join(f"{k}:{(b[k] - t0) / 1e3:.2f}" for k in (27, 28, 29) if b[k] >= t0))
