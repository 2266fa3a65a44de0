"""MTTKRP of every mode through a given libcpfit_gpu.so against numpy (einsum) for one shape.
usage: python tools/check_mttkrp.py LIB I0,I1,I2 R"""
import ctypes as C
import sys

import numpy as np

L = C.CDLL(sys.argv[1])
dims = tuple(int(x) for x in sys.argv[2].split(","))
R = int(sys.argv[3])
rng = np.random.default_rng(0)
T = rng.random(int(np.prod(dims))) * 2 - 1
u = rng.random(sum(dims) * R) * 2 - 1
d = np.array(dims, dtype=np.int64)
h = C.c_void_p()
assert L.cpfit_tensor_create_dense(len(dims), d.ctypes.data_as(C.c_void_p), T.ctypes.data_as(C.c_void_p), C.byref(h)) == 0
Tt = T.reshape(dims[::-1]).transpose()  # first-mode-fastest
facs, off = [], 0
for n in dims:
    facs.append(u[off:off + n * R].reshape(R, n).T)
    off += n * R
letters = "ijkl"[:len(dims)]
for mode in range(len(dims)):
    out = np.empty(dims[mode] * R)
    rc = L.cpfit_mttkrp(h, C.c_int64(R), u.ctypes.data_as(C.c_void_p), mode, out.ctypes.data_as(C.c_void_p))
    others = [m for m in range(len(dims)) if m != mode]
    expr = letters + "," + ",".join(letters[m] + "r" for m in others) + "->" + letters[mode] + "r"
    ref = np.einsum(expr, Tt, *[facs[m] for m in others])
    got = out.reshape(R, dims[mode]).T
    print(f"mode {mode}: rc {rc} rel {np.linalg.norm(got - ref) / np.linalg.norm(ref):.3e}")
