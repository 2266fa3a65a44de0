"""A/B of the fiber-pass kernels between two builds of libcpfit_gpu.so on the same box:
alternating rounds of cpfit_bench_kernel (kinds as in tools/prof_fiber.py) at DIMS / RANK.
usage: python tools/ab_kernels.py LIB_A LIB_B [ROUNDS]"""
import ctypes as C
import os
import sys

import numpy as np

dims = tuple(int(x) for x in os.environ.get("DIMS", "400,400,400").split(","))
R = int(os.environ.get("RANK", "16"))
kinds = [int(k) for k in os.environ.get("KINDS", "5,4,3").split(",")]
libs = [C.CDLL(p) for p in sys.argv[1:3]]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rng = np.random.default_rng(0)
T = rng.random(int(np.prod(dims)))
u = rng.random(sum(dims) * R)
d = np.array(dims, dtype=np.int64)
hs = []
for L in libs:
    h = C.c_void_p()
    rc = L.cpfit_tensor_create_dense(len(dims), d.ctypes.data_as(C.c_void_p), T.ctypes.data_as(C.c_void_p), C.byref(h))
    assert rc == 0, rc
    hs.append(h)
res = {(i, k): [] for i in range(2) for k in kinds}
for _ in range(rounds):
    for i, L in enumerate(libs):
        for k in kinds:
            ms = C.c_float()
            rc = L.cpfit_bench_kernel(hs[i], C.c_int64(R), u.ctypes.data_as(C.c_void_p), k, 0, 10, 0, C.byref(ms))
            assert rc == 0, rc
            res[(i, k)].append(ms.value)
for k in kinds:
    a, b = np.median(res[(0, k)]), np.median(res[(1, k)])
    print(f"kind {k}: A {a:.4f} ms  B {b:.4f} ms  B/A {b / a:.3f}")
