"""§8(f) row 4 timings at BASELINE config-4 scale (10M nonzeros, 10000^3): the seeded generator,
the parallel .tns writer and reader, the binary sidecar, and the oracle's sequential restatement of
the reference reader (io.cpp) on the same file; then DataTensor construction (canonicalisation +
per-mode sorts + upload). Prints one JSON line. usage: python tools/tns_speed.py [dir]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P
from oracle import pyoracle as O

d = sys.argv[1] if len(sys.argv) > 1 else tempfile.mkdtemp()
dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
out = {"host_cores": os.cpu_count()}
t = time.time()
coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
out["generate_s"] = round(time.time() - t, 3)
t = time.time()
Tc, _, _ = P.dense_test_problem((400, 400, 400), 16, 0.5, 1.0, 1.0, 0, noise_mode=1)
out["generate_c2_s"] = round(time.time() - t, 3)
del Tc
path = os.path.join(d, "c4.tns")
t = time.time()
P.write_tns(path, dims, coords, vals)
out["write_s"] = round(time.time() - t, 3)
out["file_mb"] = round(os.path.getsize(path) / 2**20, 1)
t = time.time()
dd, c, v = P.read_tns(path, sidecar=2)
out["read_text_s"] = round(time.time() - t, 3)
assert np.array_equal(c, coords) and np.array_equal(v, vals)
t = time.time()
dd, c, v = P.read_tns(path, sidecar=1)
out["read_sidecar_s"] = round(time.time() - t, 3)
assert P.read_tns.last_from_sidecar and np.array_equal(v, vals)
t = time.time()
od, oc, ov = O.tns_read(path)
out["oracle_read_s"] = round(time.time() - t, 3)
assert np.array_equal(oc, coords) and np.array_equal(ov, vals)
if P.device_count() > 0:
    t = time.time()
    tt = P.DataTensor.coo(dims, c, v)
    out["tensor_create_s"] = round(time.time() - t, 3)
    assert tt.nnz() == nnz
os.remove(path)
os.remove(path + ".cpfbin")
print(json.dumps(out), flush=True)
