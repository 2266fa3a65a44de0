"""Per-config evidence on the B200 for every BASELINE.json config:
device N-GMRES solves to the BASELINE stopping rule (C0, C1, C3), 100 iterations of the sparse
C4, kernel timings, and oracle comparisons where the CPU can afford them."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1105_5331_b200 as P
from oracle import pyoracle as O

which = sys.argv[1:] or ["c0", "c1", "c3", "c4"]
out = {}


def dense_case(name, tol, oracle_full):
    # (wall clock for the batched sweeps: host sync per wave is part of the cost)
    cfg = bench.CONFIGS[name]
    dims, R = cfg["dims"], cfg["rank"]
    nu = float(sum(dims) * R)
    T, u0 = bench.make_problem(P, cfg, 0)
    t = P.DataTensor.dense(T, dims)
    opts = P.NgmresOptions(window=20, max_iters=2000, tol_grad=tol, gradient_scale=nu)
    s = P.Solver(t, R, opts, 0)
    ms = s.restart(u0, 2000)
    st = s.state()
    tr = s.trace(st["iters"] + 1)
    rec = {"iters": st["iters"], "stop": st["stop"], "f": st["best_f"], "h": tr[-1]["h"], "ms": ms,
           "iters_per_s": st["iters"] / (ms / 1e3), "fevals": st["fevals"]}
    res = P.ngmres_solve(t, u0, opts)
    rec["ngmres_solve_api_iters"] = len(res.trace) - 1
    if oracle_full:
        o = O.Tensor.dense(dims, T)
        t0 = time.time()
        ref = o.ngmres(u0, window=20, max_iters=2000, tol_grad=tol, gradient_scale=nu)
        cpu_s = time.time() - t0
        n_ref = len(ref["trace"]) - 1
        rec["oracle"] = {"iters": n_ref, "stop": ref["stop"], "f": ref["f"], "seconds": cpu_s,
                         "iters_per_s": n_ref / cpu_s}
        rec["parity"] = {"f_rel": abs(st["best_f"] - ref["f"]) / ref["f"],
                         "iters_rel": abs(st["iters"] - n_ref) / max(n_ref, 1)}
    if name in ("c0", "c1"):
        # seed sweep (bench.cpp:80-158) as concurrent device solves: 64 starts, aggregate iters/s
        starts = np.stack([P.uniform_initial_guess(dims, R, 1000 + i) for i in range(64)])
        for conc in (1, 8, 32):
            P.solve_batch(t, starts[:conc], opts, 0, conc)  # solver pool + graphs built
            t0 = time.perf_counter()
            b = P.solve_batch(t, starts, opts, 0, conc)
            dt = time.perf_counter() - t0
            rec[f"batch64_conc{conc}"] = {"iters": int(b.iters.sum()), "seconds": dt,
                                          "iters_per_s": float(b.iters.sum()) / dt,
                                          "solves_per_s": 64 / dt, "all_grad_tol": bool((b.stop_reason == 0).all())}
    kk = int(np.prod(dims))
    for kind, nm in ((3, "fused_pass_ms"), (4, "m0_pass_ms"), (5, "s_pass_ms"), (7, "eval_ms")):
        rec[nm] = P.bench_kernel(t, u0, kind=kind, reps=10, flush_l2=True)
    rec["mttkrp_GBps"] = [round((8.0 * kk + 8.0 * R * sum(dims)) / (P.bench_kernel(t, u0, 0, m, 10, True) * 1e-3) / 1e9, 1)
                          for m in range(len(dims))]
    return rec


def sparse_case():
    dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
    t0 = time.time()
    coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
    gen_s = time.time() - t0
    t0 = time.time()
    t = P.DataTensor.coo(dims, coords, vals)
    up_s = time.time() - t0
    u0 = P.uniform_initial_guess(dims, R, 0)
    rec = {"generate_s": gen_s, "upload_s": up_s, "nnz": t.nnz()}
    bytes_mode = nnz * (2 * 4 + 8) + 8.0 * R * sum(dims)
    rec["mttkrp_ms"] = [P.bench_kernel(t, u0, 0, m, 10, True) for m in range(3)]
    rec["mttkrp_GBps_streamed"] = [round(bytes_mode / (x * 1e-3) / 1e9, 1) for x in rec["mttkrp_ms"]]
    rec["mttkrp_GBps_coo32"] = [round((32.0 * nnz + 8.0 * R * sum(dims)) / (x * 1e-3) / 1e9, 1) for x in rec["mttkrp_ms"]]
    rec["eval_ms"] = P.bench_kernel(t, u0, 1, 0, 5, True)
    opts = P.NgmresOptions(window=20, max_iters=100, tol_grad=1e-300, gradient_scale=float(sum(dims) * R))
    s = P.Solver(t, R, opts, 0)
    ms = s.restart(u0, 100)
    st = s.state()
    rec.update({"iters": st["iters"], "stop": st["stop"], "ms": ms, "iters_per_s": st["iters"] / (ms / 1e3),
                "f": st["best_f"], "fevals": st["fevals"]})
    # per-call parity at full size against the oracle (MTTKRP every mode, gradient, f)
    o = O.Tensor.coo(dims, coords, vals)
    for m in range(3):
        a, b = t.mttkrp(u0, m), o.mttkrp(u0, m)
        rec[f"mttkrp{m}_rel"] = float(np.linalg.norm(a - b) / np.linalg.norm(b))
    f, g = P.objective_and_gradient(t, u0)
    fo, go = o.eval(u0)
    rec["f_rel"] = abs(f - fo) / abs(fo)
    rec["g_rel"] = float(np.linalg.norm(g - go) / np.linalg.norm(go))
    return rec


for name in which:
    if name == "c4":
        out[name] = sparse_case()
    else:
        tol = 1e-9 if name == "c3" else 1e-10
        out[name] = dense_case(name, tol, oracle_full=(name in ("c0", "c1")))
    print(name, json.dumps(out[name]), flush=True)
