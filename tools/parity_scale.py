"""Device vs oracle at BASELINE scale (diagnostic; the gated versions live in tests/test_gpu_scale.py).

usage: python tools/parity_scale.py [c2pc] [c2it] [c3] [c4] [c1]
Prints one JSON line per check plus, for trajectories, the first row where the device and the
oracle disagree on a discrete decision (restart flag, evaluation count) or on f beyond 1e-10.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P
from oracle import pyoracle as O

CFG = {
    "c0": ((20, 20, 20), 3, 0.5, 1.0, 1.0, 1e-10),
    "c1": ((50, 50, 50), 5, 0.9, 10.0, 5.0, 1e-10),
    "c2": ((400, 400, 400), 16, 0.5, 1.0, 1.0, 1e-10),
    "c3": ((64, 64, 64, 64), 10, 0.7, 5.0, 0.0, 1e-9),
}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def problem(name):
    dims, R, c, l1, l2, tol = CFG[name]
    T, truth, _ = P.dense_test_problem(dims, R, c, l1, l2, 0, noise_mode=1, want_truth=True)
    u0 = P.uniform_initial_guess(dims, R, 0)
    return dims, R, tol, T, truth, u0


def first_divergence(dev, ref):
    for i in range(1, min(len(dev), len(ref))):
        a, b = dev[i], ref[i]
        if a["restart"] != b["restart"] or a["fevals"] != b["fevals"] or abs(a["f"] - b["f"]) > 1e-10 * abs(b["f"]):
            return i
    return None


def show(dev, ref, at, n=4):
    for i in range(max(1, at - 2), min(at + n, len(dev), len(ref))):
        a, b = dev[i], ref[i]
        print(f"  it {i}: dev f={a['f']:.15e} g={a['gnorm_rel']:.3e} fe={a['fevals']} rs={int(a['restart'])} "
              f"b={a['beta']:.8g} | ora f={b['f']:.15e} g={b['gnorm_rel']:.3e} fe={b['fevals']} "
              f"rs={int(b['restart'])} b={b['beta']:.8g}")


def c2_percall():
    dims, R, tol, T, truth, u0 = problem("c2")
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    out = {"norm_rel": abs(t.norm() - o.norm()) / o.norm()}
    for tag, u in (("u0", u0), ("truth", truth)):
        for m in range(3):
            out[f"{tag}_mttkrp{m}"] = rel(t.mttkrp(u, m), o.mttkrp(u, m))
        fo, go = o.eval(u)
        for form in (0, 1):
            f, g = P.objective_and_gradient_form(t, u, form)
            out[f"{tag}_form{form}_f"] = abs(f - fo) / abs(fo)
            out[f"{tag}_form{form}_g"] = rel(g, go)
        out[f"{tag}_h"] = float(np.sqrt(2 * fo) / o.norm())
    print("c2_percall", json.dumps(out), flush=True)


def iterates(name, k=20, **kw):
    dims, R, tol, T, truth, u0 = problem(name)
    nu = float(sum(dims) * R)
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    t0 = time.time()
    ref = o.ngmres(u0, window=20, max_iters=k, tol_grad=tol, gradient_scale=nu, record_iterates=k + 1)
    cpu = time.time() - t0
    s = P.Solver(t, R, P.NgmresOptions(window=20, max_iters=k, tol_grad=tol, gradient_scale=nu, **kw), 0)
    s.set_initial(u0)
    s.init()
    rows = []
    for it in range(1, len(ref["iterates"])):
        s.run(it)
        st = s.state()
        tr = s.trace(it + 1)
        ro = ref["trace"][it]
        rows.append({"it": it, "iterate_rel": rel(s.iterate(), ref["iterates"][it]),
                     "f_rel": abs(tr[it]["f"] - ro["f"]) / abs(ro["f"]), "restart": [tr[it]["restart"], ro["restart"]],
                     "fevals": [tr[it]["fevals"], ro["fevals"]], "beta": [tr[it]["beta"], ro["beta"]]})
        if st["stop"] >= 0:
            break
    print(f"{name}_iterates", json.dumps({"oracle_s": cpu, "opts": kw,
                                           "max_iterate_rel": max(r["iterate_rel"] for r in rows),
                                           "max_f_rel": max(r["f_rel"] for r in rows)}), flush=True)
    for r in rows:
        print("   ", json.dumps(r))


def full_solve(name, variants=((False, False),)):
    dims, R, tol, T, truth, u0 = problem(name)
    nu = float(sum(dims) * R)
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    t0 = time.time()
    ref = o.ngmres(u0, window=20, max_iters=2000 if name != "c3" else 1000, tol_grad=tol, gradient_scale=nu)
    cpu = time.time() - t0
    for reeval, resid in variants:
        res = P.ngmres_solve(t, u0, P.NgmresOptions(window=20, max_iters=2000 if name != "c3" else 1000, tol_grad=tol,
                                                    gradient_scale=nu, reeval_accepted=reeval,
                                                    residual_objective=resid))
        n, nr = len(res.trace) - 1, len(ref["trace"]) - 1
        fd = first_divergence(res.trace, ref["trace"])
        print(f"{name}_solve", json.dumps({"reeval": reeval, "resid": resid, "iters": n, "oracle_iters": nr,
                                           "stop": [res.stop_reason, ref["stop"]],
                                           "f_rel": abs(res.f - ref["f"]) / abs(ref["f"]), "oracle_s": cpu,
                                           "first_divergence": fd}), flush=True)
        if fd:
            show(res.trace, ref["trace"], fd)


def c4(k=20):
    dims, nnz, R = (10000, 10000, 10000), 10_000_000, 10
    coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 0)
    t = P.DataTensor.coo(dims, coords, vals)
    t0 = time.time()
    o = O.Tensor.coo(dims, coords, vals)
    build = time.time() - t0
    u0 = P.uniform_initial_guess(dims, R, 0)
    out = {"oracle_build_s": build}
    for m in range(3):
        out[f"mttkrp{m}"] = rel(t.mttkrp(u0, m), o.mttkrp(u0, m))
    f, g = P.objective_and_gradient(t, u0)
    fo, go = o.eval(u0)
    out["f"] = abs(f - fo) / abs(fo)
    out["g"] = rel(g, go)
    print("c4_percall", json.dumps(out), flush=True)
    nu = float(sum(dims) * R)
    t0 = time.time()
    ref = o.ngmres(u0, window=20, max_iters=k, tol_grad=1e-300, gradient_scale=nu)
    cpu = time.time() - t0
    res = P.ngmres_solve(t, u0, P.NgmresOptions(window=20, max_iters=k, tol_grad=1e-300, gradient_scale=nu))
    worst = max(abs(a["f"] - b["f"]) / abs(b["f"]) for a, b in zip(res.trace, ref["trace"]))
    fd = first_divergence(res.trace, ref["trace"])
    print("c4_trace", json.dumps({"rows": len(res.trace), "oracle_rows": len(ref["trace"]), "max_f_rel": worst,
                                  "oracle_s": cpu, "first_divergence": fd}), flush=True)
    if fd:
        show(res.trace, ref["trace"], fd)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c2pc", "c2it", "c3", "c4", "c1"]
    for w in which:
        if w == "c2pc":
            c2_percall()
        elif w == "c2it":
            iterates("c2")
        elif w == "c1it":
            iterates("c1")
        elif w == "c3":
            full_solve("c3", ((False, False), (True, True)))
        elif w == "c4":
            c4()
        elif w == "c1":
            full_solve("c1", ((False, False), (True, True), (True, False), (False, True)))
