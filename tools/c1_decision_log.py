"""Decision log for BASELINE config 1 (50^3 R=5, collinearity 0.9 swamp): where the device and the
oracle trajectories part, and how wide the oracle's own iteration count spreads when its input
moves by rounding. Output: profiles/r02_c1_decision_log.txt (run on the GPU box).

For each device objective mode (default; literal = reeval_accepted + residual_objective) it prints
the rows around (a) the first f difference above 1e-12, (b) the first line-search step (beta)
difference above 1e-8 and (c) the first discrete decision that differs (restart flag = the
slope >= 0 test of ngmres.cpp:111, or the Moré–Thuente trial count, line_search.cpp:157-183).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P
from oracle import pyoracle as O


def row(tag, r):
    return (f"{tag} f={r['f']:.16e} gnorm_rel={r['gnorm_rel']:.4e} fevals={r['fevals']} restart={int(r['restart'])} "
            f"beta={r['beta']:.12g}")


def first(dev, ref, pred):
    for i in range(1, min(len(dev), len(ref))):
        if pred(dev[i], ref[i]):
            return i
    return None


def main(out):
    dims, R = (50, 50, 50), 5
    nu = float(sum(dims) * R)
    T, _, _ = P.dense_test_problem(dims, R, 0.9, 10.0, 5.0, 0, noise_mode=1)
    u0 = P.uniform_initial_guess(dims, R, 0)
    t = P.DataTensor.dense(T, dims)
    o = O.Tensor.dense(dims, T)
    ref = o.ngmres(u0, window=20, max_iters=2000, tol_grad=1e-10, gradient_scale=nu)
    nr = len(ref["trace"]) - 1
    print(f"oracle: {nr} iterations to ||g||/{nu:g} < 1e-10, f = {ref['f']:.16e}", file=out)
    for name, kw in (("default", {}), ("literal (reeval_accepted=1, residual_objective=1)",
                                       dict(reeval_accepted=True, residual_objective=True))):
        res = P.ngmres_solve(t, u0, P.NgmresOptions(window=20, max_iters=2000, tol_grad=1e-10, gradient_scale=nu, **kw))
        dev = res.trace
        print(f"\n== device {name}: {len(dev) - 1} iterations, f = {res.f:.16e} "
              f"(rel {abs(res.f - ref['f']) / ref['f']:.2e})", file=out)
        marks = (("first f difference > 1e-12 relative", lambda a, b: abs(a["f"] - b["f"]) > 1e-12 * abs(b["f"])),
                 ("first beta difference > 1e-8 relative",
                  lambda a, b: abs(a["beta"] - b["beta"]) > 1e-8 * max(abs(b["beta"]), 1e-300)),
                 ("first discrete decision difference (restart flag or Moré–Thuente trial count)",
                  lambda a, b: a["restart"] != b["restart"] or a["fevals"] != b["fevals"]))
        for what, pred in marks:
            i = first(dev, ref["trace"], pred)
            print(f"-- {what}: iteration {i}", file=out)
            if i is None:
                continue
            for j in range(max(1, i - 2), min(i + 3, len(dev), len(ref["trace"]))):
                print("   it %3d  %s" % (j, row("dev", dev[j])), file=out)
                print("           %s" % row("ora", ref["trace"][j]), file=out)
    # the oracle's own sensitivity: the same problem, start perturbed by 1e-15 relative
    rng = np.random.default_rng(1)
    counts = []
    for _ in range(40):
        r = o.ngmres(u0 * (1 + 1e-15 * rng.standard_normal(u0.size)), window=20, max_iters=2000, tol_grad=1e-10,
                     gradient_scale=nu)
        counts.append(len(r["trace"]) - 1)
    counts = np.array(sorted(counts))
    within = float(np.mean(np.abs(counts - nr) <= max(1, int(0.02 * nr))))
    print(f"\n== oracle with its start perturbed by 1e-15 relative (40 draws): iterations {counts.min()}..{counts.max()}, "
          f"median {np.median(counts):g}; {100 * within:.0f}% of the oracle's own perturbed runs land within "
          f"+-2% of its unperturbed count\n   {counts.tolist()}", file=out)


if __name__ == "__main__":
    path = sys.argv[1] if len(sys.argv) > 1 else None
    if path:
        with open(path, "w") as f:
            main(f)
        print(open(path).read())
    else:
        main(sys.stdout)
