"""Side-by-side device vs oracle N-GMRES traces for a dense BASELINE config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1105_5331_b200 as P
from oracle import pyoracle as O

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = bench.CONFIGS[name]
dims, R = cfg["dims"], cfg["rank"]
nu = float(sum(dims) * R)
T, u0 = bench.make_problem(P, cfg, 0)
t = P.DataTensor.dense(T, dims)
o = O.Tensor.dense(dims, T)
ref = o.ngmres(u0, window=20, max_iters=2000, tol_grad=1e-10, gradient_scale=nu)
for reeval, resid in ((0, 0), (1, 1), (1, 0), (0, 1)):
    res = P.ngmres_solve(t, u0, P.NgmresOptions(window=20, max_iters=2000, tol_grad=1e-10, gradient_scale=nu,
                                                reeval_accepted=bool(reeval), residual_objective=bool(resid)))
    tr = res.trace
    first = None
    for i in range(1, min(len(tr), len(ref["trace"]))):
        a, b = tr[i], ref["trace"][i]
        if a["restart"] != b["restart"] or a["fevals"] != b["fevals"] or abs(a["f"] - b["f"]) > 1e-10 * b["f"]:
            first = i
            break
    print(f"reeval={reeval} resid={resid}: iters {len(tr) - 1} vs oracle {len(ref['trace']) - 1}; first divergence {first}")
    if first:
        for i in range(max(1, first - 2), min(first + 4, len(tr), len(ref["trace"]))):
            a, b = tr[i], ref["trace"][i]
            print(f"  it {i}: dev f={a['f']:.15e} g={a['gnorm_rel']:.3e} fe={a['fevals']} rs={int(a['restart'])} b={a['beta']:.6g}"
                  f" | ora f={b['f']:.15e} g={b['gnorm_rel']:.3e} fe={b['fevals']} rs={int(b['restart'])} b={b['beta']:.6g}")
