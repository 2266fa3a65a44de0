"""Randomised parity sweep on the GPU: random shapes (order 2-5, I_0 up to 416) and ranks 1-32,
per-call MTTKRP (every mode), f and gradient, and one ALS sweep against the CPU oracle; prints
the cases over tolerance. usage: python tools/sweep_parity.py [CASES] [SEED]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1105_5331_b200 as P
from oracle import pyoracle as O

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


for case in range(n_cases):
    order = int(rng.integers(2, 6))
    I0 = int(rng.choice([1, 3, 8, 17, 32, 33, 64, 100, 128, 129, 200, 256, 300, 416]))
    rest = [int(rng.integers(1, 40 if order <= 3 else 12)) for _ in range(order - 1)]
    dims = tuple([I0] + rest)
    if np.prod(dims) > 4_000_000:
        continue
    R = int(rng.integers(1, 33))
    T = rng.random(int(np.prod(dims))) * 2 - 1
    u = (rng.random(sum(dims) * R) * 2 - 1)
    try:
        t = P.DataTensor.dense(T, dims)
        o = O.Tensor.dense(dims, T)
        errs = {}
        for m in range(order):
            errs[f"mttkrp{m}"] = rel(t.mttkrp(u, m), o.mttkrp(u, m))
        f, g = P.objective_and_gradient(t, u)
        fo, go = o.eval(u)
        errs["f"] = abs(f - fo) / abs(fo)
        errs["g"] = rel(g, go)
        # the ALS normal matrix Gamma_n (Hadamard of the other Grams, rank <= prod_{m != n} I_m)
        # is singular when R exceeds that product: the ridge retry then makes the update
        # arbitrarily sensitive to rounding (an ill-posed case, not compared)
        if all(R <= int(np.prod([dims[m] for m in range(order) if m != n])) for n in range(order)):
            errs["als"] = rel(P.als_sweep(t, u), o.als_sweep(u))
    except Exception as e:  # noqa: BLE001
        print(f"case {case} dims {dims} R {R}: exception {type(e).__name__}: {e}")
        bad += 1
        continue
    worst = {k: v for k, v in errs.items() if v > (1e-9 if k == "als" else 1e-12)}
    if worst:
        bad += 1
        print(f"case {case} dims {dims} R {R}: " + ", ".join(f"{k} {v:.2e}" for k, v in worst.items()))
print(f"{n_cases} cases, {bad} over tolerance")
