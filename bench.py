#!/usr/bin/env python
"""bench.py — ALS-preconditioned N-GMRES for rank-R CP (arxiv/paper_1105_5331) on one B200.

Workload (BASELINE.json configs[2], the scale case the metric's roofline target is quoted on):
dense 400x400x400 fp64 tensor (512 MB), R=16, collinearity 0.5, l1=l2=1 (BASELINE l/100 noise
scaling), U[0,1] start from seed; a "step" is one N-GMRES iteration (ALS sweep, evaluation at
u_bar, windowed least squares with w=20, Moré–Thuente line search, acceptance re-evaluation).
Inputs are synthetic and generated from seeds (there is no dataset); T (512 MB) is larger than
L2 (126 MB), so no L2 flush is needed between steps.

  value  : iterations/s of the device-resident loop, inputs resident in HBM, CUDA-event timed
  e2e    : the same metric through the public C-ABI (cpfit_tensor_create_dense +
           cpfit_ngmres_solve) from pinned host buffers, uploads/downloads inside the timed region
  roofline: the dominant kernel (the fused fiber pass: S = T x1 A, M0 = T W and the per-fiber
           objective on the fp64 tensor cores) timed alone with CUDA events, against the DMMA
           fp64 peak measured in-process; HBM fraction reported beside it
  cpu_baseline: the CPU oracle (restated reference, single-threaded like the reference build)
           on a bounded sample of the same workload

`--impl reference` times the reference's own CPU algorithm (the oracle port; the reference
cannot be compiled here — Eigen3 is absent) on the same config and prints its line.
Multi-GPU (torchrun): one independent solve per rank (different seeds), weak scaling, no
collective on the data path (the reference's parallelism is across independent solves).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c0": dict(dims=(20, 20, 20), rank=3, c=0.5, l1=1.0, l2=1.0),
    "c1": dict(dims=(50, 50, 50), rank=5, c=0.9, l1=10.0, l2=5.0),
    "c2": dict(dims=(400, 400, 400), rank=16, c=0.5, l1=1.0, l2=1.0),
    "c3": dict(dims=(64, 64, 64, 64), rank=10, c=0.7, l1=5.0, l2=0.0),
}
METRIC = "ALS+N-GMRES iters/sec"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        rows = [r for (t, r) in self.rows if (t0 is None or t >= t0 - 0.05) and (t1 is None or t <= t1 + 0.05)]
        if not rows:
            rows = [r for (_, r) in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        smax = max((float(r[1]) for r in rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


def reduce_max(x, dist, device):
    """Max over ranks of a host float (identity without torch.distributed)."""
    if dist is None:
        return float(x)
    import torch
    v = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())


def aggregate(steps, world, ms_max):
    """Whole-job throughput: every rank ran `steps` iterations of its own solve (weak scaling)."""
    return world * steps / (ms_max / 1e3)


def rank_seed(rank):
    """Independent replicas: rank r solves the configuration's problem generated from seed r."""
    return rank


def make_problem(G, cfg, seed):
    """Seeded BASELINE inputs: G is the product package (repo arm) or the oracle module (reference
    arm); both restate proj/core/src/problems.cpp:63-95 / :137-145 with BASELINE's l/100 noise."""
    if hasattr(G, "DataTensor"):
        T, _, _ = G.dense_test_problem(cfg["dims"], cfg["rank"], cfg["c"], cfg["l1"], cfg["l2"], seed, noise_mode=1)
    else:
        T, _ = G.dense_test_problem(cfg["dims"], cfg["rank"], cfg["c"], cfg["l1"], cfg["l2"], seed, 1)
    u0 = G.uniform_initial_guess(cfg["dims"], cfg["rank"], seed)
    return T, u0


def stop_tol(name):
    # BASELINE stopping rule: ||g||_2 / (R sum I_n) < 1e-10 (configs 0-2; 1e-9 for config 3)
    return 1e-9 if name == "c3" else 1e-10


def config_dict(name, cfg, ws):
    """The `config` object both arms print (identical for the same --config and N)."""
    dims = cfg["dims"]
    return {"workload": f"{name}: dense {'x'.join(map(str, dims))} fp64 R={cfg['rank']} c={cfg['c']} "
                        f"l1={cfg['l1']} l2={cfg['l2']} (BASELINE configs[{name[1:]}]); ALS-preconditioned N-GMRES "
                        f"w=20, More-Thuente; consecutive solves from seeded U[0,1] starts (warm-up: seed 0; timed: "
                        f"seeds 1, 2, ...) to ||g||/(R sum I_n) < {stop_tol(name):g}, each solve's init inside the "
                        "timed region",
            "inputs": f"T = {8 * int(np.prod(dims)) / 1e6:.0f} MB" +
                      (" > L2 126 MB (no flush needed)" if 8 * int(np.prod(dims)) > 126e6 else " (L2-resident)"),
            "parallelism": f"{ws} independent replica(s), one solve stream per GPU"}


def cpu_oracle_rate(cfg, T, u0, warmup_iters, iters):
    """Oracle (single-threaded restatement of the reference) iterations/s on the host."""
    from oracle import pyoracle as O
    dims, rank = cfg["dims"], cfg["rank"]
    nu = float(sum(dims) * rank)
    o = O.Tensor.dense(dims, T)
    total = warmup_iters + iters
    res = O.Tensor.ngmres(o, u0, window=20, max_iters=total, tol_grad=1e-300, gradient_scale=nu)
    tr = res["trace"]
    last = len(tr) - 1
    t_a = tr[min(warmup_iters, last)]["time_s"]
    t_b = tr[last]["time_s"]
    n = last - min(warmup_iters, last)
    rate = n / (t_b - t_a) if n > 0 and t_b > t_a else float("nan")
    return rate, n, res


def oracle_solves(O, o, cfg, seeds, total_iters, tol):
    """The repo arm's run_solves on the oracle: consecutive reference-structured solves (init
    included) from seeded starts until total_iters iterations; wall-clock seconds."""
    dims, R = cfg["dims"], cfg["rank"]
    nu = float(sum(dims) * R)
    it, secs, n = 0, 0.0, 0
    while it < total_iters:
        u0 = O.uniform_initial_guess(dims, R, next(seeds))
        t0 = time.perf_counter()
        res = o.ngmres(u0, window=20, max_iters=total_iters - it, tol_grad=tol, gradient_scale=nu)
        secs += time.perf_counter() - t0
        it += len(res["trace"]) - 1
        n += 1
    return it, secs, n


def seed_pool_rate(O, o, cfg, tol, threads, iters_each):
    """The reference's only parallelism (bench.cpp:88-120): independent seed solves on a
    std::thread pool; here `threads` oracle solves of the same tensor at once (ctypes drops the
    GIL), aggregate iterations / wall second."""
    dims, R = cfg["dims"], cfg["rank"]
    nu = float(sum(dims) * R)
    starts = [O.uniform_initial_guess(dims, R, 5_000_000 + i) for i in range(threads)]
    done = [0] * threads

    def work(i):
        r = o.ngmres(starts[i], window=20, max_iters=iters_each, tol_grad=tol, gradient_scale=nu)
        done[i] = len(r["trace"]) - 1

    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return sum(done) / (time.perf_counter() - t0)


def run_reference(args, cfg):
    """--impl reference: the reference's CPU algorithm (the oracle restatement; the reference
    itself cannot be compiled here, Eigen3 is absent) on this arm's config, seeds and start
    sequence: W warm-up iterations of the seed-0 solve, then exactly K timed iterations of
    consecutive solves from seeds 1, 2, ... . Only oracle/ is loaded (no product library)."""
    import itertools

    from oracle import pyoracle as O
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    dims = cfg["dims"]
    tol = stop_tol(args.config)
    T, _ = make_problem(O, cfg, 0)
    o = O.Tensor.dense(dims, T)
    oracle_solves(O, o, cfg, iter([0]), args.warmup, tol)  # warm-up (untimed), seed 0 as the repo arm
    iters, secs, nsolves = oracle_solves(O, o, cfg, itertools.count(1), args.steps, tol)
    rate = iters / secs
    cores = os.cpu_count() or 1
    pool = seed_pool_rate(O, o, cfg, tol, min(cores, 8), 2 if dims[0] >= 200 else 20)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / iters,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, cfg, ws),
        "timed": {"iterations": iters, "solves": nsolves, "seconds": secs},
        "cpu_baseline": {"value": rate, "unit": "iters/s", "cores": 1, "kind": "port",
                         "sample": f"{iters} N-GMRES iterations in {nsolves} solve(s) after {args.warmup} warm-up "
                                   "iterations: oracle/ restatement of proj/core (-O3, no -march, single-threaded "
                                   "like the reference build; one solve has no intra-solve parallelism in the "
                                   "reference); the reference itself is unbuildable here (Eigen3 absent)"},
        "seed_pool": {"threads": min(cores, 8), "host_cores": cores, "iters/s": round(pool, 4),
                      "note": "aggregate of independent oracle solves on a thread pool (bench.cpp:88-120 style)"},
        "e2e": {"value": rate, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_solves(P, solver, dims, R, seeds, total_iters):
    """Consecutive device solves (BASELINE stopping rule), new seeded start each; returns
    (iterations, CUDA-event ms including every solve's init, solves, launches)."""
    it = 0
    ms = 0.0
    n = 0
    l0 = solver.launches()
    while it < total_iters:
        u0 = P.uniform_initial_guess(dims, R, next(seeds))
        ms += solver.restart(u0, total_iters - it)
        st = solver.state()
        if st["stop"] >= 100:
            raise RuntimeError(f"numerical failure in solve: {st}")
        it += st["iters"]
        n += 1
    return it, ms, n, solver.launches() - l0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    ws, rank, local = dist_env()
    if ws > 1:
        os.environ["CUDA_VISIBLE_DEVICES"] = str(local)
    import itertools

    import numpy as np

    import paper_1105_5331_b200 as P
    dist = None
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("nccl")

    def barrier():
        if dist is not None:
            dist.barrier()

    dims, R = cfg["dims"], cfg["rank"]
    nu = sum(dims) * R
    T, u0 = make_problem(P, cfg, rank_seed(rank))
    t = P.DataTensor.dense(T, dims)
    tol = stop_tol(args.config)
    cap = max(args.steps, args.warmup, 2000)
    opts = P.NgmresOptions(window=20, max_iters=cap, tol_grad=tol, gradient_scale=float(nu))
    solver = P.Solver(t, R, opts, 0)
    # seeds for the start points: rank-disjoint streams
    seeds = itertools.count(1_000_000 * rank + 1)
    run_solves(P, solver, dims, R, iter([1_000_000 * rank]), args.warmup)  # warm-up (untimed)
    clocks = ClockSampler(local if ws > 1 else int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
    clocks.start()
    time.sleep(0.3)
    barrier()
    tw0 = time.time()
    iters, ms, nsolves, launches = run_solves(P, solver, dims, R, seeds, args.steps)
    tw1 = time.time()
    barrier()
    ms_max = reduce_max(ms, dist, "cuda")
    value = aggregate(iters, ws, ms_max)

    extras = {}
    roof = None
    if not args.no_extras:
        # dominant kernel of the step: the S pass S = T x1 A0 (sreg_kernel; 1.5 launches per
        # iteration: the ALS sweep's S' and the line search's S_d), timed alone on its stream with
        # CUDA events; HBM-bound (it streams T once). The M0 pass (fiber_ws_kernel) runs as often.
        k_elems = int(np.prod(dims))
        s_ms = P.bench_kernel(t, u0, kind=5, reps=20, flush_l2=False)
        fused_ms = P.bench_kernel(t, u0, kind=3, reps=10, flush_l2=False)
        s_bytes = 8.0 * k_elems + 8.0 * R * dims[0] + 8.0 * R * (k_elems // dims[0])  # T + A0 in, S out
        s_flops = 2.0 * k_elems * R
        dmma_peak, dfma_peak = P.measure_fp64_peak()
        try:
            hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
            hbm_src = "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
        except (OSError, KeyError, ValueError):
            hbm_peak, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
        try:  # DRAM bytes per launch of this kernel from the committed ncu capture (profiles/)
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["s_pass_c2"]
            traffic = tr["bytes_per_launch"] if tuple(dims) == (400, 400, 400) and R == 16 else None
        except (OSError, KeyError, ValueError):
            traffic = None
        gbs = s_bytes / (s_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": "sreg_kernel<16,16> (S = T x1 A0, DMMA fp64 with A0 fragments in registers)",
                "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s", "frac": round(gbs / hbm_peak, 4),
                "traffic": traffic,
                "traffic_source": "profiles/traffic.json (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                "peak_source": hbm_src, "ms_per_launch": round(s_ms, 5), "alg_bytes_per_launch": s_bytes,
                "dmma": {"achieved_tflops": round(s_flops / (s_ms * 1e-3) / 1e12, 3), "peak_tflops": round(dmma_peak, 3),
                         "peak_source": "DMMA m8n8k4 f64 issue loop measured in-process"},
                "fused_pass": {"kernel": "fiber_ws_kernel<16,16> S + M0 + per-fiber f (init / residual phase)",
                               "ms_per_launch": round(fused_ms, 5),
                               "TFLOP/s": round(4.0 * k_elems * R / (fused_ms * 1e-3) / 1e12, 3)},
                "dfma_peak_tflops": round(dfma_peak, 3)}
        kern = {}
        for mode in range(len(dims)):
            mms = P.bench_kernel(t, u0, kind=0, mode=mode, reps=10, flush_l2=True)
            b = 8.0 * k_elems + 8.0 * R * sum(dims)
            kern[f"mttkrp_mode{mode}"] = {"ms": round(mms, 5), "GB/s": round(b / (mms * 1e-3) / 1e9, 1),
                                          "hbm_frac": round(b / (mms * 1e-3) / 1e9 / hbm_peak, 4)}
        # the fused gradient reads T once but contracts it twice (S = T x1 A0 and M0 = T_(0) KR):
        # 4KR flops (+2KR for the residual form) on the fp64 tensor pipe take longer than the
        # 8K bytes take on HBM at R = 16, so it is bounded by the DMMA peak, not by HBM
        for kind, name, fl in ((7, "objective_and_gradient_perfiber_f", 4.0),
                               (1, "objective_and_gradient_residual_f", 6.0)):
            gms = P.bench_kernel(t, u0, kind=kind, reps=10, flush_l2=True)
            b = 8.0 * k_elems + 8.0 * R * 2 * sum(dims)
            flops = fl * k_elems * R
            tf = flops / (gms * 1e-3) / 1e12
            kern[name] = {"ms": round(gms, 5), "GB/s": round(b / (gms * 1e-3) / 1e9, 1),
                          "hbm_frac": round(b / (gms * 1e-3) / 1e9 / hbm_peak, 4),
                          "bound": "fp64 tensor" if flops / (dmma_peak * 1e12) > b / (hbm_peak * 1e9) else "hbm",
                          "TFLOP/s": round(tf, 3), "dmma_frac": round(tf / dmma_peak, 4),
                          "floor_ms": round(max(flops / (dmma_peak * 1e12), b / (hbm_peak * 1e9)) * 1e3, 5)}
        for kind, name in ((4, "fiber_m0_pass_plus_reduce"), (5, "fiber_s_only")):
            fm = P.bench_kernel(t, u0, kind=kind, reps=10, flush_l2=False)
            kern[name] = {"ms": round(fm, 5), "GB/s": round(8.0 * k_elems / (fm * 1e-3) / 1e9, 1),
                          "hbm_frac": round(8.0 * k_elems / (fm * 1e-3) / 1e9 / hbm_peak, 4)}
        extras["kernels"] = kern
        # time to tolerance (the paper's tables are iterations / seconds to a target): one full solve
        # from the seed-1 start; and the rate over 200 iterations of consecutive solves
        ttt_ms = solver.restart(P.uniform_initial_guess(dims, R, 1_000_000 * rank + 1), cap)
        tst = solver.state()
        extras["time_to_tolerance"] = {"iterations": tst["iters"], "stop_reason": tst["stop"], "ms": round(ttt_ms, 4),
                                       "solves/s": round(1e3 / ttt_ms, 3), "f": tst["best_f"],
                                       "note": f"one solve from the seed-1 start to ||g||/(R sum I_n) < {tol:g}, init included"}
        i200, ms200, n200, _ = run_solves(P, solver, dims, R, itertools.count(2_000_000 * (rank + 1)), 200)
        extras["iters_per_s_200"] = {"value": round(i200 / (ms200 * 1e-3), 3), "iterations": i200, "solves": n200,
                                     "ms": round(ms200, 4)}
        # N-CG (ncg.cpp) through the same device loop machinery: 100 iterations from the first
        # start (restart() includes the init's canonicalisation + evaluation)
        ncg = P.Solver(t, R, P.NgmresOptions(max_iters=400, tol_grad=tol, gradient_scale=float(nu)), method=2)
        ncg.restart(u0, 20)
        n_ms = ncg.restart(u0, 100)
        nst = ncg.state()
        # the reference's seed pool (bench.cpp:88-120) on one GPU: independent solves of this
        # tensor in flight together (cpfit_solve_batch); aggregate iterations / s, wall clock
        cstarts = np.stack([P.uniform_initial_guess(dims, R, 7_000_000 + i) for i in range(8)])
        copts = P.NgmresOptions(window=20, max_iters=25, tol_grad=tol, gradient_scale=float(nu))
        conc = {}
        for cc in (1, 4):
            P.solve_batch(t, cstarts[:cc], copts, 0, cc)
            tc0 = time.perf_counter()
            bb = P.solve_batch(t, cstarts, copts, 0, cc)
            conc[f"in_flight_{cc}"] = round(float(bb.iters.sum()) / (time.perf_counter() - tc0), 1)
        extras["concurrent_solves"] = {"iters/s": conc, "solves": 8, "iters_each": 25,
                                       "note": "aggregate over independent solves of the same tensor (seed sweep)"}
        extras["ncg"] = {"iters/s": round(nst["iters"] / (n_ms * 1e-3), 1), "iters": nst["iters"],
                         "fevals": nst["fevals"], "ms": round(n_ms, 3),
                         "note": "device N-CG (Polak-Ribiere+, More-Thuente on the exact line polynomial for dense order 3, trial evaluations otherwise), init included"}
        if ws == 1:
            # the other BASELINE configs that carry a throughput: config 3 (dense 64^4, R = 10, one solve
            # to ||g|| / (R sum I_n) < 1e-9) and config 4 (sparse 10000^3, 10M nnz, R = 10, 100
            # iterations); CUDA-event time of the graph-launched solve, second run
            oc = {}
            try:
                c3 = CONFIGS["c3"]
                T3, u3 = make_problem(P, c3, 0)
                t3 = P.DataTensor.dense(T3, c3["dims"])
                nu3 = float(sum(c3["dims"]) * c3["rank"])
                s3 = P.Solver(t3, c3["rank"], P.NgmresOptions(window=20, max_iters=1000, tol_grad=stop_tol("c3"),
                                                               gradient_scale=nu3), 0)
                s3.restart(u3, 1000)
                ms3 = s3.restart(u3, 1000)
                st3 = s3.state()
                oc["c3"] = {"iters/s": round(st3["iters"] / (ms3 * 1e-3), 1), "iterations": st3["iters"],
                            "stop_reason": st3["stop"], "ms": round(ms3, 3), "f": st3["f"]}
                s3.close()
                del t3, T3
                dims4, R4 = (10000, 10000, 10000), 10
                co4, va4, _ = P.random_sparse_problem(dims4, 10_000_000, R4, 0.01, 0)
                t4 = P.DataTensor.coo(dims4, co4, va4)
                u4 = P.uniform_initial_guess(dims4, R4, 0)
                s4 = P.Solver(t4, R4, P.NgmresOptions(window=20, max_iters=100, tol_grad=1e-300,
                                                       gradient_scale=float(sum(dims4) * R4)), 0)
                s4.restart(u4, 100)
                ms4 = s4.restart(u4, 100)
                st4 = s4.state()
                oc["c4"] = {"iters/s": round(st4["iters"] / (ms4 * 1e-3), 1), "iterations": st4["iters"],
                            "ms": round(ms4, 3), "f": st4["f"]}
                del t4, co4, va4
            except Exception as e:  # the headline line must still print
                oc["error"] = str(e)[:200]
            extras["other_configs"] = oc

    # end to end through the public C-ABI from pinned host buffers: tensor upload + solves
    T_pin = np.ascontiguousarray(T)
    P.host_register(T_pin)
    e_seeds = itertools.count(1_000_000 * rank + 1)
    starts = [np.ascontiguousarray(P.uniform_initial_guess(dims, R, next(e_seeds))) for _ in range(64)]
    for s in starts:
        P.host_register(s)
    # one untimed cycle of the same calls first (W warm-up steps of the e2e leg): first-touch
    # costs of this process (device memory pool growth, lazily loaded modules) stay out of the
    # timed region; the timed region still builds the new tensor handle's graphs
    tw = P.DataTensor.dense(T_pin, dims)
    P.ngmres_solve(tw, starts[-1], P.NgmresOptions(window=20, max_iters=max(args.warmup, 3), tol_grad=tol,
                                                   gradient_scale=float(nu)))
    tw.close()  # parked (capi.cu tensor pool): the timed handle below takes over its buffers and graphs
    barrier()
    te0 = time.perf_counter()
    te = P.DataTensor.dense(T_pin, dims)
    e_it, e_solves, d2h = 0, 0, 0
    while e_it < args.steps:
        res = P.ngmres_solve(te, starts[e_solves % len(starts)],
                             P.NgmresOptions(window=20, max_iters=args.steps - e_it, tol_grad=tol,
                                             gradient_scale=float(nu)))
        e_it += len(res.trace) - 1
        e_solves += 1
        d2h += res.solution.nbytes + len(res.trace) * 72 + 8
    te1 = time.perf_counter()
    barrier()
    te.close()
    P.host_unregister(T_pin)
    for s in starts:
        P.host_unregister(s)
    e2e_s = reduce_max(te1 - te0, dist, "cuda")
    e2e_value = aggregate(e_it, ws, e2e_s * 1e3)
    h2d = T_pin.nbytes + e_solves * starts[0].nbytes

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, n, _ = cpu_oracle_rate(cfg, T, u0, 1, 2 if dims[0] >= 200 else 10)
        cpu = {"value": rate, "unit": "iters/s", "cores": 1, "kind": "port",
               "sample": f"{n} N-GMRES iterations (2..{n + 1}) of the seed-0 solve, CPU oracle "
                         "(restated proj/core, -O3, single-threaded like the reference build)"}
    clocks.stop()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / iters, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, cfg, ws),
            "timed": {"iterations": iters, "solves": nsolves, "ms": round(ms_max, 4)},
            "e2e": {"value": round(e2e_value, 3), "unit": "iters/s", "h2d_bytes_per_step": h2d // max(e_it, 1),
                    "d2h_bytes_per_step": d2h // max(e_it, 1),
                    "note": f"cpfit_tensor_create_dense + {e_solves} cpfit_ngmres_solve calls from pinned host "
                            "buffers (graphs built on the first call, cached on the tensor handle), wall clock"},
            "gpu_launches": launches,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(tw0, tw1),
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
