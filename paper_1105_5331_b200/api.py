"""Python host mirror of the reference solver API over the C-ABI (include/cpfit_gpu.h).

Names, argument meaning and error behaviour follow proj/core/include/cpfit/*.hpp:
``DataTensor`` (tensor.hpp:129-148), ``mttkrp`` (tensor.hpp:119-120), ``gram_hadamard``
(tensor.hpp:124), ``objective`` / ``objective_and_gradient`` / ``normalize_and_reorder`` /
``pack`` / ``unpack`` (kruskal.hpp:29-58), ``als_sweep`` / ``als_solve`` (als.hpp:14,23),
``accelerate`` / ``ngmres_solve`` (ngmres.hpp:44-127), ``ncg_solve`` (ncg.hpp:29),
``more_thuente`` (line_search.hpp:41).
std::invalid_argument -> ValueError, cpfit::numerical_error -> NumericalError.

All compute goes through libcpfit_gpu.so (sm_100a kernels). There is no CPU fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPFIT_GPU_LIB") or os.path.join(_HERE, "lib", "libcpfit_gpu.so")  # override: A/B builds


class NumericalError(RuntimeError):
    """cpfit::numerical_error (errors.hpp:9-12)."""


class CudaError(RuntimeError):
    pass


class CpfitIOError(OSError):
    """cpfit::io_error (errors.hpp:15-18): file and parse failures naming the file and line."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    return C.CDLL(LIB_PATH)


lib = _load()

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class TraceRow(C.Structure):
    _fields_ = [("iter", C.c_int32), ("restart", C.c_int32), ("time_s", C.c_double), ("f", C.c_double),
                ("h", C.c_double), ("gnorm_rel", C.c_double), ("beta", C.c_double), ("fevals", C.c_int64),
                ("gevals", C.c_int64), ("precond_calls", C.c_int64)]


class NgmresOptionsC(C.Structure):
    _fields_ = [("window", C.c_int32), ("max_iters", C.c_int32), ("epsilon_reg", C.c_double),
                ("tol_grad", C.c_double), ("gradient_scale", C.c_double), ("ftol", C.c_double),
                ("gtol", C.c_double), ("initial_step", C.c_double), ("max_evals", C.c_int32),
                ("restart_on_ascent", C.c_int32), ("step_min", C.c_double), ("step_max", C.c_double),
                ("reeval_accepted", C.c_int32), ("residual_objective", C.c_int32)]


class LsParamsC(C.Structure):
    _fields_ = [("ftol", C.c_double), ("gtol", C.c_double), ("initial_step", C.c_double),
                ("max_evals", C.c_int32), ("step_min", C.c_double), ("step_max", C.c_double)]


class LsResultC(C.Structure):
    _fields_ = [("step", C.c_double), ("f", C.c_double), ("dg", C.c_double), ("status", C.c_int32),
                ("evals", C.c_int32)]


PHI_FN = C.CFUNCTYPE(None, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)

# symbol table: name -> (restype, argtypes)
_SIGS = {
    "cpfit_last_error": (C.c_char_p, []),
    "cpfit_device_count": (C.c_int, []),
    "cpfit_tensor_create_dense": (C.c_int, [C.c_int, _i64p, _f64p, C.POINTER(C.c_void_p)]),
    "cpfit_tensor_create_coo": (C.c_int, [C.c_int, _i64p, C.c_int64, _i64p, _f64p, C.POINTER(C.c_void_p)]),
    "cpfit_tensor_destroy": (C.c_int, [C.c_void_p]),
    "cpfit_tensor_norm": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "cpfit_tensor_nnz": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "cpfit_mttkrp": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_int, _f64p]),
    "cpfit_objective": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.POINTER(C.c_double)]),
    "cpfit_objective_and_gradient": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _f64p, C.POINTER(C.c_double)]),
    "cpfit_objective_and_gradient_form": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_int, _f64p,
                                                    C.POINTER(C.c_double)]),
    "cpfit_gram_hadamard": (C.c_int, [C.c_int, _i64p, C.c_int64, _f64p, C.c_int, _f64p]),
    "cpfit_normalize_and_reorder": (C.c_int, [C.c_int, _i64p, C.c_int64, _f64p, _f64p]),
    "cpfit_als_sweep": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _f64p]),
    "cpfit_accelerate": (C.c_int, [C.c_int64, C.c_int64, _f64p, _f64p, _f64p, _f64p, C.c_double, _f64p, _f64p,
                                   C.POINTER(C.c_double)]),
    "cpfit_more_thuente": (C.c_int, [PHI_FN, C.c_void_p, C.c_double, C.c_double, C.POINTER(LsParamsC),
                                     C.POINTER(LsResultC)]),
    "cpfit_ngmres_solve": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.POINTER(NgmresOptionsC), _f64p,
                                     C.POINTER(C.c_double), C.POINTER(TraceRow), C.c_int64, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int)]),
    "cpfit_als_solve": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_double, C.c_int, _f64p, C.POINTER(C.c_double),
                                  C.POINTER(TraceRow), C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "cpfit_ncg_solve": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_double, C.c_int, C.POINTER(LsParamsC), _f64p,
                                  C.POINTER(C.c_double), C.POINTER(TraceRow), C.c_int64, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int)]),
    "cpfit_solve_batch": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int64, _f64p, C.POINTER(NgmresOptionsC), C.c_int,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cpfit_solver_create": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(NgmresOptionsC), C.c_int,
                                      C.POINTER(C.c_void_p)]),
    "cpfit_solver_set_initial": (C.c_int, [C.c_void_p, _f64p]),
    "cpfit_solver_init": (C.c_int, [C.c_void_p]),
    "cpfit_solver_run": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_float)]),
    "cpfit_solver_restart": (C.c_int, [C.c_void_p, _f64p, C.c_int, C.POINTER(C.c_float)]),
    "cpfit_solver_state": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "cpfit_solver_trace": (C.c_int, [C.c_void_p, C.POINTER(TraceRow), C.c_int64]),
    "cpfit_solver_best": (C.c_int, [C.c_void_p, _f64p]),
    "cpfit_solver_iterate": (C.c_int, [C.c_void_p, _f64p]),
    "cpfit_ngmres_init": (C.c_int, [C.c_void_p, _f64p, C.POINTER(C.c_double)]),
    "cpfit_ngmres_step": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]),
    "cpfit_solver_launches": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "cpfit_line_polynomial": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _f64p, _f64p, C.c_int64, _f64p, _f64p]),
    "cpfit_solver_phase_times": (C.c_int, [C.c_void_p, _f64p, C.POINTER(C.c_int64)]),
    "cpfit_debug_guard_check": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "cpfit_measure_fp64_peak": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "cpfit_host_register": (C.c_int, [C.c_void_p, C.c_int64]),
    "cpfit_host_unregister": (C.c_int, [C.c_void_p]),
    "cpfit_default_ngmres_options": (None, [C.POINTER(NgmresOptionsC)]),
    "cpfit_solver_destroy": (C.c_int, [C.c_void_p]),
    "cpfit_bench_kernel": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_float)]),
    # io (host, include/cpfit_io.h)
    "cpfit_io_last_error": (C.c_char_p, []),
    "cpfit_format_double": (C.c_int, [C.c_double, C.c_char_p, C.c_int]),
    "cpfit_tns_read": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), _i64p, C.POINTER(C.c_int64), C.c_void_p,
                                 C.c_void_p, C.c_int64, C.POINTER(C.c_int)]),
    "cpfit_tns_read_dense": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), _i64p, C.POINTER(C.c_int64),
                                       C.c_void_p, C.c_int64]),
    "cpfit_tns_write": (C.c_int, [C.c_char_p, C.c_int, _i64p, C.c_int64, _i64p, _f64p]),
    "cpfit_tns_write_dense": (C.c_int, [C.c_char_p, C.c_int, _i64p, _f64p]),
    # problems (host)
    "cpfit_problems_last_error": (C.c_char_p, []),
    "cpfit_rng_draws": (C.c_int, [C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cpfit_rng_mix": (C.c_uint64, [C.c_uint64]),
    "cpfit_collinear_factors": (C.c_int, [C.c_int, _i64p, C.c_int64, C.c_double, C.c_uint64, _f64p]),
    "cpfit_full": (C.c_int, [C.c_int, _i64p, C.c_int64, _f64p, _f64p]),
    "cpfit_dense_test_problem": (C.c_int, [C.c_int, _i64p, C.c_int64, C.c_double, C.c_double, C.c_double,
                                           C.c_uint64, C.c_int, _f64p, C.c_void_p, C.c_void_p]),
    "cpfit_uniform_initial_guess": (C.c_int, [C.c_int, _i64p, C.c_int64, C.c_uint64, _f64p]),
    "cpfit_laplacian_tensor": (C.c_int, [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "cpfit_random_sparse_problem": (C.c_int, [C.c_int, _i64p, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                              _i64p, _f64p, C.c_void_p]),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED_SYMBOLS = sorted(_SIGS)


def _check(rc: int, problems: bool = False, io: bool = False):
    if rc == 0:
        return
    err = lib.cpfit_io_last_error if io else (lib.cpfit_problems_last_error if problems else lib.cpfit_last_error)
    msg = err().decode(errors="replace")
    if rc == 4:
        raise CpfitIOError(msg)
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise NumericalError(msg)
    raise CudaError(msg)


def device_count() -> int:
    return int(lib.cpfit_device_count())


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _dims(d) -> np.ndarray:
    return np.ascontiguousarray(d, dtype=np.int64)


def _vec(x, n: int, what: str) -> np.ndarray:
    """Contiguous float64 vector of exactly n entries (the C side reads and writes n doubles);
    kruskal.cpp:208-209 unpack() rejects other lengths the same way."""
    x = _f64(x).reshape(-1)
    if x.size != n:
        raise ValueError(f"{what}: vector length does not match shape and rank")
    return x


def _packed_len(dims, rank) -> int:
    if rank < 1:
        raise ValueError("KruskalTensor: rank must be >= 1")
    return int(sum(int(d) for d in dims)) * int(rank)


# ---- pack / unpack (kruskal.cpp:195-221) ---------------------------------------------------

def pack(factors) -> np.ndarray:
    return np.concatenate([np.asarray(a, dtype=np.float64).reshape(-1, order="F") for a in factors])


def unpack(u, dims, rank):
    u = _f64(u)
    total = sum(int(d) * rank for d in dims)
    if u.size != total:
        raise ValueError("unpack: vector length does not match shape and rank")
    out, at = [], 0
    for d in dims:
        out.append(u[at:at + d * rank].reshape((d, rank), order="F"))
        at += d * rank
    return out


# ---- tensors --------------------------------------------------------------------------------

class DataTensor:
    """Device-resident DataTensor (tensor.hpp:129-148). T is uploaded once (dense values in
    first-mode-fastest order, or COO with nnz x N int64 coordinates)."""

    def __init__(self, handle, dims, sparse):
        self._h = handle
        self.dims = tuple(int(d) for d in dims)
        self.order = len(self.dims)
        self.is_sparse = sparse

    @classmethod
    def dense(cls, values, dims=None):
        values = np.asarray(values, dtype=np.float64)
        if dims is None:
            dims = values.shape
            flat = np.ascontiguousarray(values.reshape(-1, order="F"))
        else:
            flat = _f64(values).reshape(-1)
        dims = _dims(dims)
        if flat.size != int(np.prod(dims)):
            raise ValueError("DenseTensor: value count does not match shape")
        h = C.c_void_p()
        _check(lib.cpfit_tensor_create_dense(len(dims), dims, flat, C.byref(h)))
        return cls(h, dims, False)

    @classmethod
    def coo(cls, dims, coords, values):
        dims = _dims(dims)
        coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1)
        values = _f64(values).reshape(-1)
        if coords.size != values.size * len(dims):
            raise ValueError("SparseTensor: coords/values size mismatch")
        h = C.c_void_p()
        _check(lib.cpfit_tensor_create_coo(len(dims), dims, values.size, coords, values, C.byref(h)))
        return cls(h, dims, True)

    def close(self):
        if self._h:
            lib.cpfit_tensor_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def norm(self) -> float:
        v = C.c_double()
        _check(lib.cpfit_tensor_norm(self._h, C.byref(v)))
        return v.value

    def nnz(self) -> int:
        v = C.c_int64()
        _check(lib.cpfit_tensor_nnz(self._h, C.byref(v)))
        return v.value

    def nu(self, rank):
        return sum(d * rank for d in self.dims)

    def _rank(self, u):
        u = _f64(u)
        s = sum(self.dims)
        if u.size % s:
            raise ValueError("tensor and Kruskal model shapes must match")
        return u, u.size // s

    def mttkrp(self, u, mode):
        u, r = self._rank(u)
        if not 0 <= mode < self.order:
            raise ValueError("mttkrp: mode out of range")
        out = np.empty(self.dims[mode] * r)
        _check(lib.cpfit_mttkrp(self._h, r, u, mode, out))
        return out.reshape((self.dims[mode], r), order="F")


def mttkrp(t: DataTensor, u, mode):
    return t.mttkrp(u, mode)


def objective(t: DataTensor, u) -> float:
    u, r = t._rank(u)
    f = C.c_double()
    _check(lib.cpfit_objective(t._h, r, u, C.byref(f)))
    return f.value


def objective_and_gradient(t: DataTensor, u):
    u, r = t._rank(u)
    g = np.empty(u.size)
    f = C.c_double()
    _check(lib.cpfit_objective_and_gradient(t._h, r, u, g, C.byref(f)))
    return f.value, g


def objective_and_gradient_form(t: DataTensor, u, form: int):
    """form 0: the reference's residual objective (= objective_and_gradient); form 1: the
    per-fibre three-term objective the device solver loop evaluates with (dense tensors)."""
    u, r = t._rank(u)
    g = np.empty(u.size)
    f = C.c_double()
    _check(lib.cpfit_objective_and_gradient_form(t._h, r, u, int(form), g, C.byref(f)))
    return f.value, g


def gradient(t, u):
    return objective_and_gradient(t, u)[1]


def line_polynomial(t: DataTensor, u_bar, d, alphas):
    """(phi, dphi) at alphas from the device line-search polynomial (dense order 3)."""
    ub, r = t._rank(u_bar)
    dv = _vec(d, ub.size, "line_polynomial")
    al = _f64(alphas)
    phi, dphi = np.zeros(al.size), np.zeros(al.size)
    _check(lib.cpfit_line_polynomial(t._h, r, ub, dv, al if al.size else np.zeros(1), al.size, phi, dphi))
    return phi, dphi


def fit_h(t: DataTensor, u) -> float:
    n = t.norm()
    if not n > 0.0:
        raise ValueError("fit_h: data tensor must be nonzero")
    return float(np.sqrt(max(2.0 * objective(t, u), 0.0)) / n)


def gram_hadamard(dims, rank, u, skip=-1):
    dims = _dims(dims)
    u = _vec(u, _packed_len(dims, rank), "gram_hadamard")
    out = np.empty(rank * rank)
    _check(lib.cpfit_gram_hadamard(len(dims), dims, rank, u, skip, out))
    return out.reshape((rank, rank), order="F")


def normalize_and_reorder(dims, rank, u):
    dims = _dims(dims)
    u = _vec(u, _packed_len(dims, rank), "normalize_and_reorder")
    out = np.empty_like(u)
    _check(lib.cpfit_normalize_and_reorder(len(dims), dims, rank, u, out))
    return out


def als_sweep(t: DataTensor, u):
    u, r = t._rank(u)
    out = np.empty_like(u)
    _check(lib.cpfit_als_sweep(t._h, r, u, out))
    return out


@dataclass
class AccelOutcome:
    u_hat: np.ndarray
    alpha: np.ndarray
    system_residual_rel: float


def accelerate(window_u, window_g, u_bar, g_bar, epsilon_reg=1e-12) -> AccelOutcome:
    """accelerate(window, u_bar, g_bar, eps) — window lists oldest first (ngmres.hpp:44)."""
    wu = np.ascontiguousarray(np.asarray(window_u, dtype=np.float64).reshape(len(window_u), -1))
    wg = np.ascontiguousarray(np.asarray(window_g, dtype=np.float64).reshape(len(window_g), -1))
    m, n = wu.shape
    if wg.shape != wu.shape:
        raise ValueError("accelerate: window iterates and gradients must have the same shape")
    u_bar = _vec(u_bar, n, "accelerate")
    g_bar = _vec(g_bar, n, "accelerate")
    uh = np.empty(n)
    al = np.empty(max(m, 1))
    rr = C.c_double()
    _check(lib.cpfit_accelerate(n, m, wu.reshape(-1), wg.reshape(-1), u_bar, g_bar, epsilon_reg, uh, al,
                                C.byref(rr)))
    return AccelOutcome(uh, al[:m], rr.value)


# ---- line search ----------------------------------------------------------------------------

CONVERGED, MAX_EVALS, NOT_DESCENT, NUMERICAL_STALL = 0, 1, 2, 3


@dataclass
class LineSearchParams:
    ftol: float = 1e-4
    gtol: float = 1e-2
    initial_step: float = 1.0
    max_evals: int = 20
    step_min: float = 0.0
    step_max: float = 1e20


@dataclass
class LineSearchResult:
    step: float
    f: float
    dg: float
    status: int
    evals: int


def more_thuente(phi, phi0, dphi0, params: LineSearchParams = None) -> LineSearchResult:
    """phi(step) -> (f, dg). Same state machine the device line search runs."""
    p = params or LineSearchParams()
    err = []

    def cb(step, fp, gp, _ctx):
        try:
            f, g = phi(step)
            fp[0] = f
            gp[0] = g
        except Exception as e:  # pragma: no cover
            err.append(e)
            fp[0] = float("nan")
            gp[0] = float("nan")

    fn = PHI_FN(cb)
    cp = LsParamsC(p.ftol, p.gtol, p.initial_step, p.max_evals, p.step_min, p.step_max)
    out = LsResultC()
    _check(lib.cpfit_more_thuente(fn, None, phi0, dphi0, C.byref(cp), C.byref(out)))
    if err:
        raise err[0]
    return LineSearchResult(out.step, out.f, out.dg, out.status, out.evals)


# ---- solvers --------------------------------------------------------------------------------

GRAD_TOL, MAX_ITERS, STALLED = 0, 1, 2


@dataclass
class NgmresOptions:
    window: int = 20
    epsilon_reg: float = 1e-12
    tol_grad: float = 1e-9
    max_iters: int = 2000
    line_search: LineSearchParams = field(default_factory=LineSearchParams)
    restart_on_ascent: bool = True
    gradient_scale: float = 0.0  # <= 0: ||T||_F as in ngmres_solve
    reeval_accepted: bool = False  # True: the reference's extra evaluation after acceptance
    residual_objective: bool = False  # True: residual-form f for every evaluation

    def c(self):
        ls = self.line_search
        return NgmresOptionsC(self.window, self.max_iters, self.epsilon_reg, self.tol_grad, self.gradient_scale,
                              ls.ftol, ls.gtol, ls.initial_step, ls.max_evals, int(self.restart_on_ascent),
                              ls.step_min, ls.step_max, int(self.reeval_accepted), int(self.residual_objective))


@dataclass
class SolveResult:
    solution: np.ndarray  # best-f iterate, pack layout
    f: float
    trace: list
    stop_reason: int


def _trace_list(buf, rows):
    return [dict(iter=r.iter, time_s=r.time_s, f=r.f, h=r.h, gnorm_rel=r.gnorm_rel, fevals=r.fevals,
                 gevals=r.gevals, precond_calls=r.precond_calls, restart=bool(r.restart), beta=r.beta)
            for r in buf[:rows]]


def ngmres_solve(t: DataTensor, u0, opts: NgmresOptions = None) -> SolveResult:
    o = opts or NgmresOptions()
    u0, r = t._rank(u0)
    cap = o.max_iters + 1
    trace = (TraceRow * cap)()
    ub = np.empty_like(u0)
    fb = C.c_double()
    rows = C.c_int64()
    stop = C.c_int()
    oc = o.c()
    _check(lib.cpfit_ngmres_solve(t._h, r, u0, C.byref(oc), ub, C.byref(fb), trace, cap, C.byref(rows),
                                  C.byref(stop)))
    return SolveResult(ub, fb.value, _trace_list(trace, rows.value), stop.value)


def als_solve(t: DataTensor, u0, tol_grad=1e-9, max_iters=2000) -> SolveResult:
    u0, r = t._rank(u0)
    cap = max_iters + 1
    trace = (TraceRow * cap)()
    ub = np.empty_like(u0)
    fb = C.c_double()
    rows = C.c_int64()
    stop = C.c_int()
    _check(lib.cpfit_als_solve(t._h, r, u0, tol_grad, max_iters, ub, C.byref(fb), trace, cap, C.byref(rows),
                               C.byref(stop)))
    return SolveResult(ub, fb.value, _trace_list(trace, rows.value), stop.value)


@dataclass
class NcgOptions:
    """ncg.hpp:14-18"""
    tol_grad: float = 1e-9
    max_iters: int = 2000
    line_search: LineSearchParams = field(default_factory=LineSearchParams)


def ncg_solve(t: DataTensor, u0, opts: NcgOptions = None) -> SolveResult:
    """ncg_solve (ncg.hpp:29, ncg.cpp:111-122): N-CG on the CP objective, device resident.
    Stalled iterations write no trace row (ncg.cpp:60-67)."""
    o = opts or NcgOptions()
    u0, r = t._rank(u0)
    cap = o.max_iters + 1
    trace = (TraceRow * cap)()
    ub = np.empty_like(u0)
    fb = C.c_double()
    rows = C.c_int64()
    stop = C.c_int()
    ls = o.line_search
    cp = LsParamsC(ls.ftol, ls.gtol, ls.initial_step, ls.max_evals, ls.step_min, ls.step_max)
    _check(lib.cpfit_ncg_solve(t._h, r, u0, o.tol_grad, o.max_iters, C.byref(cp), ub, C.byref(fb), trace, cap,
                               C.byref(rows), C.byref(stop)))
    return SolveResult(ub, fb.value, _trace_list(trace, rows.value), stop.value)


@dataclass
class BatchResult:
    solutions: np.ndarray  # nsolves x n best iterates
    f: np.ndarray
    iters: np.ndarray
    stop_reason: np.ndarray
    fevals: np.ndarray


def solve_batch(t: DataTensor, u0s, opts: NgmresOptions = None, method: int = 0, concurrency: int = 16) -> BatchResult:
    """Independent solves of t from each row of u0s, `concurrency` at a time on their own streams
    (the reference's seed sweeps, bench.cpp:80-158). method 0 N-GMRES, 1 ALS, 2 N-CG."""
    o = opts or NgmresOptions()
    u0s = np.ascontiguousarray(np.atleast_2d(np.asarray(u0s, dtype=np.float64)))
    ns, n = u0s.shape
    _, r = t._rank(u0s[0])
    ub = np.empty((ns, n))
    fb = np.empty(ns)
    it = np.empty(ns, dtype=np.int32)
    st = np.empty(ns, dtype=np.int32)
    fe = np.empty(ns, dtype=np.int64)
    oc = o.c()
    _check(lib.cpfit_solve_batch(t._h, r, method, ns, u0s.reshape(-1), C.byref(oc), concurrency,
                                 ub.ctypes.data, fb.ctypes.data, it.ctypes.data, st.ctypes.data, fe.ctypes.data))
    return BatchResult(ub, fb, it, st, fe)


class Solver:
    """Persistent device solver (measurement surface): init once, then timed loop launches."""

    def __init__(self, t: DataTensor, rank: int, opts: NgmresOptions, method: int = 0):
        self.t = t
        h = C.c_void_p()
        oc = opts.c()
        _check(lib.cpfit_solver_create(t._h, rank, C.byref(oc), method, C.byref(h)))
        self._h = h
        self.rank = rank
        self.max_iters = opts.max_iters

    def set_initial(self, u0):
        _check(lib.cpfit_solver_set_initial(self._h, _vec(u0, self.t.nu(self.rank), "Solver.set_initial")))

    def init(self):
        _check(lib.cpfit_solver_init(self._h))

    def run(self, max_iters_total) -> float:
        ms = C.c_float()
        _check(lib.cpfit_solver_run(self._h, int(max_iters_total), C.byref(ms)))
        return ms.value

    def restart(self, u0, max_iters_total) -> float:
        """New start point + init + loop; CUDA-event ms for init + loop."""
        ms = C.c_float()
        u0 = _vec(u0, self.t.nu(self.rank), "Solver.restart")
        _check(lib.cpfit_solver_restart(self._h, u0, int(max_iters_total), C.byref(ms)))
        return ms.value

    def state(self):
        it, st, fe = C.c_int(), C.c_int(), C.c_int64()
        f, bf = C.c_double(), C.c_double()
        _check(lib.cpfit_solver_state(self._h, C.byref(it), C.byref(st), C.byref(f), C.byref(bf), C.byref(fe)))
        return dict(iters=it.value, stop=st.value, f=f.value, best_f=bf.value, fevals=fe.value)

    def trace(self, rows):
        if not 0 <= rows <= self.max_iters + 1:
            raise ValueError("Solver.trace: rows must be in [0, max_iters + 1]")
        buf = (TraceRow * max(rows, 1))()
        _check(lib.cpfit_solver_trace(self._h, buf, rows))
        return _trace_list(buf, rows)

    def best(self):
        out = np.empty(self.t.nu(self.rank))
        _check(lib.cpfit_solver_best(self._h, out))
        return out

    def iterate(self):
        out = np.empty(self.t.nu(self.rank))
        _check(lib.cpfit_solver_iterate(self._h, out))
        return out

    def ngmres_init(self, u0) -> float:
        """ngmres_init (ngmres.hpp:101-103): canonicalize, evaluate, seed the window; returns f."""
        f = C.c_double()
        _check(lib.cpfit_ngmres_init(self._h, _vec(u0, self.t.nu(self.rank), "ngmres_init"), C.byref(f)))
        return f.value

    def ngmres_step(self):
        """ngmres_step (ngmres.hpp:109-117): one iteration; the NgmresStepReport and f."""
        rs, st, b, f = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        _check(lib.cpfit_ngmres_step(self._h, C.byref(rs), C.byref(st), C.byref(b), C.byref(f)))
        return dict(restart=bool(rs.value), stalled=bool(st.value), beta=b.value, f=f.value)

    def launches(self) -> int:
        n = C.c_int64()
        _check(lib.cpfit_solver_launches(self._h, C.byref(n)))
        return n.value

    PHASES = ("als_sweep", "eval_bar", "accel_ls_init", "ls_trial_eval", "ls_update", "accepted_step", "commit",
              "loop_reentry")

    def phase_times(self):
        """{phase: (us, visits)} — needs CPFIT_PHASE_PROFILE=1 before the Solver is created."""
        us = np.zeros(8)
        cnt = (C.c_int64 * 8)()
        _check(lib.cpfit_solver_phase_times(self._h, us, cnt))
        return {k: (float(us[i]), int(cnt[i])) for i, k in enumerate(self.PHASES)}

    def close(self):
        if self._h:
            lib.cpfit_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def debug_guard_check():
    """(violations, live allocations) of the guard-band build (make guard; CPFIT_GPU_LIB pointing
    at libcpfit_gpu_guard.so); violations = -1 for a normal build."""
    v, n = C.c_int64(), C.c_int64()
    _check(lib.cpfit_debug_guard_check(C.byref(v), C.byref(n)))
    return v.value, n.value


def measure_fp64_peak():
    """(DMMA TFLOP/s, DFMA TFLOP/s) measured on the current device."""
    a, b = C.c_double(), C.c_double()
    _check(lib.cpfit_measure_fp64_peak(C.byref(a), C.byref(b)))
    return a.value, b.value


def host_register(arr: np.ndarray):
    _check(lib.cpfit_host_register(arr.ctypes.data, arr.nbytes))


def host_unregister(arr: np.ndarray):
    _check(lib.cpfit_host_unregister(arr.ctypes.data))


def bench_kernel(t: DataTensor, u, kind: int, mode: int = 0, reps: int = 10, flush_l2: bool = True) -> float:
    u, r = t._rank(u)
    ms = C.c_float()
    _check(lib.cpfit_bench_kernel(t._h, r, u, kind, mode, reps, int(flush_l2), C.byref(ms)))
    return ms.value


# ---- .tns files (io.hpp:14-30; host, multi-threaded) -----------------------------------------

def format_double(x: float) -> str:
    """format_double (io.cpp:15-19): shortest round-trip decimal form."""
    buf = C.create_string_buffer(64)
    _check(lib.cpfit_format_double(float(x), buf, 64), io=True)
    return buf.value.decode()


def read_tns(path, sidecar: int = 1):
    """read_tns_file (io.hpp:27): (dims, coords nnz x N 0-based, values) in file order.
    sidecar 0: text only; 1: use <path>.cpfbin when it matches the file; 2: also write it."""
    order = C.c_int()
    dims = np.zeros(8, dtype=np.int64)
    nnz = C.c_int64()
    p = str(path).encode()
    # header (or a matching sidecar's header) first; the body call below parses / writes the sidecar
    _check(lib.cpfit_tns_read(p, min(int(sidecar), 1), C.byref(order), dims, C.byref(nnz), None, None, 0, None),
           io=True)
    n, k = order.value, nnz.value
    coords = np.empty((max(k, 1), n), dtype=np.int64)
    vals = np.empty(max(k, 1))
    used = C.c_int()
    _check(lib.cpfit_tns_read(p, int(sidecar), C.byref(order), dims, C.byref(nnz), coords.ctypes.data,
                              vals.ctypes.data, max(k, 1), C.byref(used)), io=True)
    read_tns.last_from_sidecar = bool(used.value)
    return tuple(int(d) for d in dims[:n]), coords[:k], vals[:k]


def read_tns_dense(path, sidecar: int = 1):
    """read_tns_dense_file (io.hpp:30): (dims, values first-mode-fastest)."""
    order = C.c_int()
    dims = np.zeros(8, dtype=np.int64)
    K = C.c_int64()
    p = str(path).encode()
    _check(lib.cpfit_tns_read_dense(p, int(sidecar), C.byref(order), dims, C.byref(K), None, 0), io=True)
    vals = np.empty(max(K.value, 1))
    _check(lib.cpfit_tns_read_dense(p, int(sidecar), C.byref(order), dims, C.byref(K), vals.ctypes.data, K.value),
           io=True)
    return tuple(int(d) for d in dims[:order.value]), vals[:K.value]


def write_tns(path, dims, coords, values):
    """write_tns_file(SparseTensor) (io.hpp:24): entries as given (1-based on disk)."""
    dims = _dims(dims)
    values = _f64(values).reshape(-1)
    coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1)
    if coords.size != values.size * len(dims):
        raise ValueError("SparseTensor: coords/values size mismatch")
    _check(lib.cpfit_tns_write(str(path).encode(), len(dims), dims, values.size, coords, values), io=True)


def write_tns_dense(path, values, dims=None):
    """write_tns_file(DenseTensor) (io.hpp:25)."""
    values = np.asarray(values, dtype=np.float64)
    if dims is None:
        dims = values.shape
        values = values.reshape(-1, order="F")
    dims = _dims(dims)
    flat = _vec(values, int(np.prod(dims)), "write_tns_dense")
    _check(lib.cpfit_tns_write_dense(str(path).encode(), len(dims), dims, flat), io=True)


def data_tensor_from_tns(path, dense: bool = False, sidecar: int = 1) -> "DataTensor":
    """DataTensor(read_tns_file(path)) / DataTensor(read_tns_dense_file(path)) on the device."""
    if dense:
        dims, vals = read_tns_dense(path, sidecar)
        return DataTensor.dense(vals, dims)
    dims, coords, vals = read_tns(path, sidecar)
    return DataTensor.coo(dims, coords, vals)


# ---- problems (host generators) ---------------------------------------------------------------

def rng_draws(seed, n):
    u64 = np.empty(n, dtype=np.uint64)
    uni = np.empty(n)
    nor = np.empty(n)
    _check(lib.cpfit_rng_draws(seed, n, u64.ctypes.data, uni.ctypes.data, nor.ctypes.data), True)
    return u64, uni, nor


def rng_mix(x):
    return int(lib.cpfit_rng_mix(x))


def collinear_factors(dims, rank, c, seed):
    dims = _dims(dims)
    out = np.empty(int(dims.sum()) * rank)
    _check(lib.cpfit_collinear_factors(len(dims), dims, rank, c, seed, out), True)
    return out


def full(dims, rank, u):
    dims = _dims(dims)
    u = _vec(u, _packed_len(dims, rank), "full")
    out = np.empty(int(np.prod(dims)))
    _check(lib.cpfit_full(len(dims), dims, rank, u, out), True)
    return out


def dense_test_problem(dims, rank, c, l1, l2, seed, noise_mode=1, want_truth=False, want_noise_free=False):
    """Returns (T flat first-mode-fastest, truth packed or None, noise-free T or None).
    noise_mode 0: reference scaling (100/l-1)^(-1/2); 1: BASELINE l/100."""
    dims = _dims(dims)
    K = int(np.prod(dims))
    t = np.empty(K)
    truth = np.empty(int(dims.sum()) * rank) if want_truth else None
    nf = np.empty(K) if want_noise_free else None
    _check(lib.cpfit_dense_test_problem(len(dims), dims, rank, c, l1, l2, seed, noise_mode, t,
                                        truth.ctypes.data if truth is not None else None,
                                        nf.ctypes.data if nf is not None else None), True)
    return t, truth, nf


def uniform_initial_guess(dims, rank, seed):
    dims = _dims(dims)
    out = np.empty(int(dims.sum()) * rank)
    _check(lib.cpfit_uniform_initial_guess(len(dims), dims, rank, seed, out), True)
    return out


def laplacian_tensor(d, s):
    n = C.c_int64()
    _check(lib.cpfit_laplacian_tensor(d, s, None, None, C.byref(n)), True)
    coords = np.empty(n.value * 2 * d, dtype=np.int64)
    vals = np.empty(n.value)
    _check(lib.cpfit_laplacian_tensor(d, s, coords.ctypes.data, vals.ctypes.data, C.byref(n)), True)
    return (s,) * (2 * d), coords.reshape(-1, 2 * d), vals


def random_sparse_problem(dims, nnz, rank, noise, seed, want_truth=False):
    dims = _dims(dims)
    coords = np.empty(nnz * len(dims), dtype=np.int64)
    vals = np.empty(nnz)
    truth = np.empty(int(dims.sum()) * rank) if want_truth else None
    _check(lib.cpfit_random_sparse_problem(len(dims), dims, nnz, rank, noise, seed, coords, vals,
                                           truth.ctypes.data if truth is not None else None), True)
    return coords.reshape(-1, len(dims)), vals, truth
