"""ORACLE — TEST INFRASTRUCTURE ONLY. ctypes binding of oracle/_build/liboracle.so, the CPU
restatement of the reference (proj/core/src/*.cpp). Used only as the parity checker and the
CPU baseline; the product never imports it."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load():
    if not os.path.exists(LIB_PATH):
        build()
    return C.CDLL(LIB_PATH)


lib = _load()
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class TraceOut(C.Structure):
    _fields_ = [("iter", C.c_int32), ("restart", C.c_int32), ("f", C.c_double), ("h", C.c_double),
                ("gnorm_rel", C.c_double), ("beta", C.c_double), ("fevals", C.c_int64), ("gevals", C.c_int64),
                ("precond_calls", C.c_int64), ("time_s", C.c_double)]


class Opts(C.Structure):
    _fields_ = [("window", C.c_int32), ("max_iters", C.c_int32), ("epsilon_reg", C.c_double),
                ("tol_grad", C.c_double), ("ftol", C.c_double), ("gtol", C.c_double), ("initial_step", C.c_double),
                ("max_evals", C.c_int32), ("restart_on_ascent", C.c_int32), ("step_min", C.c_double),
                ("step_max", C.c_double)]


PHI = C.CFUNCTYPE(None, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)

_SIGS = {
    "oracle_last_error": (C.c_char_p, []),
    "oracle_tensor_dense": (C.c_int, [C.c_int, _i64p, _f64p, C.POINTER(C.c_void_p)]),
    "oracle_tensor_sparse": (C.c_int, [C.c_int, _i64p, C.c_int64, _i64p, _f64p, C.POINTER(C.c_void_p)]),
    "oracle_tensor_nnz": (C.c_int64, [C.c_void_p]),
    "oracle_tensor_sparse_contents": (C.c_int, [C.c_void_p, _i64p, _f64p]),
    "oracle_tensor_free": (None, [C.c_void_p]),
    "oracle_tensor_norm": (C.c_double, [C.c_void_p]),
    "oracle_mttkrp": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_int, _f64p]),
    "oracle_objective": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.POINTER(C.c_double)]),
    "oracle_eval": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _f64p, C.POINTER(C.c_double)]),
    "oracle_gram_hadamard": (C.c_int, [C.c_int, _i64p, C.c_int64, _f64p, C.c_int, _f64p]),
    "oracle_normalize": (C.c_int, [C.c_int, _i64p, C.c_int64, _f64p, _f64p]),
    "oracle_full": (C.c_int, [C.c_int, _i64p, C.c_int64, _f64p, _f64p]),
    "oracle_als_sweep": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _f64p]),
    "oracle_accelerate": (C.c_int, [C.c_int64, C.c_int64, _f64p, _f64p, _f64p, _f64p, C.c_double, _f64p, _f64p,
                                    C.POINTER(C.c_double)]),
    "oracle_ngmres_cp": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.POINTER(Opts), C.c_double, C.c_int, _f64p,
                                   C.POINTER(C.c_double), C.POINTER(TraceOut), C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int), C.c_void_p, C.POINTER(C.c_double)]),
    "oracle_als_solve": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_double, C.c_int, _f64p, C.POINTER(TraceOut),
                                   C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "oracle_more_thuente": (C.c_int, [PHI, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_int, C.c_double, C.c_double, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int)]),
    "oracle_ngmres_linear": (C.c_int, [C.c_int64, _f64p, _f64p, C.c_double, _f64p, C.c_int, C.c_int, C.c_double,
                                       C.c_double, C.c_int, C.c_double, C.c_int, _f64p, _f64p,
                                       C.POINTER(C.c_int64)]),
    "oracle_problems_last_error": (C.c_char_p, []),
    "oracle_dense_test_problem": (C.c_int, [C.c_int, _i64p, C.c_int64, C.c_double, C.c_double, C.c_double,
                                            C.c_uint64, C.c_int, _f64p, C.c_void_p]),
    "oracle_uniform_initial_guess": (C.c_int, [C.c_int, _i64p, C.c_int64, C.c_uint64, _f64p]),
    "oracle_random_sparse_problem": (C.c_int, [C.c_int, _i64p, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                               _i64p, _f64p]),
    "oracle_io_last_error": (C.c_char_p, []),
    "oracle_tns_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), _i64p, C.POINTER(C.c_int64), C.c_void_p,
                                  C.c_void_p]),
    "oracle_tns_write": (C.c_int, [C.c_char_p, C.c_int, _i64p, C.c_int64, _i64p, _f64p]),
    "oracle_ncg_cp": (C.c_int, [C.c_void_p, C.c_int64, _f64p, C.c_double, C.c_int, _f64p, C.POINTER(TraceOut),
                                C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
}
for _n, (_r, _a) in _SIGS.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a


class OracleError(RuntimeError):
    pass


class OracleNumericalError(OracleError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = lib.oracle_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise OracleNumericalError(msg)
    raise OracleError(msg)


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


class Tensor:
    def __init__(self, h, dims):
        self.h = h
        self.dims = tuple(int(d) for d in dims)

    @classmethod
    def dense(cls, dims, flat):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        flat = _f64(flat).reshape(-1)
        if flat.size != int(np.prod(dims)):
            raise ValueError("DenseTensor: value count does not match shape")
        h = C.c_void_p()
        _check(lib.oracle_tensor_dense(len(dims), dims, flat, C.byref(h)))
        return cls(h, dims)

    @classmethod
    def coo(cls, dims, coords, vals):
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1)
        vals = _f64(vals).reshape(-1)
        h = C.c_void_p()
        _check(lib.oracle_tensor_sparse(len(dims), dims, vals.size, coords, vals, C.byref(h)))
        return cls(h, dims)

    def __del__(self):
        if getattr(self, "h", None):
            lib.oracle_tensor_free(self.h)
            self.h = None

    def norm(self):
        return lib.oracle_tensor_norm(self.h)

    def rank_of(self, u):
        return _f64(u).size // sum(self.dims)

    def sparse_contents(self):
        n = lib.oracle_tensor_nnz(self.h)
        c = np.empty(n * len(self.dims), dtype=np.int64)
        v = np.empty(n)
        _check(lib.oracle_tensor_sparse_contents(self.h, c, v))
        return c.reshape(n, -1), v

    def mttkrp(self, u, mode):
        r = self.rank_of(u)
        out = np.empty(self.dims[mode] * r)
        _check(lib.oracle_mttkrp(self.h, r, _f64(u), mode, out))
        return out.reshape((self.dims[mode], r), order="F")

    def objective(self, u):
        f = C.c_double()
        _check(lib.oracle_objective(self.h, self.rank_of(u), _f64(u), C.byref(f)))
        return f.value

    def eval(self, u):
        g = np.empty(_f64(u).size)
        f = C.c_double()
        _check(lib.oracle_eval(self.h, self.rank_of(u), _f64(u), g, C.byref(f)))
        return f.value, g

    def als_sweep(self, u):
        out = np.empty(_f64(u).size)
        _check(lib.oracle_als_sweep(self.h, self.rank_of(u), _f64(u), out))
        return out

    def ngmres(self, u0, window=20, max_iters=2000, epsilon_reg=1e-12, tol_grad=1e-9, gradient_scale=None,
               restart_on_ascent=True, record_iterates=0, ftol=1e-4, gtol=1e-2, initial_step=1.0, max_evals=20):
        u0 = _f64(u0)
        r = self.rank_of(u0)
        o = Opts(window, max_iters, epsilon_reg, tol_grad, ftol, gtol, initial_step, max_evals,
                 int(restart_on_ascent), 0.0, 1e20)
        cap = max_iters + 1
        tr = (TraceOut * cap)()
        ub = np.empty_like(u0)
        fb = C.c_double()
        rows = C.c_int64()
        stop = C.c_int()
        secs = C.c_double()
        its = np.empty((max(record_iterates, 1), u0.size))
        gs = self.norm() if gradient_scale is None else gradient_scale
        _check(lib.oracle_ngmres_cp(self.h, r, u0, C.byref(o), gs, record_iterates, ub, C.byref(fb), tr, cap,
                                    C.byref(rows), C.byref(stop), its.ctypes.data if record_iterates else None,
                                    C.byref(secs)))
        return dict(u=ub, f=fb.value, trace=_trace(tr, rows.value), stop=stop.value, seconds=secs.value,
                    iterates=its[:min(record_iterates, rows.value)] if record_iterates else None)

    def als_solve(self, u0, tol_grad=1e-9, max_iters=2000):
        u0 = _f64(u0)
        cap = max_iters + 1
        tr = (TraceOut * cap)()
        ub = np.empty_like(u0)
        rows = C.c_int64()
        stop = C.c_int()
        _check(lib.oracle_als_solve(self.h, self.rank_of(u0), u0, tol_grad, max_iters, ub, tr, cap, C.byref(rows),
                                    C.byref(stop)))
        return dict(u=ub, trace=_trace(tr, rows.value), stop=stop.value)

    def ncg(self, u0, tol_grad=1e-9, max_iters=2000):
        u0 = _f64(u0)
        cap = max_iters + 1
        tr = (TraceOut * cap)()
        ub = np.empty_like(u0)
        rows = C.c_int64()
        stop = C.c_int()
        _check(lib.oracle_ncg_cp(self.h, self.rank_of(u0), u0, tol_grad, max_iters, ub, tr, cap, C.byref(rows),
                                 C.byref(stop)))
        return dict(u=ub, trace=_trace(tr, rows.value), stop=stop.value)


def _check_problems(rc):
    if rc == 0:
        return
    msg = lib.oracle_problems_last_error().decode()
    raise (ValueError if rc == 1 else OracleError)(msg)


def dense_test_problem(dims, rank, c, l1, l2, seed, noise_mode=1, want_truth=False):
    """problems.cpp:63-95 restated (noise_mode 1: BASELINE's l/100 scaling). Returns (T flat
    first-mode-fastest, truth factors in pack order or None)."""
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    t = np.empty(int(np.prod(dims)))
    truth = np.empty(int(dims.sum()) * rank) if want_truth else None
    _check_problems(lib.oracle_dense_test_problem(len(dims), dims, rank, c, l1, l2, seed, noise_mode, t,
                                                  truth.ctypes.data if truth is not None else None))
    return t, truth


def uniform_initial_guess(dims, rank, seed):
    """problems.cpp:137-145 restated."""
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    out = np.empty(int(dims.sum()) * rank)
    _check_problems(lib.oracle_uniform_initial_guess(len(dims), dims, rank, seed, out))
    return out


def random_sparse_problem(dims, nnz, rank, noise, seed):
    """BASELINE.json configs[4] generator. Returns (coords nnz x N, values)."""
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    coords = np.empty(nnz * len(dims), dtype=np.int64)
    vals = np.empty(nnz)
    _check_problems(lib.oracle_random_sparse_problem(len(dims), dims, nnz, rank, noise, seed, coords, vals))
    return coords.reshape(-1, len(dims)), vals


class OracleIOError(OracleError):
    """cpfit::io_error"""


def tns_read(path):
    """read_tns_file restated (io.cpp:104-147, 179-188): (dims, coords nnz x N, values) as written,
    or OracleIOError with the reference's message."""
    order = C.c_int()
    dims = np.zeros(16, dtype=np.int64)
    nnz = C.c_int64()
    if lib.oracle_tns_read(str(path).encode(), C.byref(order), dims, C.byref(nnz), None, None):
        raise OracleIOError(lib.oracle_io_last_error().decode())
    n = order.value
    coords = np.empty(max(nnz.value, 1) * n, dtype=np.int64)
    vals = np.empty(max(nnz.value, 1))
    if lib.oracle_tns_read(str(path).encode(), C.byref(order), dims, C.byref(nnz), coords.ctypes.data,
                           vals.ctypes.data):
        raise OracleIOError(lib.oracle_io_last_error().decode())
    return tuple(int(d) for d in dims[:n]), coords[:nnz.value * n].reshape(-1, n), vals[:nnz.value]


def tns_write(path, dims, coords, values):
    """write_tns_file(SparseTensor) restated (io.cpp:151-159)."""
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    coords = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1)
    values = _f64(values).reshape(-1)
    if lib.oracle_tns_write(str(path).encode(), len(dims), dims, values.size, coords, values):
        raise OracleIOError(lib.oracle_io_last_error().decode())


def _trace(tr, rows):
    return [dict(iter=t.iter, f=t.f, h=t.h, gnorm_rel=t.gnorm_rel, fevals=t.fevals, gevals=t.gevals,
                 precond_calls=t.precond_calls, restart=bool(t.restart), beta=t.beta, time_s=t.time_s)
            for t in tr[:rows]]


def gram_hadamard(dims, rank, u, skip=-1):
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    out = np.empty(rank * rank)
    _check(lib.oracle_gram_hadamard(len(dims), dims, rank, _f64(u), skip, out))
    return out.reshape((rank, rank), order="F")


def normalize(dims, rank, u):
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    out = np.empty(_f64(u).size)
    _check(lib.oracle_normalize(len(dims), dims, rank, _f64(u), out))
    return out


def full(dims, rank, u):
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    out = np.empty(int(np.prod(dims)))
    _check(lib.oracle_full(len(dims), dims, rank, _f64(u), out))
    return out


def accelerate(window_u, window_g, u_bar, g_bar, eps=1e-12):
    wu = np.ascontiguousarray(np.asarray(window_u, dtype=np.float64).reshape(len(window_u), -1))
    wg = np.ascontiguousarray(np.asarray(window_g, dtype=np.float64).reshape(len(window_g), -1))
    m, n = wu.shape
    uh = np.empty(n)
    al = np.empty(m)
    rr = C.c_double()
    _check(lib.oracle_accelerate(n, m, wu.reshape(-1), wg.reshape(-1), _f64(u_bar), _f64(g_bar), eps, uh, al,
                                 C.byref(rr)))
    return uh, al, rr.value


def more_thuente(phi, phi0, dphi0, ftol=1e-4, gtol=1e-2, initial_step=1.0, max_evals=20, step_min=0.0,
                 step_max=1e20):
    def cb(s, fp, gp, _):
        f, g = phi(s)
        fp[0] = f
        gp[0] = g

    fn = PHI(cb)
    st, f, g = C.c_double(), C.c_double(), C.c_double()
    status, ev = C.c_int(), C.c_int()
    _check(lib.oracle_more_thuente(fn, None, phi0, dphi0, ftol, gtol, initial_step, max_evals, step_min, step_max,
                                   C.byref(st), C.byref(f), C.byref(g), C.byref(status), C.byref(ev)))
    return dict(step=st.value, f=f.value, dg=g.value, status=status.value, evals=ev.value)


def ngmres_linear(a, b, omega, u0, window, max_iters, epsilon_reg, tol_grad, restart_on_ascent=False,
                  fixed_step=None):
    n = len(b)
    u = np.empty(n)
    obs = np.empty(max_iters + 2)
    cnt = C.c_int64()
    _check(lib.oracle_ngmres_linear(n, _f64(np.asarray(a).reshape(-1, order="F")), _f64(b), omega, _f64(u0), window,
                                    max_iters, epsilon_reg, tol_grad, int(restart_on_ascent),
                                    0.0 if fixed_step is None else fixed_step, int(fixed_step is not None), u, obs,
                                    C.byref(cnt)))
    return u, obs[:cnt.value]
