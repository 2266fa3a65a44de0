// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp). extern "C" surface for the pytest
// checkers and bench.py's CPU baseline leg (ctypes). Status: 0 ok, 1 invalid_argument,
// 2 numerical_error, 3 other.
#include "oracle.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const numerical_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

Shape make_shape(int n, const int64_t* dims) { return Shape(std::vector<index_t>(dims, dims + n)); }

KruskalTensor kt(const DataTensor& t, int64_t rank, const double* u) {
    const Shape& s = t.shape();
    index_t total = 0;
    for (int n = 0; n < s.order(); ++n) total += s.dim(n) * rank;
    return unpack(Vector(u, u + total), s, rank);
}

void copy_out(const Vector& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(double)); }

struct TraceOut {
    int32_t iter;
    int32_t restart;
    double f, h, gnorm_rel, beta;
    int64_t fevals, gevals;
    int64_t precond_calls;
    double time_s;
};

void write_trace(const std::vector<TraceRecord>& tr, TraceOut* out, int64_t cap, int64_t* rows) {
    *rows = static_cast<int64_t>(tr.size());
    for (size_t i = 0; i < tr.size() && static_cast<int64_t>(i) < cap; ++i)
        out[i] = {tr[i].iter, tr[i].restart ? 1 : 0, tr[i].f, tr[i].h, tr[i].gnorm_rel, tr[i].beta,
                  tr[i].fevals, tr[i].gevals, tr[i].precond_calls, tr[i].time_s};
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

int oracle_tensor_dense(int n, const int64_t* dims, const double* vals, void** out) {
    return guard([&] {
        Shape s = make_shape(n, dims);
        std::vector<double> v(vals, vals + s.num_elements());
        *out = new DataTensor(DenseTensor(s, std::move(v)));
    });
}

int oracle_tensor_sparse(int n, const int64_t* dims, int64_t nnz, const int64_t* coords, const double* vals,
                         void** out) {
    return guard([&] {
        Shape s = make_shape(n, dims);
        *out = new DataTensor(SparseTensor(s, std::vector<index_t>(coords, coords + nnz * n),
                                           std::vector<double>(vals, vals + nnz)));
    });
}

// Canonicalized sparse contents (after sort/sum/drop): nnz then copy.
int64_t oracle_tensor_nnz(void* h) {
    auto* t = static_cast<DataTensor*>(h);
    return t->is_sparse() ? t->sparse().nnz() : t->shape().num_elements();
}
int oracle_tensor_sparse_contents(void* h, int64_t* coords, double* vals) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        const auto& sp = t->sparse();
        std::memcpy(coords, sp.coords.data(), sp.coords.size() * sizeof(int64_t));
        std::memcpy(vals, sp.values.data(), sp.values.size() * sizeof(double));
    });
}

void oracle_tensor_free(void* h) { delete static_cast<DataTensor*>(h); }
double oracle_tensor_norm(void* h) { return static_cast<DataTensor*>(h)->norm(); }

int oracle_mttkrp(void* h, int64_t rank, const double* u, int mode, double* out) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        const Matrix m = t->mttkrp(kt(*t, rank, u).factors, mode);
        std::memcpy(out, m.v.data(), m.v.size() * sizeof(double));
    });
}

int oracle_objective(void* h, int64_t rank, const double* u, double* f) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        *f = objective(*t, kt(*t, rank, u));
    });
}

int oracle_eval(void* h, int64_t rank, const double* u, double* g, double* f) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        Vector gv;
        *f = objective_and_gradient(*t, kt(*t, rank, u), gv);
        copy_out(gv, g);
    });
}

int oracle_gram_hadamard(int n, const int64_t* dims, int64_t rank, const double* u, int skip, double* out) {
    return guard([&] {
        Shape s = make_shape(n, dims);
        index_t total = 0;
        for (int k = 0; k < n; ++k) total += dims[k] * rank;
        const KruskalTensor k = unpack(Vector(u, u + total), s, rank);
        const Matrix g = gram_hadamard(k.factors, skip);
        std::memcpy(out, g.v.data(), g.v.size() * sizeof(double));
    });
}

int oracle_normalize(int n, const int64_t* dims, int64_t rank, const double* u, double* out) {
    return guard([&] {
        Shape s = make_shape(n, dims);
        index_t total = 0;
        for (int k = 0; k < n; ++k) total += dims[k] * rank;
        copy_out(pack(normalize_and_reorder(unpack(Vector(u, u + total), s, rank))), out);
    });
}

int oracle_full(int n, const int64_t* dims, int64_t rank, const double* u, double* out) {
    return guard([&] {
        Shape s = make_shape(n, dims);
        index_t total = 0;
        for (int k = 0; k < n; ++k) total += dims[k] * rank;
        const DenseTensor d = full(unpack(Vector(u, u + total), s, rank));
        std::memcpy(out, d.values.data(), d.values.size() * sizeof(double));
    });
}

int oracle_als_sweep(void* h, int64_t rank, const double* u, double* out) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        copy_out(pack(als_sweep(*t, kt(*t, rank, u))), out);
    });
}

// window_u / window_g: m x n row blocks, oldest first.
int oracle_accelerate(int64_t n, int64_t m, const double* wu, const double* wg, const double* ub, const double* gb,
                      double eps, double* uhat, double* alpha, double* resid) {
    return guard([&] {
        AccelWindow w(static_cast<size_t>(m));
        for (int64_t j = 0; j < m; ++j) w.push(Vector(wu + j * n, wu + (j + 1) * n), Vector(wg + j * n, wg + (j + 1) * n));
        const AccelOutcome o = accelerate(w, Vector(ub, ub + n), Vector(gb, gb + n), eps);
        copy_out(o.u_hat, uhat);
        copy_out(o.alpha, alpha);
        *resid = o.system_residual_rel;
    });
}

struct OracleNgmresOpts {
    int32_t window;
    int32_t max_iters;
    double epsilon_reg;
    double tol_grad;
    double ftol, gtol, initial_step;
    int32_t max_evals;
    int32_t restart_on_ascent;
    double step_min, step_max;
};

int oracle_ngmres_cp(void* h, int64_t rank, const double* u0, const OracleNgmresOpts* o, double gradient_scale,
                     int record_iterates, double* u_best, double* f_best, TraceOut* trace, int64_t trace_cap,
                     int64_t* rows, int* stop, double* iterates, double* seconds) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        NgmresOptions opts;
        opts.window = o->window;
        opts.max_iters = o->max_iters;
        opts.epsilon_reg = o->epsilon_reg;
        opts.tol_grad = o->tol_grad;
        opts.line_search = {o->ftol, o->gtol, o->initial_step, o->max_evals, o->step_min, o->step_max};
        opts.restart_on_ascent = o->restart_on_ascent != 0;
        const auto t0 = std::chrono::steady_clock::now();
        const MinimizeResult r = ngmres_cp(*t, kt(*t, rank, u0), opts, gradient_scale, record_iterates);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        copy_out(r.u, u_best);
        *f_best = r.f;
        write_trace(r.trace, trace, trace_cap, rows);
        *stop = static_cast<int>(r.stop);
        if (iterates)
            for (size_t i = 0; i < r.iterates.size(); ++i) copy_out(r.iterates[i], iterates + i * r.u.size());
    });
}

int oracle_als_solve(void* h, int64_t rank, const double* u0, double tol_grad, int max_iters, double* u_best,
                     TraceOut* trace, int64_t trace_cap, int64_t* rows, int* stop) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        const SolveResult r = als_solve(*t, kt(*t, rank, u0), {tol_grad, max_iters});
        copy_out(pack(r.solution), u_best);
        write_trace(r.trace, trace, trace_cap, rows);
        *stop = static_cast<int>(r.stop);
    });
}

// Moré–Thuente with a C callback phi(step, &f, &dg, ctx).
typedef void (*oracle_phi_fn)(double, double*, double*, void*);
int oracle_more_thuente(oracle_phi_fn phi, void* ctx, double phi0, double dphi0, double ftol, double gtol,
                        double initial_step, int max_evals, double step_min, double step_max, double* step,
                        double* f, double* dg, int* status, int* evals) {
    return guard([&] {
        LineSearchParams p{ftol, gtol, initial_step, max_evals, step_min, step_max};
        const LineSearchResult r = more_thuente(
            [&](double s, double& fv, double& g) { phi(s, &fv, &g, ctx); }, phi0, dphi0, p);
        *step = r.step;
        *f = r.f;
        *dg = r.dg;
        *status = static_cast<int>(r.status);
        *evals = r.evals;
    });
}

// Generic N-GMRES on a quadratic f = 1/2 u^T A u - b^T u with M(u) = u + omega (b - A u)
// (the reference's own linear test seam, test_ngmres.cpp:94-102).
int oracle_ngmres_linear(int64_t n, const double* a, const double* b, double omega, const double* u0,
                         int window, int max_iters, double epsilon_reg, double tol_grad, int restart_on_ascent,
                         double fixed_step, int use_fixed, double* u_out, double* ghat_norms, int64_t* n_obs) {
    return guard([&] {
        Matrix A(n, n);
        std::memcpy(A.v.data(), a, static_cast<size_t>(n * n) * sizeof(double));
        Vector B(b, b + n);
        auto mv = [&](const Vector& u) {
            Vector y(static_cast<size_t>(n), 0.0);
            for (int64_t j = 0; j < n; ++j)
                for (int64_t i = 0; i < n; ++i) y[static_cast<size_t>(i)] += A(i, j) * u[static_cast<size_t>(j)];
            return y;
        };
        NgmresProblem p;
        p.eval = [&](const Vector& u, Vector& g) {
            const Vector au = mv(u);
            g.resize(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) g[static_cast<size_t>(i)] = au[static_cast<size_t>(i)] - B[static_cast<size_t>(i)];
            return 0.5 * dot(u, au) - dot(B, u);
        };
        p.precondition = [&](const Vector& u) {
            const Vector au = mv(u);
            Vector y = u;
            for (int64_t i = 0; i < n; ++i) y[static_cast<size_t>(i)] += omega * (B[static_cast<size_t>(i)] - au[static_cast<size_t>(i)]);
            return y;
        };
        if (use_fixed) p.fixed_step = fixed_step;
        int64_t cnt = 0;
        p.observer = [&](const AccelWindow&, const Vector&, const Vector&, const Vector& uh) {
            const Vector au = mv(uh);
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) {
                const double r = au[static_cast<size_t>(i)] - B[static_cast<size_t>(i)];
                s += r * r;
            }
            ghat_norms[cnt++] = std::sqrt(s);
        };
        NgmresOptions o;
        o.window = window;
        o.max_iters = max_iters;
        o.epsilon_reg = epsilon_reg;
        o.tol_grad = tol_grad;
        o.restart_on_ascent = restart_on_ascent != 0;
        const MinimizeResult r = ngmres_minimize(p, Vector(u0, u0 + n), o);
        copy_out(r.u, u_out);
        *n_obs = cnt;
    });
}

int oracle_ncg_cp(void* h, int64_t rank, const double* u0, double tol_grad, int max_iters, double* u_best,
                  TraceOut* trace, int64_t trace_cap, int64_t* rows, int* stop) {
    return guard([&] {
        auto* t = static_cast<DataTensor*>(h);
        const Shape s = t->shape();
        auto eval = [&](const Vector& u, Vector& g) { return objective_and_gradient(*t, unpack(u, s, rank), g); };
        NcgOptions o;
        o.tol_grad = tol_grad;
        o.max_iters = max_iters;
        const double sc = t->norm();
        const MinimizeResult r = ncg_minimize(eval, pack(normalize_and_reorder(kt(*t, rank, u0))), o, sc,
                                              [sc](double f) { return std::sqrt(std::max(2.0 * f, 0.0)) / sc; });
        copy_out(pack(normalize_and_reorder(unpack(r.u, s, rank))), u_best);
        write_trace(r.trace, trace, trace_cap, rows);
        *stop = static_cast<int>(r.stop);
    });
}

}  // extern "C"
