// extern "C" surface (include/cpfit_gpu.h). Exceptions become status codes here.
#include "../../include/cpfit_gpu.h"
#include "device.cuh"
#include "linesearch.cuh"
#include "solver.cuh"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

using namespace cpfit_gpu;

namespace cpfit_gpu {
void dense_fiber(const DevTensor& t, EvalWork& w, const double* u, bool do_s, bool do_m0, cudaStream_t st);
void dense_fiber_fused(const DevTensor& t, EvalWork& w, const double* u, cudaStream_t st, const int* resid_flag);
}  // namespace cpfit_gpu

struct cpfit_tensor_s {
    DevTensor* t = nullptr;
    cudaStream_t st = nullptr;
    std::map<int, EvalWork*> works;
    std::mutex mu;
    double* scratch = nullptr;  // device buffers for per-call ops
    size_t scratch_n = 0;
    int* one_ = nullptr;        // device int 1: residual-form objective for per-call evaluations
    const int* one() {
        if (!one_) {
            CPFIT_CUDA(cudaMalloc(&one_, sizeof(int)));
            const int v = 1;
            CPFIT_CUDA(cudaMemcpy(one_, &v, sizeof(int), cudaMemcpyHostToDevice));
        }
        return one_;
    }
    // solvers of the one-shot solve calls, kept between calls (graph capture and instantiation
    // cost milliseconds): one per method, reused while rank and graph-baked options match
    std::unique_ptr<Solver> solvers[3];
    Solver& solver(int R, const SolverOptions& o, int method) {
        std::unique_ptr<Solver>& s = solvers[method];
        if (!s || s->rank() != R || !s->options().serves(o)) {
            s.reset();
            s = std::make_unique<Solver>(t, R, o, method);
        }
        return *s;
    }
    // concurrent solvers of the batched solve calls (own streams and workspaces each), kept
    // while rank, method and graph-baked options match
    std::vector<std::unique_ptr<Solver>> pool;
    int pool_method = -1;
    std::vector<Solver*> batch(int R, const SolverOptions& o, int method, int n) {
        if (!pool.empty() && (pool_method != method || pool[0]->rank() != R || !pool[0]->options().serves(o)))
            pool.clear();
        pool_method = method;
        while ((int)pool.size() < n) pool.push_back(std::make_unique<Solver>(t, R, o, method));
        std::vector<Solver*> v;
        for (int k = 0; k < n; ++k) v.push_back(pool[(size_t)k].get());
        return v;
    }
    ~cpfit_tensor_s() {
        pool.clear();
        for (auto& sv : solvers) sv.reset();
        for (auto& kv : works) work_destroy(kv.second);
        cudaFree(one_);
        cudaFree(scratch);
        tensor_destroy(t);
        if (st) cudaStreamDestroy(st);
    }
    EvalWork& work(int R) {
        auto it = works.find(R);
        if (it != works.end()) return *it->second;
        EvalWork* w = work_create(*t, R);
        works[R] = w;
        return *w;
    }
    double* buf(size_t n) {
        if (n > scratch_n) {
            cudaFree(scratch);
            CPFIT_CUDA(cudaMalloc(&scratch, sizeof(double) * n));
            scratch_n = n;
        }
        return scratch;
    }
};

// Dense tensor handles of a destroyed DataTensor are parked here (up to CPFIT_TENSOR_POOL_MB of
// device memory, default 8192; 0 disables) with their workspaces and captured solver graphs, and
// a new dense tensor of the same shape and kind takes one over: its values are uploaded into the
// same device buffers (tensor_fill_dense), so the graphs — which read T, the fibre norms and
// ||T|| through those buffers — stay valid and the new handle pays only the upload, not the
// workspace allocation or graph capture/instantiation (tens of ms at 400^3). Graph caches are
// thus keyed by (shape, rank, options), not by handle.
namespace {
struct TensorPool {
    std::mutex mu;
    std::vector<cpfit_tensor_s*> items;  // oldest first
    size_t bytes = 0;
};
TensorPool& tensor_pool() {
    static TensorPool* p = new TensorPool();  // never destroyed: outlives static destructors
    return *p;
}
size_t pool_cap_bytes() {
    static const size_t cap = [] {
        const char* e = std::getenv("CPFIT_TENSOR_POOL_MB");
        return (size_t)(e ? std::strtoull(e, nullptr, 10) : 8192ull) << 20;
    }();
    return cap;
}
size_t handle_bytes(const cpfit_tensor_s* h) { return sizeof(double) * (size_t)h->t->ldT * (size_t)h->t->J; }
bool same_dense_kind(const DevTensor& a, int order, const int64_t* dims, bool generic) {
    if (a.sparse || a.order != order || a.generic != generic) return false;
    for (int n = 0; n < order; ++n)
        if (a.dims[n] != dims[n]) return false;
    return true;
}
}  // namespace

struct cpfit_solver_s {
    std::unique_ptr<Solver> s;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~cpfit_solver_s() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

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
    } catch (const cpfit_gpu::numerical_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

int64_t packed_len(int order, const int64_t* dims, int64_t R) {
    int64_t s = 0;
    for (int n = 0; n < order; ++n) s += dims[n] * R;
    return s;
}

void check_rank(int64_t R) {
    if (R < 1) throw std::invalid_argument("KruskalTensor: rank must be >= 1");
    if (R > kMaxRankWide) throw std::invalid_argument("device path supports rank <= 64");
}

void check_finite(const double* u, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(u[i])) throw std::invalid_argument("KruskalTensor: entries must be finite");
}

// Factor-only context (gram_hadamard / normalize need no tensor).
struct FactorCtx {
    DevTensor t;
    EvalWork* w = nullptr;
    cudaStream_t st = nullptr;
    FactorCtx(int order, const int64_t* dims, int R) {
        if (order < 1 || order > kMaxOrder) throw std::invalid_argument("order must be in [1, 8] on device");
        t.order = order;
        t.sparse = true;
        for (int n = 0; n < order; ++n) {
            if (dims[n] < 1) throw std::invalid_argument("Shape: every mode size must be >= 1");
            t.dims[n] = dims[n];
        }
        CPFIT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        w = work_create(t, R);
    }
    ~FactorCtx() {
        work_destroy(w);
        cudaStreamDestroy(st);
    }
};

struct DevBuf {
    double* p = nullptr;
    explicit DevBuf(size_t n) { CPFIT_CUDA(cudaMalloc(&p, sizeof(double) * std::max<size_t>(n, 1))); }
    ~DevBuf() { cudaFree(p); }
};

SolverOptions to_opts(const cpfit_ngmres_options* o, double tnorm) {
    SolverOptions s;
    s.window = o->window;
    s.max_iters = o->max_iters;
    s.epsilon_reg = o->epsilon_reg;
    s.tol_grad = o->tol_grad;
    s.gradient_scale = (o->gradient_scale > 0.0) ? o->gradient_scale : tnorm;
    s.ftol = o->ftol;
    s.gtol = o->gtol;
    s.initial_step = o->initial_step;
    s.max_evals = o->max_evals;
    s.step_min = o->step_min;
    s.step_max = o->step_max;
    s.restart_on_ascent = o->restart_on_ascent;
    s.reeval_accepted = o->reeval_accepted;
    s.residual_objective = o->residual_objective;
    if (s.window < 1) throw std::invalid_argument("ngmres: window must be >= 1");
    if (!(s.tol_grad > 0.0)) throw std::invalid_argument("ngmres: tol_grad must be > 0");
    if (s.epsilon_reg < 0.0) throw std::invalid_argument("ngmres: epsilon_reg must be >= 0");
    if (!(s.ftol > 0.0 && s.ftol < s.gtol && s.gtol < 1.0))
        throw std::invalid_argument("more_thuente: need 0 < ftol < gtol < 1");
    if (!(s.initial_step > 0.0)) throw std::invalid_argument("more_thuente: initial_step must be > 0");
    if (s.max_evals < 1) throw std::invalid_argument("more_thuente: max_evals must be >= 1");
    if (!(s.step_min >= 0.0 && s.step_min < s.step_max))
        throw std::invalid_argument("more_thuente: need 0 <= step_min < step_max");
    if (s.max_iters < 0) throw std::invalid_argument("ngmres: max_iters must be >= 0");
    return s;
}

void finish_solve(Solver& sv, double* u_best, double* f_best, cpfit_trace_row* trace, int64_t cap, int64_t* rows,
                  int* stop) {
    const SolverSummary sm = sv.summary();
    if (sm.status) {
        if (sm.status & 1)
            throw cpfit_gpu::numerical_error(
                "als_sweep: normal matrix is singular after regularization (structurally rank-deficient iterate)");
        throw cpfit_gpu::numerical_error("als_sweep: non-finite solution of the normal equations");
    }
    const int nrows = sm.rows;
    if (rows) *rows = nrows;
    if (trace && cap > 0) {
        std::vector<TraceRow> tr((size_t)nrows);
        sv.copy_trace(tr.data(), nrows);
        for (int64_t i = 0; i < std::min<int64_t>(cap, nrows); ++i) std::memcpy(&trace[i], &tr[(size_t)i], sizeof(TraceRow));
    }
    if (u_best) {
        sv.copy_best(u_best, true);
        sv.sync();
    }
    if (f_best) *f_best = sm.best_f;
    if (stop) *stop = (sm.stop < 0) ? 1 : sm.stop;
}
}  // namespace

static_assert(sizeof(cpfit_trace_row) == sizeof(TraceRow), "trace row layout");

extern "C" {

const char* cpfit_last_error(void) { return g_err.c_str(); }

int cpfit_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

void cpfit_default_ngmres_options(cpfit_ngmres_options* o) {
    *o = cpfit_ngmres_options{20, 2000, 1e-12, 1e-9, 0.0, 1e-4, 1e-2, 1.0, 20, 1, 0.0, 1e20, 0, 0};
}

int cpfit_tensor_create_dense(int order, const int64_t* dims, const double* values, cpfit_tensor* out) {
    return guard([&] {
        if (order >= 1 && order <= kMaxOrder) {
            bool dims_ok = true;
            for (int n = 0; n < order; ++n) dims_ok = dims_ok && dims[n] >= 1;
            if (dims_ok) {
                const char* fg = std::getenv("CPFIT_FORCE_GENERIC");
                const bool generic = !fiber_path_fits(order, dims[0]) || (fg && fg[0] == '1');
                cpfit_tensor_s* reuse = nullptr;
                {
                    TensorPool& p = tensor_pool();
                    std::lock_guard<std::mutex> lk(p.mu);
                    for (size_t i = 0; i < p.items.size(); ++i)
                        if (same_dense_kind(*p.items[i]->t, order, dims, generic)) {
                            reuse = p.items[i];
                            p.bytes -= handle_bytes(reuse);
                            p.items.erase(p.items.begin() + (std::ptrdiff_t)i);
                            break;
                        }
                }
                if (reuse) {
                    std::unique_ptr<cpfit_tensor_s> h(reuse);  // deleted if the new values are rejected
                    tensor_fill_dense(*h->t, values, h->st);
                    *out = h.release();
                    return;
                }
            }
        }
        auto h = std::make_unique<cpfit_tensor_s>();
        CPFIT_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
        h->t = tensor_create_dense(order, dims, values, h->st);
        *out = h.release();
    });
}

int cpfit_tensor_create_coo(int order, const int64_t* dims, int64_t nnz, const int64_t* coords, const double* values,
                            cpfit_tensor* out) {
    return guard([&] {
        if (nnz < 0) throw std::invalid_argument("SparseTensor: coords/values size mismatch");
        auto h = std::make_unique<cpfit_tensor_s>();
        CPFIT_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
        h->t = tensor_create_coo(order, dims, nnz, coords, values, h->st);
        *out = h.release();
    });
}

int cpfit_tensor_destroy(cpfit_tensor t) {
    return guard([&] {
        if (!t) return;
        const size_t cap = pool_cap_bytes();
        if (t->t && !t->t->sparse && handle_bytes(t) <= cap) {
            // wait for this handle's work before another thread may refill it
            CPFIT_CUDA(cudaStreamSynchronize(t->st));
            std::vector<cpfit_tensor_s*> evict;
            {
                TensorPool& p = tensor_pool();
                std::lock_guard<std::mutex> lk(p.mu);
                p.items.push_back(t);
                p.bytes += handle_bytes(t);
                while (p.bytes > cap && !p.items.empty()) {
                    p.bytes -= handle_bytes(p.items.front());
                    evict.push_back(p.items.front());
                    p.items.erase(p.items.begin());
                }
            }
            for (cpfit_tensor_s* e : evict) delete e;
            return;
        }
        delete t;
    });
}

int cpfit_tensor_norm(cpfit_tensor t, double* norm) {
    return guard([&] { *norm = t->t->norm; });
}

int cpfit_tensor_nnz(cpfit_tensor t, int64_t* nnz) {
    return guard([&] { *nnz = t->t->sparse ? t->t->nnz : t->t->K; });
}

int cpfit_mttkrp(cpfit_tensor t, int64_t rank, const double* u, int mode, double* out) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        if (mode < 0 || mode >= t->t->order) throw std::invalid_argument("mttkrp: mode out of range");
        EvalWork& w = t->work((int)rank);
        check_finite(u, w.nu);
        double* du = t->buf((size_t)w.nu + (size_t)t->t->dims[mode] * rank);
        double* dout = du + w.nu;
        CPFIT_CUDA(cudaMemcpyAsync(du, u, sizeof(double) * w.nu, cudaMemcpyHostToDevice, t->st));
        mttkrp_device(*t->t, w, du, mode, dout, t->st);
        CPFIT_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * t->t->dims[mode] * rank, cudaMemcpyDeviceToHost, t->st));
        CPFIT_CUDA(cudaStreamSynchronize(t->st));
    });
}

static int eval_impl(cpfit_tensor t, int64_t rank, const double* u, double* grad, double* f, int form = 0) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        EvalWork& w = t->work((int)rank);
        check_finite(u, w.nu);
        double* du = t->buf(2 * (size_t)w.nu + 8);
        double* dg = du + w.nu;
        EvalScalars* sc = reinterpret_cast<EvalScalars*>(dg + w.nu);
        CPFIT_CUDA(cudaMemcpyAsync(du, u, sizeof(double) * w.nu, cudaMemcpyHostToDevice, t->st));
        // per-call objective uses the reference's residual form (kruskal.cpp:83-102); form 1 selects
        // the per-fibre three-term form the solver loop evaluates with (dense only)
        if (form != 0 && form != 1) throw std::invalid_argument("objective form must be 0 (residual) or 1 (per-fibre)");
        eval_device(*t->t, w, du, dg, sc, nullptr, nullptr, t->st, grad != nullptr, form == 1 ? nullptr : t->one());
        EvalScalars hs;
        CPFIT_CUDA(cudaMemcpyAsync(&hs, sc, sizeof(EvalScalars), cudaMemcpyDeviceToHost, t->st));
        if (grad) CPFIT_CUDA(cudaMemcpyAsync(grad, dg, sizeof(double) * w.nu, cudaMemcpyDeviceToHost, t->st));
        CPFIT_CUDA(cudaStreamSynchronize(t->st));
        *f = hs.f;
    });
}

int cpfit_objective(cpfit_tensor t, int64_t rank, const double* u, double* f) { return eval_impl(t, rank, u, nullptr, f); }

int cpfit_objective_and_gradient(cpfit_tensor t, int64_t rank, const double* u, double* grad, double* f) {
    return eval_impl(t, rank, u, grad, f);
}

int cpfit_objective_and_gradient_form(cpfit_tensor t, int64_t rank, const double* u, int form, double* grad,
                                      double* f) {
    return eval_impl(t, rank, u, grad, f, form);
}

int cpfit_gram_hadamard(int order, const int64_t* dims, int64_t rank, const double* u, int skip, double* out) {
    return guard([&] {
        check_rank(rank);
        FactorCtx c(order, dims, (int)rank);
        const int64_t n = packed_len(order, dims, rank);
        DevBuf du((size_t)n + (size_t)rank * rank);
        CPFIT_CUDA(cudaMemcpyAsync(du.p, u, sizeof(double) * n, cudaMemcpyHostToDevice, c.st));
        grams_device(*c.w, du.p, c.st);
        gram_hadamard_device(*c.w, skip, du.p + n, c.st);
        CPFIT_CUDA(cudaMemcpyAsync(out, du.p + n, sizeof(double) * rank * rank, cudaMemcpyDeviceToHost, c.st));
        CPFIT_CUDA(cudaStreamSynchronize(c.st));
    });
}

int cpfit_normalize_and_reorder(int order, const int64_t* dims, int64_t rank, const double* u, double* out) {
    return guard([&] {
        check_rank(rank);
        FactorCtx c(order, dims, (int)rank);
        const int64_t n = packed_len(order, dims, rank);
        DevBuf du(2 * (size_t)n);
        CPFIT_CUDA(cudaMemcpyAsync(du.p, u, sizeof(double) * n, cudaMemcpyHostToDevice, c.st));
        grams_device(*c.w, du.p, c.st);
        normalize_device(*c.w, du.p, du.p + n, c.st);
        CPFIT_CUDA(cudaMemcpyAsync(out, du.p + n, sizeof(double) * n, cudaMemcpyDeviceToHost, c.st));
        CPFIT_CUDA(cudaStreamSynchronize(c.st));
    });
}

int cpfit_als_sweep(cpfit_tensor t, int64_t rank, const double* u, double* out) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        EvalWork& w = t->work((int)rank);
        check_finite(u, w.nu);
        int64_t maxI = 1;
        for (int k = 0; k < t->t->order; ++k) maxI = std::max(maxI, t->t->dims[k]);
        DevBuf b(3 * (size_t)w.nu + (size_t)maxI * rank + 1);
        double* du = b.p;
        double* dout = du + w.nu;
        double* work = dout + w.nu;
        double* mbuf = work + w.nu;
        int* status = reinterpret_cast<int*>(mbuf + maxI * rank);
        CPFIT_CUDA(cudaMemsetAsync(status, 0, sizeof(int), t->st));
        CPFIT_CUDA(cudaMemcpyAsync(du, u, sizeof(double) * w.nu, cudaMemcpyHostToDevice, t->st));
        als_sweep_device_ws(*t->t, w, du, dout, work, mbuf, status, t->st);
        int hs = 0;
        CPFIT_CUDA(cudaMemcpyAsync(&hs, status, sizeof(int), cudaMemcpyDeviceToHost, t->st));
        CPFIT_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * w.nu, cudaMemcpyDeviceToHost, t->st));
        CPFIT_CUDA(cudaStreamSynchronize(t->st));
        if (hs & 1)
            throw cpfit_gpu::numerical_error(
                "als_sweep: normal matrix is singular after regularization (structurally rank-deficient iterate)");
        if (hs) throw cpfit_gpu::numerical_error("als_sweep: non-finite solution of the normal equations");
    });
}

int cpfit_accelerate(int64_t n, int64_t m, const double* wu, const double* wg, const double* ub, const double* gb,
                     double eps, double* u_hat, double* alpha, double* residual_rel) {
    return guard([&] {
        if (m < 1) throw std::invalid_argument("accelerate: window must be nonempty");
        cudaStream_t st;
        CPFIT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        struct S {
            cudaStream_t s;
            ~S() { cudaStreamDestroy(s); }
        } sg{st};
        std::unique_ptr<AccelWork, void (*)(AccelWork*)> a(accel_create(n, (int)m), accel_destroy);
        DevBuf b(2 * (size_t)(n * m) + 4 * (size_t)n + 2);
        double* dwu = b.p;
        double* dwg = dwu + n * m;
        double* dub = dwg + n * m;
        double* dgb = dub + n;
        double* duh = dgb + n;
        double* dd_ = duh + n;
        int* ring = reinterpret_cast<int*>(dd_ + n);
        const int hr[2] = {(int)m, 0};
        CPFIT_CUDA(cudaMemcpyAsync(dwu, wu, sizeof(double) * n * m, cudaMemcpyHostToDevice, st));
        CPFIT_CUDA(cudaMemcpyAsync(dwg, wg, sizeof(double) * n * m, cudaMemcpyHostToDevice, st));
        CPFIT_CUDA(cudaMemcpyAsync(dub, ub, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        CPFIT_CUDA(cudaMemcpyAsync(dgb, gb, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        CPFIT_CUDA(cudaMemcpyAsync(ring, hr, sizeof(hr), cudaMemcpyHostToDevice, st));
        accelerate_device(*a, dwu, dwg, ring, dub, dgb, eps, duh, dd_, st);
        CPFIT_CUDA(cudaMemcpyAsync(u_hat, duh, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CPFIT_CUDA(cudaMemcpyAsync(alpha, a->alpha, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
        double sc[3];
        CPFIT_CUDA(cudaMemcpyAsync(sc, a->scal, sizeof(sc), cudaMemcpyDeviceToHost, st));
        CPFIT_CUDA(cudaStreamSynchronize(st));
        *residual_rel = sc[0];
    });
}

int cpfit_more_thuente(cpfit_phi_fn phi, void* ctx, double phi0, double dphi0, const cpfit_line_search_params* p,
                       cpfit_line_search_result* out) {
    return guard([&] {
        if (!(p->ftol > 0.0 && p->ftol < p->gtol && p->gtol < 1.0))
            throw std::invalid_argument("more_thuente: need 0 < ftol < gtol < 1");
        if (!(p->initial_step > 0.0)) throw std::invalid_argument("more_thuente: initial_step must be > 0");
        if (p->max_evals < 1) throw std::invalid_argument("more_thuente: max_evals must be >= 1");
        if (!(p->step_min >= 0.0 && p->step_min < p->step_max))
            throw std::invalid_argument("more_thuente: need 0 <= step_min < step_max");
        MoreThuente mt;
        LsParams lp{p->ftol, p->gtol, p->initial_step, p->max_evals, p->step_min, p->step_max};
        if (mt.begin(lp, phi0, dphi0)) {
            for (;;) {
                double f = 0.0, g = 0.0;
                phi(mt.stp, &f, &g, ctx);
                if (mt.update(f, g)) break;
            }
        }
        *out = cpfit_line_search_result{mt.out_step, mt.out_f, mt.out_g, mt.status, mt.evals};
    });
}

int cpfit_ngmres_solve(cpfit_tensor t, int64_t rank, const double* u0, const cpfit_ngmres_options* o, double* u_best,
                       double* f_best, cpfit_trace_row* trace, int64_t cap, int64_t* rows, int* stop_reason) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        const SolverOptions so = to_opts(o, t->t->norm);
        Solver& sv = t->solver((int)rank, so, 0);
        check_finite(u0, sv.n());
        sv.set_initial(u0, true);
        sv.run_init();
        sv.run_loop(so.max_iters);
        finish_solve(sv, u_best, f_best, trace, cap, rows, stop_reason);
    });
}

int cpfit_als_solve(cpfit_tensor t, int64_t rank, const double* u0, double tol_grad, int max_iters, double* u_best,
                    double* f_best, cpfit_trace_row* trace, int64_t cap, int64_t* rows, int* stop_reason) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        SolverOptions so;
        so.tol_grad = tol_grad;
        so.max_iters = max_iters;
        so.gradient_scale = t->t->norm;  // als.cpp:74 (||g|| / ||T||)
        Solver& sv = t->solver((int)rank, so, 1);
        check_finite(u0, sv.n());
        sv.set_initial(u0, true);
        sv.run_init();
        sv.run_loop(so.max_iters);
        finish_solve(sv, u_best, f_best, trace, cap, rows, stop_reason);
    });
}

int cpfit_ncg_solve(cpfit_tensor t, int64_t rank, const double* u0, double tol_grad, int max_iters,
                    const cpfit_line_search_params* ls, double* u_best, double* f_best, cpfit_trace_row* trace,
                    int64_t cap, int64_t* rows, int* stop_reason) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        if (!(tol_grad > 0.0)) throw std::invalid_argument("ncg: tol_grad must be > 0");  // ncg.cpp:12
        cpfit_ngmres_options o;
        cpfit_default_ngmres_options(&o);
        o.tol_grad = tol_grad;
        o.max_iters = max_iters;
        o.gradient_scale = t->t->norm;  // ncg_solve passes ||T|| (ncg.cpp:119)
        if (ls) {
            o.ftol = ls->ftol;
            o.gtol = ls->gtol;
            o.initial_step = ls->initial_step;
            o.max_evals = ls->max_evals;
            o.step_min = ls->step_min;
            o.step_max = ls->step_max;
        }
        const SolverOptions so = to_opts(&o, t->t->norm);
        Solver& sv = t->solver((int)rank, so, 2);
        check_finite(u0, sv.n());
        sv.set_initial(u0, true);
        sv.run_init();
        sv.run_loop(so.max_iters);
        finish_solve(sv, u_best, f_best, trace, cap, rows, stop_reason);
    });
}

int cpfit_solve_batch(cpfit_tensor t, int64_t rank, int method, int64_t nsolves, const double* u0s,
                      const cpfit_ngmres_options* o, int concurrency, double* u_best, double* f_best, int* iters,
                      int* stop_reason, int64_t* fevals) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        if (method < 0 || method > 2) throw std::invalid_argument("solve_batch: method must be 0, 1 or 2");
        if (nsolves < 0) throw std::invalid_argument("solve_batch: nsolves must be >= 0");
        if (nsolves == 0) return;
        SolverOptions so = to_opts(o, t->t->norm);
        if (method == 2 && !(o->gradient_scale > 0.0)) so.gradient_scale = t->t->norm;
        const int conc = (int)std::max<int64_t>(1, std::min<int64_t>(nsolves, concurrency > 0 ? concurrency : 16));
        std::vector<Solver*> sv = t->batch((int)rank, so, method, conc);
        const int64_t n = sv[0]->n();
        check_finite(u0s, n * nsolves);
        // waves of `conc` solves: every solver's init + loop graphs are queued on its own stream
        // before any result is read back, so the solves of a wave run concurrently
        for (int64_t w0 = 0; w0 < nsolves; w0 += conc) {
            const int64_t w1 = std::min<int64_t>(nsolves, w0 + conc);
            for (int64_t i = w0; i < w1; ++i) {
                Solver& s = *sv[(size_t)(i - w0)];
                s.set_initial(u0s + i * n, true);
                s.run_init();
                s.run_loop(so.max_iters);
            }
            for (int64_t i = w0; i < w1; ++i) {
                Solver& s = *sv[(size_t)(i - w0)];
                const SolverSummary sm = s.summary();
                if (sm.status) throw cpfit_gpu::numerical_error("solve_batch: numerical failure in the ALS normal equations");
                if (u_best) s.copy_best(u_best + i * n, true);
                if (f_best) f_best[i] = sm.best_f;
                if (iters) iters[i] = sm.iters;
                if (stop_reason) stop_reason[i] = (sm.stop < 0) ? 1 : sm.stop;
                if (fevals) fevals[i] = sm.fevals;
            }
            for (Solver* s : sv) s->sync();
        }
    });
}

int cpfit_solver_create(cpfit_tensor t, int64_t rank, const cpfit_ngmres_options* o, int method, cpfit_solver* out) {
    return guard([&] {
        check_rank(rank);
        if (method < 0 || method > 2) throw std::invalid_argument("solver: method must be 0 (N-GMRES), 1 (ALS) or 2 (N-CG)");
        SolverOptions so = to_opts(o, t->t->norm);
        if (method == 1) so.gradient_scale = (o->gradient_scale > 0.0) ? o->gradient_scale : t->t->norm;
        auto h = std::make_unique<cpfit_solver_s>();
        h->s = std::make_unique<Solver>(t->t, (int)rank, so, method);
        CPFIT_CUDA(cudaEventCreate(&h->e0));
        CPFIT_CUDA(cudaEventCreate(&h->e1));
        *out = h.release();
    });
}

int cpfit_solver_set_initial(cpfit_solver s, const double* u0) {
    return guard([&] {
        s->s->set_initial(u0, true);
        s->s->sync();
    });
}

int cpfit_solver_init(cpfit_solver s) {
    return guard([&] {
        s->s->run_init();
        s->s->sync();
    });
}

int cpfit_solver_run(cpfit_solver s, int max_iters_total, float* ms) {
    return guard([&] {
        Solver& sv = *s->s;
        CPFIT_CUDA(cudaEventRecord(s->e0, sv.stream()));
        sv.run_loop(max_iters_total);
        CPFIT_CUDA(cudaEventRecord(s->e1, sv.stream()));
        CPFIT_CUDA(cudaEventSynchronize(s->e1));
        float t = 0.f;
        CPFIT_CUDA(cudaEventElapsedTime(&t, s->e0, s->e1));
        if (ms) *ms = t;
    });
}

int cpfit_solver_restart(cpfit_solver s, const double* u0, int max_iters_total, float* ms) {
    return guard([&] {
        Solver& sv = *s->s;
        sv.set_initial(u0, true);
        sv.sync();
        CPFIT_CUDA(cudaEventRecord(s->e0, sv.stream()));
        sv.run_init();
        sv.run_loop(max_iters_total);
        CPFIT_CUDA(cudaEventRecord(s->e1, sv.stream()));
        CPFIT_CUDA(cudaEventSynchronize(s->e1));
        float t = 0.f;
        CPFIT_CUDA(cudaEventElapsedTime(&t, s->e0, s->e1));
        if (ms) *ms = t;
    });
}

int cpfit_solver_state(cpfit_solver s, int* iters, int* stop_reason, double* f, double* best_f, int64_t* fevals) {
    return guard([&] {
        const SolverSummary sm = s->s->summary();
        if (iters) *iters = sm.iters;
        if (stop_reason) *stop_reason = sm.stop;
        if (f) *f = sm.f;
        if (best_f) *best_f = sm.best_f;
        if (fevals) *fevals = sm.fevals;
        if (sm.status) throw cpfit_gpu::numerical_error("solver: numerical failure in the ALS normal equations");
    });
}

int cpfit_solver_trace(cpfit_solver s, cpfit_trace_row* trace, int64_t rows) {
    return guard([&] { s->s->copy_trace(reinterpret_cast<TraceRow*>(trace), (int)rows); });
}

int cpfit_solver_best(cpfit_solver s, double* u) {
    return guard([&] {
        s->s->copy_best(u, true);
        s->s->sync();
    });
}

int cpfit_solver_launches(cpfit_solver s, int64_t* launches) {
    return guard([&] { *launches = s->s->summary().launches; });
}

int cpfit_line_polynomial(cpfit_tensor t, int64_t rank, const double* u_bar, const double* d, const double* alphas,
                          int64_t n, double* phi, double* dphi) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        if (!cpfit_gpu::poly_supported(*t->t) || rank > cpfit_gpu::kMaxRank)
            throw std::invalid_argument(
                "line polynomial: order-3 (dense or sparse) or dense order-4 tensors, rank <= 32, only");
        if (n < 0) throw std::invalid_argument("line polynomial: n >= 0");
        EvalWork& w = t->work((int)rank);
        check_finite(u_bar, w.nu);
        check_finite(d, w.nu);
        DevBuf b(3 * (size_t)w.nu + 3 * (size_t)std::max<int64_t>(n, 1) + 16);
        double* du = b.p;
        double* dd_ = du + w.nu;
        double* dg = dd_ + w.nu;
        double* da = dg + w.nu;
        double* dphi_d = da + std::max<int64_t>(n, 1);
        double* dd2 = dphi_d + std::max<int64_t>(n, 1);
        EvalScalars* sc = reinterpret_cast<EvalScalars*>(dd2 + std::max<int64_t>(n, 1));
        int* status = reinterpret_cast<int*>(sc + 1);
        CPFIT_CUDA(cudaMemcpyAsync(du, u_bar, sizeof(double) * w.nu, cudaMemcpyHostToDevice, t->st));
        CPFIT_CUDA(cudaMemcpyAsync(dd_, d, sizeof(double) * w.nu, cudaMemcpyHostToDevice, t->st));
        if (n > 0) CPFIT_CUDA(cudaMemcpyAsync(da, alphas, sizeof(double) * n, cudaMemcpyHostToDevice, t->st));
        // the evaluation at u_bar leaves S(u_bar) in w.S
        eval_device(*t->t, w, du, dg, sc, nullptr, status, t->st, true, t->one());
        std::unique_ptr<cpfit_gpu::PolyWork, void (*)(cpfit_gpu::PolyWork*)> pw(cpfit_gpu::poly_create(*t->t, w),
                                                                               cpfit_gpu::poly_destroy);
        cpfit_gpu::poly_build_device(*t->t, w, *pw, du, dd_, t->st);
        if (n > 0) {
            cpfit_gpu::poly_eval_device(*pw, da, (int)n, dphi_d, dd2, t->st);
            CPFIT_CUDA(cudaMemcpyAsync(phi, dphi_d, sizeof(double) * n, cudaMemcpyDeviceToHost, t->st));
            CPFIT_CUDA(cudaMemcpyAsync(dphi, dd2, sizeof(double) * n, cudaMemcpyDeviceToHost, t->st));
        }
        CPFIT_CUDA(cudaStreamSynchronize(t->st));
    });
}

int cpfit_fiber_prof(uint64_t* out, int reset) {
    return guard([&] {
        unsigned long long* b = cpfit_gpu::fiber_prof_buffer();
        CPFIT_CUDA(cudaDeviceSynchronize());
        CPFIT_CUDA(cudaMemcpy(out, b, sizeof(unsigned long long) * cpfit_gpu::kFiberProfSlots, cudaMemcpyDeviceToHost));
        if (reset) CPFIT_CUDA(cudaMemset(b, 0, sizeof(unsigned long long) * cpfit_gpu::kFiberProfSlots));
    });
}

int cpfit_solver_phase_times(cpfit_solver s, double* us, int64_t* visits) {
    return guard([&] {
        if (!s->s->phase_times(us, visits))
            throw std::invalid_argument("phase profiling is off (set CPFIT_PHASE_PROFILE=1 before cpfit_solver_create)");
    });
}

int cpfit_solver_iterate(cpfit_solver s, double* u) {
    return guard([&] {
        s->s->copy_current(u);
        s->s->sync();
    });
}

int cpfit_ngmres_init(cpfit_solver s, const double* u0, double* f) {
    return guard([&] {
        if (s->s->method() != 0) throw std::invalid_argument("ngmres_init: the solver was created for another method");
        check_finite(u0, s->s->n());
        s->s->set_initial(u0, true);
        s->s->run_init();
        const SolverSummary sm = s->s->summary();
        if (f) *f = sm.f;
    });
}

int cpfit_ngmres_step(cpfit_solver s, int* restart, int* stalled, double* beta, double* f) {
    return guard([&] {
        if (s->s->method() != 0) throw std::invalid_argument("ngmres_step: the solver was created for another method");
        const SolverSummary before = s->s->summary();
        if (before.stop >= 0)
            throw std::invalid_argument("ngmres_step: the solve has stopped (gradient tolerance, stalls or budget)");
        s->s->run_loop(before.iters + 1);
        const SolverSummary sm = s->s->summary();
        if (sm.status) throw cpfit_gpu::numerical_error("ngmres_step: numerical failure in the ALS normal equations");
        if (restart) *restart = sm.restart;
        if (stalled) *stalled = sm.stalled;
        if (beta) *beta = sm.beta;
        if (f) *f = sm.f;
    });
}

int cpfit_solver_destroy(cpfit_solver s) {
    return guard([&] { delete s; });
}

}  // extern "C"

namespace {
__global__ void l2_flush_read(const double2* __restrict__ p, int64_t n, double* sink) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = p[i];
        acc += v.x + v.y;
    }
    if (acc == 1.2345e300) *sink = acc;  // never true for the zeroed buffer; keeps the loads
}
}  // namespace

extern "C" {
int cpfit_bench_kernel(cpfit_tensor t, int64_t rank, const double* u, int kind, int mode, int reps, int flush_l2,
                       float* ms_per_call) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(t->mu);
        check_rank(rank);
        EvalWork& w = t->work((int)rank);
        int64_t maxI = 1;
        for (int k = 0; k < t->t->order; ++k) maxI = std::max(maxI, t->t->dims[k]);
        DevBuf b(4 * (size_t)w.nu + (size_t)maxI * rank + 16);
        double* du = b.p;
        double* dg = du + w.nu;
        double* work = dg + w.nu;
        double* dout = work + w.nu;
        double* mbuf = dout + w.nu;
        EvalScalars* sc = reinterpret_cast<EvalScalars*>(mbuf + maxI * rank);
        int* status = reinterpret_cast<int*>(sc + 1);
        CPFIT_CUDA(cudaMemcpyAsync(du, u, sizeof(double) * w.nu, cudaMemcpyHostToDevice, t->st));
        CPFIT_CUDA(cudaMemsetAsync(status, 0, sizeof(int), t->st));
        const size_t flush_bytes = 256ull << 20;  // > 126 MB L2
        DevBuf flush(flush_l2 ? flush_bytes / 8 : 1);
        if (flush_l2) CPFIT_CUDA(cudaMemsetAsync(flush.p, 0, flush_bytes, t->st));
        cudaEvent_t e0, e1;
        CPFIT_CUDA(cudaEventCreate(&e0));
        CPFIT_CUDA(cudaEventCreate(&e1));
        if (kind >= 3 && (rowwise(*t->t) || rank > kMaxRank))
            throw std::invalid_argument("fiber-pass kinds need a dense tensor and rank <= 32");
        if (kind >= 3) grams_device(w, du, t->st);
        auto call = [&] {
            switch (kind) {
                case 0: mttkrp_device(*t->t, w, du, mode, dout, t->st); break;
                case 1: eval_device(*t->t, w, du, dg, sc, nullptr, status, t->st, true, t->one()); break;
                case 7: eval_device(*t->t, w, du, dg, sc, nullptr, status, t->st, true, nullptr); break;
                case 2: als_sweep_device_ws(*t->t, w, du, dout, work, mbuf, status, t->st); break;
                case 3: dense_fiber_fused(*t->t, w, du, t->st, nullptr); break;   // S + M0 + per-fiber f
                case 6: dense_fiber_fused(*t->t, w, du, t->st, t->one()); break;  // S + M0 + residual f
                case 4: dense_fiber(*t->t, w, du, false, true, t->st); break;   // M0 only
                case 5: dense_fiber(*t->t, w, du, true, false, t->st); break;   // S only
                case 8: mttkrp3_last_only(w, du, dout, t->st); break;           // last-mode contraction of S
                default: throw std::invalid_argument("bench kind");
            }
        };
        for (int i = 0; i < 3; ++i) call();
        float total = 0.f;
        for (int i = 0; i < reps; ++i) {
            if (flush_l2) {  // evict L2 by reading a buffer twice its size (no dirty lines left behind)
                l2_flush_read<<<592, 256, 0, t->st>>>(reinterpret_cast<const double2*>(flush.p), flush_bytes / 16,
                                                       flush.p + flush_bytes / 8 - 1);
                CPFIT_CUDA(cudaGetLastError());
            }
            CPFIT_CUDA(cudaEventRecord(e0, t->st));
            call();
            CPFIT_CUDA(cudaEventRecord(e1, t->st));
            CPFIT_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            CPFIT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            total += ms;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_per_call = total / std::max(1, reps);
    });
}

}  // extern "C"
