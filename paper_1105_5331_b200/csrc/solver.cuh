// Device-resident CP solvers (C++ side of the C-ABI; see solver.cu).
#pragma once

#include "device.cuh"

#include <algorithm>

namespace cpfit_gpu {

// Mirrors cpfit::NgmresOptions (ngmres.hpp:50-57) + LineSearchParams (line_search.hpp:7-14)
// and AlsOptions (als.hpp:16-19); gradient_scale is NgmresProblem::gradient_scale.
struct SolverOptions {
    int window = 20;
    int max_iters = 2000;
    double epsilon_reg = 1e-12;
    double tol_grad = 1e-9;
    double gradient_scale = 1.0;
    double ftol = 1e-4, gtol = 1e-2, initial_step = 1.0;
    int max_evals = 20;
    double step_min = 0.0, step_max = 1e20;
    int restart_on_ascent = 1;
    // 1: re-evaluate at the canonicalized accepted point as ngmres.cpp:139-140 does;
    // 0: map the accepted trial's (f, g) through the exact normalisation rescale (default)
    int reeval_accepted = 0;
    // 1: every evaluation uses the residual objective (kruskal.cpp:83-102); 0: per-fiber
    // three-term form until f stagnates, then residual (sticky)
    int residual_objective = 0;

    // a solver built for *this can run a solve with options o (graphs bake in everything but
    // the iteration budget, which only needs to fit the trace buffer)
    bool serves(const SolverOptions& o) const {
        return window == o.window && o.max_iters <= std::max(max_iters, 2000) && epsilon_reg == o.epsilon_reg &&
               tol_grad == o.tol_grad && gradient_scale == o.gradient_scale && ftol == o.ftol && gtol == o.gtol &&
               initial_step == o.initial_step && max_evals == o.max_evals && step_min == o.step_min &&
               step_max == o.step_max && restart_on_ascent == o.restart_on_ascent &&
               reeval_accepted == o.reeval_accepted && residual_objective == o.residual_objective;
    }
};

// One trace row (trace.hpp:18-29); layout shared with the C-ABI cpfit_trace_row.
struct TraceRow {
    int32_t iter;
    int32_t restart;
    double time_s, f, h, gnorm_rel, beta;
    int64_t fevals, gevals, precond_calls;
};

struct SolverSummary {
    int iters, stop, status;
    double f, best_f;
    long long fevals, gevals;
    long long launches;  // kernels launched by the loop graphs since init
    int rows;            // trace rows written (N-CG writes none for stalled iterations)
    int restart, stalled;  // the last iteration's NgmresStepReport (ngmres.hpp:109-113)
    double beta;
};

class Solver {
public:
    // method 0: ALS-preconditioned N-GMRES, 1: stand-alone ALS, 2: N-CG (ncg.cpp)
    Solver(DevTensor* t, int R, const SolverOptions& o, int method);
    ~Solver();
    void set_initial(const double* u0, bool host);
    void run_init();
    void run_loop(int max_iters_total);
    void sync();
    SolverSummary summary();
    void copy_trace(TraceRow* out, int rows);
    void copy_best(double* out, bool host);
    void copy_current(double* out);
    // CPFIT_PHASE_PROFILE=1 at construction: globaltimer stamps between the phases of each
    // iteration; out[k] = accumulated us, cnt[k] = visits (kPhases entries each)
    static constexpr int kPhases = 8;
    bool phase_times(double* out, int64_t* cnt);
    cudaStream_t stream() const { return st_; }
    int rank() const { return R_; }
    int method() const { return method_; }
    const SolverOptions& options() const { return opt_; }
    int64_t n() const { return n_; }

private:
    void construct(DevTensor* t, int R, const SolverOptions& o);
    void release();
    void build_graphs();
    void run_loop_eager();
    void emit_poly_accept(cudaStream_t st, const void* ctl);
    void emit_bar(cudaStream_t st, const void* ctl);
    void emit_ncg_end(cudaStream_t st, const void* ctl, unsigned long long loop_h);
    void emit_ncg_poly(cudaStream_t st, const void* ctl);
    PolyWork* pw_ = nullptr;  // exact line search (poly.cu), when it applies
    bool gout_ = false;       // normalisations hand on their output's Grams
    bool defer_ = false;      // eval at the sweep's own point, then normalise (no S rescale)
    int norm_nb_ = 0;         // normalize_grad blocks (partials of ||g_bar||^2 in red_)
    double* gram_bar_ = nullptr;
    int64_t gram_n() const { return (int64_t)w_->order * w_->RP * w_->RP; }
    size_t gram_bytes() const { return sizeof(double) * (size_t)gram_n(); }
    int n_poly_ = 0, n_accp_ = 0, n_direct_ = 0;
    bool eager_ = false;
    alignas(16) unsigned char ctl_blob_[512] = {};  // the control-kernel parameters (solver.cu Ctl)
    DevTensor* t_;
    int R_;
    SolverOptions opt_;
    int method_;
    EvalWork* w_ = nullptr;
    AccelWork* a_ = nullptr;
    int64_t n_ = 0;
    int cap_ = 1;
    cudaStream_t st_{}, st2_{}, st3_{}, st4_{};
    double *u_ = nullptr, *g_ = nullptr, *ub_ = nullptr, *gb_ = nullptr, *d_ = nullptr, *ut_ = nullptr,
           *gt_ = nullptr, *un_ = nullptr, *gn_ = nullptr, *u0_ = nullptr, *ubest_ = nullptr, *work_ = nullptr,
           *mbuf_ = nullptr, *wu_ = nullptr, *wg_ = nullptr, *ubl_ = nullptr, *gbl_ = nullptr, *red_ = nullptr;
    // dense N-GMRES: M0 = T x KR(modes >= 1) at u (cur), u_bar (bar), the best trial (best) and
    // the accepted trial (sel), so the ALS sweep reuses the evaluation's mode-0 contraction
    double *m0_cur_ = nullptr, *m0_bar_ = nullptr, *m0_best_ = nullptr, *m0_sel_ = nullptr;
    // where an evaluation leaves M0: w.m0 ([RP][32 nchunk], fibre passes) or the mode-0 block of
    // w.sp_part ([I_0][RP], rowwise tensors)
    double* m0_src() const { return w_->m0_rowwise ? w_->sp_part : w_->m0; }
    int64_t m0_n_ = 0;
    unsigned long long* phase_ = nullptr;  // [kPhases] ns, [kPhases] counts, [1] last stamp
    void* sc_ = nullptr;
    void* state_ = nullptr;
    TraceRow* trace_ = nullptr;
    int trace_cap_ = 0;
    int host_max_ = 0;
    int n_prelude_ = 0, n_body_ = 0, n_ls_ = 0, n_acc_ = 0, n_init_ = 0;
    long long init_launches_ = 0, launches_done_ = 0;
    long long pending_loop_launches();
    long long loop_launches_ = 0;
    cudaGraph_t g_init_ = nullptr, g_loop_ = nullptr;
    cudaGraphExec_t x_init_ = nullptr, x_loop_ = nullptr;
};

}  // namespace cpfit_gpu
