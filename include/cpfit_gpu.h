/*
 * cpfit_gpu.h — C-ABI of the B200-native cpfit hot path (libcpfit_gpu.so).
 *
 * Drop-in boundary for the reference's solver API in proj/core/include/cpfit/ (C++20,
 * Eigen). Every entry point below replaces one reference function; the citation names the
 * reference declaration it stands for. Conventions:
 *   - host pointers in and out (the library does the H2D/D2H copies); a tensor handle is
 *     uploaded once and keeps T resident in HBM (DataTensor, tensor.hpp:129-148);
 *   - factor sets cross the ABI in the reference's pack() layout (kruskal.cpp:195-206):
 *     factors in mode order, each column-major I_n x R, total length R * sum I_n;
 *   - return codes mirror the reference's exceptions: 0 ok, 1 std::invalid_argument,
 *     2 cpfit::numerical_error (errors.hpp:9-12), 3 CUDA / other failure; the message is
 *     available from cpfit_last_error() (thread-local);
 *   - distinct tensor handles may be used from different threads concurrently.
 * Device limits: order <= 8, rank <= 64 (ranks above 32 on the per-mode path), N-GMRES window <= 112, sparse mode sizes < 2^31,
 * R * sum(I_n) < 2^31. Dense shapes of any mode sizes: the fibre-tile passes take mode-0 lengths
 * up to 416 (order >= 2); order-1 tensors and longer mode-0 fibres run the generic per-mode
 * kernels (csrc/generic.cu) with the same results and error behaviour. Shapes beyond the limits
 * return 1 (std::invalid_argument) at the first call that needs them.
 * Destroyed dense handles are pooled (CPFIT_TENSOR_POOL_MB, default 8192; 0 disables): a new
 * dense tensor of the same shape reuses the device buffers and captured solver graphs.
 */
#ifndef CPFIT_GPU_H
#define CPFIT_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cpfit_tensor_s* cpfit_tensor;
typedef struct cpfit_solver_s* cpfit_solver;

/* trace.hpp:18-29 TraceRecord */
typedef struct {
    int32_t iter;
    int32_t restart;
    double time_s, f, h, gnorm_rel, beta;
    int64_t fevals, gevals, precond_calls;
} cpfit_trace_row;

/* ngmres.hpp:50-57 NgmresOptions + line_search.hpp:7-14 LineSearchParams.
 * gradient_scale: NgmresProblem::gradient_scale (ngmres.hpp:71); <= 0 selects ||T||_F as in
 * ngmres_solve (ngmres.cpp:219). */
typedef struct {
    int32_t window;
    int32_t max_iters;
    double epsilon_reg;
    double tol_grad;
    double gradient_scale;
    double ftol, gtol, initial_step;
    int32_t max_evals;
    int32_t restart_on_ascent;
    double step_min, step_max;
    /* 1: re-evaluate at the canonicalized accepted point (ngmres.cpp:139-140) — one more pass
     * over T per accepted step; 0 (default): map the accepted trial's f and gradient through
     * the exact normalisation rescale (f invariant, G_n -> G_n D_n^-1). Counters are identical. */
    int32_t reeval_accepted;
    /* 1: every evaluation uses the residual objective 1/2 sum (T - model)^2 (kruskal.cpp:83-102,
     * 6KR flops); 0 (default): the per-fiber three-term form (4KR, ~1e-14 relative at h ~ 1e-2)
     * until f stagnates (relative decrease < 1e-8) or h < 1e-3, then the residual form. */
    int32_t residual_objective;
} cpfit_ngmres_options;

/* line_search.hpp:7-14 / 23-29 */
typedef struct {
    double ftol, gtol, initial_step;
    int32_t max_evals;
    double step_min, step_max;
} cpfit_line_search_params;
typedef struct {
    double step, f, dg;
    int32_t status; /* 0 Converged, 1 MaxEvals, 2 NotDescent, 3 NumericalStall */
    int32_t evals;
} cpfit_line_search_result;
typedef void (*cpfit_phi_fn)(double step, double* f, double* dg, void* ctx);

const char* cpfit_last_error(void);
int cpfit_device_count(void);
void cpfit_default_ngmres_options(cpfit_ngmres_options* o);

/* DataTensor(DenseTensor) — tensor.hpp:46-60, 129-148 (values first-mode-fastest). */
int cpfit_tensor_create_dense(int order, const int64_t* dims, const double* values, cpfit_tensor* out);
/* DataTensor(SparseTensor) — tensor.hpp:66-88: coords nnz*N AoS, canonicalised like the
 * reference constructor (tensor.cpp:56-103). */
int cpfit_tensor_create_coo(int order, const int64_t* dims, int64_t nnz, const int64_t* coords,
                            const double* values, cpfit_tensor* out);
int cpfit_tensor_destroy(cpfit_tensor t);
/* DataTensor::norm() — tensor.hpp:139 */
int cpfit_tensor_norm(cpfit_tensor t, double* norm);
/* SparseTensor::nnz() after canonicalisation — tensor.hpp:75 */
int cpfit_tensor_nnz(cpfit_tensor t, int64_t* nnz);

/* DataTensor::mttkrp(factors, mode) — tensor.hpp:142; out is I_mode x R column-major. */
int cpfit_mttkrp(cpfit_tensor t, int64_t rank, const double* u, int mode, double* out);
/* objective(t, k) — kruskal.hpp:36 */
int cpfit_objective(cpfit_tensor t, int64_t rank, const double* u, double* f);
/* objective_and_gradient(t, k, grad) — kruskal.hpp:43; grad in pack() layout. */
int cpfit_objective_and_gradient(cpfit_tensor t, int64_t rank, const double* u, double* grad, double* f);
/* objective_and_gradient with the device's objective form selected: form 0 is the reference's
 * residual form 1/2 sum (T - model)^2 (kruskal.cpp:83-102; what cpfit_objective_and_gradient
 * computes); form 1 is the per-fibre three-term form the solver loop evaluates with until f
 * stagnates (dense tensors; sparse tensors always use the three-term form of kruskal.cpp:146-148).
 * Parity hook for the loop's default objective. */
int cpfit_objective_and_gradient_form(cpfit_tensor t, int64_t rank, const double* u, int form, double* grad,
                                      double* f);
/* gram_hadamard(factors, skip) — tensor.hpp:124; out R x R column-major. */
int cpfit_gram_hadamard(int order, const int64_t* dims, int64_t rank, const double* u, int skip, double* out);
/* normalize_and_reorder(k) — kruskal.hpp:54 */
int cpfit_normalize_and_reorder(int order, const int64_t* dims, int64_t rank, const double* u, double* out);
/* als_sweep(t, k) — als.hpp:14 */
int cpfit_als_sweep(cpfit_tensor t, int64_t rank, const double* u, double* out);
/* accelerate(window, u_bar, g_bar, eps) — ngmres.hpp:44-45. window_u / window_g hold m
 * vectors of length n, oldest first (AccelWindow order, ngmres.hpp:16-35). */
int cpfit_accelerate(int64_t n, int64_t m, const double* window_u, const double* window_g, const double* u_bar,
                     const double* g_bar, double epsilon_reg, double* u_hat, double* alpha, double* residual_rel);
/* more_thuente(eval, phi0, dphi0, params) — line_search.hpp:41-42 (host state machine shared
 * with the device line search). */
int cpfit_more_thuente(cpfit_phi_fn phi, void* ctx, double phi0, double dphi0, const cpfit_line_search_params* p,
                       cpfit_line_search_result* out);
/* ngmres_solve(t, initial, opts) — ngmres.hpp:126-127; the whole solve is device resident.
 * u_best receives the best-f iterate (pack layout), trace up to `cap` rows. */
int cpfit_ngmres_solve(cpfit_tensor t, int64_t rank, const double* u0, const cpfit_ngmres_options* o, double* u_best,
                       double* f_best, cpfit_trace_row* trace, int64_t cap, int64_t* rows, int* stop_reason);
/* als_solve(t, initial, opts) — als.hpp:23 */
int cpfit_als_solve(cpfit_tensor t, int64_t rank, const double* u0, double tol_grad, int max_iters, double* u_best,
                    double* f_best, cpfit_trace_row* trace, int64_t cap, int64_t* rows, int* stop_reason);

/* ncg_solve(t, initial, opts) — ncg.hpp:29 (NcgOptions ncg.hpp:14-18: tol_grad, max_iters,
 * line_search; ls may be NULL for the defaults). Device-resident like cpfit_ngmres_solve;
 * u_best is the best-f iterate, normalised once (ncg.cpp:122). Stalled iterations write no
 * trace row (ncg.cpp:60-67), so *rows can be below iterations + 1. */
int cpfit_ncg_solve(cpfit_tensor t, int64_t rank, const double* u0, double tol_grad, int max_iters,
                    const cpfit_line_search_params* ls, double* u_best, double* f_best, cpfit_trace_row* trace,
                    int64_t cap, int64_t* rows, int* stop_reason);

/* Batched solves (bench.cpp:80-158 runs seeds on a thread pool): nsolves independent solves of
 * the same tensor from the starts u0s (nsolves x n, pack layout), `concurrency` of them in
 * flight at once (<= 0: 16), each on its own stream and workspace. method 0 N-GMRES, 1 ALS,
 * 2 N-CG (gradient_scale <= 0 means ||T|| as in the single-solve calls). Per solve: best
 * iterate (u_best, may be NULL), best f, iterations, stop reason, f evaluations. */
int cpfit_solve_batch(cpfit_tensor t, int64_t rank, int method, int64_t nsolves, const double* u0s,
                      const cpfit_ngmres_options* o, int concurrency, double* u_best, double* f_best, int* iters,
                      int* stop_reason, int64_t* fevals);

/* Persistent solver handle for measurement (the same device loop as cpfit_ngmres_solve,
 * split into init + timed loop launches). method 0: N-GMRES, 1: ALS, 2: N-CG. */
int cpfit_solver_create(cpfit_tensor t, int64_t rank, const cpfit_ngmres_options* o, int method, cpfit_solver* out);
int cpfit_solver_set_initial(cpfit_solver s, const double* u0);
int cpfit_solver_init(cpfit_solver s);
/* runs until max_iters_total iterations (or a stop); *ms = CUDA-event time on the solver stream */
int cpfit_solver_run(cpfit_solver s, int max_iters_total, float* ms);
/* new start point (host), init (canonicalize + evaluate + seed window) and run; *ms covers
 * init + loop on the solver stream */
int cpfit_solver_restart(cpfit_solver s, const double* u0, int max_iters_total, float* ms);
int cpfit_solver_state(cpfit_solver s, int* iters, int* stop_reason, double* f, double* best_f, int64_t* fevals);
int cpfit_solver_trace(cpfit_solver s, cpfit_trace_row* trace, int64_t rows);
int cpfit_solver_best(cpfit_solver s, double* u);
/* current (last accepted, canonical) iterate */
int cpfit_solver_iterate(cpfit_solver s, double* u);
/* ngmres_init(problem, initial, opts) — ngmres.hpp:101-103, for the CP problem ngmres_solve builds
 * (ngmres.cpp:209-222) on a method-0 solver: canonicalize, evaluate, seed the window; *f = f(u).
 * The state (NgmresState, ngmres.hpp:92-99: u, g, f, window, counters) stays on the device. */
int cpfit_ngmres_init(cpfit_solver s, const double* u0, double* f);
/* ngmres_step(problem, state, opts) — ngmres.hpp:109-117: one device iteration; the
 * NgmresStepReport (restart, stalled, beta) and the accepted f. The device loop also applies
 * ngmres_minimize's stop tests (ngmres.cpp:185-197): a step after a stop returns 1. */
int cpfit_ngmres_step(cpfit_solver s, int* restart, int* stalled, double* beta, double* f);
int cpfit_solver_destroy(cpfit_solver s);

/* kernels of this library launched by the solver's loop graphs since cpfit_solver_init
 * (counted from the captured graph bodies x the device-side iteration / line-search counters) */
int cpfit_solver_launches(cpfit_solver s, int64_t* launches);
/* phi(a) = f(u_bar + a d) and phi'(a) = g(u_bar + a d).d at the n steps alphas[], evaluated from
 * the degree-6 polynomial the device line search uses (dense order-3 tensors; the reference
 * evaluates objective_and_gradient at each trial, ngmres.cpp:113-126). Parity / diagnostics. */
int cpfit_line_polynomial(cpfit_tensor t, int64_t rank, const double* u_bar, const double* d, const double* alphas,
                          int64_t n, double* phi, double* dphi);
/* Diagnostic: fiber-pass barrier-wait cycles by role (12 counters; nonzero only in a library
 * built with -DCPFIT_FIBER_PROF, see tools/fiber_prof.py); reset != 0 clears them. */
int cpfit_fiber_prof(uint64_t* out, int reset);
/* Diagnostic: per-phase device time of the solver loop (8 phases: ALS sweep, eval(u_bar),
 * accelerate + LS init, LS trial eval, LS update, accepted step, commit, loop re-entry), in us,
 * and visit counts. Only when CPFIT_PHASE_PROFILE=1 was set before cpfit_solver_create (the
 * stamps add one tiny kernel per phase); otherwise returns 1 (invalid_argument). */
int cpfit_solver_phase_times(cpfit_solver s, double* us, int64_t* visits);

/* Device-resident kernel timing (inputs already in HBM): average ms per call over `reps`
 * calls timed with CUDA events on the launching stream, L2 flushed between calls when
 * flush_l2 != 0. kind: 0 mttkrp(mode), 1 objective_and_gradient, 2 als_sweep,
 * 3 fused fiber pass alone (S + M0 + per-fiber f), 4 fiber pass M0 only, 5 fiber pass S only. */
int cpfit_bench_kernel(cpfit_tensor t, int64_t rank, const double* u, int kind, int mode, int reps, int flush_l2,
                       float* ms_per_call);

/* Diagnostic: in the guard-band build (make guard, -DCPFIT_GUARD) every device allocation carries
 * 4 KB guard bands; checks them all now. *violations = guard bands found changed so far (frees
 * included), -1 when this is not a guard build; *live_allocations = device buffers alive. */
int cpfit_debug_guard_check(int64_t* violations, int64_t* live_allocations);

/* fp64 peaks measured on the current device (DMMA m8n8k4 and DFMA issue loops), TFLOP/s */
int cpfit_measure_fp64_peak(double* dmma_tflops, double* dfma_tflops);
/* page-lock / unlock a host buffer (pinned H2D copies for end-to-end runs) */
int cpfit_host_register(void* p, int64_t bytes);
int cpfit_host_unregister(void* p);

#ifdef __cplusplus
}
#endif
#endif /* CPFIT_GPU_H */
