// Internal device-side API of the cpfit B200 path (not part of the C-ABI).
//
// Data layout in HBM:
//   * dense T: first-mode-fastest like the reference (tensor.hpp:42-60), but each mode-0
//     fiber is padded to ldT = round_up(I_0, 4) doubles (zeros) so every fiber starts
//     32-byte aligned and can be moved by one bulk async copy;
//   * iterates u / gradients g: the reference's packed layout (pack(), kruskal.cpp:195-206):
//     factors in mode order, each column-major — vectors cross the C-ABI unchanged;
//   * S = T x_1 A^(0) (per mode-0 fiber, RP doubles, row-major [fiber][r]) is materialised
//     by the fiber pass and consumed by the level contractions for modes >= 1;
//   * sparse T: canonical COO (sorted lexicographically, tensor.cpp:56-103) uploaded as
//     structure-of-arrays int64 indices + fp64 values.
#pragma once

#include "common.cuh"
#include "gram.cuh"

#include <vector>

namespace cpfit_gpu {

struct DevTensor {
    int order = 0;
    int64_t dims[kMaxOrder] = {};
    int64_t K = 0;
    bool sparse = false;
    // dense, but evaluated per mode by the generic kernels (generic.cu) like a sparse tensor:
    // order 1, or mode-0 fibres too long for the fibre tiles (see fiber_path_fits)
    bool generic = false;
    double norm = 0.0, norm_sq = 0.0, norm_sq_lo = 0.0;  // ||T||^2 = norm_sq + norm_sq_lo (dense)
    // the same three scalars in device memory: captured graphs read them from here, so a
    // pooled tensor refilled with new values (capi.cu) keeps its graphs valid
    double* dscal = nullptr;
    // dense
    double* T = nullptr;
    int64_t ldT = 0;  // padded fiber stride
    int64_t J = 0;    // number of mode-0 fibers (K / I_0)
    double* fiber_norm2 = nullptr;  // ||t_f||^2 per fiber (dd-accurate), for the per-fiber objective
    // sparse: canonical nnz and the per-mode sorted copies (sparse.cuh)
    int64_t nnz = 0;
    struct SparseModes* modes = nullptr;
};

// per-mode ("rowwise") evaluation: sparse tensors and generic dense tensors
inline bool rowwise(const DevTensor& t) { return t.sparse || t.generic; }
// the fibre-tile passes take a dense tensor of this order and mode-0 length for every rank
bool fiber_path_fits(int order, int64_t I0);

int sm_count();  // SMs of the current device (cached)
struct EvalWork;
// slab.cu: the M0 pass of short-fibre tensors with 16 | I_1 (false: shape does not qualify)
// resid_flag: a device flag; when nonzero at run time the slab kernels exit without writing
bool dense_m0_slab(const DevTensor& t, EvalWork& w, const double* u, cudaStream_t st, const int* resid_flag);
bool m0_slab_applies(const DevTensor& t, const EvalWork& w);
// the per-fibre objective partials (w.f_part) of the slab shapes with S given
void dense_fobj_slab(const DevTensor& t, EvalWork& w, const double* u, const double* S, const double* gamma0,
                     cudaStream_t st, const int* resid_flag);
// fiber-pass barrier-wait counters (filled only by a -DCPFIT_FIBER_PROF build)
constexpr int kFiberProfSlots = 12;
unsigned long long* fiber_prof_buffer();

DevTensor* tensor_create_dense(int order, const int64_t* dims, const double* host_vals, cudaStream_t st);
DevTensor* tensor_create_coo(int order, const int64_t* dims, int64_t nnz, const int64_t* coords_aos,
                             const double* vals, cudaStream_t st);
void tensor_destroy(DevTensor* t);
// new values into an existing dense tensor of the same shape (upload, finite check, norms)
void tensor_fill_dense(DevTensor& t, const double* host_vals, cudaStream_t st);

// last-block-done counters (one per kernel family; each resets its own after use)
constexpr int kLvlCounters = 1024;
constexpr int kCounterGrad = 0, kCounterGram = 1, kCounterSolve = 2, kCounterNorm = 3, kCounters = 4;
// normalisations can hand on the Grams of their output when order * RP^2 <= kGramsOutMax
constexpr int kGramsOutMax = 4096;

// Scratch for one evaluation context (sized from tensor + rank).
struct EvalWork {
    int R = 0, RP = 0;
    int64_t nu = 0;              // R * sum I_n
    int order = 0;
    int64_t dims[kMaxOrder] = {};
    int64_t off[kMaxOrder + 1] = {};  // packed offsets (R * prefix sum)
    // dense fiber pass
    int fiber_grid = 0, fiber_F = 16, fiber_nchunk = 0, fiber_nst = 3;
    // short fibres (row pitch <= 256 doubles): one TMA box of 16 fibres per tile instead of 16
    // bulk copies, for the fused/M0 kernel's pitch and the S pass's pitch
    bool fiber_tmap = false;
    int sreg_groups = 0;  // S pass tile groups for short fibres (0: K split)
    CUtensorMap tmap_fws{}, tmap_sreg{};
    // slab M0 pass (slab.cu): a box of 16 fibres x half a (padded) row; -1 not tried, 0 none, 1 ok
    CUtensorMap tmap_slab{};
    int slab_tmap = -1;
    size_t fiber_smem = 0;
    double* S = nullptr;        // J x RP
    double* S2 = nullptr;       // (dense order 3) a second J x RP right after S: the line search's S_d
    double* m0_part = nullptr;  // fiber_grid x RP x (32*nchunk)
    double* f_part = nullptr;   // fiber_grid (+ sparse/other scalars)
    double* m0 = nullptr;       // reduced M0 [RP][32*nchunk]
    // level contractions (modes 1..N-2 heads)
    int lvl_nx[kMaxOrder] = {}, lvl_ny[kMaxOrder] = {}, lvl_km[kMaxOrder] = {};  // grid, pairs/thread
    int64_t lvl_spc[kMaxOrder] = {};   // slabs per CTA
    bool lvl_bulk[kMaxOrder] = {};     // the last level: bulk-copy kernel (grid ny x nx)
    double* lvl_part[kMaxOrder] = {};  // M_h partials (nx x I_h x RP)
    double* lvl_spart[kMaxOrder] = {}; // Sout partials over pair chunks (ny x Jt x RP; ny > 1 only)
    double* lvl_m[kMaxOrder] = {};     // reduced M_h [i][r]
    double* lvl_S[kMaxOrder] = {};     // S_{h} outputs (slabs x RP)
    unsigned int* counter = nullptr;   // last-block-done counters [kCounters]
    unsigned int* lvl_cnt = nullptr;   // per pair tile counters of the level kernel's M finish
    // Grams (gram.cuh): per-mode row chunks, dd partials [global chunk][R(R+1)/2]
    int gram_nchunk[kMaxOrder] = {}, gram_chunk0[kMaxOrder] = {};
    dd* gram_part = nullptr;
    double* gram = nullptr;     // [mode][RP*RP] (rounded from dd; padded entries 0)
    // sparse
    double* sp_part = nullptr;  // per-mode outputs I_n x RP
    bool m0_rowwise = false;    // M0 of an evaluation lives in sp_part ([i][RP]), not m0 ([RP][ld])
    double* frows = nullptr;    // row-major RP-padded factor copies (sum I_n x RP)
    // generic dense (generic.cu): column-range partials of one mode, residual partials count
    double* gen_part = nullptr;
    int gen_fgrid = 0;
    // reductions
    double* red = nullptr;      // per-CTA partials for norms/dots
    double* rg_red = nullptr;   // reduce_grad block partials [rg_blocks][3] (dense)
    int64_t rg_blocks = 0;
    int red_grid = 0;
    // ALS: Cholesky factors of Gamma_n per mode (als.cu chol_kernel) and the side stream the
    // factorisations run on, overlapping the streaming passes
    double* chol = nullptr;
    int64_t chol_stride = 0;
    int* nperm = nullptr;            // last normalisation: permutation, mode-0 scales
    double* nscale0 = nullptr;
    dd* solve_part = nullptr;        // per-mode Gram partials of the ALS solves
    int64_t solve_part_stride = 0;   // dd per mode ([blocks][npair])
    cudaStream_t side = nullptr;
    cudaEvent_t ev_gram = nullptr;  // finalize_gram_side done
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

EvalWork* work_create(const DevTensor& t, int R);
void work_destroy(EvalWork* w);

// Device scalars written by the evaluation and read by control kernels.
struct EvalScalars {
    double f;      // objective
    double gnorm2; // ||g||^2
    double gdotd;  // g . d (when a direction is supplied)
    double inner;  // <M0, A0>
};

// objective_and_gradient (kruskal.cpp:127-149) at device iterate u; writes g (packed),
// scalars->f, ->gnorm2 and (if d != nullptr) ->gdotd.  Grams of u are computed first.
// mode = 0 gradient+f; mode = 1 f only (objective()).
// grad_dep (dense, order >= 3): an event the gradient step waits for (a Gram finalised beside
// the T pass)
void eval_device(const DevTensor& t, EvalWork& w, const double* u, double* g, EvalScalars* sc, const double* d,
                 int* status, cudaStream_t st, bool need_grad = true, const int* resid_flag = nullptr,
                 bool s_given = false, bool grams_given = false, cudaEvent_t grad_dep = nullptr,
                 int rowwise_skip = -1);
// rowwise tensors: M0 at u_bar + beta d from the four mixed mode-0 products the sparse line
// contractions leave (PolyWork::m0xy): AA + beta (AD + DA) + beta^2 DD -> w.sp_part (mode 0)
void sparse_m0_at_point(EvalWork& w, const double* m0xy, int64_t I0, const double* beta, cudaStream_t st);

// mttkrp(T, factors(u), mode) (tensor.cpp:206-259) -> out (I_mode x R col-major).
void mttkrp3_last_only(EvalWork& w, const double* u, double* out, cudaStream_t st);
void mttkrp_device(const DevTensor& t, EvalWork& w, const double* u, int mode, double* out, cudaStream_t st);

// Grams G_n = A_n^T A_n for all modes (double-double accumulation) -> w.gram.
void grams_device(EvalWork& w, const double* u, cudaStream_t st);
// gram_hadamard(factors(u), skip) (tensor.cpp:261-274) -> out (R x R col-major), from w.gram.
void gram_hadamard_device(EvalWork& w, int skip, double* out, cudaStream_t st);
// normalize_and_reorder (kruskal.cpp:156-193): u -> out, Grams in w.gram updated to match.
// out_grams: leave the Grams of out in w.gram (rescaled/permuted input Grams)
void normalize_device(EvalWork& w, const double* u, double* out, cudaStream_t st, int pending = -1,
                      bool save_perm = false, bool out_grams = false);
// normalize u -> uout and map the gradient g at u to the normalised point (G_n D_n^-1,
// permuted) -> gout; writes per-block partial ||gout||^2 to red, returns the block count.
// save_perm: the permutation and mode-0 scales into w.nperm / w.nscale0; gram_copy: a second
// copy of the output Grams (with out_grams)
int normalize_grad_device(EvalWork& w, const double* u, const double* g, double* uout, double* gout, double* red,
                          cudaStream_t st, const double* m0 = nullptr, double* m0out = nullptr, bool out_grams = false,
                          bool save_perm = false, double* gram_copy = nullptr);
// One ALS sweep (als.cpp:38-48): u -> out (normalized); work: n_u scratch, mbuf: max I_n x R
// scratch. status: bit0 singular normal matrix after the ridge retry, bit1 non-finite solve.
// keep_s: leave S(out) = T x_1 A0(out) in w.S (dense; for an evaluation with s_given)
// grams_given: w.gram already holds the Grams of u; then the Grams of out are left in w.gram
// defer_norm (dense): stop before the normalisation — the unnormalised sweep result stays in
// work with S' = T x_1 A0' in w.S and its Grams in w.gram except the last mode's, still in
// solve partials (finalize_gram_side); out is not written.
void als_sweep_device_ws(const DevTensor& t, EvalWork& w, const double* u, double* out, double* work, double* mbuf,
                         int* status, cudaStream_t st, const double* m0_given = nullptr, bool keep_s = false,
                         bool grams_given = false, bool defer_norm = false);
void gram_mode_device(EvalWork& w, const double* u, int mode, cudaStream_t st);
// G_mode <- its pending ALS-solve partials, one block on w.side after the work queued on st;
// records `done` on w.side
void finalize_gram_side(EvalWork& w, int mode, cudaStream_t st, cudaEvent_t done);

// Dense pieces for the exact line search (poly.cu): S = T x_1 A (first factor of u) into S_out;
// and the evaluation at u when T x_1 A0(u) = w.S (+ *beta Sd when Sd is given) (order 3: M0
// pass + level + gradient; scalars->f is NOT the objective — the caller supplies it).
void dense_s_pass(const DevTensor& t, EvalWork& w, const double* u, double* S_out, cudaStream_t st);
// perm / sc0: w.S holds S' with S(u_bar)[j][r] = S'[j][perm r] sc0[r] (the iterate's
// normalisation after the evaluation; null: w.S is S(u_bar) itself)
void eval_given_s_device(const DevTensor& t, EvalWork& w, const double* u, double* g, EvalScalars* sc,
                         cudaStream_t st, const double* Sd = nullptr, const double* beta = nullptr,
                         bool grams_given = false, const int* perm = nullptr, const double* sc0 = nullptr);

// Exact line search along d for order-3 dense tensors (poly.cu): phi(a) = f(u_bar + a d) is a
// degree-6 polynomial whose coefficients follow from S(u_bar) (in w.S), S_d = T x_1 D0, the
// factor/direction Grams and ||T||^2; they are built in double-double.
struct PolyWork {
    int64_t nchunk_total = 0;
    double* S_d = nullptr;    // J x RP
    dd* gpart = nullptr;      // cross-Gram task partials
    dd* grams = nullptr;      // [3 modes][3 kinds AA, AD, DD][RP*RP]
    dd* s8part = nullptr;     // per-block partials of the 8 contractions
    dd* s8 = nullptr;         // the 8 contractions <T, [[X0, X1, X2]]>
    dd* coef = nullptr;       // phi coefficients [7]
    unsigned int* counter = nullptr;
    int s8_grid = 0;
    double* drows = nullptr;  // sparse: row-major copy of d's factors
    double* m0xy = nullptr;   // sparse: the mode-0 products with (X1, X2) in {AA, AD, DA, DD} [4][I0][RP]
    // the cross Grams run beside the S_d pass on their own stream (graph branch)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};
bool poly_supported(const DevTensor& t);
constexpr int kSparseLineBlocks = 592;
// sparse order 3: the eight contractions of the line polynomial into part[nblocks][8] (sparse.cu)
void sparse_line_contractions(const DevTensor& t, EvalWork& w, const double* ub, const double* d, double* drows,
                              dd* part, int nblocks, cudaStream_t st, double* m0xy = nullptr);
PolyWork* poly_create(const DevTensor& t, const EvalWork& w);
void poly_destroy(PolyWork* p);
// coefficients of phi from u_bar (its S in w.S) and d
// (perm / sc0 as for eval_given_s_device)
void poly_build_device(const DevTensor& t, EvalWork& w, PolyWork& pw, const double* ub, const double* d,
                       cudaStream_t st, const int* perm = nullptr, const double* sc0 = nullptr);
// the accepted point u* = u_bar + beta d (beta on the device) and its Grams (into w.gram) from
// the double-double cross Grams of the last build: A^T A + beta (A^T D + D^T A) + beta^2 D^T D
void poly_point_device(EvalWork& w, const PolyWork& pw, const double* ub, const double* d, const double* beta,
                       double* ut, cudaStream_t st);
// phi(alphas[i]), phi'(alphas[i]) (device arrays)
void poly_eval_device(const PolyWork& pw, const double* alphas, int n, double* phi, double* dphi, cudaStream_t st);

// Routing with the workspace's rank: ranks above kMaxRank (RP = 64) take the per-mode path on
// every tensor (a dense one through the generic kernels, csrc/generic.cu)
inline bool rowwise(const DevTensor& t, const EvalWork& w) { return rowwise(t) || w.RP > kMaxRank; }
inline bool generic_dense(const DevTensor& t, const EvalWork& w) { return t.generic || (!t.sparse && w.RP > kMaxRank); }

// Accelerate (ngmres.cpp:27-63) on device.
struct AccelWork {
    int64_t n = 0;
    int cap = 0;
    int leaf_grid = 0, leaf_rows = 0;
    double* rbuf[2] = {nullptr, nullptr};
    double* alpha = nullptr;  // cap
    double* scal = nullptr;   // [0] residual_rel, [1] slope, [2] delta, [3] m
    double* red = nullptr;
};
AccelWork* accel_create(int64_t n, int cap);
void accel_destroy(AccelWork* a);
// Window as ring slots: wu/wg base pointers with slot stride n; order[j] = slot of j-th
// oldest entry; m entries (device int). Produces uhat and d = uhat - ubar, slope = gbar.d.
// slope_by_caller: leave slope = sum of a.red[0 .. accel_update_blocks(a)) to the caller
void accelerate_device(AccelWork& a, const double* wu, const double* wg, const int* ring, const double* ub,
                       const double* gb, double eps, double* uhat, double* d, cudaStream_t st,
                       bool slope_by_caller = false);
inline int accel_update_blocks(const AccelWork& a) { return (int)std::min<int64_t>(1024, (a.n + 255) / 256); }

}  // namespace cpfit_gpu
