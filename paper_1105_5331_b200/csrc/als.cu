// ALS preconditioner M(.) on device (als.cpp:16-48) and normalize_and_reorder
// (kruskal.cpp:156-193).
//
// One sweep is Gauss-Seidel over modes 0..N-1 exactly as the reference; the dense
// right-hand sides come from a dimension tree instead of N independent MTTKRPs:
//   mode 0      : tail contraction of T with KR(A1..A_{N-1})          (T pass 1)
//   mode 1      : S' = T x_1 A0'  (stored) then the level contraction   (T pass 2)
//   modes >= 2  : level contractions of S' with the freshly solved heads (no T pass)
// so a sweep streams T twice instead of N times. The R x R normal matrix
// Gamma_n = *_{m!=n} A_m^T A_m is factored by a one-warp left-looking Cholesky in the column
// order of Eigen's unblocked LLT, with the reference's one ridge retry (1e-12 * trace) before
// reporting numerical failure; the factorisation of Gamma_n runs on a side stream while the
// pass producing M_n streams (its Grams are final once mode n-1 is solved).
#include "device.cuh"


#include <algorithm>

#ifdef CPFIT_NORM_STAMPS
__device__ unsigned long long g_norm_stamps[32];
#define NSTAMP(k)                                                                              \
    do {                                                                                       \
        if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) {            \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
            g_norm_stamps[(blockIdx.x == 0 ? 0 : 16) + (k)] = t_;                              \
        }                                                                                      \
    } while (0)
#define NSTAMPL(k)                                                                             \
    do {                                                                                       \
        if (threadIdx.x == 0) {                                                                \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
            g_norm_stamps[k] = t_;                                                             \
        }                                                                                      \
    } while (0)
extern "C" int cpfit_debug_norm_stamps(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_norm_stamps, sizeof(unsigned long long) * 32);
}
#else
#define NSTAMP(k) \
    do {          \
    } while (0)
#define NSTAMPL(k) \
    do {           \
    } while (0)
#endif

namespace cpfit_gpu {


void dense_fiber(const DevTensor& t, EvalWork& w, const double* u, bool do_s, bool do_m0, cudaStream_t st);
void dense_level(const DevTensor& t, EvalWork& w, int h, const double* Sin, const double* u, bool do_m, bool do_s,
                 double* Sout, cudaStream_t st, bool defer);
void gather_m(int64_t In, EvalWork& w, const double* part, int grid, int ld, int layout, double* out,
              cudaStream_t st);
void gram_mode_device(EvalWork& w, const double* u, int mode, cudaStream_t st);
void rowwise_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st,
                   int skip_mode = -1);

namespace {

// Mode update (als.cpp:38-48 for one mode) in two kernels:
//   chol_kernel       finalise the Gram the previous mode's solve left as block partials,
//                     Gamma_n = *_{m != n} G_m, and its Cholesky factor;
//   solve_gram_kernel A_n <- M_n Gamma_n^-1 (RP lanes per row, substitution by shuffles) and
//                     per-block dd partials of the Gram of the new A_n.
// The factorisation is a serial chain of R reciprocal square roots, so it runs on a side stream
// as soon as the Grams it needs exist, overlapping the streaming pass that produces M_n; the
// solve has no grid-wide step (its Gram is finished by the next consumer).
constexpr int kCholThreads = 256;
constexpr int kSolveThreads = 256;
constexpr int kSolveWideRows = 64;  // rows per block step of solve_gram_wide_kernel (ranks > 32)
constexpr int kSolveMaxBlocks = 148;

struct GramPending {
    int mode;          // mode whose Gram is still in block partials (-1: none)
    const dd* part;    // [nblk][npair]
    int nblk;
};

struct CholParams {
    int order, R, RP, mode;
    double* gram;        // [mode][RP*RP] (the pending mode is finalised in place)
    GramPending pend;
    double* fac;         // [R*R] L row-major, [R] 1 / l_kk, [1] ok flag (1.0 / 0.0)
    int* status;
};

// dd sum over blocks (in order) of one Gram pair, loads batched ahead of the serial chain
__device__ __forceinline__ double pending_pair(const GramPending& g, int npair, int p) {
    constexpr int B = 32;  // one round of loads in flight for the usual <= 32 partials
    dd s{0.0, 0.0};
    for (int b0 = 0; b0 < g.nblk; b0 += B) {
        dd v[B];
#pragma unroll
        for (int j = 0; j < B; ++j) v[j] = (b0 + j < g.nblk) ? g.part[(size_t)(b0 + j) * npair + p] : dd{0.0, 0.0};
#pragma unroll
        for (int j = 0; j < B; ++j)
            if (b0 + j < g.nblk) s = dd_add(s, v[j]);
    }
    return s.hi + s.lo;
}
// all threads of the block: G_pending <- rounded sum of its partials (pads zero)
__device__ void finalize_pending(const GramPending& g, int R, int RP, double* gram) {
    if (g.mode < 0) return;
    const int npair = R * (R + 1) / 2;
    double* out = gram + (size_t)g.mode * RP * RP;
    gram_zero_pads(R, RP, out);
    for (int p = threadIdx.x; p < npair; p += blockDim.x) {
        const double v = pending_pair(g, npair, p);
        int r, q;
        pair_rq(p, R, r, q);
        out[r * RP + q] = v;
        out[q * RP + r] = v;
    }
}

// Left-looking LLT (Eigen's unblocked llt_inplace order: l_ik = (g_ik - sum_{j<k} l_ij l_kj)
// / l_kk, j ascending; the pivot likewise, the ridge added to g_kk first), one warp: lane i
// keeps row i of Gamma and of L in registers and receives row k by shuffles, so a column costs
// one k-long DFMA chain plus one reciprocal square root. The division by l_kk = sqrt(x) is a
// multiplication by rsqrt(x) (<= 1 ulp from the quotient) and l_kk = x rsqrt(x). Returns false
// (uniformly) on a pivot <= 0; a NaN pivot passes as in Eigen and surfaces as a non-finite solve.
template <int RP>
__device__ bool warp_llt(const double (&gr)[RP], double (&lr)[RP], double& dinv, int R, double ridge) {
    const int lane = threadIdx.x & 31;
    bool ok = true;
#pragma unroll
    for (int j = 0; j < RP; ++j) lr[j] = 0.0;
#pragma unroll
    for (int k = 0; k < RP; ++k) {
        if (k < R) {
            double s = gr[k] + (lane == k ? ridge : 0.0);
#pragma unroll
            for (int j = 0; j < k; ++j) s -= lr[j] * __shfl_sync(0xffffffffu, lr[j], k);
            const double x = __shfl_sync(0xffffffffu, s, k);
            if (x <= 0.0) ok = false;
            const double inv = rsqrt(x);
            if (lane == k) {
                lr[k] = x * inv;
                dinv = inv;
            } else if (lane > k) {
                lr[k] = s * inv;
            }
        }
    }
    return ok;
}

template <int RP>
__global__ void __launch_bounds__(kCholThreads) chol_kernel(const CholParams p) {
    __shared__ double gam[RP * RP];
    const int R = p.R, tid = threadIdx.x, lane = tid & 31;
    finalize_pending(p.pend, R, RP, p.gram);
    __syncthreads();
    // Gamma_n = Hadamard product of the other modes' Grams (independent loads, one per thread)
    for (int e = tid; e < RP * RP; e += blockDim.x) {
        const int q = e / RP, r = e % RP;
        double v = 0.0;
        if (q < R && r < R) {
            v = 1.0;
            for (int m = 0; m < p.order; ++m)
                if (m != p.mode) v *= p.gram[(size_t)m * RP * RP + e];
        }
        gam[e] = v;
    }
    __syncthreads();
    if (tid >= 32) return;
    const bool row = lane < R;
    double gr[RP], lr[RP], dinv = 0.0;
#pragma unroll
    for (int j = 0; j < RP; ++j) gr[j] = row ? gam[lane * RP + j] : 0.0;
    bool ok = warp_llt<RP>(gr, lr, dinv, R, 0.0);
    if (!ok) {
        // one ridge retry (1e-12 trace), as the reference's solve_spd
        double tr = 0.0;
#pragma unroll
        for (int j = 0; j < RP; ++j) tr += __shfl_sync(0xffffffffu, gr[j], j);  // diagonal, j ascending
        const double ridge = 1e-12 * tr;
        ok = (ridge > 0.0) && warp_llt<RP>(gr, lr, dinv, R, ridge);
    }
    if (row) {
#pragma unroll
        for (int j = 0; j < RP; ++j)
            if (j < R) p.fac[lane * R + j] = (j <= lane) ? lr[j] : 0.0;
        p.fac[R * R + lane] = dinv;
    }
    if (lane == 0) {
        p.fac[R * R + R] = ok ? 1.0 : 0.0;
        if (!ok) atomicOr(p.status, 1);
    }
}

// Ranks above 32 (RP = 64): the same left-looking LLT with the same operation order (l_ik =
// (g_ik - sum_{j<k} l_ij l_kj) / l_kk, j ascending, the division a multiplication by rsqrt, one
// ridge retry), a column per step over the block's threads with L in shared memory instead of a
// lane per row. Latency-bound (R dependent steps); only the wide-rank path uses it.
__global__ void __launch_bounds__(kCholThreads) chol_wide_kernel(const CholParams p) {
    constexpr int RP = kMaxRankWide;
    extern __shared__ double cwsm[];  // gam [RP * RP], l [RP * RP]
    double* gam = cwsm;
    double* l = cwsm + RP * RP;
    __shared__ double dv[RP];
    __shared__ int okf;
    const int R = p.R, tid = threadIdx.x;
    finalize_pending(p.pend, R, RP, p.gram);
    __syncthreads();
    for (int e = tid; e < RP * RP; e += blockDim.x) {
        const int q = e / RP, r = e % RP;
        double v = 0.0;
        if (q < R && r < R) {
            v = 1.0;
            for (int m = 0; m < p.order; ++m)
                if (m != p.mode) v *= p.gram[(size_t)m * RP * RP + e];
        }
        gam[e] = v;
    }
    __syncthreads();
    double ridge = 0.0;
    bool ok = false;
    for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
        if (attempt == 1) {
            double tr = 0.0;
            for (int j = 0; j < R; ++j) tr += gam[j * RP + j];  // diagonal, j ascending
            ridge = 1e-12 * tr;
            if (!(ridge > 0.0)) break;
        }
        if (tid == 0) okf = 1;
        for (int e = tid; e < RP * RP; e += blockDim.x) l[e] = 0.0;
        __syncthreads();
        for (int k = 0; k < R; ++k) {
            // pivot (thread 0) then column k below it, every row against the finished columns j < k
            if (tid == 0) {
                double s2 = gam[k * RP + k] + ridge;
                for (int j = 0; j < k; ++j) s2 -= l[k * RP + j] * l[k * RP + j];
                if (s2 <= 0.0) okf = 0;
                const double inv = rsqrt(s2);
                l[k * RP + k] = s2 * inv;
                dv[k] = inv;
            }
            __syncthreads();
            if (!okf) break;
            for (int i = k + 1 + tid; i < R; i += blockDim.x) {
                double s2 = gam[i * RP + k];
                for (int j = 0; j < k; ++j) s2 -= l[i * RP + j] * l[k * RP + j];
                l[i * RP + k] = s2 * dv[k];
            }
            __syncthreads();
        }
        __syncthreads();
        ok = okf != 0;
    }
    for (int e = tid; e < R * R; e += blockDim.x) {
        const int i = e / R, j = e % R;
        p.fac[e] = (j <= i) ? l[i * RP + j] : 0.0;
    }
    for (int i = tid; i < R; i += blockDim.x) p.fac[R * R + i] = dv[i];
    if (tid == 0) {
        p.fac[R * R + R] = ok ? 1.0 : 0.0;
        if (!ok) atomicOr(p.status, 1);
    }
}

struct SolveGramParams {
    int R, mode;
    int64_t In;
    const double* fac;   // chol_kernel output for this mode
    const double* M;     // layout 0: M[r * ld + i]; layout 1: M[i * RP + r]
    int layout;
    int64_t ld;
    int nparts;          // M = sum of nparts partial vectors M + c * pstride (fixed order)
    int64_t pstride;
    // optional: the last block to finish sums the Gram partials into gram (this mode's slot)
    unsigned int* fin_counter;
    double* gram;
    int RP;
    double* out;         // col-major In x R (block of the packed iterate)
    int* status;
    dd* part;            // this mode's Gram partials [gridDim.x][npair]
};

// RP lanes own one row i (lane r holds m_ir): L y = m by columns (y_j on lane j, broadcast,
// lanes r > j subtract l_rj y_j — the same j-ascending operation order as the dot-product
// form), then L^T x = y by columns (j descending). The block's rows are staged in shared memory
// and its Gram partial is accumulated in double-double, one upper-triangle pair per thread.
template <int RP>
__global__ void __launch_bounds__(kSolveThreads) solve_gram_kernel(const SolveGramParams p) {
    constexpr int RPB = kSolveThreads / RP;  // rows per block step
    constexpr int NPT = (RP * (RP + 1) / 2 + kSolveThreads - 1) / kSolveThreads;
    __shared__ double l[RP * RP];
    __shared__ double dinv[RP];
    __shared__ double xs[RPB][RP + 1];
    const int R = p.R;
    const int tid = threadIdx.x;
    if (p.fac[R * R + R] == 0.0) return;  // factorisation failed (status set): uniform exit
    for (int e = tid; e < R * R; e += blockDim.x) l[e] = p.fac[e];
    for (int e = tid; e < R; e += blockDim.x) dinv[e] = p.fac[R * R + e];
    const int npair = R * (R + 1) / 2;
    int pa[NPT], pb[NPT];
    dd acc[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        acc[k] = dd{0.0, 0.0};
        const int q = tid + k * kSolveThreads;
        if (q < npair) {
            pair_rq(q, R, pa[k], pb[k]);
        } else {
            pa[k] = pb[k] = -1;
        }
    }
    __syncthreads();
    const int r = tid % RP, rl = tid / RP;
    bool fin = true;
    for (int64_t i0 = (int64_t)blockIdx.x * RPB; i0 < p.In; i0 += (int64_t)gridDim.x * RPB) {
        const int64_t i = i0 + rl;
        const bool live = i < p.In && r < R;
        double s = 0.0;
        if (live) {
            const double* m = p.M + (p.layout == 0 ? (int64_t)r * p.ld + i : i * RP + r);
            for (int c0 = 0; c0 < p.nparts; c0 += 32) {  // one round of loads for <= 32 partials
                double x[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) x[u] = c0 + u < p.nparts ? m[(int64_t)(c0 + u) * p.pstride] : 0.0;
#pragma unroll
                for (int u = 0; u < 32; ++u) s += x[u];
            }
        }
        double y = 0.0;
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            if (j < R) {
                const double yj = __shfl_sync(0xffffffffu, s * dinv[j], j, RP);
                if (r == j) y = yj;
                if (r > j) s -= l[r * R + j] * yj;
            }
        }
        double t = y, x = 0.0;
#pragma unroll
        for (int j = RP - 1; j >= 0; --j) {
            if (j < R) {
                const double xj = __shfl_sync(0xffffffffu, t * dinv[j], j, RP);
                if (r == j) x = xj;
                if (r < j) t -= l[j * R + r] * xj;
            }
        }
        if (live) {
            p.out[(int64_t)r * p.In + i] = x;
            fin = fin && isfinite(x);
        }
        __syncthreads();  // previous step's Gram reads of xs are done
        xs[rl][r] = live ? x : 0.0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NPT; ++k)
            if (pa[k] >= 0)
                for (int rr = 0; rr < RPB; ++rr) acc[k] = dd_fma(acc[k], xs[rr][pa[k]], xs[rr][pb[k]]);
    }
    if (!fin) atomicOr(p.status, 2);
#pragma unroll
    for (int k = 0; k < NPT; ++k)
        if (pa[k] >= 0) p.part[(size_t)blockIdx.x * npair + tid + k * kSolveThreads] = acc[k];
    if (p.fin_counter && last_block_arrives(p.fin_counter)) {
        GramPending g{};
        g.mode = p.mode;
        g.part = p.part;
        g.nblk = (int)gridDim.x;
        finalize_pending(g, R, p.RP, p.gram);
    }
}

// Ranks above 32: a thread per row i with the row in registers (m_i summed from the partials in
// order, then L y = m and L^T x = y by columns in the same operation order as solve_gram_kernel),
// the block's rows staged in shared memory for the double-double Gram partials of the output.
__global__ void __launch_bounds__(kSolveWideRows) solve_gram_wide_kernel(const SolveGramParams p) {
    constexpr int RP = kMaxRankWide;
    extern __shared__ double swsm[];  // l [RP * RP], then xs [kSolveWideRows][RP + 1]
    double* l = swsm;
    double (*xs)[RP + 1] = reinterpret_cast<double (*)[RP + 1]>(swsm + RP * RP);
    __shared__ double dinv[RP];
    const int R = p.R, tid = threadIdx.x;
    if (p.fac[R * R + R] == 0.0) return;  // factorisation failed (status set): uniform exit
    for (int e = tid; e < R * R; e += blockDim.x) l[(e / R) * RP + e % R] = p.fac[e];
    for (int e = tid; e < R; e += blockDim.x) dinv[e] = p.fac[R * R + e];
    const int npair = R * (R + 1) / 2;
    constexpr int NPT = (RP * (RP + 1) / 2 + kSolveWideRows - 1) / kSolveWideRows;
    dd acc[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) acc[k] = dd{0.0, 0.0};
    __syncthreads();
    bool fin = true;
    for (int64_t i0 = (int64_t)blockIdx.x * kSolveWideRows; i0 < p.In; i0 += (int64_t)gridDim.x * kSolveWideRows) {
        const int64_t i = i0 + tid;
        const bool live = i < p.In;
        double s[RP];
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            double v = 0.0;
            if (live && r < R) {
                const double* m = p.M + (p.layout == 0 ? (int64_t)r * p.ld + i : i * p.RP + r);
                for (int c = 0; c < p.nparts; ++c) v += m[(int64_t)c * p.pstride];
            }
            s[r] = v;
        }
        double y[RP];
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            y[j] = 0.0;
            if (j < R) {
                y[j] = s[j] * dinv[j];
#pragma unroll
                for (int r = j + 1; r < RP; ++r)
                    if (r < R) s[r] -= l[r * RP + j] * y[j];
            }
        }
#pragma unroll
        for (int j = RP - 1; j >= 0; --j) {
            if (j < R) {
                const double xj = y[j] * dinv[j];
#pragma unroll
                for (int r = 0; r < j; ++r) y[r] -= l[j * RP + r] * xj;
                y[j] = xj;
            }
        }
        __syncthreads();  // the previous step's Gram reads of xs are done
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const double x = (live && r < R) ? y[r] : 0.0;
            if (live && r < R) {
                p.out[(int64_t)r * p.In + i] = x;
                fin = fin && isfinite(x);
            }
            xs[tid][r] = x;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NPT; ++k) {
            const int q = tid + k * kSolveWideRows;
            if (q < npair) {
                int a, b;
                pair_rq(q, R, a, b);
                for (int rr = 0; rr < kSolveWideRows; ++rr) acc[k] = dd_fma(acc[k], xs[rr][a], xs[rr][b]);
            }
        }
    }
    if (!fin) atomicOr(p.status, 2);
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int q = tid + k * kSolveWideRows;
        if (q < npair) p.part[(size_t)blockIdx.x * npair + q] = acc[k];
    }
    if (p.fin_counter && last_block_arrives(p.fin_counter)) {
        GramPending g{};
        g.mode = p.mode;
        g.part = p.part;
        g.nblk = (int)gridDim.x;
        finalize_pending(g, R, p.RP, p.gram);
    }
}

struct NormParams {
    int order, R, RP;
    int64_t dims[kMaxOrder];
    int64_t off[kMaxOrder + 1];
    const double* gram;
    const double* u;
    double* out;
    // optional: the gradient at u, mapped to the normalised point (G -> G D^-1, permuted),
    // and per-block partial sums of its squares
    const double* g;
    double* gout;
    double* red;
    // optional: M0 = T x KR(modes >= 1) at u ([RP][ld]), mapped to the normalised point:
    // M0'(:, r) = M0(:, perm r) / s_0(r)  (prod_n s_n = 1 for every nonzero term)
    const double* m0;
    double* m0out;
    int m0_ld;
    int m0_rowmajor;  // M0 as [i][RP] (rowwise tensors, m0_ld = I_0 rows) instead of [r][m0_ld]
    // optional: a Gram still in block partials (the last mode of an ALS sweep): its diagonal is
    // summed from the partials here, and block 0 finalises it into gram_w
    GramPending pend;
    double* gram_w;
    // optional: the permutation and the mode-0 scales of the normalisation (block 0 writes)
    int* perm_out;
    double* scale0_out;
    // optional: the last block rewrites gram_w as the Grams of the output,
    // G'_n(q, r) = s_n(q) s_n(r) G_n(perm q, perm r) (and into gram_copy when given)
    unsigned int* counter;
    double* gram_copy;
};

// normalize_and_reorder: norms from the (double-double) Gram diagonals, lambda_r =
// prod_n ||a_r^(n)||, stable sort by decreasing lambda, scale to lambda^(1/N); zero-lambda
// terms keep their columns and sort last (kruskal.cpp:156-193).
__global__ void normalize_kernel(const NormParams p) {
    __shared__ double nrm[kMaxOrder][kMaxRankWide];
    __shared__ double lam[kMaxRankWide];
    __shared__ int perm[kMaxRankWide];
    __shared__ double scale[kMaxOrder][kMaxRankWide];
    __shared__ double diag[kMaxOrder][kMaxRankWide];
    const int tid = threadIdx.x;
    NSTAMP(0);
    for (int e = tid; e < p.order * p.R; e += blockDim.x) {  // Gram diagonals, independent loads
        const int n = e / p.R, r = e % p.R;
        diag[n][r] = (n == p.pend.mode) ? pending_pair(p.pend, p.R * (p.R + 1) / 2, r * p.R - r * (r - 1) / 2)
                                        : p.gram[(size_t)n * p.RP * p.RP + r * (p.RP + 1)];
    }
    if (blockIdx.x == 0) finalize_pending(p.pend, p.R, p.RP, p.gram_w);
    __syncthreads();
    NSTAMP(1);
    if (p.R > 32) {
        // ranks above 32: thread r, the same stable descending order through shared memory
        const int r = tid;
        const bool on = r < p.R;
        double l = 1.0;
        if (on) {
            for (int n = 0; n < p.order; ++n) {
                const double v = sqrt(diag[n][r]);
                nrm[n][r] = v;
                l *= v;
            }
            lam[r] = l;
        }
        __syncthreads();
        if (on) {
            int pos = 0;
            for (int q = 0; q < p.R; ++q) {
                const double lq = lam[q];
                if (lq > l || (q < r && !(l > lq) && !(lq > l))) ++pos;
            }
            perm[pos] = r;
        }
        __syncthreads();
        if (on) {
            const int src = perm[r];
            const double ls = lam[src];
            const double root = (ls == 0.0) ? 0.0 : (p.order == 3 ? cbrt(ls) : pow(ls, 1.0 / p.order));
            for (int n = 0; n < p.order; ++n) scale[n][r] = (ls == 0.0) ? 1.0 : root / nrm[n][src];
            if (blockIdx.x == 0 && p.perm_out) {
                p.perm_out[r] = src;
                p.scale0_out[r] = scale[0][r];
            }
        }
    } else if (tid < 32) {
        // warp 0, lane r: rank r's norms (shared memory) and lambda, the stable sort by shuffles
        const int r = tid;
        const bool on = r < p.R;
        double l = 1.0;
        if (on)
            for (int n = 0; n < p.order; ++n) {
                const double v = sqrt(diag[n][r]);
                nrm[n][r] = v;
                l *= v;
            }
        if (on) lam[r] = l;
        // stable descending rank: count entries that must precede this one
        int pos = 0;
        for (int q = 0; q < p.R; ++q) {
            const double lq = __shfl_sync(0xffffffffu, l, q);
            if (lq > l || (q < r && !(l > lq) && !(lq > l))) ++pos;
        }
        if (on) perm[pos] = r;
        __syncwarp();
        const int src = on ? perm[r] : 0;
        const double ls = __shfl_sync(0xffffffffu, l, src);
        if (on) {
            // lambda^(1/N): cbrt for N = 3 (one root instead of pow's log / exp)
            const double root = (ls == 0.0) ? 0.0 : (p.order == 3 ? cbrt(ls) : pow(ls, 1.0 / p.order));
            for (int n = 0; n < p.order; ++n) scale[n][r] = (ls == 0.0) ? 1.0 : root / nrm[n][src];
            if (blockIdx.x == 0 && p.perm_out) {
                p.perm_out[r] = src;
                p.scale0_out[r] = scale[0][r];
            }
        }
    }
    __syncthreads();
    NSTAMP(4);
    const int64_t total = p.off[p.order];
    const int64_t tm = p.m0 ? (int64_t)p.RP * p.m0_ld : 0;
    double g2 = 0.0;
    // the iterate / gradient element and the M0 element of one index together (their loads overlap)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + tid; e < total || e < tm; e += (int64_t)gridDim.x * blockDim.x) {
        if (e < tm) {
            // 32-bit index math (tm, total < 2^31 for any iterate that fits a solve): 64-bit
            // division costs ~100 instructions and dominated the kernel at n_u = 3e5
            int r, i;
            if (p.m0_rowmajor) {
                i = (int)e / p.RP;
                r = (int)e - i * p.RP;
            } else {
                r = (int)e / p.m0_ld;
                i = (int)e - r * p.m0_ld;
            }
            double v = 0.0;
            if (r < p.R) {
                const int src = perm[r];
                v = p.m0_rowmajor ? p.m0[(int64_t)i * p.RP + src] : p.m0[(int64_t)src * p.m0_ld + i];
                if (lam[src] != 0.0) v /= scale[0][r];
            }
            p.m0out[e] = v;
        }
        if (e < total) {
            int n = 0;
            while (e >= p.off[n + 1]) ++n;
            const int loc = (int)(e - p.off[n]);
            const int In = (int)p.dims[n];
            const int r = loc / In;
            const int i = loc - r * In;
            const int src = perm[r];
            const int64_t at = p.off[n] + (int64_t)src * In + i;
            const double v = p.u[at];
            const bool keep = (lam[src] == 0.0);
            p.out[e] = keep ? v : v * scale[n][r];
            if (p.g) {
                const double gv = keep ? p.g[at] : p.g[at] / scale[n][r];
                p.gout[e] = gv;
                g2 += gv * gv;
            }
        }
    }
    if (p.g) {
        __shared__ double red[32];
        g2 = warp_sum(g2);
        if ((tid & 31) == 0) red[tid >> 5] = g2;
        __syncthreads();
        NSTAMP(5);
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
            p.red[blockIdx.x] = s;
        }
    }
    if (p.counter) {
        // every block has read the input Grams once the last one arrives: rewrite them as the
        // Grams of the normalised output (the next evaluation / sweep then skips the Gram pass)
        NSTAMP(10);
        if (!last_block_arrives(p.counter)) return;
        NSTAMPL(27);
        __shared__ double gin[kGramsOutMax];  // callers check order * RP * RP <= kGramsOutMax
        const int RR = p.RP * p.RP;
        {
            for (int e = tid; e < p.order * RR; e += blockDim.x) gin[e] = p.gram_w[e];
            __syncthreads();
            NSTAMPL(28);
            for (int e = tid; e < p.order * RR; e += blockDim.x) {
                const int n = e / RR, q = (e % RR) / p.RP, r = e % p.RP;
                double v = 0.0;
                if (q < p.R && r < p.R) v = scale[n][q] * scale[n][r] * gin[n * RR + perm[q] * p.RP + perm[r]];
                p.gram_w[e] = v;
                if (p.gram_copy) p.gram_copy[e] = v;
            }
        }
    }
    NSTAMP(12);
    if (p.counter) NSTAMPL(29);
}

__global__ void gram_hadamard_kernel(const double* gram, int order, int R, int RP, int skip, double* out) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int q = e % R, r = e / R;  // out col-major (q, r)
        double v = 1.0;
        for (int m = 0; m < order; ++m)
            if (m != skip) v *= gram[(size_t)m * RP * RP + q * RP + r];
        out[e] = v;
    }
}

}  // namespace

namespace {
int solve_blocks(const EvalWork& w, int n) {
    const int rpb = w.RP > kMaxRank ? kSolveWideRows : kSolveThreads / w.RP;
    return (int)std::max<int64_t>(1, std::min<int64_t>((w.dims[n] + rpb - 1) / rpb, kSolveMaxBlocks));
}
GramPending pending_of(const EvalWork& w, int n) {
    GramPending g{};
    g.mode = n;
    g.part = w.solve_part + (size_t)n * w.solve_part_stride;
    g.nblk = n >= 0 ? solve_blocks(w, n) : 0;
    if (n < 0) g.part = nullptr;
    return g;
}

}  // namespace

void gram_hadamard_device(EvalWork& w, int skip, double* out, cudaStream_t st) {
    gram_hadamard_kernel<<<1, 256, 0, st>>>(w.gram, w.order, w.R, w.RP, skip, out);
    CPFIT_CUDA(cudaGetLastError());
}

void normalize_device(EvalWork& w, const double* u, double* out, cudaStream_t st, int pending, bool save_perm,
                      bool out_grams) {
    NormParams p{};
    p.pend = pending_of(w, pending);
    p.gram_w = w.gram;
    if (out_grams) p.counter = w.counter + kCounterNorm;
    if (save_perm) {
        p.perm_out = w.nperm;
        p.scale0_out = w.nscale0;
    }
    p.order = w.order;
    p.R = w.R;
    p.RP = w.RP;
    for (int n = 0; n < w.order; ++n) {
        p.dims[n] = w.dims[n];
        p.off[n] = w.off[n];
    }
    p.off[w.order] = w.off[w.order];
    p.gram = w.gram;
    p.u = u;
    p.out = out;
    const int blocks = (int)std::min<int64_t>(296, (w.nu + 255) / 256);
    normalize_kernel<<<blocks, 256, 0, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
}

int normalize_grad_device(EvalWork& w, const double* u, const double* g, double* uout, double* gout, double* red,
                          cudaStream_t st, const double* m0, double* m0out, bool out_grams, bool save_perm,
                          double* gram_copy) {
    NormParams p{};
    p.pend.mode = -1;
    p.gram_w = w.gram;
    if (out_grams) p.counter = w.counter + kCounterNorm;
    p.gram_copy = gram_copy;
    if (save_perm) {
        p.perm_out = w.nperm;
        p.scale0_out = w.nscale0;
    }
    p.order = w.order;
    p.R = w.R;
    p.RP = w.RP;
    for (int n = 0; n < w.order; ++n) {
        p.dims[n] = w.dims[n];
        p.off[n] = w.off[n];
    }
    p.off[w.order] = w.off[w.order];
    p.gram = w.gram;
    p.u = u;
    p.out = uout;
    p.g = g;
    p.gout = gout;
    p.red = red;
    p.m0 = m0;
    p.m0out = m0out;
    p.m0_rowmajor = w.m0_rowwise ? 1 : 0;
    p.m0_ld = w.m0_rowwise ? (int)w.dims[0] : 32 * w.fiber_nchunk;
    const int blocks = (int)std::min<int64_t>(296, (w.nu + 255) / 256);
    normalize_kernel<<<blocks, 256, 0, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
    return blocks;
}

namespace {
// Cholesky factor of Gamma_n -> w.chol + mode slot; first finalises mode `pending`'s Gram
void chol_mode(EvalWork& w, int n, int pending, int* status, cudaStream_t st) {
    CholParams p{};
    p.order = w.order;
    p.R = w.R;
    p.RP = w.RP;
    p.mode = n;
    p.gram = w.gram;
    p.pend = pending_of(w, pending);
    p.fac = w.chol + (size_t)n * w.chol_stride;
    p.status = status;
    switch (w.RP) {
        case 8: chol_kernel<8><<<1, kCholThreads, 0, st>>>(p); break;
        case 16: chol_kernel<16><<<1, kCholThreads, 0, st>>>(p); break;
        case 32: chol_kernel<32><<<1, kCholThreads, 0, st>>>(p); break;
        default: {
            const size_t sm = sizeof(double) * 2 * kMaxRankWide * kMaxRankWide;
            CPFIT_CUDA(cudaFuncSetAttribute(chol_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            chol_wide_kernel<<<1, kCholThreads, sm, st>>>(p);
            break;
        }
    }
    CPFIT_CUDA(cudaGetLastError());
}

// A_n <- M_n Gamma_n^-1 (factor from chol_mode); G_n left as block partials (pending)
void solve_gram(EvalWork& w, int n, const double* M, int layout, int64_t ld, double* ublock, int* status,
                cudaStream_t st, int nparts = 1, int64_t pstride = 0, bool finalize = false) {
    SolveGramParams p{};
    p.nparts = nparts;
    p.pstride = pstride;
    p.RP = w.RP;
    if (finalize) {
        p.fin_counter = w.counter + kCounterSolve;
        p.gram = w.gram;
    }
    p.R = w.R;
    p.mode = n;
    p.In = w.dims[n];
    p.fac = w.chol + (size_t)n * w.chol_stride;
    p.M = M;
    p.layout = layout;
    p.ld = ld;
    p.out = ublock;
    p.status = status;
    p.part = w.solve_part + (size_t)n * w.solve_part_stride;
    const int grid = solve_blocks(w, n);
    switch (w.RP) {
        case 8: solve_gram_kernel<8><<<grid, kSolveThreads, 0, st>>>(p); break;
        case 16: solve_gram_kernel<16><<<grid, kSolveThreads, 0, st>>>(p); break;
        case 32: solve_gram_kernel<32><<<grid, kSolveThreads, 0, st>>>(p); break;
        default: {
            const size_t sm = sizeof(double) * (kMaxRankWide * kMaxRankWide + kSolveWideRows * (kMaxRankWide + 1));
            CPFIT_CUDA(cudaFuncSetAttribute(solve_gram_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            solve_gram_wide_kernel<<<grid, kSolveWideRows, sm, st>>>(p);
            break;
        }
    }
    CPFIT_CUDA(cudaGetLastError());
}

__global__ void finalize_gram_kernel(const GramPending g, int R, int RP, double* gram) {
    finalize_pending(g, R, RP, gram);
}

// chol_mode(n) on the side stream once everything queued on st so far is done; the next
// solve_gram(n) on st waits for it (join_chol)
void fork_chol(EvalWork& w, int n, int* status, cudaStream_t st) {
    CPFIT_CUDA(cudaEventRecord(w.ev_fork, st));
    CPFIT_CUDA(cudaStreamWaitEvent(w.side, w.ev_fork, 0));
    chol_mode(w, n, n - 1, status, w.side);
    CPFIT_CUDA(cudaEventRecord(w.ev_join, w.side));
}
void join_chol(EvalWork& w, cudaStream_t st) { CPFIT_CUDA(cudaStreamWaitEvent(st, w.ev_join, 0)); }
}  // namespace

namespace {
// S(u_bar)[j][r] = S'[j][perm r] * s_0(r): the sweep's S' = T x_1 A0' mapped to the normalised
// iterate (its mode-0 factor is A0' permuted and scaled), for the evaluation that follows
template <int RP>
__global__ void s_rescale_kernel(double* S, int64_t J, int R, const int* perm, const double* sc) {
    // one element per lane; a row (RP <= 32 lanes) lives in one warp, so the permutation is a
    // shuffle after every lane has loaded its element
    const int64_t n = J * RP;
    const int lane = threadIdx.x & 31;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x; e0 < n; e0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = e0 + threadIdx.x;
        const int r = (int)(e % RP);
        const double v = e < n ? S[e] : 0.0;
        const int src = (lane & ~(RP - 1)) + (r < R ? perm[r] : 0);
        const double o = __shfl_sync(0xffffffffu, v, src);
        if (e < n) S[e] = r < R ? o * sc[r] : 0.0;
    }
}
}  // namespace

// work: n_u scratch (pre-normalisation iterate), mbuf: max(I_n)*R scratch
void als_sweep_device_ws(const DevTensor& t, EvalWork& w, const double* u, double* out, double* work, double* mbuf,
                         int* status, cudaStream_t st, const double* m0_given, bool keep_s, bool grams_given,
                         bool defer_norm) {
    CPFIT_CUDA(cudaMemcpyAsync(work, u, sizeof(double) * w.nu, cudaMemcpyDeviceToDevice, st));
    if (!grams_given) grams_device(w, work, st);
    const int N = t.order;
    // Gamma_0 from the Grams of u; each later Gamma_n as soon as G_{n-1}' exists (side stream)
    chol_mode(w, 0, -1, status, st);
    if (rowwise(t, w)) {
        for (int n = 0; n < N; ++n) {
            if (n > 0) fork_chol(w, n, status, st);
            // mode 0: the M0 the evaluation of this iterate produced ([i][RP]), when given
            if (!(n == 0 && m0_given)) rowwise_modes(t, w, work, n, st);
            int64_t off = 0;
            for (int m = 0; m < n; ++m) off += t.dims[m] * w.RP;
            if (n > 0) join_chol(w, st);
            solve_gram(w, n, (n == 0 && m0_given) ? m0_given : w.sp_part + off, 1, 0, work + w.off[n], status, st);
        }
    } else {
        // mode 0: tail contraction with the old modes >= 1 — or, inside the N-GMRES loop, the
        // M0 the evaluation of this iterate already produced (m0_given, [RP][32 NC])
        if (!m0_given) dense_fiber(t, w, work, false, true, st);
        solve_gram(w, 0, m0_given ? m0_given : w.m0, 0, 32 * w.fiber_nchunk, work + w.off[0], status, st);
        fork_chol(w, 1, status, st);
        // S' = T x_1 A0'
        dense_fiber(t, w, work, true, false, st);
        const double* Sin = w.S;
        for (int n = 1; n < N; ++n) {
            // the solves sum the level partials themselves (no reduction launches)
            if (n < N - 1) {
                dense_level(t, w, n, Sin, work, true, false, nullptr, st, true);
                join_chol(w, st);
                solve_gram(w, n, w.lvl_part[n], 1, 0, work + w.off[n], status, st, w.lvl_nx[n], t.dims[n] * w.RP);
                fork_chol(w, n + 1, status, st);
                const bool last_level = (n == N - 2);
                dense_level(t, w, n, Sin, work, false, true, w.lvl_S[n], st, last_level);
                Sin = w.lvl_S[n];
                if (last_level && w.lvl_ny[n] > 1) {
                    join_chol(w, st);
                    solve_gram(w, N - 1, w.lvl_spart[n], 1, 0, work + w.off[N - 1], status, st, w.lvl_ny[n],
                               t.dims[N - 1] * w.RP);
                    break;
                }
            } else {
                join_chol(w, st);
                solve_gram(w, n, Sin, 1, 0, work + w.off[n], status, st);
            }
        }
    }
    // deferred: the caller evaluates the sweep's own point (work, S' in w.S; the last mode's
    // Gram still in solve partials: finalize_gram_side) and normalises afterwards
    // (normalize_grad), so S never needs the rescale below
    if (defer_norm) return;
    normalize_device(w, work, out, st, N - 1, keep_s && !rowwise(t, w), grams_given);
    if (keep_s && !rowwise(t, w)) {
        const int blocks = (int)std::min<int64_t>(8 * 148, (t.J * w.RP + 255) / 256);
        switch (w.RP) {
            case 8: s_rescale_kernel<8><<<blocks, 256, 0, st>>>(w.S, t.J, w.R, w.nperm, w.nscale0); break;
            case 16: s_rescale_kernel<16><<<blocks, 256, 0, st>>>(w.S, t.J, w.R, w.nperm, w.nscale0); break;
            default: s_rescale_kernel<32><<<blocks, 256, 0, st>>>(w.S, t.J, w.R, w.nperm, w.nscale0); break;
        }
        CPFIT_CUDA(cudaGetLastError());
    }
}

// G_mode <- the sum of its pending solve partials, as one block on the side stream (forked
// after everything queued on st); `done` is recorded on the side stream when it has finished
void finalize_gram_side(EvalWork& w, int mode, cudaStream_t st, cudaEvent_t done) {
    CPFIT_CUDA(cudaEventRecord(w.ev_fork, st));
    CPFIT_CUDA(cudaStreamWaitEvent(w.side, w.ev_fork, 0));
    finalize_gram_kernel<<<1, 256, 0, w.side>>>(pending_of(w, mode), w.R, w.RP, w.gram);
    CPFIT_CUDA(cudaGetLastError());
    CPFIT_CUDA(cudaEventRecord(done, w.side));
}

}  // namespace cpfit_gpu
