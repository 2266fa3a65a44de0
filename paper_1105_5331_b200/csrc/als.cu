// ALS preconditioner M(.) on device (als.cpp:16-48) and normalize_and_reorder
// (kruskal.cpp:156-193).
//
// One sweep is Gauss-Seidel over modes 0..N-1 exactly as the reference; the dense
// right-hand sides come from a dimension tree instead of N independent MTTKRPs:
//   mode 0      : tail contraction of T with KR(A1..A_{N-1})          (T pass 1)
//   mode 1      : S' = T x_1 A0'  (stored) then the level contraction   (T pass 2)
//   modes >= 2  : level contractions of S' with the freshly solved heads (no T pass)
// so a sweep streams T twice instead of N times. The R x R normal matrix
// Gamma_n = *_{m!=n} A_m^T A_m is factored by a warp-parallel left-looking Cholesky in the
// column order of Eigen's unblocked LLT, with the reference's one ridge retry
// (1e-12 * trace) before reporting numerical failure.
#include "device.cuh"

#include <algorithm>

namespace cpfit_gpu {

void dense_fiber(const DevTensor& t, EvalWork& w, const double* u, bool do_s, bool do_m0, cudaStream_t st);
void dense_level(const DevTensor& t, EvalWork& w, int h, const double* Sin, const double* u, bool do_m, bool do_s,
                 double* Sout, cudaStream_t st);
void gather_m(int64_t In, EvalWork& w, const double* part, int grid, int ld, int layout, double* out,
              cudaStream_t st);
void gram_mode_device(EvalWork& w, const double* u, int mode, cudaStream_t st);
void sparse_all_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st);

namespace {

struct SolveParams {
    int order, R, RP, mode;
    int64_t In;
    const double* gram;  // [mode][RP*RP]
    const double* M;     // col-major In x R
    double* out;         // col-major In x R (block of the packed iterate)
    int* status;
};

// Left-looking LLT of g (R x R, row-major in smem) into l; returns false on pivot <= 0.
__device__ bool warp_llt(const double* g, double* l, int R, double ridge) {
    const int lane = threadIdx.x & 31;
    bool ok = true;
    for (int k = 0; k < R; ++k) {
        // pivot: x = a_kk - sum_j l_kj^2  (j ascending, as Eigen's A10.squaredNorm())
        double x = g[k * R + k] + ridge;
        for (int j = 0; j < k; ++j) x -= l[k * R + j] * l[k * R + j];
        if (!(x > 0.0)) {
            if (x <= 0.0) ok = false;  // NaN passes Eigen's (x <= 0) test
        }
        if (x <= 0.0) return false;
        x = sqrt(x);
        __syncwarp();
        for (int i = k + 1 + lane; i < R; i += 32) {
            double s = g[i * R + k];
            for (int j = 0; j < k; ++j) s -= l[i * R + j] * l[k * R + j];
            l[i * R + k] = s / x;
        }
        if (lane == 0) l[k * R + k] = x;
        __syncwarp();
    }
    return ok;
}

__global__ void solve_kernel(const SolveParams p) {
    __shared__ double g[kMaxRank * kMaxRank];
    __shared__ double l[kMaxRank * kMaxRank];
    __shared__ int ok_s;
    const int R = p.R;
    const int tid = threadIdx.x;
    for (int e = tid; e < R * R; e += blockDim.x) {
        const int q = e / R, r = e % R;
        double v = 1.0;
        for (int m = 0; m < p.order; ++m)
            if (m != p.mode) v *= p.gram[(size_t)m * p.RP * p.RP + q * p.RP + r];
        g[e] = v;
        l[e] = 0.0;
    }
    __syncthreads();
    if (tid < 32) {
        bool ok = warp_llt(g, l, R, 0.0);
        if (!ok) {
            double tr = 0.0;
            for (int i = 0; i < R; ++i) tr += g[i * R + i];
            const double ridge = 1e-12 * tr;
            __syncwarp();
            for (int e = tid; e < R * R; e += 32) l[e] = 0.0;
            __syncwarp();
            ok = (ridge > 0.0) && warp_llt(g, l, R, ridge);
        }
        if (tid == 0) ok_s = ok ? 1 : 0;
    }
    __syncthreads();
    if (!ok_s) {
        if (tid == 0 && blockIdx.x == 0) atomicOr(p.status, 1);
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + tid; i < p.In; i += (int64_t)gridDim.x * blockDim.x) {
        double y[kMaxRank];
        for (int r = 0; r < R; ++r) {  // L y = m_i
            double s = p.M[(int64_t)r * p.In + i];
            for (int j = 0; j < r; ++j) s -= l[r * R + j] * y[j];
            y[r] = s / l[r * R + r];
        }
        for (int r = R - 1; r >= 0; --r) {  // L^T x = y
            double s = y[r];
            for (int j = r + 1; j < R; ++j) s -= l[j * R + r] * y[j];
            y[r] = s / l[r * R + r];
        }
        bool fin = true;
        for (int r = 0; r < R; ++r) {
            p.out[(int64_t)r * p.In + i] = y[r];
            fin = fin && isfinite(y[r]);
        }
        if (!fin) atomicOr(p.status, 2);
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
};

// normalize_and_reorder: norms from the (double-double) Gram diagonals, lambda_r =
// prod_n ||a_r^(n)||, stable sort by decreasing lambda, scale to lambda^(1/N); zero-lambda
// terms keep their columns and sort last (kruskal.cpp:156-193).
__global__ void normalize_kernel(const NormParams p) {
    __shared__ double nrm[kMaxOrder][kMaxRank];
    __shared__ double lam[kMaxRank];
    __shared__ int perm[kMaxRank];
    __shared__ double scale[kMaxOrder][kMaxRank];
    const int tid = threadIdx.x;
    if (tid < p.R) {
        double l = 1.0;
        for (int n = 0; n < p.order; ++n) {
            const double v = sqrt(p.gram[(size_t)n * p.RP * p.RP + tid * p.RP + tid]);
            nrm[n][tid] = v;
            l *= v;
        }
        lam[tid] = l;
    }
    __syncthreads();
    if (tid < p.R) {
        // stable descending rank: count entries that must precede this one
        int pos = 0;
        for (int q = 0; q < p.R; ++q)
            if (lam[q] > lam[tid] || (q < tid && !(lam[tid] > lam[q]) && !(lam[q] > lam[tid]))) ++pos;
        perm[pos] = tid;
    }
    __syncthreads();
    if (tid < p.R) {
        const int src = perm[tid];
        const double l = lam[src];
        for (int n = 0; n < p.order; ++n) scale[n][tid] = (l == 0.0) ? 1.0 : pow(l, 1.0 / p.order) / nrm[n][src];
    }
    __syncthreads();
    const int64_t total = p.off[p.order];
    double g2 = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + tid; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int n = 0;
        while (e >= p.off[n + 1]) ++n;
        const int64_t loc = e - p.off[n];
        const int64_t In = p.dims[n];
        const int r = (int)(loc / In);
        const int64_t i = loc % In;
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
    if (p.m0) {
        const int64_t tm = (int64_t)p.RP * p.m0_ld;
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + tid; e < tm; e += (int64_t)gridDim.x * blockDim.x) {
            const int r = (int)(e / p.m0_ld);
            const int64_t i = e % p.m0_ld;
            double v = 0.0;
            if (r < p.R) {
                const int src = perm[r];
                v = p.m0[(int64_t)src * p.m0_ld + i];
                if (lam[src] != 0.0) v /= scale[0][r];
            }
            p.m0out[e] = v;
        }
    }
    if (p.g) {
        __shared__ double red[32];
        g2 = warp_sum(g2);
        if ((tid & 31) == 0) red[tid >> 5] = g2;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
            p.red[blockIdx.x] = s;
        }
    }
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

void gram_hadamard_device(EvalWork& w, int skip, double* out, cudaStream_t st) {
    gram_hadamard_kernel<<<1, 256, 0, st>>>(w.gram, w.order, w.R, w.RP, skip, out);
    CPFIT_CUDA(cudaGetLastError());
}

void normalize_device(EvalWork& w, const double* u, double* out, cudaStream_t st) {
    NormParams p{};
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
                          cudaStream_t st, const double* m0, double* m0out) {
    NormParams p{};
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
    p.m0_ld = 32 * w.fiber_nchunk;
    const int blocks = (int)std::min<int64_t>(296, (w.nu + 255) / 256);
    normalize_kernel<<<blocks, 256, 0, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
    return blocks;
}

namespace {
void solve_mode(EvalWork& w, int n, const double* M, double* ublock, int* status, cudaStream_t st) {
    SolveParams p{};
    p.order = w.order;
    p.R = w.R;
    p.RP = w.RP;
    p.mode = n;
    p.In = w.dims[n];
    p.gram = w.gram;
    p.M = M;
    p.out = ublock;
    p.status = status;
    const int blocks = (int)std::min<int64_t>(296, (p.In + 127) / 128);
    solve_kernel<<<blocks, 128, 0, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
}
}  // namespace

// work: n_u scratch (pre-normalisation iterate), mbuf: max(I_n)*R scratch
void als_sweep_device_ws(const DevTensor& t, EvalWork& w, const double* u, double* out, double* work, double* mbuf,
                         int* status, cudaStream_t st, const double* m0_given) {
    CPFIT_CUDA(cudaMemcpyAsync(work, u, sizeof(double) * w.nu, cudaMemcpyDeviceToDevice, st));
    grams_device(w, work, st);
    const int N = t.order;
    if (t.sparse) {
        for (int n = 0; n < N; ++n) {
            sparse_all_modes(t, w, work, n, st);
            int64_t off = 0;
            for (int m = 0; m < n; ++m) off += t.dims[m] * w.RP;
            gather_m(t.dims[n], w, w.sp_part + off, 1, 0, 1, mbuf, st);
            solve_mode(w, n, mbuf, work + w.off[n], status, st);
            gram_mode_device(w, work, n, st);
        }
    } else {
        // mode 0: tail contraction with the old modes >= 1 — or, inside the N-GMRES loop, the
        // M0 the evaluation of this iterate already produced (m0_given, [RP][32 NC])
        if (!m0_given) dense_fiber(t, w, work, false, true, st);
        gather_m(t.dims[0], w, m0_given ? m0_given : w.m0, 1, 32 * w.fiber_nchunk, 0, mbuf, st);
        solve_mode(w, 0, mbuf, work + w.off[0], status, st);
        gram_mode_device(w, work, 0, st);
        // S' = T x_1 A0'
        dense_fiber(t, w, work, true, false, st);
        const double* Sin = w.S;
        for (int n = 1; n < N; ++n) {
            if (n < N - 1) {
                dense_level(t, w, n, Sin, work, true, false, nullptr, st);
                gather_m(t.dims[n], w, w.lvl_m[n], 1, 0, 1, mbuf, st);
            } else {
                gather_m(t.dims[n], w, Sin, 1, 0, 1, mbuf, st);
            }
            solve_mode(w, n, mbuf, work + w.off[n], status, st);
            gram_mode_device(w, work, n, st);
            if (n < N - 1) {
                dense_level(t, w, n, Sin, work, false, true, w.lvl_S[n], st);
                Sin = w.lvl_S[n];
            }
        }
    }
    normalize_device(w, work, out, st);
}

}  // namespace cpfit_gpu
