// N-GMRES Step II on device (accelerate, ngmres.cpp:27-63).
//
// The reference solves min ||P a + g||^2 + delta ||a||^2 (P columns g_bar - g_j, delta =
// eps * max diag P^T P) by a column-pivoted Householder QR of the stacked n_u+m by m matrix.
// Here the tall part is reduced first by a communication-avoiding TSQR of X = [P | -g_bar]
// (one streaming pass over the window, Householder in shared memory per row block, then a
// tree of merges of the (m+1)x(m+1) R factors). Because Q is orthogonal,
//   ||P a + g_bar||^2 = ||R_P a - r_c||^2 + rho^2,  ||P e_j|| = ||R_P e_j||,  P^T g_bar = -R_P^T r_c,
// so delta, the right-hand side and the damped problem are recovered exactly from R, and the
// small (2m x m) stacked system [R_P; sqrt(delta) I] a = [r_c; 0] is solved with the same
// column-pivoted Householder algorithm (pivot order by column norms, which equal the tall
// matrix's) in one warp. u_hat = u_bar + sum_j a_j (u_bar - u_j), d = u_hat - u_bar and the
// descent slope g_bar.d are formed in a final streaming pass.
#include "device.cuh"

#include <algorithm>
#include <string>

namespace cpfit_gpu {

namespace {

constexpr int kLeafRows = 256;
constexpr int kTsqrThreads = 512;
constexpr size_t kTsqrSmem = 220 * 1024;  // dynamic shared memory of one TSQR block
constexpr int kQrMaxRows = 320;           // smem_qr: kQrMaxRpl rows per lane

// Leaf rows for windows of C = m + 1 columns: 256 up to C = 64 (the stacked running R + leaf rows
// fit smem_qr's 320 rows), fewer above so (C + rows) x C doubles stay in shared memory.
int tsqr_leaf_rows(int C) {
    if (C <= 64) return kLeafRows;
    return std::min<int>(kQrMaxRows - C, (int)(kTsqrSmem / (sizeof(double) * C)) - C);
}
// R factors stacked per merge block: (C + per C) rows within both limits, at least one
int tsqr_merge_per(int C) {
    if (C <= 64) return std::max(1, kLeafRows / C);
    const int rows = std::min<int>(kQrMaxRows, (int)(kTsqrSmem / (sizeof(double) * C)));
    return std::max(1, (rows - C) / C);
}

struct TsqrParams {
    int64_t n;
    int cap;
    const int* ring;  // [0] = m, [1] = head slot
    const double* wg;
    const double* gb;
    const double* rin;   // merge input (stacked R's) or null for leaf
    int64_t nin;         // number of input R's (merge)
    double* rout;        // output R's [cta][C*C] (col-major C x C, ld = C)
    int64_t blocks_per_cta;
    int64_t nblocks;
    int per_block;       // rows (leaf) or R's (merge) per block
};

// Householder QR (no pivoting; Eigen makeHouseholder / applyHouseholderOnTheLeft) of the
// H x C column-major smem matrix x (ld = H, H <= 32 kQrMaxRpl); upper triangle left in rows
// 0..C-1, the rest zeroed. Latency-bound (C sequential steps): one warp forms each reflector,
// then every warp updates its columns with the reflector and the column cached in registers
// (lanes over rows, loads issued before the dot product).
constexpr int kQrMaxRpl = 10;

__device__ void smem_qr(double* x, int H, int C, double* tau_s /* [3] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int K = min(H, C);
    for (int k = 0; k < K; ++k) {
        double* col = x + (size_t)k * H;
        if (warp == 0) {
            double cv[kQrMaxRpl];
#pragma unroll
            for (int u = 0; u < kQrMaxRpl; ++u) {
                const int i = k + 1 + lane + 32 * u;
                cv[u] = i < H ? col[i] : 0.0;
            }
            double tail = 0.0;
#pragma unroll
            for (int u = 0; u < kQrMaxRpl; ++u) tail += cv[u] * cv[u];
            tail = warp_sum(tail);
            const double c0 = col[k];
            double tau, beta;
            if (tail <= 2.2250738585072014e-308) {
                tau = 0.0;
                beta = c0;
                for (int i = k + 1 + lane; i < H; i += 32) col[i] = 0.0;
            } else {
                beta = sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                tau = (beta - c0) / beta;
            }
            __syncwarp();
            if (lane == 0) {
                tau_s[0] = tau;
                tau_s[1] = beta;
                tau_s[2] = c0 - beta;  // essential part = tail / (c0 - beta)
            }
        }
        __syncthreads();
        const double tau = tau_s[0];
        if (tau != 0.0) {
            // essential part of the reflector, every thread one division
            const double inv = tau_s[2];
            for (int i = k + 1 + threadIdx.x; i < H; i += blockDim.x) col[i] /= inv;
            __syncthreads();
            double vr[kQrMaxRpl];
#pragma unroll
            for (int u = 0; u < kQrMaxRpl; ++u) {
                const int i = k + 1 + lane + 32 * u;
                vr[u] = i < H ? col[i] : 0.0;
            }
            for (int j = k + 1 + warp; j < C; j += nw) {
                double* cj = x + (size_t)j * H;
                double cr[kQrMaxRpl];
                double t = 0.0;
#pragma unroll
                for (int u = 0; u < kQrMaxRpl; ++u) {
                    const int i = k + 1 + lane + 32 * u;
                    cr[u] = i < H ? cj[i] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kQrMaxRpl; ++u) t += vr[u] * cr[u];
                t = warp_sum(t) + cj[k];
#pragma unroll
                for (int u = 0; u < kQrMaxRpl; ++u) {
                    const int i = k + 1 + lane + 32 * u;
                    if (i < H) cj[i] = cr[u] - tau * vr[u] * t;
                }
                if (lane == 0) cj[k] -= tau * t;
            }
        }
        if (threadIdx.x == 0) col[k] = tau_s[1];
        __syncthreads();
    }
    // zero everything below the diagonal (essential parts)
    for (int e = threadIdx.x; e < H * C; e += blockDim.x) {
        const int j = e / H, i = e % H;
        if (i > j) x[e] = 0.0;
    }
    __syncthreads();
}

__global__ void tsqr_kernel(const TsqrParams p) {
    extern __shared__ double xs[];
    __shared__ double tau_s[3];
    const int m = p.ring[0], head = p.ring[1];
    const int C = m + 1;
    const int H = C + p.per_block * (p.rin ? C : 1);
    const int64_t b0 = blockIdx.x * p.blocks_per_cta;
    const int64_t b1 = imin64(p.nblocks, b0 + p.blocks_per_cta);
    bool have = false;
    for (int e = threadIdx.x; e < H * C; e += blockDim.x) xs[e] = 0.0;
    __syncthreads();
    for (int64_t b = b0; b < b1; ++b) {
        const int top = have ? C : 0;
        if (!p.rin) {
            // leaves hold per_block rows; column j of the window sits in ring slot head + j (mod cap)
            const int lr = p.per_block;
            const int64_t r0 = b * lr;
#pragma unroll 4
            for (int e = threadIdx.x; e < lr * C; e += blockDim.x) {
                const int j = e / lr, ii = e % lr;
                const int64_t i = r0 + ii;
                double v = 0.0;
                if (i < p.n) {
                    const double g = p.gb[i];
                    if (j < m) {
                        const int slot = head + j < p.cap ? head + j : head + j - p.cap;
                        v = g - p.wg[(int64_t)slot * p.n + i];
                    } else {
                        v = -g;
                    }
                }
                xs[(size_t)j * H + top + ii] = v;
            }
            for (int e = threadIdx.x; e < (H - top - p.per_block) * C; e += blockDim.x) {
                const int rows = H - top - p.per_block;
                const int j = e / rows, ii = e % rows;
                xs[(size_t)j * H + top + p.per_block + ii] = 0.0;
            }
        } else {
            const int64_t k0 = b * p.per_block;
            for (int e = threadIdx.x; e < p.per_block * C * C; e += blockDim.x) {
                const int kk = e / (C * C), rem = e % (C * C);
                const int j = rem / C, i = rem % C;
                const int64_t src = k0 + kk;
                xs[(size_t)j * H + top + kk * C + i] = (src < p.nin) ? p.rin[src * C * C + (size_t)j * C + i] : 0.0;
            }
            for (int e = threadIdx.x; e < (H - top - p.per_block * C) * C; e += blockDim.x) {
                const int rows = H - top - p.per_block * C;
                const int j = e / rows, ii = e % rows;
                xs[(size_t)j * H + top + p.per_block * C + ii] = 0.0;
            }
        }
        __syncthreads();
        smem_qr(xs, H, C, tau_s);
        have = true;
    }
    double* out = p.rout + (size_t)blockIdx.x * C * C;
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
        const int j = e / C, i = e % C;
        out[e] = have ? xs[(size_t)j * H + i] : 0.0;
    }
}

// Damped least squares from the final R with Eigen ColPivHouseholderQR semantics (pivot on the
// largest updated column norm, LAPACK-style norm downdating with recomputation, threshold rank),
// one block of kSolveThreads: R staged in shared memory once; each Householder step is one warp's
// norm + scalars, then the remaining columns are updated one warp per column (lanes over rows).
constexpr int kSolveThreads = 512;

__global__ void __launch_bounds__(kSolveThreads) accel_solve_kernel(const double* rfin, const int* ring, double eps,
                                                                    double* alpha, double* scal) {
    extern __shared__ double sm[];  // a: 2m x m stacked system (col-major); the C x C R factor stays in global
    __shared__ double bvec[2 * kMaxWindow], cvec[2 * kMaxWindow], upd[kMaxWindow], dir[kMaxWindow], hc[kMaxWindow],
        rhs[kMaxWindow], al[kMaxWindow], colsq[kMaxWindow], yv[kMaxWindow];
    __shared__ int perm[kMaxWindow], transp[kMaxWindow];
    __shared__ double sh_delta, sh_rn, sh_thr_help, sh_maxpivot, sh_tau;
    __shared__ int sh_nzp, sh_nz;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int m = ring[0];
    const int C = m + 1;
    const int rows = 2 * m;
    double* a = sm;
    const double* __restrict__ rf = rfin;  // L2-resident; read a few times
    // ||R_P e_j||^2 and rhs_j = R_P(:, j) . r_c = -(P^T g_bar)_j
    for (int j = tid; j < m; j += blockDim.x) {
        double s2 = 0.0, r = 0.0;
        for (int i = 0; i <= j; ++i) {
            const double v = rf[(size_t)j * C + i];
            s2 += v * v;
            r += v * rf[(size_t)m * C + i];
        }
        colsq[j] = s2;
        rhs[j] = r;
    }
    __syncthreads();
    if (tid == 0) {
        double dmax = 0.0, rn = 0.0;
        for (int j = 0; j < m; ++j) {
            dmax = (j == 0) ? colsq[j] : fmax(dmax, colsq[j]);
            rn += rhs[j] * rhs[j];
        }
        sh_delta = (dmax > 0.0) ? eps * dmax : eps;
        sh_rn = sqrt(rn);
    }
    __syncthreads();
    const double delta = sh_delta, rn = sh_rn;
    if (rn == 0.0) {
        for (int j = tid; j < m; j += blockDim.x) alpha[j] = 0.0;
        if (tid == 0) {
            scal[0] = 0.0;
            scal[2] = delta;
        }
        return;
    }
    const double sd = sqrt(delta);
    for (int e = tid; e < rows * m; e += blockDim.x) {
        const int j = e / rows, i = e % rows;
        double v;
        if (i < m)
            v = (i <= j) ? rf[(size_t)j * C + i] : 0.0;
        else
            v = (i - m == j) ? sd : 0.0;
        a[(size_t)j * rows + i] = v;
    }
    for (int i = tid; i < rows; i += blockDim.x) bvec[i] = (i < m) ? rf[(size_t)m * C + i] : 0.0;
    __syncthreads();
    const double epsm = 2.220446049250313e-16;
    for (int j = warp; j < m; j += nw) {
        double s2 = 0.0;
        for (int i = lane; i < rows; i += 32) s2 += a[(size_t)j * rows + i] * a[(size_t)j * rows + i];
        s2 = warp_sum(s2);
        if (lane == 0) {
            upd[j] = dir[j] = sqrt(s2);
            perm[j] = j;
        }
    }
    __syncthreads();
    if (tid == 0) {
        double maxcol = 0.0;
        for (int j = 0; j < m; ++j) maxcol = fmax(maxcol, upd[j]);
        sh_thr_help = (maxcol * epsm) * (maxcol * epsm) / rows;
        sh_nzp = m;
        sh_maxpivot = 0.0;
    }
    __syncthreads();
    const double down_thr = sqrt(epsm);
    const int size = m;
    for (int k = 0; k < size; ++k) {
        double* col = a + (size_t)k * rows;
        if (warp == 0) {
            // pivot: first column of largest updated norm among k..m-1 (lane-strided candidates,
            // then a shuffle argmax that keeps the smallest index on ties)
            double bv = -1.0;
            int bi = m;
            for (int j = k + lane; j < m; j += 32)
                if (upd[j] > bv) {
                    bv = upd[j];
                    bi = j;
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            const int big = bi;
            if (lane == 0) {
                const double bsq = upd[big] * upd[big];
                if (sh_nzp == size && bsq < sh_thr_help * (rows - k)) sh_nzp = k;
                transp[k] = big;
                if (k != big) {
                    double t = upd[k];
                    upd[k] = upd[big];
                    upd[big] = t;
                    t = dir[k];
                    dir[k] = dir[big];
                    dir[big] = t;
                }
            }
            if (k != big)
                for (int i = lane; i < rows; i += 32) {
                    const double t = col[i];
                    col[i] = a[(size_t)big * rows + i];
                    a[(size_t)big * rows + i] = t;
                }
            __syncwarp();
            // Householder on column k rows k..rows-1 (Eigen makeHouseholder)
            double tail = 0.0;
            for (int i = k + 1 + lane; i < rows; i += 32) tail += col[i] * col[i];
            tail = warp_sum(tail);
            const double c0 = col[k];
            double tau, beta, inv = 0.0;
            if (tail <= 2.2250738585072014e-308) {
                tau = 0.0;
                beta = c0;
            } else {
                beta = sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                inv = c0 - beta;
                tau = (beta - c0) / beta;
            }
            for (int i = k + 1 + lane; i < rows; i += 32) col[i] = (inv == 0.0) ? 0.0 : col[i] / inv;
            __syncwarp();
            if (lane == 0) {
                col[k] = beta;
                sh_tau = tau;
                hc[k] = tau;
                sh_maxpivot = fmax(sh_maxpivot, fabs(beta));
            }
        }
        __syncthreads();
        const double tau = sh_tau;
        // apply to columns k+1.. (one warp per column, lanes over rows) + norm downdate
        for (int j = k + 1 + warp; j < m; j += nw) {
            double* cj = a + (size_t)j * rows;
            if (rows - k == 1) {
                if (lane == 0) cj[k] *= (1.0 - tau);
            } else if (tau != 0.0) {
                double t = 0.0;
                for (int i = k + 1 + lane; i < rows; i += 32) t += col[i] * cj[i];
                t = warp_sum(t) + cj[k];
                for (int i = k + 1 + lane; i < rows; i += 32) cj[i] -= tau * col[i] * t;
                __syncwarp();
                if (lane == 0) cj[k] -= tau * t;
            }
            __syncwarp();
            if (upd[j] != 0.0) {
                double t = fabs(cj[k]) / upd[j];
                t = (1.0 + t) * (1.0 - t);
                if (t < 0.0) t = 0.0;
                const double ratio = upd[j] / dir[j];
                const double t2 = t * ratio * ratio;
                if (t2 <= down_thr) {
                    double s2 = 0.0;
                    for (int i = k + 1 + lane; i < rows; i += 32) s2 += cj[i] * cj[i];
                    s2 = warp_sum(s2);
                    __syncwarp();
                    if (lane == 0) upd[j] = dir[j] = sqrt(s2);
                } else {
                    __syncwarp();
                    if (lane == 0) upd[j] *= sqrt(t);
                }
            }
            __syncwarp();
        }
        __syncthreads();
    }
    if (tid == 0) {
        for (int k = 0; k < size; ++k) {
            const int t = perm[k];
            perm[k] = perm[transp[k]];
            perm[transp[k]] = t;
        }
        const double thr = sh_maxpivot * epsm * size;
        int nz = 0;
        for (int i = 0; i < sh_nzp; ++i) nz += (fabs(a[(size_t)i * rows + i]) > thr) ? 1 : 0;
        sh_nz = nz;
    }
    for (int i = tid; i < rows; i += blockDim.x) cvec[i] = bvec[i];
    for (int j = tid; j < m; j += blockDim.x) al[j] = 0.0;
    __syncthreads();
    const int nz = sh_nz;
    // c <- Q^T b (the nz reflectors in order), then back substitution on the leading nz x nz
    for (int k = 0; k < nz; ++k) {
        const double tk = hc[k];
        const int n = rows - k;
        if (n == 1) {
            if (tid == 0) cvec[k] *= (1.0 - tk);
            __syncthreads();
            continue;
        }
        if (tk == 0.0) continue;
        if (warp == 0) {
            double t = 0.0;
            for (int i = 1 + lane; i < n; i += 32) t += a[(size_t)k * rows + k + i] * cvec[k + i];
            t = warp_sum(t) + cvec[k];
            if (lane == 0) sh_tau = t;
        }
        __syncthreads();
        const double t = sh_tau;
        for (int i = 1 + tid; i < n; i += blockDim.x) cvec[k + i] -= tk * a[(size_t)k * rows + k + i] * t;
        if (tid == 0) cvec[k] -= tk * t;
        __syncthreads();
    }
    for (int i = nz - 1; i >= 0; --i) {
        if (warp == 0) {
            double s2 = 0.0;
            for (int j = i + 1 + lane; j < nz; j += 32) s2 += a[(size_t)j * rows + i] * cvec[j];
            s2 = warp_sum(s2);
            if (lane == 0) cvec[i] = (cvec[i] - s2) / a[(size_t)i * rows + i];
        }
        __syncthreads();
    }
    for (int i = tid; i < nz; i += blockDim.x) al[perm[i]] = cvec[i];
    __syncthreads();
    // residual_rel = ||(R_P^T R_P + delta I) alpha - rhs|| / ||rhs||  via y = R_P alpha
    for (int i = tid; i < m; i += blockDim.x) {
        double y = 0.0;
        for (int j = i; j < m; ++j) y += rf[(size_t)j * C + i] * al[j];
        yv[i] = y;
    }
    __syncthreads();
    if (warp == 0) {
        double rr = 0.0;
        for (int j = lane; j < m; j += 32) {
            double z = delta * al[j];
            for (int i = 0; i <= j; ++i) z += rf[(size_t)j * C + i] * yv[i];
            z -= rhs[j];
            rr += z * z;
        }
        rr = warp_sum(rr);
        if (lane == 0) {
            scal[0] = sqrt(rr) / rn;
            scal[2] = delta;
        }
    }
    for (int j = tid; j < m; j += blockDim.x) alpha[j] = al[j];
}

struct UpdParams {
    int64_t n;
    int cap;
    const int* ring;
    const double* wu;
    const double* ub;
    const double* gb;
    const double* alpha;
    double* uhat;
    double* d;
    double* red;
};

__global__ void accel_update_kernel(const UpdParams p) {
    __shared__ double red[32];
    const int m = p.ring[0], head = p.ring[1];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
        const double ub = p.ub[i];
        double uh = ub;
        for (int j = 0; j < m; ++j) {
            const int slot = (head + j) % p.cap;
            uh += p.alpha[j] * (ub - p.wu[(int64_t)slot * p.n + i]);
        }
        if (p.uhat) p.uhat[i] = uh;
        const double dv = uh - ub;
        p.d[i] = dv;
        s += p.gb[i] * dv;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        p.red[blockIdx.x] = t;
    }
}

__global__ void accel_slope_kernel(const double* red, int nblk, double* scal) {
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int b = 0; b < nblk; ++b) t += red[b];
        scal[1] = t;
    }
}

}  // namespace

AccelWork* accel_create(int64_t n, int cap) {
    if (cap < 1 || cap > kMaxWindow)
        throw std::invalid_argument("device accelerate supports window 1.." + std::to_string(kMaxWindow));
    auto* a = new AccelWork();
    a->n = n;
    a->cap = cap;
    const int C = cap + 1;
    a->leaf_rows = tsqr_leaf_rows(C);
    const int64_t nblocks = (n + a->leaf_rows - 1) / a->leaf_rows;
    a->leaf_grid = (int)std::min<int64_t>(nblocks, 148);
    const size_t rsz = sizeof(double) * (size_t)std::max<int64_t>(a->leaf_grid, 1) * C * C;
    CPFIT_CUDA(cudaMalloc(&a->rbuf[0], rsz));
    CPFIT_CUDA(cudaMalloc(&a->rbuf[1], rsz));
    CPFIT_CUDA(cudaMalloc(&a->alpha, sizeof(double) * std::max(64, cap)));
    CPFIT_CUDA(cudaMalloc(&a->scal, sizeof(double) * 8));
    CPFIT_CUDA(cudaMalloc(&a->red, sizeof(double) * 1024));
    return a;
}

void accel_destroy(AccelWork* a) {
    if (!a) return;
    cudaFree(a->rbuf[0]);
    cudaFree(a->rbuf[1]);
    cudaFree(a->alpha);
    cudaFree(a->scal);
    cudaFree(a->red);
    delete a;
}

void accelerate_device(AccelWork& a, const double* wu, const double* wg, const int* ring, const double* ub,
                       const double* gb, double eps, double* uhat, double* d, cudaStream_t st, bool slope_by_caller) {
    const int C = a.cap + 1;  // smem sized for the full window
    TsqrParams p{};
    p.n = a.n;
    p.cap = a.cap;
    p.ring = ring;
    p.wg = wg;
    p.gb = gb;
    p.per_block = a.leaf_rows;
    p.nblocks = (a.n + a.leaf_rows - 1) / a.leaf_rows;
    p.blocks_per_cta = (p.nblocks + a.leaf_grid - 1) / a.leaf_grid;
    p.rout = a.rbuf[0];
    size_t smem = sizeof(double) * (size_t)(C + a.leaf_rows) * C;
    CPFIT_CUDA(cudaFuncSetAttribute(tsqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int g0 = (int)((p.nblocks + p.blocks_per_cta - 1) / p.blocks_per_cta);
    tsqr_kernel<<<g0, kTsqrThreads, smem, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
    int64_t cnt = g0;
    int src = 0;
    const int per = tsqr_merge_per(C);
    while (cnt > 1) {
        TsqrParams q = p;
        q.rin = a.rbuf[src];
        q.nin = cnt;
        q.rout = a.rbuf[src ^ 1];
        q.per_block = per;
        q.nblocks = (cnt + per - 1) / per;
        // one R per block (wide windows): every CTA merges at least two blocks so cnt shrinks
        const int64_t gmax = per == 1 ? std::max<int64_t>(1, q.nblocks / 2) : 148;
        q.blocks_per_cta = (q.nblocks + gmax - 1) / gmax;
        const int g = (int)((q.nblocks + q.blocks_per_cta - 1) / q.blocks_per_cta);
        smem = sizeof(double) * (size_t)(C + per * C) * C;
        tsqr_kernel<<<g, kTsqrThreads, smem, st>>>(q);
        CPFIT_CUDA(cudaGetLastError());
        cnt = g;
        src ^= 1;
    }
    const size_t ssmem = sizeof(double) * (2 * (size_t)a.cap * a.cap);
    CPFIT_CUDA(cudaFuncSetAttribute(accel_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
    accel_solve_kernel<<<1, kSolveThreads, ssmem, st>>>(a.rbuf[src], ring, eps, a.alpha, a.scal);
    CPFIT_CUDA(cudaGetLastError());
    UpdParams u{};
    u.n = a.n;
    u.cap = a.cap;
    u.ring = ring;
    u.wu = wu;
    u.ub = ub;
    u.gb = gb;
    u.alpha = a.alpha;
    u.uhat = uhat;
    u.d = d;
    u.red = a.red;
    const int nb = accel_update_blocks(a);
    accel_update_kernel<<<nb, 256, 0, st>>>(u);
    if (!slope_by_caller) accel_slope_kernel<<<1, 32, 0, st>>>(a.red, nb, a.scal);
    CPFIT_CUDA(cudaGetLastError());
}

}  // namespace cpfit_gpu
