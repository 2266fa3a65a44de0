// Sparse COO MTTKRP on device (tensor.cpp:242-259) for the sparse objective/gradient
// (kruskal.cpp:106-111, 127-149).
//
// Each mode n has its own mode-n-sorted copy (built at upload), so M_n(i, :) is a
// segmented sum over rows of that copy: one warp per row, lanes strided over the row's
// nonzeros, product v * prod_{k != n} A_k(c_k, :) in the reference's mode order, then a
// warp reduction. Deterministic (no atomics); the streamed bytes per nonzero are the
// value plus N-1 int32 indices; the factor-row gathers hit L2 (row-major RP-padded
// copies of the factors, rebuilt per evaluation).
#include "sparse.cuh"

#include <algorithm>
#include <thread>

namespace cpfit_gpu {

namespace {

struct SpParams {
    int64_t In;
    int64_t nnz;
    const int64_t* rowptr;
    const int32_t* oidx;
    const double* vals;
    int nother;
    int R;  // lanes r >= R skip their (zero) factor loads: a row of R < RP doubles touches fewer sectors
    const double* frow[kMaxOrder];
    double* out;  // In x RP
};

// Warp per output row; lanes span the rank: lane = (g, r) with r = lane % RP and
// G = 32 / RP nonzeros per step, so each factor-row gather is one contiguous RP*8-byte segment
// per lane group (one L1 wavefront) instead of 32 scattered rows. Indices and values are read
// coalesced, 32 nonzeros at a time, and broadcast to the lane groups with shuffles. ORD is the
// number of other modes (N-1) when specialised, 0 generic.
template <int RP, int NO>
__global__ void __launch_bounds__(256) sp_mttkrp_kernel(const SpParams p) {
    constexpr int G = 32 / RP;
    const int lane = threadIdx.x & 31;
    const int r = lane % RP, g = lane / RP;
    const int nother = NO > 0 ? NO : p.nother;
    const bool live = r < p.R;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < p.In; i += nw) {
        double acc = 0.0;
        const int64_t j0 = p.rowptr[i], j1 = p.rowptr[i + 1];
        // the next chunk's values and indices are loaded while this chunk's gathers run
        constexpr int NK = NO > 0 ? NO : kMaxOrder;
        double vn = 0.0;
        int cn[NK];
        auto load_chunk = [&](int64_t jb) {
            const int64_t jl = jb + lane;
            const bool okl = jl < j1;
            vn = okl ? __ldg(p.vals + jl) : 0.0;
#pragma unroll
            for (int k = 0; k < NK; ++k) cn[k] = (okl && k < nother) ? __ldg(p.oidx + (int64_t)k * p.nnz + jl) : 0;
        };
        if (j0 < j1) load_chunk(j0);
        for (int64_t jb = j0; jb < j1; jb += 32) {
            const double vl = vn;
            int cl[NK];
#pragma unroll
            for (int k = 0; k < NK; ++k) cl[k] = cn[k];
            if (jb + 32 < j1) load_chunk(jb + 32);
            const int cnt = (int)imin64(32, j1 - jb);
            if (cnt == 32) {
                // full chunk: every gather of the 32 nonzeros in flight before the products
                // (the loop is L2-latency bound otherwise)
                double pr[32 / G];
#pragma unroll
                for (int t = 0; t < 32 / G; ++t) {
                    const int q = t * G + g;
                    double prod = __shfl_sync(0xffffffffu, vl, q);
#pragma unroll
                    for (int k = 0; k < (NO > 0 ? NO : kMaxOrder); ++k) {
                        if (k < nother) {
                            const int c = __shfl_sync(0xffffffffu, cl[k], q);
                            prod *= live ? __ldg(p.frow[k] + (int64_t)c * RP + r) : 0.0;
                        }
                    }
                    pr[t] = prod;
                }
#pragma unroll
                for (int t = 0; t < 32 / G; ++t) acc += pr[t];
                continue;
            }
            for (int q0 = 0; q0 < cnt; q0 += G) {
                const int q = q0 + g;
                double prod = __shfl_sync(0xffffffffu, vl, q & 31);
#pragma unroll
                for (int k = 0; k < (NO > 0 ? NO : kMaxOrder); ++k) {
                    if (k < nother) {
                        const int c = __shfl_sync(0xffffffffu, cl[k], q & 31);
                        prod *= live ? __ldg(p.frow[k] + (int64_t)c * RP + r) : 0.0;
                    }
                }
                if (q < cnt) acc += prod;
            }
        }
        // combine the G lane groups (fixed order)
#pragma unroll
        for (int o = RP; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (g == 0) p.out[i * RP + r] = acc;
    }
}

template <int RP>
void launch_sp(const SpParams& p, int blocks, int order, cudaStream_t st) {
    switch (order) {
        case 3: sp_mttkrp_kernel<RP, 2><<<blocks, 256, 0, st>>>(p); break;
        case 4: sp_mttkrp_kernel<RP, 3><<<blocks, 256, 0, st>>>(p); break;
        default: sp_mttkrp_kernel<RP, 0><<<blocks, 256, 0, st>>>(p); break;
    }
}

__global__ void frows_kernel(int order, const int64_t* dims_d, int64_t d0, int64_t d1, int64_t d2, int64_t d3,
                             int64_t d4, int64_t d5, int64_t d6, int64_t d7, int R, int RP, const double* u,
                             double* frows) {
    const int64_t dims[8] = {d0, d1, d2, d3, d4, d5, d6, d7};
    (void)dims_d;
    int64_t total = 0;
    for (int n = 0; n < order; ++n) total += dims[n] * RP;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t rem = e, uoff = 0;
        int n = 0;
        while (rem >= dims[n] * RP) {
            rem -= dims[n] * RP;
            uoff += dims[n] * R;
            ++n;
        }
        const int64_t i = rem / RP;
        const int r = (int)(rem % RP);
        frows[e] = (r < R) ? u[uoff + (int64_t)r * dims[n] + i] : 0.0;
    }
}


// The eight contractions <T, [[X0, X1, X2]]> (X_n in {A_n, D_n}, index 4 b0 + 2 b1 + b2, b_n = 1
// selects D_n) of a sparse order-3 tensor for the exact line-search polynomial (poly.cu): warp per
// mode-0 row i over the mode-0 sorted copy, lanes spanning the rank as in sp_mttkrp_kernel; per
// 32-nonzero chunk the four inner sums sum_nz v X1[j][r] X2[k][r] in fp64, folded into
// double-double with X0[i][r] in {A0, D0}; per-block partials [block][8] for coef_kernel.
template <int RP>
__global__ void __launch_bounds__(256) sp_line8_kernel(const SpParams p, const double* a0rows, const double* d0rows,
                                                       const double* a1, const double* e1, const double* a2,
                                                       const double* e2, dd* part, double* m0xy) {
    constexpr int G = 32 / RP;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = lane % RP, g = lane / RP;
    const bool live = r < p.R;
    dd acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = dd{0.0, 0.0};
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < p.In; i += nw) {
        const double x0a = live ? a0rows[i * RP + r] : 0.0, x0d = live ? d0rows[i * RP + r] : 0.0;
        const int64_t j0 = p.rowptr[i], j1 = p.rowptr[i + 1];
        double qs[4] = {0.0, 0.0, 0.0, 0.0};  // the row's mode-0 products X1 X2 (for M0 at u*)
        for (int64_t jb = j0; jb < j1; jb += 32) {
            const int64_t jl = jb + lane;
            const bool okl = jl < j1;
            const double vl = okl ? __ldg(p.vals + jl) : 0.0;
            const int cj = okl ? __ldg(p.oidx + jl) : 0, ck = okl ? __ldg(p.oidx + p.nnz + jl) : 0;
            const int cnt = (int)imin64(32, j1 - jb);
            double q[4] = {0.0, 0.0, 0.0, 0.0};  // X1 X2 in {AA, AD, DA, DD}
            for (int q0 = 0; q0 < cnt; q0 += G) {
                const int qq = q0 + g;
                const double v = __shfl_sync(0xffffffffu, vl, qq & 31);
                const int j = __shfl_sync(0xffffffffu, cj, qq & 31), k = __shfl_sync(0xffffffffu, ck, qq & 31);
                if (qq < cnt && live) {
                    const double y1a = __ldg(a1 + (int64_t)j * RP + r), y1d = __ldg(e1 + (int64_t)j * RP + r);
                    const double y2a = __ldg(a2 + (int64_t)k * RP + r), y2d = __ldg(e2 + (int64_t)k * RP + r);
                    const double va = v * y1a, vd = v * y1d;
                    q[0] = fma(va, y2a, q[0]);
                    q[1] = fma(va, y2d, q[1]);
                    q[2] = fma(vd, y2a, q[2]);
                    q[3] = fma(vd, y2d, q[3]);
                }
            }
#pragma unroll
            for (int b12 = 0; b12 < 4; ++b12) {
                acc[b12] = dd_fma(acc[b12], x0a, q[b12]);
                acc[4 + b12] = dd_fma(acc[4 + b12], x0d, q[b12]);
                qs[b12] += q[b12];
            }
        }
        if (m0xy) {  // combine the lane groups (fixed order), one row of each product
#pragma unroll
            for (int b12 = 0; b12 < 4; ++b12) {
                double v = qs[b12];
#pragma unroll
                for (int o = RP; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (g == 0) m0xy[((int64_t)b12 * p.In + i) * RP + r] = live ? v : 0.0;
            }
        }
    }
    // warp tree (fixed order), then the warps in order
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const dd t{__shfl_xor_sync(0xffffffffu, acc[k].hi, o), __shfl_xor_sync(0xffffffffu, acc[k].lo, o)};
            acc[k] = dd_add(acc[k], t);
        }
    __shared__ dd red[8][8];
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < 8; ++k) red[warp][k] = acc[k];
    __syncthreads();
    if (threadIdx.x < 8) {
        dd s{0.0, 0.0};
        for (int w8 = 0; w8 < (int)(blockDim.x >> 5); ++w8) s = dd_add(s, red[w8][threadIdx.x]);
        part[(size_t)blockIdx.x * 8 + threadIdx.x] = s;
    }
}

}  // namespace

void upload_sparse_modes(DevTensor& t, const std::vector<int64_t>& coords, const std::vector<double>& vals,
                         cudaStream_t st) {
    auto* sm = new SparseModes();
    t.modes = sm;
    const int N = t.order;
    const int64_t nnz = (int64_t)vals.size();
    // the N counting sorts are independent: one host thread each, then the uploads in order
    std::vector<std::vector<int64_t>> rowptrs((size_t)N);
    std::vector<std::vector<int32_t>> oidxs((size_t)N);
    std::vector<std::vector<double>> svs((size_t)N);
    auto sort_mode = [&](int n) {
        const int64_t In = t.dims[n];
        std::vector<int64_t>& rowptr = rowptrs[(size_t)n];
        rowptr.assign((size_t)In + 1, 0);
        for (int64_t j = 0; j < nnz; ++j) ++rowptr[(size_t)coords[(size_t)j * N + n] + 1];
        for (int64_t i = 0; i < In; ++i) rowptr[(size_t)i + 1] += rowptr[(size_t)i];
        std::vector<int64_t> pos(rowptr.begin(), rowptr.end() - 1);
        std::vector<int32_t>& oidx = oidxs[(size_t)n];
        oidx.resize((size_t)std::max(1, N - 1) * (size_t)nnz);
        std::vector<double>& sv = svs[(size_t)n];
        sv.resize((size_t)nnz);
        for (int64_t j = 0; j < nnz; ++j) {  // stable counting sort by mode-n index
            const int64_t dst = pos[(size_t)coords[(size_t)j * N + n]]++;
            sv[(size_t)dst] = vals[(size_t)j];
            int k = 0;
            for (int m = 0; m < N; ++m) {
                if (m == n) continue;
                oidx[(size_t)k * nnz + dst] = (int32_t)coords[(size_t)j * N + m];
                ++k;
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (int n = 1; n < N; ++n) th.emplace_back(sort_mode, n);
        sort_mode(0);
        for (auto& x : th) x.join();
    }
    for (int n = 0; n < N; ++n) {
        const std::vector<int64_t>& rowptr = rowptrs[(size_t)n];
        const std::vector<int32_t>& oidx = oidxs[(size_t)n];
        const std::vector<double>& sv = svs[(size_t)n];
        CPFIT_CUDA(cudaMalloc(&sm->rowptr[n], sizeof(int64_t) * rowptr.size()));
        CPFIT_CUDA(cudaMalloc(&sm->oidx[n], sizeof(int32_t) * std::max<size_t>(oidx.size(), 1)));
        CPFIT_CUDA(cudaMalloc(&sm->vals[n], sizeof(double) * std::max<size_t>(sv.size(), 1)));
        CPFIT_CUDA(cudaMemcpyAsync(sm->rowptr[n], rowptr.data(), sizeof(int64_t) * rowptr.size(), cudaMemcpyHostToDevice, st));
        if (nnz > 0) {
            CPFIT_CUDA(cudaMemcpyAsync(sm->oidx[n], oidx.data(), sizeof(int32_t) * oidx.size(), cudaMemcpyHostToDevice, st));
            CPFIT_CUDA(cudaMemcpyAsync(sm->vals[n], sv.data(), sizeof(double) * sv.size(), cudaMemcpyHostToDevice, st));
        }
        CPFIT_CUDA(cudaStreamSynchronize(st));  // host staging vectors go out of scope
    }
    t.nnz = nnz;
}

void free_sparse_modes(DevTensor& t) {
    if (!t.modes) return;
    for (int n = 0; n < kMaxOrder; ++n) {
        cudaFree(t.modes->rowptr[n]);
        cudaFree(t.modes->oidx[n]);
        cudaFree(t.modes->vals[n]);
    }
    delete t.modes;
    t.modes = nullptr;
}

void sparse_all_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st,
                      int skip_mode) {
    const int N = t.order;
    int64_t total = 0;
    for (int n = 0; n < N; ++n) total += t.dims[n] * w.RP;
    frows_kernel<<<(int)std::min<int64_t>(1024, (total + 255) / 256), 256, 0, st>>>(
        N, nullptr, t.dims[0], t.dims[1], t.dims[2], t.dims[3], t.dims[4], t.dims[5], t.dims[6], t.dims[7], w.R, w.RP,
        u, w.frows);
    CPFIT_CUDA(cudaGetLastError());
    int64_t off[kMaxOrder + 1];
    off[0] = 0;
    for (int n = 0; n < N; ++n) off[n + 1] = off[n] + t.dims[n] * w.RP;
    for (int n = 0; n < N; ++n) {
        if ((only_mode >= 0 && n != only_mode) || n == skip_mode) continue;
        SpParams p{};
        p.In = t.dims[n];
        p.nnz = t.nnz;
        p.rowptr = t.modes->rowptr[n];
        p.oidx = t.modes->oidx[n];
        p.vals = t.modes->vals[n];
        int k = 0;
        for (int m = 0; m < N; ++m)
            if (m != n) p.frow[k++] = w.frows + off[m];
        p.nother = k;
        p.R = w.R;
        p.out = w.sp_part + off[n];
        const int blocks = (int)std::min<int64_t>(148 * 8, (p.In * 32 + 255) / 256);
        switch (w.RP) {
            case 8: launch_sp<8>(p, blocks, N, st); break;
            case 16: launch_sp<16>(p, blocks, N, st); break;
            default: launch_sp<32>(p, blocks, N, st); break;
        }
        CPFIT_CUDA(cudaGetLastError());
    }
}

}  // namespace cpfit_gpu

namespace cpfit_gpu {
// Row-major copies of the factors of u_bar (w.frows) and d (drows), then the eight line
// contractions into part[nblocks][8] (poly.cu's coefficient kernel sums them in order).
void sparse_line_contractions(const DevTensor& t, EvalWork& w, const double* ub, const double* d, double* drows,
                              dd* part, int nblocks, cudaStream_t st, double* m0xy) {
    if (t.order != 3) throw std::logic_error("sparse line contractions: order 3 only");
    int64_t total = 0;
    for (int n = 0; n < 3; ++n) total += t.dims[n] * w.RP;
    const int fb = (int)std::min<int64_t>(1024, (total + 255) / 256);
    frows_kernel<<<fb, 256, 0, st>>>(3, nullptr, t.dims[0], t.dims[1], t.dims[2], 0, 0, 0, 0, 0, w.R, w.RP, ub, w.frows);
    frows_kernel<<<fb, 256, 0, st>>>(3, nullptr, t.dims[0], t.dims[1], t.dims[2], 0, 0, 0, 0, 0, w.R, w.RP, d, drows);
    CPFIT_CUDA(cudaGetLastError());
    const int64_t o1 = t.dims[0] * w.RP, o2 = o1 + t.dims[1] * w.RP;
    SpParams p{};
    p.In = t.dims[0];
    p.nnz = t.nnz;
    p.rowptr = t.modes->rowptr[0];
    p.oidx = t.modes->oidx[0];
    p.vals = t.modes->vals[0];
    p.nother = 2;
    p.R = w.R;
    switch (w.RP) {
        case 8:
            sp_line8_kernel<8><<<nblocks, 256, 0, st>>>(p, w.frows, drows, w.frows + o1, drows + o1, w.frows + o2, drows + o2, part, m0xy);
            break;
        case 16:
            sp_line8_kernel<16><<<nblocks, 256, 0, st>>>(p, w.frows, drows, w.frows + o1, drows + o1, w.frows + o2, drows + o2, part, m0xy);
            break;
        default:
            sp_line8_kernel<32><<<nblocks, 256, 0, st>>>(p, w.frows, drows, w.frows + o1, drows + o1, w.frows + o2, drows + o2, part, m0xy);
            break;
    }
    CPFIT_CUDA(cudaGetLastError());
}
}  // namespace cpfit_gpu

namespace cpfit_gpu {
namespace {
__global__ void sp_m0_point_kernel(const double* __restrict__ q, int64_t n, const double* beta, double* out) {
    const double b = *beta;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = q[e] + b * (q[n + e] + q[2 * n + e]) + (b * b) * q[3 * n + e];
}
}  // namespace

void sparse_m0_at_point(EvalWork& w, const double* m0xy, int64_t I0, const double* beta, cudaStream_t st) {
    const int64_t n = I0 * w.RP;
    sp_m0_point_kernel<<<(int)std::min<int64_t>(1184, (n + 255) / 256), 256, 0, st>>>(m0xy, n, beta, w.sp_part);
    CPFIT_CUDA(cudaGetLastError());
}
}  // namespace cpfit_gpu
