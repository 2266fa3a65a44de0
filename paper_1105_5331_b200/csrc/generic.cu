// Generic dense MTTKRP and residual objective (tensor.cpp:206-240, kruskal.cpp:83-102) for the
// dense shapes the fibre-tile passes (fiber.cuh) do not take: order 1 (tensor.cpp:214-216) and
// mode-0 fibres longer than a shared-memory tile holds. Such tensors run the per-mode
// ("rowwise") evaluation the sparse path uses: every mode's M_n into w.sp_part, then the
// gradient epilogue (dense.cu grad_kernel) with the residual f from these partials.
//
// Kernel: mode n's matricisation T_(n) (I_n rows) times W = KR(the other factors), W never
// materialised in HBM. A CTA owns a block of rows (one row per thread, R accumulators in
// registers) and a contiguous range of columns; per chunk of kCols columns it stages the W rows
// and the columns' element offsets in shared memory, then every thread streams its row's
// elements. For mode 0 consecutive threads read consecutive doubles; for n >= 1 each thread
// walks its own contiguous run of the lower modes (columns are ordered lower-modes-fastest), so
// every line it touches is reused by its next loads. Column-range partials are summed in a
// fixed order (deterministic). The mode-0 kernel can also accumulate the residual
// (T - model)^2 per element, model = A0(i,:) . W(c,:), as the reference's dense objective does.
#include "device.cuh"

#include <algorithm>
#include <stdexcept>

namespace cpfit_gpu {
namespace {

constexpr int kCols = 32;      // columns staged per chunk
constexpr int kGenThreads = 128;

struct GenParams {
    int order, n, R;
    int64_t dims[kMaxOrder];
    const double* T;
    int64_t ldT;
    const double* u;
    int64_t uoff[kMaxOrder];
    int64_t In, C;        // rows, columns (K / I_n)
    int64_t stride;       // element distance between rows i and i + 1
    int64_t Lp;           // n >= 1: prod_{1 <= m < n} I_m
    int64_t cols_per_cta;
    double* part;         // [gridDim.x][In][RP]
    double* fpart;        // [gridDim.y * gridDim.x] residual partials (mode 0), or null
};

// column c -> element offset of row 0, and the W row (product of the other modes' factor rows)
__device__ __forceinline__ int64_t column_base(const GenParams& p, int64_t c, int* idx) {
    if (p.n == 0) {
        int64_t rem = c;
        for (int m = 1; m < p.order; ++m) {
            idx[m] = (int)(rem % p.dims[m]);
            rem /= p.dims[m];
        }
        return p.ldT * c;
    }
    // c = l + L t, l = (i_0 .. i_{n-1}) (i_0 fastest), t = (i_{n+1} ..)
    int64_t rem = c;
    for (int m = 0; m < p.n; ++m) {
        idx[m] = (int)(rem % p.dims[m]);
        rem /= p.dims[m];
    }
    const int64_t t = rem;
    for (int m = p.n + 1; m < p.order; ++m) {
        idx[m] = (int)(rem % p.dims[m]);
        rem /= p.dims[m];
    }
    int64_t lp = 0, mult = 1;
    for (int m = 1; m < p.n; ++m) {
        lp += idx[m] * mult;
        mult *= p.dims[m];
    }
    return idx[0] + p.ldT * (lp + p.Lp * p.In * t);
}

// RP = 64 (ranks above 32): the residual's A_0 row lives in shared memory ([r][thread], the
// accumulators alone fill half the register file)
template <int RP>
__global__ void __launch_bounds__(kGenThreads) gen_mttkrp_kernel(const GenParams p) {
    constexpr bool A0S = RP > 32;
    __shared__ double Ws[kCols][RP + 1];
    __shared__ int64_t base[kCols];
    __shared__ int cidx[kCols][kMaxOrder];
    __shared__ double fred[kGenThreads / 32];
    extern __shared__ double a0sm[];  // A0S: [RP][blockDim.x]
    const int tid = threadIdx.x;
    const int64_t i = (int64_t)blockIdx.y * blockDim.x + tid;
    const bool row_ok = i < p.In;
    const int64_t c0 = (int64_t)blockIdx.x * p.cols_per_cta;
    const int64_t c1 = (p.C < c0 + p.cols_per_cta) ? p.C : c0 + p.cols_per_cta;
    double acc[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[r] = 0.0;
    double a0[A0S ? 1 : RP];
    double fs = 0.0;
    if (p.fpart) {
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const double v = (row_ok && r < p.R) ? p.u[p.uoff[0] + (int64_t)r * p.In + i] : 0.0;
            if (A0S)
                a0sm[r * blockDim.x + tid] = v;
            else
                a0[r] = v;
        }
    }
    auto a0v = [&](int r) { return A0S ? a0sm[r * blockDim.x + tid] : a0[r]; };
    for (int64_t cc = c0; cc < c1; cc += kCols) {
        const int nc = (int)((c1 - cc < kCols) ? c1 - cc : kCols);
        __syncthreads();  // the previous chunk's W is consumed
        if (tid < nc) base[tid] = column_base(p, cc + tid, cidx[tid]);
        __syncthreads();
        for (int e = tid; e < nc * RP; e += blockDim.x) {
            const int k = e / RP, r = e % RP;
            double w = 0.0;
            if (r < p.R) {
                w = 1.0;
                for (int m = 0; m < p.order; ++m)
                    if (m != p.n) w *= p.u[p.uoff[m] + (int64_t)r * p.dims[m] + cidx[k][m]];
            }
            Ws[k][r] = w;
        }
        __syncthreads();
        if (row_ok) {
            const double* trow = p.T + i * p.stride;
            int k = 0;
            for (; k + 4 <= nc; k += 4) {
                double x[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = trow[base[k + q]];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (p.fpart) {
                        double m = 0.0;
#pragma unroll
                        for (int r = 0; r < RP; ++r) m += a0v(r) * Ws[k + q][r];
                        const double d = x[q] - m;
                        fs += d * d;
                    }
#pragma unroll
                    for (int r = 0; r < RP; ++r) acc[r] += x[q] * Ws[k + q][r];
                }
            }
            for (; k < nc; ++k) {
                const double x = trow[base[k]];
                if (p.fpart) {
                    double m = 0.0;
#pragma unroll
                    for (int r = 0; r < RP; ++r) m += a0v(r) * Ws[k][r];
                    const double d = x - m;
                    fs += d * d;
                }
#pragma unroll
                for (int r = 0; r < RP; ++r) acc[r] += x * Ws[k][r];
            }
        }
    }
    if (row_ok) {
        double* out = p.part + ((int64_t)blockIdx.x * p.In + i) * RP;
#pragma unroll
        for (int r = 0; r < RP; ++r) out[r] = acc[r];
    }
    if (p.fpart) {
        fs = warp_sum(fs);
        if ((tid & 31) == 0) fred[tid >> 5] = fs;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < (int)blockDim.x / 32; ++w) s += fred[w];
            p.fpart[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
        }
    }
}

// out[i][r] = sum over column ranges (in order) of part[x][i][r]
__global__ void gen_reduce_kernel(const double* part, int nx, int64_t n, double* out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int x = 0; x < nx; ++x) s += part[(int64_t)x * n + e];
        out[e] = s;
    }
}

int gen_threads(int64_t In) { return (int)std::min<int64_t>(kGenThreads, (In + 31) / 32 * 32); }

}  // namespace

// Grid of mode n: gy row blocks x gx column ranges, gx sized for ~4 CTAs per SM and capped so
// the partials stay <= 4M doubles.
void generic_plan(const DevTensor& t, int RP, int n, int* gx, int64_t* cols_per_cta, int* gy) {
    const int64_t In = t.dims[n], C = t.K / In;
    const int th = gen_threads(In);
    *gy = (int)((In + th - 1) / th);
    int64_t want = std::max<int64_t>(1, (4LL * sm_count() + *gy - 1) / *gy);
    want = std::min<int64_t>(want, (C + kCols - 1) / kCols);
    want = std::min<int64_t>(want, std::max<int64_t>(1, (4LL << 20) / (In * RP)));
    const int64_t cpc = ((C + want - 1) / want + kCols - 1) / kCols * kCols;
    *cols_per_cta = cpc;
    *gx = (int)((C + cpc - 1) / cpc);
}

// M_n of every mode (only_mode < 0; mode 0 also leaves the residual partials in w.f_part) or
// of one mode, into w.sp_part [mode offset][i][RP].
void generic_all_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st,
                       int skip_mode) {
    int64_t off = 0;
    for (int n = 0; n < t.order; ++n) {
        const int64_t In = t.dims[n];
        if ((only_mode < 0 || n == only_mode) && n != skip_mode) {
            GenParams p{};
            p.order = t.order;
            p.n = n;
            p.R = w.R;
            for (int m = 0; m < t.order; ++m) {
                p.dims[m] = t.dims[m];
                p.uoff[m] = w.off[m];
            }
            p.T = t.T;
            p.ldT = t.ldT;
            p.u = u;
            p.In = In;
            p.C = t.K / In;
            int64_t lp = 1;
            for (int m = 1; m < n; ++m) lp *= t.dims[m];
            p.Lp = lp;
            p.stride = (n == 0) ? 1 : t.ldT * lp;
            int gx, gy;
            generic_plan(t, w.RP, n, &gx, &p.cols_per_cta, &gy);
            p.part = w.gen_part;
            p.fpart = (n == 0 && only_mode < 0) ? w.f_part : nullptr;
            const dim3 grid((unsigned)gx, (unsigned)gy);
            const int th = gen_threads(In);
            switch (w.RP) {
                case 8: gen_mttkrp_kernel<8><<<grid, th, 0, st>>>(p); break;
                case 16: gen_mttkrp_kernel<16><<<grid, th, 0, st>>>(p); break;
                case 32: gen_mttkrp_kernel<32><<<grid, th, 0, st>>>(p); break;
                default: {
                    const size_t sm = p.fpart ? sizeof(double) * 64 * th : 0;
                    CPFIT_CUDA(cudaFuncSetAttribute(gen_mttkrp_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)sm));
                    gen_mttkrp_kernel<64><<<grid, th, sm, st>>>(p);
                    break;
                }
            }
            CPFIT_CUDA(cudaGetLastError());
            const int64_t ne = In * w.RP;
            gen_reduce_kernel<<<(int)std::min<int64_t>(1184, (ne + 255) / 256), 256, 0, st>>>(w.gen_part, gx, ne,
                                                                                             w.sp_part + off);
            CPFIT_CUDA(cudaGetLastError());
        }
        off += In * w.RP;
    }
}

}  // namespace cpfit_gpu
