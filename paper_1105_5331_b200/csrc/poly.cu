// Exact line search along the N-GMRES direction for dense order-3 tensors.
//
// The line search of ngmres.cpp:111-147 (Moré–Thuente, line_search.cpp) evaluates
// phi(a) = f(u_bar + a d) and phi'(a) = g(u_bar + a d).d at each trial step. With
// A_n(a) = A_n + a D_n,
//   f(a) = 1/2 ||T||^2 - <T, [[A_0(a), A_1(a), A_2(a)]]> + 1/2 1^T (G_0(a) * G_1(a) * G_2(a)) 1,
//   G_n(a) = A_n^T A_n + a (A_n^T D_n + D_n^T A_n) + a^2 D_n^T D_n,
// so phi is a polynomial of degree 6 and phi' its derivative. Its coefficients need
//   * the eight contractions <T, [[X_0, X_1, X_2]]>, X_n in {A_n, D_n}, which follow from
//     S(u_bar) = T x_1 A_0 (left in w.S by the evaluation of u_bar) and S_d = T x_1 D_0 (one
//     streaming pass) by a weighted reduction over the fibres — computed in double-double;
//   * the nine R x R products A_n^T A_n, A_n^T D_n, D_n^T D_n (double-double);
//   * ||T||^2 (double-double since tensor creation).
// One S pass + reductions replace every trial evaluation of the line search (2-3 fused passes
// per iteration at the benchmark configuration); the accepted point is then evaluated once from
// S(u*) = S(u_bar) + beta S_d plus an M0 pass (eval_given_s_device). phi is a difference of
// terms of size ||T||^2, hence double-double throughout.
#include "device.cuh"
#include "poly.cuh"

#include <algorithm>

namespace cpfit_gpu {

namespace {

constexpr int kKinds = 3;  // A^T A, A^T D, D^T D

struct CrossParams {
    int R, RP;
    int64_t dims[3];
    const double* a[3];
    const double* d[3];
    int nchunk[3];
    int64_t base[3];  // first task of mode n
    int64_t rows[3];
    dd* part;         // [task]
    dd* out;          // [mode][kind][RP*RP]
    unsigned int* counter;
};

// warp task t of mode n: (chunk c, kind k, q, r) -> part
__global__ void __launch_bounds__(256) cross_gram_kernel(const CrossParams p) {
    const int RR = p.R * p.R;
    const int64_t total = p.base[2] + (int64_t)p.nchunk[2] * kKinds * RR;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    for (int64_t t = warp; t < total; t += nwarps) {
        const int n = t < p.base[1] ? 0 : (t < p.base[2] ? 1 : 2);
        const int64_t tl = t - p.base[n];
        const int c = (int)(tl / (kKinds * RR));
        const int k = (int)((tl / RR) % kKinds);
        const int e = (int)(tl % RR);
        const int q = e / p.R, r = e % p.R;
        const int64_t In = p.dims[n];
        const double* x = (k == 2 ? p.d[n] : p.a[n]) + (int64_t)q * In;
        const double* y = (k == 0 ? p.a[n] : p.d[n]) + (int64_t)r * In;
        const int64_t i0 = (int64_t)c * p.rows[n];
        const dd s = warp_dot_dd(x, y, i0, imin64(In, i0 + p.rows[n]));
        if ((threadIdx.x & 31) == 0) p.part[t] = s;
    }
    if (!last_block_arrives(p.counter)) return;
    for (int f = threadIdx.x; f < 3 * kKinds * p.RP * p.RP; f += blockDim.x) {
        const int n = f / (kKinds * p.RP * p.RP);
        const int k = (f / (p.RP * p.RP)) % kKinds;
        const int e = f % (p.RP * p.RP);
        const int q = e / p.RP, r = e % p.RP;
        dd s{0.0, 0.0};
        if (q < p.R && r < p.R)
            for (int c = 0; c < p.nchunk[n]; ++c)
                s = dd_add(s, p.part[p.base[n] + ((int64_t)c * kKinds + k) * RR + q * p.R + r]);
        p.out[f] = s;
    }
}

struct S8Params {
    const double* S;   // S(u_bar), J x RP
    const double* Sd;  // S_d
    int64_t J, I1;
    int R, RP;
    const double *A1, *D1, *A2, *D2;
    dd* part;          // [block][8]
    dd* out;           // [8]
    unsigned int* counter;
};

__device__ __forceinline__ dd dd_shfl_xor(dd v, int o) {
    return dd{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
}

// the eight <T, [[X0, X1, X2]]> (index 4 b0 + 2 b1 + b2, b_n = 1 selects D_n): fp64 sums over
// the R ranks of one fibre (FMA), folded into double-double accumulators per fibre — a fibre's
// sum carries the same ~1e-15 relative error as the DMMA-computed S it is built from

// Thread (i1, r) walks a chunk of i2 (fibre j = i1 + I1 i2): the S reads are coalesced over
// (i1, r), X1 is loaded once, and X2[i2][r] comes from a shared-memory copy of the chunk's
// rows of A2 and D2. fp64 FMA partial sums over kS8Run fibres are folded into double-double.
constexpr int kS8Run = 16;
constexpr int kS8I2 = 64;  // i2 per block chunk

__global__ void __launch_bounds__(256) s8_kernel(const S8Params p) {
    __shared__ dd red[8][8];
    __shared__ double x2s[2][kS8I2][33];
    dd acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = dd{0.0, 0.0};
    const int I1 = (int)p.I1, I2 = (int)(p.J / p.I1);
    const int npr = I1 * p.RP;                           // (i1, r) pairs
    const int ngx = (npr + blockDim.x - 1) / blockDim.x;  // blocks over pairs
    const int pr = (blockIdx.x % ngx) * blockDim.x + threadIdx.x;
    const int i2a = (blockIdx.x / ngx) * kS8I2;
    const int i2b = min(I2, i2a + kS8I2);
    for (int e = threadIdx.x; e < (i2b - i2a) * p.RP; e += blockDim.x) {
        const int ii = e / p.RP, r = e % p.RP;
        const bool ok = r < p.R;
        x2s[0][ii][r] = ok ? p.A2[(int64_t)r * I2 + i2a + ii] : 0.0;
        x2s[1][ii][r] = ok ? p.D2[(int64_t)r * I2 + i2a + ii] : 0.0;
    }
    __syncthreads();
    const int i1 = pr / p.RP, r = pr % p.RP;
    if (pr < npr && r < p.R) {
        const double x1a = p.A1[(int64_t)r * I1 + i1], x1d = p.D1[(int64_t)r * I1 + i1];
        for (int i0 = i2a; i0 < i2b; i0 += kS8Run) {
            double part[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) part[k] = 0.0;
            const int iend = min(i2b, i0 + kS8Run);
            for (int i2 = i0; i2 < iend; ++i2) {
                const int64_t e = ((int64_t)i2 * I1 + i1) * p.RP + r;
                const double sa = p.S[e], sd = p.Sd[e];
                const double x2a = x2s[0][i2 - i2a][r], x2d = x2s[1][i2 - i2a][r];
                const double aa = x1a * x2a, ad = x1a * x2d, da = x1d * x2a, dd2 = x1d * x2d;
                part[0] = fma(sa, aa, part[0]);
                part[1] = fma(sa, ad, part[1]);
                part[2] = fma(sa, da, part[2]);
                part[3] = fma(sa, dd2, part[3]);
                part[4] = fma(sd, aa, part[4]);
                part[5] = fma(sd, ad, part[5]);
                part[6] = fma(sd, da, part[6]);
                part[7] = fma(sd, dd2, part[7]);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] = dd_add(acc[k], dd{part[k], 0.0});
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[k] = dd_add(acc[k], dd_shfl_xor(acc[k], o));
        if (lane == 0) red[warp][k] = acc[k];
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        dd s{0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = dd_add(s, red[w][threadIdx.x]);
        p.part[(size_t)blockIdx.x * 8 + threadIdx.x] = s;
    }
    if (!last_block_arrives(p.counter)) return;
    // blocks' partials: thread t folds blocks t, t + 256, ... (fixed order), then a shared tree
    __shared__ dd tr[256];
    for (int k = 0; k < 8; ++k) {
        dd s{0.0, 0.0};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s = dd_add(s, p.part[(size_t)b * 8 + k]);
        tr[threadIdx.x] = s;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) tr[threadIdx.x] = dd_add(tr[threadIdx.x], tr[threadIdx.x + w]);
            __syncthreads();
        }
        if (threadIdx.x == 0) p.out[k] = tr[0];
        __syncthreads();
    }
}

struct CoefParams {
    int R, RP;
    const dd* grams;  // [mode][kind][RP*RP]
    const dd* s8;
    dd half_norm_sq;
    dd* coef;         // [kPolyDeg + 1]
};

// phi coefficients: 1/2 ||T||^2 - sum_S a^|S| s8[S] + 1/2 sum_qr prod_n G_n(a)_qr
__global__ void __launch_bounds__(256) coef_kernel(const CoefParams p) {
    __shared__ dd red[256][kPolyDeg + 1];
    dd c[kPolyDeg + 1];
#pragma unroll
    for (int k = 0; k <= kPolyDeg; ++k) c[k] = dd{0.0, 0.0};
    const int RR = p.RP * p.RP;
    for (int e = threadIdx.x; e < p.R * p.R; e += blockDim.x) {
        const int q = e / p.R, r = e % p.R;
        dd prod[kPolyDeg + 1];
#pragma unroll
        for (int k = 0; k <= kPolyDeg; ++k) prod[k] = dd{k == 0 ? 1.0 : 0.0, 0.0};
        int deg = 0;
        for (int n = 0; n < 3; ++n) {
            const dd* g = p.grams + (size_t)n * kKinds * RR;
            const dd q0 = g[q * p.RP + r];
            const dd q1 = dd_add(g[RR + q * p.RP + r], g[RR + r * p.RP + q]);
            const dd q2 = g[2 * RR + q * p.RP + r];
            dd nx[kPolyDeg + 1];
#pragma unroll
            for (int k = 0; k <= kPolyDeg; ++k) nx[k] = dd{0.0, 0.0};
            for (int k = 0; k <= deg; ++k) {
                nx[k] = dd_add(nx[k], dd_mul(prod[k], q0));
                nx[k + 1] = dd_add(nx[k + 1], dd_mul(prod[k], q1));
                nx[k + 2] = dd_add(nx[k + 2], dd_mul(prod[k], q2));
            }
            deg += 2;
#pragma unroll
            for (int k = 0; k <= kPolyDeg; ++k) prod[k] = nx[k];
        }
#pragma unroll
        for (int k = 0; k <= kPolyDeg; ++k) c[k] = dd_add(c[k], prod[k]);
    }
#pragma unroll
    for (int k = 0; k <= kPolyDeg; ++k) red[threadIdx.x][k] = c[k];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {  // fixed-order tree
        if ((int)threadIdx.x < w)
#pragma unroll
            for (int k = 0; k <= kPolyDeg; ++k) red[threadIdx.x][k] = dd_add(red[threadIdx.x][k], red[threadIdx.x + w][k]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        // <T, model(a)>: a^|S| s8[S]
        dd a[4] = {p.s8[0], dd_add(dd_add(p.s8[4], p.s8[2]), p.s8[1]), dd_add(dd_add(p.s8[6], p.s8[5]), p.s8[3]),
                   p.s8[7]};
        for (int k = 0; k <= kPolyDeg; ++k) {
            dd v = dd_mul(dd{0.5, 0.0}, red[0][k]);
            if (k <= 3) v = dd_sub(v, a[k]);
            if (k == 0) v = dd_add(v, p.half_norm_sq);
            p.coef[k] = v;
        }
    }
}

}  // namespace

namespace {
__global__ void poly_eval_many_kernel(const dd* coef, const double* alphas, int n, double* phi, double* dphi) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double f, g;
        poly_eval(coef, alphas[i], f, g);
        phi[i] = f;
        dphi[i] = g;
    }
}
}  // namespace

void poly_eval_device(const PolyWork& pw, const double* alphas, int n, double* phi, double* dphi, cudaStream_t st) {
    poly_eval_many_kernel<<<(n + 127) / 128, 128, 0, st>>>(pw.coef, alphas, n, phi, dphi);
    CPFIT_CUDA(cudaGetLastError());
}

bool poly_supported(const DevTensor& t) { return !t.sparse && t.order == 3; }

PolyWork* poly_create(const DevTensor& t, const EvalWork& w) {
    auto* p = new PolyWork();
    int64_t tasks = 0;
    for (int n = 0; n < 3; ++n) tasks += (int64_t)gram_chunks(t.dims[n]) * kKinds * w.R * w.R;
    p->nchunk_total = tasks;
    p->s8_grid = (int)(((t.dims[1] * w.RP + 255) / 256) * ((t.dims[2] + kS8I2 - 1) / kS8I2));
    CPFIT_CUDA(cudaMalloc(&p->S_d, sizeof(double) * (size_t)t.J * w.RP));
    CPFIT_CUDA(cudaMalloc(&p->gpart, sizeof(dd) * (size_t)std::max<int64_t>(tasks, 1)));
    CPFIT_CUDA(cudaMalloc(&p->grams, sizeof(dd) * 3 * kKinds * (size_t)w.RP * w.RP));
    CPFIT_CUDA(cudaMalloc(&p->s8part, sizeof(dd) * 8 * (size_t)p->s8_grid));
    CPFIT_CUDA(cudaMalloc(&p->coef, sizeof(dd) * (kPolyDeg + 1)));
    CPFIT_CUDA(cudaMalloc(&p->s8, sizeof(dd) * 8));
    CPFIT_CUDA(cudaMalloc(&p->counter, sizeof(unsigned int) * 2));
    CPFIT_CUDA(cudaMemset(p->counter, 0, sizeof(unsigned int) * 2));
    return p;
}

void poly_destroy(PolyWork* p) {
    if (!p) return;
    cudaFree(p->S_d);
    cudaFree(p->gpart);
    cudaFree(p->grams);
    cudaFree(p->s8part);
    cudaFree(p->coef);
    cudaFree(p->s8);
    cudaFree(p->counter);
    delete p;
}

void poly_build_device(const DevTensor& t, EvalWork& w, PolyWork& pw, const double* ub, const double* d,
                       cudaStream_t st) {
    // S_d = T x_1 D_0 (the direction's first block)
    dense_s_pass(t, w, d, pw.S_d, st);
    CrossParams c{};
    c.R = w.R;
    c.RP = w.RP;
    int64_t base = 0;
    for (int n = 0; n < 3; ++n) {
        c.dims[n] = t.dims[n];
        c.a[n] = ub + w.off[n];
        c.d[n] = d + w.off[n];
        c.nchunk[n] = gram_chunks(t.dims[n]);
        c.rows[n] = gram_chunk_rows(t.dims[n]);
        c.base[n] = base;
        base += (int64_t)c.nchunk[n] * kKinds * w.R * w.R;
    }
    c.part = pw.gpart;
    c.out = pw.grams;
    c.counter = pw.counter;
    const int cgrid = (int)std::max<int64_t>(1, std::min<int64_t>((base + 7) / 8, 4 * sm_count()));
    cross_gram_kernel<<<cgrid, 256, 0, st>>>(c);
    CPFIT_CUDA(cudaGetLastError());
    S8Params s{};
    s.S = w.S;
    s.Sd = pw.S_d;
    s.J = t.J;
    s.I1 = t.dims[1];
    s.R = w.R;
    s.RP = w.RP;
    s.A1 = ub + w.off[1];
    s.D1 = d + w.off[1];
    s.A2 = ub + w.off[2];
    s.D2 = d + w.off[2];
    s.part = pw.s8part;
    s.out = pw.s8;
    s.counter = pw.counter + 1;
    const int ngx = (int)((t.dims[0 + 1] * w.RP + 255) / 256);
    const int ngy = (int)((t.dims[2] + kS8I2 - 1) / kS8I2);
    s8_kernel<<<ngx * ngy, 256, 0, st>>>(s);
    CPFIT_CUDA(cudaGetLastError());
    CoefParams q{};
    q.R = w.R;
    q.RP = w.RP;
    q.grams = pw.grams;
    q.s8 = pw.s8;
    q.half_norm_sq = dd{0.5 * t.norm_sq, 0.5 * t.norm_sq_lo};
    q.coef = pw.coef;
    coef_kernel<<<1, 256, 0, st>>>(q);
    CPFIT_CUDA(cudaGetLastError());
}

}  // namespace cpfit_gpu
