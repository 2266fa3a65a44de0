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
    int R, RP, nmodes;
    int64_t dims[4];
    const double* a[4];
    const double* d[4];
    dd* out;          // [mode][kind][RP*RP]
};

// one warp per (mode n, kind k, q, r) over all rows of the mode (lane-strided dd accumulation,
// fixed xor tree); padded entries are written as zero by warps with q or r >= R
__global__ void __launch_bounds__(256) cross_gram_kernel(const CrossParams p) {
    const int RR = p.RP * p.RP;
    const int total = p.nmodes * kKinds * RR;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    for (int t = warp; t < total; t += nwarps) {
        const int n = t / (kKinds * RR), k = (t / RR) % kKinds, e = t % RR;
        const int q = e / p.RP, r = e % p.RP;
        dd s{0.0, 0.0};
        if (q < p.R && r < p.R) {
            const int64_t In = p.dims[n];
            const double* x = (k == 2 ? p.d[n] : p.a[n]) + (int64_t)q * In;
            const double* y = (k == 0 ? p.a[n] : p.d[n]) + (int64_t)r * In;
            s = warp_dot_dd(x, y, 0, In);
        }
        if ((threadIdx.x & 31) == 0) p.out[t] = s;
    }
}

struct S8Params {
    int i2c;           // i2 per block (<= kS8I2)
    const double* S;   // S(u_bar), J x RP
    const double* Sd;  // S_d
    int64_t J, I1;
    int R, RP;
    const double *A1, *D1, *A2, *D2;
    dd* part;          // [block][8]
    dd* out;           // [8]
    unsigned int* counter;
    const int* perm;   // S(u_bar)[j][r] = S[j][perm r] sc0[r] when set
    const double* sc0;
};

__device__ __forceinline__ dd dd_shfl_xor(dd v, int o) {
    return dd{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
}

// the eight <T, [[X0, X1, X2]]> (index 4 b0 + 2 b1 + b2, b_n = 1 selects D_n) as
//   sum_{i1, r} X1[i1][r] sum_{i2} S_{b0}[i1 + I1 i2][r] X2[i2][r]:
// thread (i1, r) walks a chunk of i2 (fibre j = i1 + I1 i2) accumulating the four inner sums
// (S or S_d against A2 or D2); the X1 factors multiply in once per chunk, in double-double. The
// S reads are coalesced over (i1, r) and X2[i2][r] comes from a shared-memory copy of the chunk's
// rows of A2 and D2. fp64 FMA partial sums over kS8Run fibres are folded into double-double —
// a run's sum carries the same ~1e-15 relative error as the DMMA-computed S it is built from.
constexpr int kS8Run = 8;
constexpr int kS8I2 = 48;  // max i2 per block chunk (the chunk is sized so the grid is one wave)

// a += b for a double-double accumulator without renormalising (lo collects the rounding errors
// of hi; dd_norm once at the end)
__device__ __forceinline__ void dd_acc(dd& a, double b) {
    const double s = a.hi + b;
    const double bb = s - a.hi;
    a.lo += (a.hi - (s - bb)) + (b - bb);
    a.hi = s;
}

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
    const int i2a = (blockIdx.x / ngx) * p.i2c;
    const int i2b = min(I2, i2a + p.i2c);
    const int i1 = pr / p.RP, r = pr % p.RP;
    const bool active = pr < npr && r < p.R;
    // S(u_bar) column r = sc0[r] x S column perm[r]: coalesced loads, then a shuffle from the
    // lane holding column perm[r] of the same row (a row of RP pairs lies in one warp)
    const int lane0 = threadIdx.x & 31;
    const int src = (lane0 & ~(p.RP - 1)) + ((p.perm && r < p.R) ? p.perm[r] : r);
    const double scl = (active && p.perm) ? p.sc0[r] : 1.0;
    // the first run's S loads and the X1 factors go out before the X2 staging barrier
    double sav[kS8Run], sdv[kS8Run];
    auto load_run = [&](int i0) {
#pragma unroll
        for (int u = 0; u < kS8Run; ++u) {
            const int i2 = i0 + u;
            const int64_t e = ((int64_t)i2 * I1 + i1) * p.RP;
            sav[u] = active && i2 < i2b ? p.S[e + r] : 0.0;
            sdv[u] = active && i2 < i2b ? p.Sd[e + r] : 0.0;
        }
    };
    load_run(i2a);
    const dd x1a{active ? p.A1[(int64_t)r * I1 + i1] : 0.0, 0.0};
    const dd x1d{active ? p.D1[(int64_t)r * I1 + i1] : 0.0, 0.0};
    for (int e = threadIdx.x; e < (i2b - i2a) * p.RP; e += blockDim.x) {
        const int n = i2b - i2a, ii = e % n, rr = e / n;  // coalesced over i2
        const bool ok = rr < p.R;
        x2s[0][ii][rr] = ok ? p.A2[(int64_t)rr * I2 + i2a + ii] : 0.0;
        x2s[1][ii][rr] = ok ? p.D2[(int64_t)rr * I2 + i2a + ii] : 0.0;
    }
    __syncthreads();
    {  // every lane (the shuffles); inactive lanes hold zeros
        dd q[4];  // S.A2, S.D2, S_d.A2, S_d.D2 over the chunk
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = dd{0.0, 0.0};
        for (int i0 = i2a; i0 < i2b; i0 += kS8Run) {
            if (i0 > i2a) load_run(i0);  // the run's loads issue together
            double part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int u = 0; u < kS8Run; ++u) {
                const int i2 = i0 + u;
                if (i2 >= i2b) break;
                const double x2a = x2s[0][i2 - i2a][r], x2d = x2s[1][i2 - i2a][r];
                const double sa = p.perm ? __shfl_sync(0xffffffffu, sav[u], src) : sav[u];
                part[0] = fma(sa, x2a, part[0]);
                part[1] = fma(sa, x2d, part[1]);
                part[2] = fma(sdv[u], x2a, part[2]);
                part[3] = fma(sdv[u], x2d, part[3]);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) dd_acc(q[k], part[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = dd_two_sum(q[k].hi, q[k].lo);
        // S(u_bar) column r = sc0[r] x S column perm[r]: the scale applies to the S sums
        if (p.perm) {
            q[0] = dd_mul(q[0], dd{scl, 0.0});
            q[1] = dd_mul(q[1], dd{scl, 0.0});
        }
        // k = 4 b0 + 2 b1 + b2: q index 2 b0 + b2, X1 by b1
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = dd_mul(q[2 * (k >> 2) + (k & 1)], (k & 2) ? x1d : x1a);
    }
    // transposing warp reduction: each xor step halves the values a lane holds (4 + 2 + 1 + 1 + 1
    // double-double adds per lane); contraction k ends in lane 4 k
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        const bool b = lane & 16;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const dd mine = b ? acc[j + 4] : acc[j], other = b ? acc[j] : acc[j + 4];
            acc[j] = dd_add(mine, dd_shfl_xor(other, 16));
        }
    }
    {
        const bool c = lane & 8;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const dd mine = c ? acc[j + 2] : acc[j], other = c ? acc[j] : acc[j + 2];
            acc[j] = dd_add(mine, dd_shfl_xor(other, 8));
        }
    }
    {
        const bool d = lane & 4;
        const dd mine = d ? acc[1] : acc[0], other = d ? acc[0] : acc[1];
        acc[0] = dd_add(mine, dd_shfl_xor(other, 4));
    }
    acc[0] = dd_add(acc[0], dd_shfl_xor(acc[0], 2));
    acc[0] = dd_add(acc[0], dd_shfl_xor(acc[0], 1));
    if ((lane & 3) == 0) red[warp][lane >> 2] = acc[0];
    __syncthreads();
    if (threadIdx.x < 8) {
        dd s{0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = dd_add(s, red[w][threadIdx.x]);
        p.part[(size_t)blockIdx.x * 8 + threadIdx.x] = s;
    }
}

// s8 grid: (i1, r) pair blocks x i2 chunks, the chunk sized so all blocks are resident at once
// (a second, mostly empty wave doubled the kernel time); returns (blocks, pair blocks, chunk)
int3 s8_grid_dims(const DevTensor& t, const EvalWork& w) {
    static int per_sm = [] {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, s8_kernel, 256, 0) != cudaSuccess || b < 1) {
            (void)cudaGetLastError();
            b = 1;
        }
        return b;
    }();
    int sms = 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        sms = 148;
    }
    const int64_t I2 = t.dims[2];
    const int ngx = (int)((t.dims[1] * w.RP + 255) / 256);
    int64_t ngy = std::max<int64_t>(1, (int64_t)sms * per_sm / ngx);
    int64_t i2c = std::min<int64_t>(kS8I2, (I2 + ngy - 1) / ngy);
    ngy = (I2 + i2c - 1) / i2c;
    return make_int3((int)(ngx * ngy), ngx, (int)i2c);
}

struct CoefParams {
    int R, RP;
    const dd* grams;   // [mode][kind][RP*RP]
    const dd* s8part;  // [block][8] partials of the eight contractions
    int s8_blocks;
    const double* tn;  // device [||T||, ||T||^2 hi, lo] (DevTensor::dscal)
    dd* coef;          // [kPolyDeg + 1]
};

// phi coefficients: 1/2 ||T||^2 - sum_S a^|S| s8[S] + 1/2 sum_qr prod_n G_n(a)_qr
__global__ void __launch_bounds__(256) coef_kernel(const CoefParams p) {
    dd c8[8];
#pragma unroll
    for (int k = 0; k <= kPolyDeg3; ++k) c8[k] = dd{0.0, 0.0};
    const int RR = p.RP * p.RP;
    for (int e = threadIdx.x; e < p.R * p.R; e += blockDim.x) {
        const int q = e / p.R, r = e % p.R;
        dd qc[3][3];
#pragma unroll
        for (int n = 0; n < 3; ++n) {
            const dd* g = p.grams + (size_t)n * kKinds * RR;
            qc[n][0] = g[q * p.RP + r];
            qc[n][1] = dd_add(g[RR + q * p.RP + r], g[RR + r * p.RP + q]);
            qc[n][2] = g[2 * RR + q * p.RP + r];
        }
        // (q0 + q1 a + q2 a^2) for modes 0, 1, 2 multiplied out (degrees 4 then 6), unrolled
        dd p4[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) p4[k] = dd{0.0, 0.0};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) p4[i + j] = dd_add(p4[i + j], dd_mul(qc[0][i], qc[1][j]));
#pragma unroll
        for (int i = 0; i < 5; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) c8[i + j] = dd_add(c8[i + j], dd_mul(p4[i], qc[2][j]));
    }
    // the eight contractions: s8_kernel's block partials, thread t folding blocks b = t / 8 mod 32
    // of contraction t % 8 (loads issued together)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    dd v8{0.0, 0.0};
    {
        const int k = threadIdx.x & 7, g = threadIdx.x >> 3;
        for (int b0 = g; b0 < p.s8_blocks; b0 += 32 * 16) {
            dd x[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int b = b0 + 32 * u;
                x[u] = b < p.s8_blocks ? p.s8part[(size_t)b * 8 + k] : dd{0.0, 0.0};
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) v8 = dd_add(v8, x[u]);
        }
    }
    // fixed-order trees: a transposing shuffle reduction of the seven coefficients (plus a zero)
    // that ends with coefficient k in lane 4 k, the s8 sums over the warp's four groups, then the
    // warps in order
    c8[kPolyDeg3 + 1] = dd{0.0, 0.0};
    {
        const bool b = lane & 16;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const dd mine = b ? c8[j + 4] : c8[j], other = b ? c8[j] : c8[j + 4];
            c8[j] = dd_add(mine, dd_shfl_xor(other, 16));
        }
    }
    {
        const bool cc = lane & 8;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const dd mine = cc ? c8[j + 2] : c8[j], other = cc ? c8[j] : c8[j + 2];
            c8[j] = dd_add(mine, dd_shfl_xor(other, 8));
        }
    }
    {
        const bool d = lane & 4;
        const dd mine = d ? c8[1] : c8[0], other = d ? c8[0] : c8[1];
        c8[0] = dd_add(mine, dd_shfl_xor(other, 4));
    }
    c8[0] = dd_add(c8[0], dd_shfl_xor(c8[0], 2));
    c8[0] = dd_add(c8[0], dd_shfl_xor(c8[0], 1));
#pragma unroll
    for (int o = 16; o >= 8; o >>= 1) v8 = dd_add(v8, dd_shfl_xor(v8, o));
    __shared__ dd red[8][kPolyDeg3 + 1 + 8];
    if ((lane & 3) == 0 && (lane >> 2) <= kPolyDeg3) red[warp][lane >> 2] = c8[0];
    if (lane < 8) red[warp][kPolyDeg3 + 1 + lane] = v8;
    __syncthreads();
    __shared__ dd tot[kPolyDeg3 + 1 + 8];
    if (threadIdx.x < kPolyDeg3 + 1 + 8) {
        dd v{0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = dd_add(v, red[w][threadIdx.x]);
        tot[threadIdx.x] = v;
    }
    __syncthreads();
    const dd* s8v = tot + kPolyDeg3 + 1;
    if (threadIdx.x == 0) {
        // <T, model(a)>: a^|S| s8[S]
        dd a[4] = {s8v[0], dd_add(dd_add(s8v[4], s8v[2]), s8v[1]), dd_add(dd_add(s8v[6], s8v[5]), s8v[3]), s8v[7]};
        for (int k = 0; k <= kPolyDeg3; ++k) {
            dd v = dd_mul(dd{0.5, 0.0}, tot[k]);
            if (k <= 3) v = dd_sub(v, a[k]);
            if (k == 0) v = dd_add(v, dd{0.5 * p.tn[1], 0.5 * p.tn[2]});
            p.coef[k] = v;
        }
        for (int k = kPolyDeg3 + 1; k <= kPolyDeg; ++k) p.coef[k] = dd{0.0, 0.0};
    }
}


// ---- order 4 (degree 8) ---------------------------------------------------------------------
// the sixteen <T, [[X0, X1, X2, X3]]> (index 8 b0 + 4 b1 + 2 b2 + b3, b_n = 1 selects D_n) as
//   sum_{i1, r} X1[i1][r] sum_{o} S_{b0}[i1 + I1 o][r] (X2 X3)[o][r],  o = i2 + I2 i3:
// thread (i1, r) walks a chunk of o with the chunk's four X2[i2] X3[i3] row products (AA, AD, DA,
// DD) staged in shared memory; fp64 runs folded into double-double as in s8_kernel.
constexpr int kS16O = 40;  // max outer indices per block chunk (static shared memory)
struct S16Params {
    int oc;            // outer indices per block
    const double* S;
    const double* Sd;
    int64_t I1, I2, I3;
    int R, RP;
    const double *A1, *D1, *A2, *D2, *A3, *D3;
    dd* part;          // [block][16]
    const int* perm;
    const double* sc0;
};

__global__ void __launch_bounds__(256) s16_kernel(const S16Params p) {
    __shared__ double x23[4][kS16O][33];
    __shared__ dd red[8][16];
    const int I1 = (int)p.I1, I2 = (int)p.I2;
    const int NO = (int)(p.I2 * p.I3);
    const int npr = I1 * p.RP;
    const int ngx = (npr + blockDim.x - 1) / blockDim.x;
    const int pr = (blockIdx.x % ngx) * blockDim.x + threadIdx.x;
    const int oa = (blockIdx.x / ngx) * p.oc;
    const int ob = min(NO, oa + p.oc);
    const int i1 = pr / p.RP, r = pr % p.RP;
    const bool active = pr < npr && r < p.R;
    const int lane0 = threadIdx.x & 31;
    const int src = (lane0 & ~(p.RP - 1)) + ((p.perm && r < p.R) ? p.perm[r] : r);
    const double scl = (active && p.perm) ? p.sc0[r] : 1.0;
    for (int e = threadIdx.x; e < (ob - oa) * p.RP; e += blockDim.x) {
        const int n = ob - oa, ii = e % n, rr = e / n;
        const int o = oa + ii, i2 = o % I2, i3 = o / I2;
        const bool ok = rr < p.R;
        const double a2 = ok ? p.A2[(int64_t)rr * p.I2 + i2] : 0.0, d2 = ok ? p.D2[(int64_t)rr * p.I2 + i2] : 0.0;
        const double a3 = ok ? p.A3[(int64_t)rr * p.I3 + i3] : 0.0, d3 = ok ? p.D3[(int64_t)rr * p.I3 + i3] : 0.0;
        x23[0][ii][rr] = a2 * a3;
        x23[1][ii][rr] = a2 * d3;
        x23[2][ii][rr] = d2 * a3;
        x23[3][ii][rr] = d2 * d3;
    }
    const double x1a = active ? p.A1[(int64_t)r * p.I1 + i1] : 0.0;
    const double x1d = active ? p.D1[(int64_t)r * p.I1 + i1] : 0.0;
    __syncthreads();
    dd q[2][4];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[b][c] = dd{0.0, 0.0};
    for (int o0 = oa; o0 < ob; o0 += 8) {
        double run[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
        double sv[8], dv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t f = (int64_t)i1 + (int64_t)I1 * (o0 + u);
            const bool ok = pr < npr && o0 + u < ob;
            sv[u] = ok ? p.S[f * p.RP + r] : 0.0;
            dv[u] = ok ? p.Sd[f * p.RP + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (o0 + u >= ob) break;
            const double sa = p.perm ? __shfl_sync(0xffffffffu, sv[u], src) : sv[u];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const double x = x23[c][o0 + u - oa][r];
                run[0][c] = fma(sa, x, run[0][c]);
                run[1][c] = fma(dv[u], x, run[1][c]);
            }
        }
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < 4; ++c) dd_acc(q[b][c], run[b][c]);
    }
    dd acc[16];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            dd v = dd_two_sum(q[b][c].hi, q[b][c].lo);
            if (b == 0 && p.perm) v = dd_mul(v, dd{scl, 0.0});
            if (!active) v = dd{0.0, 0.0};
            acc[8 * b + c] = dd_mul(v, dd{x1a, 0.0});
            acc[8 * b + 4 + c] = dd_mul(v, dd{x1d, 0.0});
        }
    // transposing warp reduction (as in s8_kernel): each xor step halves the values a lane holds
    // (8 + 4 + 2 + 1 + 1 double-double adds per lane instead of 16 x 5); contraction k ends in
    // lanes 2k, 2k + 1
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const dd mine = up ? acc[j + h] : acc[j], other = up ? acc[j] : acc[j + h];
            acc[j] = dd_add(mine, dd_shfl_xor(other, o));
        }
    }
    acc[0] = dd_add(acc[0], dd_shfl_xor(acc[0], 1));
    if ((lane & 1) == 0) red[warp][lane >> 1] = acc[0];
    __syncthreads();
    if (threadIdx.x < 16) {
        dd v{0.0, 0.0};
        for (int w8 = 0; w8 < (int)(blockDim.x >> 5); ++w8) v = dd_add(v, red[w8][threadIdx.x]);
        p.part[(size_t)blockIdx.x * 16 + threadIdx.x] = v;
    }
}

// order-4 phi coefficients: 1/2 ||T||^2 - sum_S a^|S| s16[S] + 1/2 sum_qr prod_n G_n(a)_qr
__global__ void __launch_bounds__(256) coef4_kernel(const CoefParams p) {
    dd c[kPolyDeg + 1];
#pragma unroll
    for (int k = 0; k <= kPolyDeg; ++k) c[k] = dd{0.0, 0.0};
    const int RR = p.RP * p.RP;
    for (int e = threadIdx.x; e < p.R * p.R; e += blockDim.x) {
        const int q = e / p.R, r = e % p.R;
        dd qc[4][3];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            const dd* g = p.grams + (size_t)n * kKinds * RR;
            qc[n][0] = g[q * p.RP + r];
            qc[n][1] = dd_add(g[RR + q * p.RP + r], g[RR + r * p.RP + q]);
            qc[n][2] = g[2 * RR + q * p.RP + r];
        }
        dd pa[5], pb[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) pa[k] = pb[k] = dd{0.0, 0.0};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                pa[i + j] = dd_add(pa[i + j], dd_mul(qc[0][i], qc[1][j]));
                pb[i + j] = dd_add(pb[i + j], dd_mul(qc[2][i], qc[3][j]));
            }
#pragma unroll
        for (int i = 0; i < 5; ++i)
#pragma unroll
            for (int j = 0; j < 5; ++j) c[i + j] = dd_add(c[i + j], dd_mul(pa[i], pb[j]));
    }
    // the sixteen contractions: thread t folds blocks b = t / 16 mod 16 of contraction t % 16
    dd v{0.0, 0.0};
    {
        const int k = threadIdx.x & 15, g = threadIdx.x >> 4;
        for (int b = g; b < p.s8_blocks; b += 16) v = dd_add(v, p.s8part[(size_t)b * 16 + k]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k <= kPolyDeg; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c[k] = dd_add(c[k], dd_shfl_xor(c[k], o));
    v = dd_add(v, dd_shfl_xor(v, 16));
    __shared__ dd red[8][kPolyDeg + 1 + 16];
    if (lane == 0)
#pragma unroll
        for (int k = 0; k <= kPolyDeg; ++k) red[warp][k] = c[k];
    if (lane < 16) red[warp][kPolyDeg + 1 + lane] = v;
    __syncthreads();
    __shared__ dd tot[kPolyDeg + 1 + 16];
    if (threadIdx.x < kPolyDeg + 1 + 16) {
        dd t{0.0, 0.0};
        for (int w8 = 0; w8 < (int)(blockDim.x >> 5); ++w8) t = dd_add(t, red[w8][threadIdx.x]);
        tot[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const dd* s16 = tot + kPolyDeg + 1;
        dd a[5];
        for (int j = 0; j < 5; ++j) a[j] = dd{0.0, 0.0};
        for (int k = 0; k < 16; ++k) a[__popc(k)] = dd_add(a[__popc(k)], s16[k]);
        for (int k = 0; k <= kPolyDeg; ++k) {
            dd x = dd_mul(dd{0.5, 0.0}, tot[k]);
            if (k <= 4) x = dd_sub(x, a[k]);
            if (k == 0) x = dd_add(x, dd{0.5 * p.tn[1], 0.5 * p.tn[2]});
            p.coef[k] = x;
        }
    }
}

// s16 grid: (i1, r) pair blocks x outer chunks sized for one wave; returns (blocks, pair blocks, chunk)
int3 s16_grid_dims(const DevTensor& t, const EvalWork& w) {
    int sms = 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        sms = 148;
    }
    const int64_t NO = t.dims[2] * t.dims[3];
    const int ngx = (int)((t.dims[1] * w.RP + 255) / 256);
    int64_t ngy = std::max<int64_t>(1, (int64_t)2 * sms / ngx);
    const int64_t oc = std::min<int64_t>(kS16O, (NO + ngy - 1) / ngy);
    ngy = (NO + oc - 1) / oc;
    return make_int3((int)(ngx * ngy), ngx, (int)oc);
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

namespace {
// u* = u_bar + beta d (grid-stride) and, in the first block, G_n(u*) from the cross Grams
__global__ void __launch_bounds__(256) poly_point_kernel(const double* ub, const double* d, const double* beta_p,
                                                         double* ut, int64_t n, const dd* cg, double* gram, int RP,
                                                         int nmodes) {
    const double beta = *beta_p;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ut[i] = ub[i] + beta * d[i];
    if (blockIdx.x != 0) return;
    const int RR = RP * RP;
    const dd b{beta, 0.0}, b2 = dd_mul(b, b);
    for (int e = threadIdx.x; e < nmodes * RR; e += blockDim.x) {
        const int m = e / RR, q = (e % RR) / RP, r = e % RP;
        const dd* g = cg + (size_t)m * kKinds * RR;
        const dd ad = dd_add(g[RR + q * RP + r], g[RR + r * RP + q]);
        const dd v = dd_add(dd_add(g[q * RP + r], dd_mul(b, ad)), dd_mul(b2, g[2 * RR + q * RP + r]));
        gram[e] = v.hi + v.lo;
    }
}
}  // namespace

void poly_point_device(EvalWork& w, const PolyWork& pw, const double* ub, const double* d, const double* beta,
                       double* ut, cudaStream_t st) {
    poly_point_kernel<<<(int)std::min<int64_t>(148, (w.nu + 255) / 256), 256, 0, st>>>(ub, d, beta, ut, w.nu,
                                                                                        pw.grams, w.gram, w.RP,
                                                                                        w.order);
    CPFIT_CUDA(cudaGetLastError());
}

bool poly_supported(const DevTensor& t) {
    return !t.generic && (t.order == 3 || (t.order == 4 && !t.sparse));
}

PolyWork* poly_create(const DevTensor& t, const EvalWork& w) {
    auto* p = new PolyWork();
    int64_t tasks = 0;
    for (int n = 0; n < t.order; ++n) tasks += (int64_t)gram_chunks(t.dims[n]) * kKinds * w.R * w.R;
    p->nchunk_total = tasks;
    if (t.sparse) {
        // sparse: the eight contractions in one pass over the mode-0 sorted nonzeros, reading
        // row-major copies of u_bar's and d's factors (drows holds d's)
        p->s8_grid = kSparseLineBlocks;
        int64_t rows = 0;
        for (int n = 0; n < 3; ++n) rows += t.dims[n];
        CPFIT_CUDA(cudaMalloc(&p->drows, sizeof(double) * (size_t)rows * w.RP));
        CPFIT_CUDA(cudaMalloc(&p->m0xy, sizeof(double) * 4 * (size_t)t.dims[0] * w.RP));
    } else {
        p->s8_grid = t.order == 4 ? s16_grid_dims(t, w).x : s8_grid_dims(t, w).x;
        p->S_d = w.S2;  // owned by the evaluation workspace (next to S)
    }
    CPFIT_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    CPFIT_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
    CPFIT_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
    CPFIT_CUDA(cudaMalloc(&p->gpart, sizeof(dd) * (size_t)std::max<int64_t>(tasks, 1)));
    CPFIT_CUDA(cudaMalloc(&p->grams, sizeof(dd) * 4 * kKinds * (size_t)w.RP * w.RP));
    CPFIT_CUDA(cudaMalloc(&p->s8part, sizeof(dd) * 16 * (size_t)p->s8_grid));
    CPFIT_CUDA(cudaMalloc(&p->coef, sizeof(dd) * (kPolyDeg + 1)));
    CPFIT_CUDA(cudaMalloc(&p->s8, sizeof(dd) * 8));
    CPFIT_CUDA(cudaMalloc(&p->counter, sizeof(unsigned int) * 2));
    CPFIT_CUDA(cudaMemset(p->counter, 0, sizeof(unsigned int) * 2));
    return p;
}

void poly_destroy(PolyWork* p) {
    if (!p) return;
    cudaFree(p->gpart);
    cudaFree(p->grams);
    cudaFree(p->s8part);
    cudaFree(p->coef);
    cudaFree(p->s8);
    cudaFree(p->counter);
    cudaFree(p->drows);
    cudaFree(p->m0xy);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    if (p->side) cudaStreamDestroy(p->side);
    delete p;
}

void launch_coef(const DevTensor& t, const EvalWork& w, const PolyWork& pw, int s8_blocks, cudaStream_t st) {
    CoefParams q{};
    q.R = w.R;
    q.RP = w.RP;
    q.grams = pw.grams;
    q.s8part = pw.s8part;
    q.s8_blocks = s8_blocks;
    q.tn = t.dscal;
    q.coef = pw.coef;
    coef_kernel<<<1, 256, 0, st>>>(q);
    CPFIT_CUDA(cudaGetLastError());
}

void poly_build_device(const DevTensor& t, EvalWork& w, PolyWork& pw, const double* ub, const double* d,
                       cudaStream_t st, const int* perm, const double* sc0) {
    // the cross Grams need only u_bar and d: on the side stream, beside the S_d pass (38
    // registers per thread: they fit next to the pass's one CTA per SM)
    CPFIT_CUDA(cudaEventRecord(pw.ev_fork, st));
    CPFIT_CUDA(cudaStreamWaitEvent(pw.side, pw.ev_fork, 0));
    CrossParams c{};
    c.R = w.R;
    c.RP = w.RP;
    c.nmodes = t.order;
    for (int n = 0; n < t.order; ++n) {
        c.dims[n] = t.dims[n];
        c.a[n] = ub + w.off[n];
        c.d[n] = d + w.off[n];
    }
    c.out = pw.grams;
    const int ctasks = t.order * kKinds * w.RP * w.RP;
    cross_gram_kernel<<<(ctasks + 7) / 8, 256, 0, pw.side>>>(c);
    CPFIT_CUDA(cudaGetLastError());
    CPFIT_CUDA(cudaEventRecord(pw.ev_join, pw.side));
    if (t.sparse) {
        sparse_line_contractions(t, w, ub, d, pw.drows, pw.s8part, pw.s8_grid, st, pw.m0xy);
        CPFIT_CUDA(cudaStreamWaitEvent(st, pw.ev_join, 0));  // cross Grams done
        launch_coef(t, w, pw, pw.s8_grid, st);
        return;
    }
    // S_d = T x_1 D_0 (the direction's first block)
    dense_s_pass(t, w, d, pw.S_d, st);
    if (t.order == 4) {
        S16Params s16{};
        const int3 sg = s16_grid_dims(t, w);
        s16.oc = sg.z;
        s16.S = w.S;
        s16.Sd = pw.S_d;
        s16.I1 = t.dims[1];
        s16.I2 = t.dims[2];
        s16.I3 = t.dims[3];
        s16.R = w.R;
        s16.RP = w.RP;
        s16.A1 = ub + w.off[1];
        s16.D1 = d + w.off[1];
        s16.A2 = ub + w.off[2];
        s16.D2 = d + w.off[2];
        s16.A3 = ub + w.off[3];
        s16.D3 = d + w.off[3];
        s16.part = pw.s8part;
        s16.perm = perm;
        s16.sc0 = sc0;
        s16_kernel<<<sg.x, 256, 0, st>>>(s16);
        CPFIT_CUDA(cudaGetLastError());
        CPFIT_CUDA(cudaStreamWaitEvent(st, pw.ev_join, 0));  // cross Grams done
        CoefParams q{};
        q.R = w.R;
        q.RP = w.RP;
        q.grams = pw.grams;
        q.s8part = pw.s8part;
        q.s8_blocks = sg.x;
        q.tn = t.dscal;
        q.coef = pw.coef;
        coef4_kernel<<<1, 256, 0, st>>>(q);
        CPFIT_CUDA(cudaGetLastError());
        return;
    }
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
    s.perm = perm;
    s.sc0 = sc0;

    const int3 sg = s8_grid_dims(t, w);
    s.i2c = sg.z;
    static bool carve = [] {  // several CTAs per SM need the shared-memory carveout
        cudaFuncSetAttribute(s8_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        return true;
    }();
    (void)carve;
    s8_kernel<<<sg.x, 256, 0, st>>>(s);
    CPFIT_CUDA(cudaGetLastError());
    CPFIT_CUDA(cudaStreamWaitEvent(st, pw.ev_join, 0));  // cross Grams done
    launch_coef(t, w, pw, sg.x, st);
}

}  // namespace cpfit_gpu
