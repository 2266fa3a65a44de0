// Sparse COO MTTKRP on device (tensor.cpp:242-259) for the sparse objective/gradient
// (kruskal.cpp:106-111, 127-149).
//
// Each mode n has its own mode-n-sorted copy (built at upload), so M_n(i, :) is a
// segmented sum over rows of that copy: one warp per row, lane groups over the row's
// nonzeros, product v * prod_{k != n} A_k(c_k, :), then a fixed-order combination of the
// groups. Deterministic (no atomics); the streamed bytes per nonzero are the value plus the
// other modes' indices (two 16-bit indices packed in one word for order 3 when they fit); the
// factor-row gathers hit L2 (row-major RP-padded copies of the factors, rebuilt per
// evaluation). At BASELINE config 4 the gathers are the bound: ~5.7 L2 sectors per nonzero
// at ~75 % of the L2 throughput cap (profiles/r02_summary.md, "Sparse").
#include "sparse.cuh"

#include <algorithm>
#include <thread>
#include <type_traits>

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

// Row-segment layout (the default). A factor row of RP doubles is one 128-byte line at RP = 16;
// it is gathered by L = RP/2 lanes with one 16-byte load each, so every quarter-warp phase of a
// 128-bit load touches exactly one line (one L1 wavefront per row; lanes past R are predicated off
// so only the sectors holding ranks < R move). One warp step covers G = 32 / L nonzeros (RP = 16: 4).
// Every lane of a group loads its nonzero's value and indices itself — for order 3 with both other
// mode sizes <= 65536 the two indices come packed in one 32-bit word (one wavefront per step) — so
// no shuffles sit between the index stream and the gathers. The previous layout (RP lanes with
// 8-byte loads, indices broadcast by 4 shuffles per 2 nonzeros) spent a third of the L1 data path
// on shuffles; a 5-lane layout for R = 10 straddled quarter-warp phases (1.5 wavefronts per row).
// U steps are issued before their products; each warp owns rows_per_warp consecutive rows and one
// lane prefetches the next row's index/value ranges into L2 with a bulk prefetch, so the dependent
// index loads of a row's first chunk hit L2. Groups are combined in fixed order at the end of a row
// (deterministic).
__device__ __forceinline__ void bulk_prefetch_l2(const void* base, int64_t bytes) {
    // the 16-byte-aligned interior only: a prefetch reaching past the allocation faults
    const uintptr_t a0 = (reinterpret_cast<uintptr_t>(base) + 15) & ~uintptr_t(15);
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(base) + (uintptr_t)bytes) & ~uintptr_t(15);
    if (a1 > a0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
}

// Loads through volatile asm keep their program order: the chunk's next index loads and all of
// its gathers issue before the first product (the compiler otherwise interleaves them with the
// multiplies to save registers, putting several L2 round trips in series per chunk).
__device__ __forceinline__ double2 ldg_d2(const double2* a, bool on) {
    double2 v;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n mov.f64 %0, 0d0000000000000000;\n"
        " mov.f64 %1, 0d0000000000000000;\n @p ld.global.nc.v2.f64 {%0, %1}, [%2];\n}"
        : "=d"(v.x), "=d"(v.y)
        : "l"(a), "r"((unsigned)on));
    return v;
}
__device__ __forceinline__ double ldg_d(const double* a, bool on) {  // 0.0 when !on
    double v;
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n mov.f64 %0, 0d0000000000000000;\n"
                 " @p ld.global.nc.f64 %0, [%1];\n}"
                 : "=d"(v)
                 : "l"(a), "r"((unsigned)on));
    return v;
}
__device__ __forceinline__ uint32_t ldg_u(const uint32_t* a) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(a));
    return v;
}

template <int RP, int NO, int U, bool PK>
__global__ void __launch_bounds__(256) sp_mttkrp2_kernel(const SpParams p, const uint32_t* __restrict__ pidx,
                                                         int64_t rows_per_warp) {
    constexpr int L = RP / 2, G = 32 / L;
    constexpr int NK = NO > 0 ? NO : kMaxOrder - 1;
    const int lane = threadIdx.x & 31;
    const int g = lane / L, c = lane % L;
    const bool live = 2 * c < p.R;
    const int nother = NO > 0 ? NO : p.nother;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t i0 = gw * rows_per_warp, i1 = imin64(p.In, i0 + rows_per_warp);
    const double2* fr[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) fr[k] = reinterpret_cast<const double2*>(k < nother ? p.frow[k] : p.frow[0]) + c;
    auto prefetch_row = [&](int64_t i) {
        const int64_t a = p.rowptr[i], b = p.rowptr[i + 1];
        if (b > a) {
            bulk_prefetch_l2(p.vals + a, (b - a) * 8);
            if (PK)
                bulk_prefetch_l2(pidx + a, (b - a) * 4);
            else
                for (int k = 0; k < nother; ++k) bulk_prefetch_l2(p.oidx + (int64_t)k * p.nnz + a, (b - a) * 4);
        }
    };
    if (lane == 0 && i0 < i1) prefetch_row(i0);
    for (int64_t i = i0; i < i1; ++i) {
        if (lane == 0 && i + 1 < i1) prefetch_row(i + 1);
        const int64_t j0 = p.rowptr[i], j1 = p.rowptr[i + 1];
        double ax = 0.0, ay = 0.0;
        if (j0 >= j1) {
            if (g == 0) reinterpret_cast<double2*>(p.out + i * RP)[c] = make_double2(0.0, 0.0);
            continue;
        }
        // Two-stage software pipeline over chunks of C = G*U nonzeros: in the iteration that
        // consumes chunk m, the gathers of chunk m+1 and the index loads of chunk m+2 are issued
        // first. Loop-carried registers keep them in flight across the products (the compiler
        // otherwise sinks each gather next to its multiply). Slots past the row's end load an
        // in-range address and carry v = 0.
        constexpr int C = G * U;
        const int n = (int)(j1 - j0);
        const double* vrow = p.vals + j0;
        const uint32_t* prow = PK ? pidx + j0 : nullptr;
        auto load_idx = [&](int64_t jb, double (&vv)[U], int (&cc)[U][NK]) {
#pragma unroll
            for (int t = 0; t < U; ++t) {
                const int q = (int)(jb - j0) + t * G + g;  // offset in the row (rows < 2^31 nonzeros)
                const bool ok = q < n;
                const int qc = ok ? q : 0;
                vv[t] = ldg_d(vrow + qc, ok);
                if (PK) {
                    cc[t][0] = (int)ldg_u(prow + qc);
                } else {
#pragma unroll
                    for (int k = 0; k < NK; ++k)
                        cc[t][k] = k < nother ? __ldg(p.oidx + (int64_t)k * p.nnz + j0 + qc) : 0;
                }
            }
        };
        auto gather = [&](const int (&cc)[U][NK], double2 (&xx)[U][NK]) {
#pragma unroll
            for (int t = 0; t < U; ++t) {
                int ci[NK];
                if (PK) {
                    const uint32_t w = (uint32_t)cc[t][0];
                    ci[0] = (int)(w & 0xffffu);
                    ci[1] = (int)(w >> 16);
                } else {
#pragma unroll
                    for (int k = 0; k < NK; ++k) ci[k] = cc[t][k];
                }
#pragma unroll
                for (int k = 0; k < NK; ++k)
                    if (k < nother) xx[t][k] = ldg_d2(fr[k] + (int64_t)ci[k] * L, live);
            }
        };
        double va[U], vb[U];
        int ca[U][NK], cb[U][NK];
        double2 xa[U][NK];
        load_idx(j0, va, ca);
        gather(ca, xa);
        load_idx(j0 + C, vb, cb);
        for (int64_t jb = j0; jb < j1; jb += C) {
            double2 xb[U][NK];
            gather(cb, xb);              // chunk m+1
            double vc[U];
#pragma unroll
            for (int t = 0; t < U; ++t) vc[t] = vb[t];
            load_idx(jb + 2 * C, vb, cb);  // chunk m+2
#pragma unroll
            for (int t = 0; t < U; ++t) {
                double px = va[t], py = va[t];
#pragma unroll
                for (int k = 0; k < NK; ++k)
                    if (k < nother) {
                        px *= xa[t][k].x;
                        py *= xa[t][k].y;
                    }
                ax += px;
                ay += py;
            }
#pragma unroll
            for (int t = 0; t < U; ++t) {
                va[t] = vc[t];
#pragma unroll
                for (int k = 0; k < NK; ++k) xa[t][k] = xb[t][k];
            }
        }
        // groups in fixed order onto group 0's lanes, which write the row (zeros past R)
#pragma unroll
        for (int o = L; o < 32; o <<= 1) {
            ax += __shfl_xor_sync(0xffffffffu, ax, o);
            ay += __shfl_xor_sync(0xffffffffu, ay, o);
        }
        if (g == 0) reinterpret_cast<double2*>(p.out + i * RP)[c] = make_double2(ax, ay);
    }
}

template <int RP>
#ifndef CPFIT_SP_U
#define CPFIT_SP_U 2
#endif
void launch_sp2(const SpParams& p, const uint32_t* pidx, int order, cudaStream_t st) {
    constexpr int U = CPFIT_SP_U;
    // rows_per_warp from a target of 32 resident warps per SM; blocks of 8 warps
#ifndef CPFIT_SP_WPS
#define CPFIT_SP_WPS 24
#endif
    const int64_t max_warps = 148 * CPFIT_SP_WPS;
    const int64_t rpw = std::max<int64_t>(1, (p.In + max_warps - 1) / max_warps);
    const int64_t nwarps = (p.In + rpw - 1) / rpw;
    const int blocks = (int)std::max<int64_t>(1, (nwarps + 7) / 8);
    if (order == 3 && pidx)
        sp_mttkrp2_kernel<RP, 2, U, true><<<blocks, 256, 0, st>>>(p, pidx, rpw);
    else if (order == 3)
        sp_mttkrp2_kernel<RP, 2, U, false><<<blocks, 256, 0, st>>>(p, nullptr, rpw);
    else if (order == 4)
        sp_mttkrp2_kernel<RP, 3, U, false><<<blocks, 256, 0, st>>>(p, nullptr, rpw);
    else
        sp_mttkrp2_kernel<RP, 0, 2, false><<<blocks, 256, 0, st>>>(p, nullptr, rpw);
}

bool sp_v1() {
    static const bool v1 = [] {
        const char* e = getenv("CPFIT_SP_V1");
        return e && e[0] == '1';
    }();
    return v1;
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
// selects D_n) of a sparse order-3 tensor for the exact line-search polynomial (poly.cu), over the
// mode-0 sorted copy in the layout and two-stage pipeline of sp_mttkrp2_kernel (RP/2 lanes per
// row, 16-byte gathers of A1[j], D1[j], A2[k], D2[k]; packed indices when they fit). Each lane
// sums v X1[j] X2[k] for its two ranks in fp64 over a window of 16 of its group's nonzeros, then
// folds the window into double-double with X0[i] in {A0, D0} (the same 16-term fp64 sums as the
// shuffle-broadcast kernel it replaces); per-block partials [block][8] for coef_kernel, and the
// row's four mode-0 products X1 X2 (for M0 at u*) when m0xy is set.
template <int RP, int U, bool PK>
__global__ void __launch_bounds__(256, 2) sp_line8_kernel(const SpParams p, const uint32_t* __restrict__ pidx,
                                                       int64_t rows_per_warp, const double* a0rows,
                                                       const double* d0rows, const double* a1, const double* e1,
                                                       const double* a2, const double* e2, dd* part, double* m0xy) {
    constexpr int L = RP / 2, G = 32 / L, C = G * U;
    constexpr int FOLD = 16 / U;  // chunks per fp64 window (16 nonzeros per lane group)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / L, c = lane % L;
    const bool live = 2 * c < p.R;
    dd acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = dd{0.0, 0.0};
    const double2* f1a = reinterpret_cast<const double2*>(a1) + c;
    const double2* f1d = reinterpret_cast<const double2*>(e1) + c;
    const double2* f2a = reinterpret_cast<const double2*>(a2) + c;
    const double2* f2d = reinterpret_cast<const double2*>(e2) + c;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t i0 = gw * rows_per_warp, i1 = imin64(p.In, i0 + rows_per_warp);
    auto prefetch_row = [&](int64_t i) {
        const int64_t a = p.rowptr[i], b = p.rowptr[i + 1];
        if (b > a) {
            bulk_prefetch_l2(p.vals + a, (b - a) * 8);
            if (PK) {
                bulk_prefetch_l2(pidx + a, (b - a) * 4);
            } else {
                bulk_prefetch_l2(p.oidx + a, (b - a) * 4);
                bulk_prefetch_l2(p.oidx + p.nnz + a, (b - a) * 4);
            }
        }
    };
    if (lane == 0 && i0 < i1) prefetch_row(i0);
    for (int64_t i = i0; i < i1; ++i) {
        if (lane == 0 && i + 1 < i1) prefetch_row(i + 1);
        const double2 x0a = live ? reinterpret_cast<const double2*>(a0rows + i * RP)[c] : make_double2(0.0, 0.0);
        const double2 x0d = live ? reinterpret_cast<const double2*>(d0rows + i * RP)[c] : make_double2(0.0, 0.0);
        const int64_t j0 = p.rowptr[i], j1 = p.rowptr[i + 1];
        double2 qs[4], q[4];  // the row's X1 X2 products (for M0 at u*) and the current fp64 window
#pragma unroll
        for (int b12 = 0; b12 < 4; ++b12) qs[b12] = q[b12] = make_double2(0.0, 0.0);
        auto fold = [&]() {
#pragma unroll
            for (int b12 = 0; b12 < 4; ++b12) {
                acc[b12] = dd_fma(dd_fma(acc[b12], x0a.x, q[b12].x), x0a.y, q[b12].y);
                acc[4 + b12] = dd_fma(dd_fma(acc[4 + b12], x0d.x, q[b12].x), x0d.y, q[b12].y);
                qs[b12].x += q[b12].x;
                qs[b12].y += q[b12].y;
                q[b12] = make_double2(0.0, 0.0);
            }
        };
        if (j0 < j1) {
            const int n = (int)(j1 - j0);
            const double* vrow = p.vals + j0;
            const uint32_t* prow = PK ? pidx + j0 : nullptr;
            auto load_idx = [&](int64_t jb, double (&vv)[U], int (&cj)[U], int (&ck)[U]) {
#pragma unroll
                for (int t = 0; t < U; ++t) {
                    const int qo = (int)(jb - j0) + t * G + g;
                    const bool ok = qo < n;
                    const int qc = ok ? qo : 0;
                    vv[t] = ldg_d(vrow + qc, ok);
                    if (PK) {
                        cj[t] = (int)ldg_u(prow + qc);
                        ck[t] = 0;
                    } else {
                        cj[t] = __ldg(p.oidx + j0 + qc);
                        ck[t] = __ldg(p.oidx + p.nnz + j0 + qc);
                    }
                }
            };
            auto gather = [&](const int (&cj)[U], const int (&ck)[U], double2 (&xx)[U][4]) {
#pragma unroll
                for (int t = 0; t < U; ++t) {
                    int j = cj[t], k = ck[t];
                    if (PK) {
                        k = (int)((uint32_t)j >> 16);
                        j = (int)((uint32_t)j & 0xffffu);
                    }
                    xx[t][0] = ldg_d2(f1a + (int64_t)j * L, live);
                    xx[t][1] = ldg_d2(f1d + (int64_t)j * L, live);
                    xx[t][2] = ldg_d2(f2a + (int64_t)k * L, live);
                    xx[t][3] = ldg_d2(f2d + (int64_t)k * L, live);
                }
            };
            auto consume = [&](const double2 (&xx)[U][4], const double (&vv)[U]) {
#pragma unroll
                for (int t = 0; t < U; ++t) {
                    const double vax = vv[t] * xx[t][0].x, vay = vv[t] * xx[t][0].y;
                    const double vdx = vv[t] * xx[t][1].x, vdy = vv[t] * xx[t][1].y;
                    q[0].x = fma(vax, xx[t][2].x, q[0].x);
                    q[0].y = fma(vay, xx[t][2].y, q[0].y);
                    q[1].x = fma(vax, xx[t][3].x, q[1].x);
                    q[1].y = fma(vay, xx[t][3].y, q[1].y);
                    q[2].x = fma(vdx, xx[t][2].x, q[2].x);
                    q[2].y = fma(vdy, xx[t][2].y, q[2].y);
                    q[3].x = fma(vdx, xx[t][3].x, q[3].x);
                    q[3].y = fma(vdy, xx[t][3].y, q[3].y);
                }
            };
            double va[U], vb[U], vx[U];
            int ja[U], ka[U], jb_[U], kb[U];
            double2 xa[U][4];
            load_idx(j0, va, ja, ka);
            gather(ja, ka, xa);
#pragma unroll
            for (int t = 0; t < U; ++t) vx[t] = va[t];
            load_idx(j0 + C, vb, jb_, kb);
            int nf = 0;
            for (int64_t jb = j0; jb < j1; jb += C) {
                double2 xb[U][4];
                gather(jb_, kb, xb);  // chunk m+1
                double vn[U];
#pragma unroll
                for (int t = 0; t < U; ++t) vn[t] = vb[t];
                load_idx(jb + 2 * C, vb, jb_, kb);  // chunk m+2
                consume(xa, vx);                     // chunk m
                if (++nf == FOLD) {
                    fold();
                    nf = 0;
                }
#pragma unroll
                for (int t = 0; t < U; ++t) {
                    vx[t] = vn[t];
#pragma unroll
                    for (int k = 0; k < 4; ++k) xa[t][k] = xb[t][k];
                }
            }
            if (nf) fold();
        }
        if (m0xy) {  // combine the lane groups (fixed order), one row of each product
#pragma unroll
            for (int b12 = 0; b12 < 4; ++b12) {
                double vx2 = qs[b12].x, vy2 = qs[b12].y;
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    vx2 += __shfl_xor_sync(0xffffffffu, vx2, o);
                    vy2 += __shfl_xor_sync(0xffffffffu, vy2, o);
                }
                if (g == 0)
                    reinterpret_cast<double2*>(m0xy + ((int64_t)b12 * p.In + i) * RP)[c] = make_double2(vx2, vy2);
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
    std::vector<std::vector<uint32_t>> pidxs((size_t)N);
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
        if (N == 3 && nnz > 0) {
            bool fits = true;
            for (int m = 0; m < 3; ++m)
                if (m != n && t.dims[m] > 65536) fits = false;
            if (fits) {
                pidxs[(size_t)n].resize((size_t)nnz);
                uint32_t* pk = pidxs[(size_t)n].data();
                const int32_t* o = oidx.data();
                for (int64_t j = 0; j < nnz; ++j) pk[j] = (uint32_t)o[j] | ((uint32_t)o[nnz + j] << 16);
                CPFIT_CUDA(cudaMalloc(&sm->pidx[n], sizeof(uint32_t) * (size_t)nnz));
                CPFIT_CUDA(cudaMemcpyAsync(sm->pidx[n], pk, sizeof(uint32_t) * (size_t)nnz, cudaMemcpyHostToDevice, st));
            }
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
        cudaFree(t.modes->pidx[n]);
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
        if (!sp_v1() || w.RP > 32) {
            const uint32_t* pk = t.modes->pidx[n];
            switch (w.RP) {
                case 8: launch_sp2<8>(p, pk, N, st); break;
                case 16: launch_sp2<16>(p, pk, N, st); break;
                case 32: launch_sp2<32>(p, pk, N, st); break;
                default: launch_sp2<64>(p, pk, N, st); break;
            }
            CPFIT_CUDA(cudaGetLastError());
            continue;
        }
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
#ifndef CPFIT_L8_U
#define CPFIT_L8_U 1
#endif
    // rows per warp so the nblocks x 8 warps cover the rows in one pass
    const int64_t rpw = std::max<int64_t>(1, (p.In + (int64_t)nblocks * 8 - 1) / ((int64_t)nblocks * 8));
    const uint32_t* pk = t.modes->pidx[0];
    auto go = [&](auto tag) {
        constexpr int RP = decltype(tag)::value;
        if (pk)
            sp_line8_kernel<RP, CPFIT_L8_U, true><<<nblocks, 256, 0, st>>>(p, pk, rpw, w.frows, drows, w.frows + o1, drows + o1,
                                                                  w.frows + o2, drows + o2, part, m0xy);
        else
            sp_line8_kernel<RP, CPFIT_L8_U, false><<<nblocks, 256, 0, st>>>(p, nullptr, rpw, w.frows, drows, w.frows + o1,
                                                                   drows + o1, w.frows + o2, drows + o2, part, m0xy);
    };
    switch (w.RP) {
        case 8: go(std::integral_constant<int, 8>{}); break;
        case 16: go(std::integral_constant<int, 16>{}); break;
        default: go(std::integral_constant<int, 32>{}); break;
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
