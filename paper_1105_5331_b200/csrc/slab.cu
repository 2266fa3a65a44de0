// Mode-0 MTTKRP for short fibres by slabs (the M0 pass of mttkrp mode 0 and of the evaluation at
// an accepted point, kruskal.cpp:127-149 / tensor.cpp:206-240).
//
// When 16 | I_1, the 16 consecutive mode-0 fibres of a tile share their tail index (i_2, ..),
// so the tile's Khatri-Rao rows are W_f = A_1(i_1, :) * c, c = prod_{m >= 2} A_m(i_m, :):
//   M0 += T_tile W_tile = (T_tile A_1(block, :)) diag(c).
// A_1 is the same for every slab (I_1 fibres with one tail index): its DMMA A-fragments stay in
// registers for the whole pass, the tile's products Y accumulate on the tensor cores over the
// slab, and one scaling by c per slab folds them into M0. No W producers, no W ring: each warp
// streams its own contiguous tile range through a private ring (one TMA box of 16 fibres x I0s
// doubles per tile — the fibre kernels' tensor map, pad columns arriving as zeros — else one
// cp.async.bulk per fibre row; rows are 4 mod 16 doubles apart so the B-fragment loads are
// conflict free),
// and the CTA's warps sum their M0 in fixed order into the same per-CTA partial layout the fibre
// kernels write (m0_part[cta][r][32 nchunk]), so the reduction downstream is unchanged.
// The fibre kernels' M0 warps wait on their two W-producer warps for short fibres (C3: 44 us for
// a pass whose HBM floor is 20.5 us, profiles/r02_summary.md); this pass has no producer role
// (C3: 29 us, DMMA sub-pipe ~60 % busy with RP = 16 for R = 10).
// The evaluation at u_bar (M0 + per-fibre objective, S given) runs this pass plus
// fobj_slab_kernel (the per-fibre objective from S, the fibre norms and the factor rows) in place
// of the fibre kernel; both exit at once when the residual form is on (a device flag read at run
// time in the captured graph), and the fibre kernel then runs instead (FiberParams::only_resid).
#include "device.cuh"

#include <cstdlib>

namespace cpfit_gpu {

namespace {

constexpr int kSlabWarps = 16;  // 8 tile ranges x 2 row halves
constexpr int kSlabStages = 2;
constexpr int kSlabTileF = 16;  // fibres per tile

struct SlabParams {
    const double* T;
    int64_t ldT;
    int I0, I0s, I1;
    int64_t ntiles;  // J / 16
    int order, R;
    int64_t dims[kMaxOrder];
    const double* fac[kMaxOrder];  // col-major I_m x R blocks of the packed iterate
    double* m0_part;               // [grid][RP][ld]
    int ld;                        // 32 * nchunk
    int64_t tiles_per_warp;
    const int* resid_flag;         // exit at once when set (the residual form runs the fibre kernel)
    int use_tmap;                  // one TMA box (I0s x 16 at column h I0h, pads arrive as zeros) per tile
    int I0h;                       // rows of M0 per warp (a half of I0)
    CUtensorMap tmap;
};

// NQ = I_1 / 16 tiles per slab, NMT = row tiles of M0 per warp: the warps of a pair take the
// same tiles and one half of the I_0 rows each (twice the warps for the same shared memory)
template <int RP, int NQ, int NMT>
__global__ void __launch_bounds__(kSlabWarps * 32, 1) m0slab_kernel(const __grid_constant__ SlabParams p) {
    constexpr int NRT = RP / 8;
    if (p.resid_flag && *p.resid_flag) return;
    extern __shared__ __align__(128) double slab_raw[];
    __shared__ uint64_t full[kSlabWarps][kSlabStages];
    // TMA destinations need 128-byte alignment (the dynamic region follows the static barriers)
    double* slab_smem = slab_raw + ((128u - (smem_u32(slab_raw) & 127u)) & 127u) / 8u;  // stays a shared pointer
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int stage_dbl = kSlabTileF * p.I0s;
    double* ring = slab_smem + (size_t)warp * kSlabStages * stage_dbl;
    if (lane == 0)
        for (int s = 0; s < kSlabStages; ++s) mbar_init(&full[warp][s], 1);
    mbar_fence_init();
    __syncwarp();

    const int half = warp & 1;
    const int64_t gw = (int64_t)blockIdx.x * (kSlabWarps / 2) + (warp >> 1);
    const int64_t t0 = gw * p.tiles_per_warp, t1 = imin64(p.ntiles, t0 + p.tiles_per_warp);
    const uint64_t pol = l2_evict_first();
    const uint32_t row_bytes = (uint32_t)p.I0h * 8u;
    auto issue = [&](int64_t tile, int s) {
        if (p.use_tmap) {
            if (lane == 0) {
                mbar_arrive_expect_tx(&full[warp][s], (uint32_t)(kSlabTileF * p.I0s * 8));
                tma_2d_g2s_hint(ring + (size_t)s * stage_dbl, &p.tmap, half * p.I0h, (int)(tile * kSlabTileF),
                                &full[warp][s], pol);
            }
            return;
        }
        if (lane == 0) mbar_arrive_expect_tx(&full[warp][s], row_bytes * kSlabTileF);
        if (lane < kSlabTileF) {
            const double* src = p.T + (tile * kSlabTileF + lane) * p.ldT + half * p.I0h;
            bulk_g2s_hint(ring + (size_t)s * stage_dbl + (size_t)lane * p.I0s, src, row_bytes, &full[warp][s], pol);
        }
    };
    for (int s = 0; s < kSlabStages; ++s)
        if (t0 + s < t1) issue(t0 + s, s);

    // A_1^T fragments, shared by the CTA's warps, lane-major (conflict-free loads):
    // a1s[rt][ks][lane] = A[m = lane/4][k = lane%4] = A_1(i_1 = 4 ks + lane%4, r = 8 rt + lane/4)
    double* a1s = slab_smem + (size_t)kSlabWarps * kSlabStages * stage_dbl;
    for (int e = threadIdx.x; e < NRT * NQ * 4 * 32; e += blockDim.x) {
        const int l = e & 31, ks = (e >> 5) % (NQ * 4), rt = (e >> 5) / (NQ * 4);
        const int r = rt * 8 + (l >> 2), i1 = ks * 4 + (l & 3);
        a1s[e] = r < p.R ? p.fac[1][(int64_t)r * p.I1 + i1] : 0.0;
    }
    __syncthreads();
    double m0[NRT][NMT][2], y[NRT][NMT][2];
#pragma unroll
    for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
        for (int nt = 0; nt < NMT; ++nt) m0[rt][nt][0] = m0[rt][nt][1] = y[rt][nt][0] = y[rt][nt][1] = 0.0;

    // c = prod_{m >= 2} A_m(i_m, r) for the lane's accumulator rows r = 8 rt + lane/4
    auto flush = [&](int64_t slab) {
        double c[NRT];
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt) c[rt] = 1.0;
        int rem = (int)slab;  // slabs < 2^31 (checked on the host)
        for (int m = 2; m < p.order; ++m) {
            const int dm = (int)p.dims[m];
            const int im = rem % dm;
            rem /= dm;
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt) {
                const int r = rt * 8 + (lane >> 2);
                c[rt] *= r < p.R ? p.fac[m][(int64_t)r * dm + im] : 0.0;
            }
        }
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
            for (int nt = 0; nt < NMT; ++nt) {
                m0[rt][nt][0] = fma(c[rt], y[rt][nt][0], m0[rt][nt][0]);
                m0[rt][nt][1] = fma(c[rt], y[rt][nt][1], m0[rt][nt][1]);
                y[rt][nt][0] = y[rt][nt][1] = 0.0;
            }
    };

    int64_t k = 0;  // local tile counter (ring position)
    if (t0 < t1) {
        const int64_t s_first = t0 / NQ, s_last = (t1 - 1) / NQ;
        for (int64_t slab = s_first; slab <= s_last; ++slab) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int64_t tile = slab * NQ + q;
                if (tile < t0 || tile >= t1) continue;  // warp-uniform
                const int s = (int)(k % kSlabStages);
                mbar_wait(&full[warp][s], (uint32_t)((k / kSlabStages) & 1));
                const double* tt = ring + (size_t)s * stage_dbl;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const double* row = tt + (size_t)(kk * 4 + (lane & 3)) * p.I0s + (lane >> 2);
                    double a[NRT];
#pragma unroll
                    for (int rt = 0; rt < NRT; ++rt) a[rt] = a1s[(rt * NQ * 4 + q * 4 + kk) * 32 + lane];
#pragma unroll
                    for (int nt = 0; nt < NMT; ++nt) {
                        const double b = row[nt * 8];  // B[k = lane%4][n = lane/4] = T(fibre, i_0)
#pragma unroll
                        for (int rt = 0; rt < NRT; ++rt) dmma_8x8x4(y[rt][nt][0], y[rt][nt][1], a[rt], b);
                    }
                }
                // the stage's reads are done (the mma.sync consumed them): hand it to the next copy
                __syncwarp();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (tile + kSlabStages < t1) issue(tile + kSlabStages, s);
                ++k;
            }
            flush(slab);
        }
    }

    // fixed-order sum of the CTA's warps (the rings are free once every warp is done)
    __syncthreads();
    double* red = slab_smem;  // [kSlabWarps / 2][RP][2 * 8 NMT]: each pair's two halves side by side
    constexpr int LDR = 2 * 8 * NMT;
#pragma unroll
    for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
        for (int nt = 0; nt < NMT; ++nt) {
            const int r = rt * 8 + (lane >> 2), i = half * p.I0h + nt * 8 + 2 * (lane & 3);
            double* d = red + ((size_t)(warp >> 1) * RP + r) * LDR + i;
            d[0] = m0[rt][nt][0];
            d[1] = m0[rt][nt][1];
        }
    __syncthreads();
    double* out = p.m0_part + (size_t)blockIdx.x * RP * p.ld;
    for (int e = threadIdx.x; e < RP * p.ld; e += blockDim.x) {
        const int r = e / p.ld, i = e % p.ld;
        double v = 0.0;
        if (i < p.I0)
            for (int w2 = 0; w2 < kSlabWarps / 2; ++w2) v += red[((size_t)w2 * RP + r) * LDR + i];
        out[e] = v;
    }
}

template <int RP, int NQ>
bool launch_nmt(const SlabParams& p, int grid, size_t smem, cudaStream_t st) {
    switch (p.I0h / 8) {
#define CPFIT_SLAB_NMT(n)                                                                                      \
    case n:                                                                                                    \
        CPFIT_CUDA(cudaFuncSetAttribute(m0slab_kernel<RP, NQ, n>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        (int)smem));                                                           \
        m0slab_kernel<RP, NQ, n><<<grid, kSlabWarps * 32, smem, st>>>(p);                                     \
        return true;
        CPFIT_SLAB_NMT(1)
        CPFIT_SLAB_NMT(2)
        CPFIT_SLAB_NMT(3)
        CPFIT_SLAB_NMT(4)
#undef CPFIT_SLAB_NMT
        default: return false;
    }
}

template <int RP>
bool launch_nq(const SlabParams& p, int grid, size_t smem, cudaStream_t st) {
    switch (p.I1 / kSlabTileF) {
        case 1: return launch_nmt<RP, 1>(p, grid, smem, st);
        case 2: return launch_nmt<RP, 2>(p, grid, smem, st);
        case 3: return launch_nmt<RP, 3>(p, grid, smem, st);
        case 4: return launch_nmt<RP, 4>(p, grid, smem, st);
        default: return false;
    }
}

// the half-row box map (16 fibres x I0s doubles starting at column h I0h; columns past ldT arrive
// as zeros), cached on the workspace
bool slab_tmap(const DevTensor& t, EvalWork& w, int I0s) {
    if (w.slab_tmap >= 0) return w.slab_tmap == 1;
    w.slab_tmap = 0;
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (t.J >= ((int64_t)1 << 31) || I0s > 256) return false;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
        (void)cudaGetLastError();
        return false;
    }
    const cuuint64_t gdim[2] = {(cuuint64_t)t.ldT, (cuuint64_t)t.J};
    const cuuint64_t gstride[1] = {(cuuint64_t)t.ldT * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)I0s, (cuuint32_t)kSlabTileF};
    const cuuint32_t estride[2] = {1, 1};
    if (reinterpret_cast<EncodeFn>(fn)(&w.tmap_slab, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)t.T, gdim, gstride, box,
                                       estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        w.slab_tmap = 1;
    return w.slab_tmap == 1;
}

}  // namespace

// The slab M0 pass applies to dense tensors of order >= 3 with I_0 <= 64, 16 | I_0, 16 | I_1,
// I_1 <= 64 and RP <= 16 (A_1's fragments in registers); CPFIT_NO_SLAB=1 disables it (A/B).
bool m0_slab_applies(const DevTensor& t, const EvalWork& w) {
    static const bool off = [] {
        const char* e = std::getenv("CPFIT_NO_SLAB");
        return e && e[0] == '1';
    }();
    if (off || rowwise(t) || t.order < 3 || w.RP > 16 || !w.m0_part || t.J / t.dims[1] >= ((int64_t)1 << 31))
        return false;
    const int64_t I0 = t.dims[0], I1 = t.dims[1];
    return I0 <= 64 && I0 % 16 == 0 && I1 % kSlabTileF == 0 && I1 <= 4 * kSlabTileF && 32 * w.fiber_nchunk >= I0;
}

// M0 partials of T x KR(modes >= 1) at u into w.m0_part (w.fiber_grid CTAs, the fibre kernels'
// layout); false when the shape does not qualify (the caller runs the fibre kernel instead)
bool dense_m0_slab(const DevTensor& t, EvalWork& w, const double* u, cudaStream_t st, const int* resid_flag) {
    if (!m0_slab_applies(t, w)) return false;
    SlabParams p{};
    p.resid_flag = resid_flag;
    p.T = t.T;
    p.ldT = t.ldT;
    p.I0 = (int)t.dims[0];
    p.I0h = p.I0 / 2;
    // rows of a half tile in shared memory: 4 mod 16 doubles apart (conflict-free B loads)
    p.I0s = (p.I0h + 15) / 16 * 16 + 4;
    p.use_tmap = slab_tmap(t, w, p.I0s) ? 1 : 0;
    if (p.use_tmap) p.tmap = w.tmap_slab;
    p.I1 = (int)t.dims[1];
    p.ntiles = t.J / kSlabTileF;
    p.order = t.order;
    p.R = w.R;
    for (int m = 0; m < t.order; ++m) {
        p.dims[m] = t.dims[m];
        p.fac[m] = u + w.off[m];
    }
    p.m0_part = w.m0_part;
    p.ld = 32 * w.fiber_nchunk;
    const int grid = w.fiber_grid;
    const int64_t nranges = (int64_t)grid * (kSlabWarps / 2);
    p.tiles_per_warp = (p.ntiles + nranges - 1) / nranges;
    const size_t ring = sizeof(double) * (size_t)kSlabWarps * kSlabStages * kSlabTileF * p.I0s;
    const size_t red = sizeof(double) * (size_t)(kSlabWarps / 2) * w.RP * p.I0;
    const size_t a1b = sizeof(double) * (size_t)(w.RP / 8) * (p.I1 / kSlabTileF) * 4 * 32;
    const size_t smem = (ring > red ? ring : red) + a1b + 128;  // + the alignment slack
    bool ok = false;
    switch (w.RP) {
        case 8: ok = launch_nq<8>(p, grid, smem, st); break;
        default: ok = launch_nq<16>(p, grid, smem, st); break;
    }
    CPFIT_CUDA(cudaGetLastError());
    return ok;
}

namespace {

constexpr int kFobjThreads = 1024;

struct FobjParams {
    int64_t J;
    int I1, order, R;
    int64_t dims[kMaxOrder];
    const double* fac[kMaxOrder];
    const double* S;       // J x RP (S = T x_1 A_0)
    const double* fnorm2;  // ||t_f||^2 per fibre
    const double* gamma0;  // A_0^T A_0, RP x RP
    double* f_part;        // [grid]
    const int* resid_flag;
};

// Per-fibre objective with S given (the fibre kernels' S-given epilogue, fiber.cuh): for fibre f
// with w_f = A_1(i_1, :) * prod_{m >= 2} A_m(i_m, :), the partial sum of
// ||t_f||^2 + w_f^T (Gamma_0 w_f - 2 s_f); RP lanes per fibre (Gamma_0 row r on lane r), the
// block's fibres contiguous, fixed-order sums -> f_part[block].
template <int RP>
__global__ void __launch_bounds__(kFobjThreads) fobj_slab_kernel(const FobjParams p) {
    if (p.resid_flag && *p.resid_flag) return;
    // lane per fibre: w_f, s_f in registers, Gamma_0 from shared memory (broadcast loads);
    // a warp takes 32 consecutive fibres of one slab (I_1 % 16 == 0: a half warp never crosses)
    __shared__ double gam[RP * RP];
    __shared__ double red[kFobjThreads / 32];
    extern __shared__ double wsh[];  // per warp [r][lane]
    for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) gam[e] = p.gamma0[e];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
    const int R = p.R;
    // fibre indices fit 32 bits (m0_slab_applies: J / I_1 < 2^31, I_1 <= 64)
    const int f_lo = (int)((int64_t)blockIdx.x * p.J / gridDim.x), f_hi = (int)((int64_t)(blockIdx.x + 1) * p.J / gridDim.x);
    double acc = 0.0;
    for (int f = f_lo + warp * 32 + lane; f - lane < f_hi; f += nw * 32) {  // warp-uniform
        const bool ok = f < f_hi;
        const int fc = ok ? f : f_lo;
        const int i1 = fc % p.I1;
        int rem = fc / p.I1;
        double w[RP];
#pragma unroll
        for (int r = 0; r < RP; ++r) w[r] = r < R ? p.fac[1][(int64_t)r * p.I1 + i1] : 0.0;
        for (int m = 2; m < p.order; ++m) {
            const int dm = (int)p.dims[m];
            const int im = rem % dm;
            rem /= dm;
            const double* am = p.fac[m] + im;
#pragma unroll
            for (int r = 0; r < RP; ++r)
                if (r < R) w[r] *= am[(int64_t)r * dm];
        }
        const double2* srow = reinterpret_cast<const double2*>(p.S + (int64_t)fc * RP);
        double t = 0.0;
#pragma unroll
        for (int r2 = 0; r2 < RP / 2; ++r2) {
            if (2 * r2 < R) {
                const double2 sv = srow[r2];
                t = fma(w[2 * r2], -2.0 * sv.x, t);
                t = fma(w[2 * r2 + 1], -2.0 * sv.y, t);
            }
        }
        // w^T Gamma_0 w: the q loop stays rolled (w_q from this lane's shared-memory copy) so the
        // Gamma_0 loads are not all hoisted into registers
        double* wq = wsh + (size_t)warp * RP * 32 + lane;
#pragma unroll
        for (int r = 0; r < RP; ++r) wq[r * 32] = w[r];
#pragma unroll 1
        for (int q = 0; q < R; ++q) {
            double g = 0.0;
#pragma unroll
            for (int r = 0; r < RP; ++r)
                if (r < R) g = fma(gam[q * RP + r], w[r], g);
            t = fma(wq[q * 32], g, t);
        }
        if (ok) acc += p.fnorm2[fc] + t;
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w2 = 0; w2 < nw; ++w2) s += red[w2];
        p.f_part[blockIdx.x] = s;
    }
}

}  // namespace

void dense_fobj_slab(const DevTensor& t, EvalWork& w, const double* u, const double* S, const double* gamma0,
                     cudaStream_t st, const int* resid_flag) {
    FobjParams p{};
    p.J = t.J;
    p.I1 = (int)t.dims[1];
    p.order = t.order;
    p.R = w.R;
    for (int m = 0; m < t.order; ++m) {
        p.dims[m] = t.dims[m];
        p.fac[m] = u + w.off[m];
    }
    p.S = S;
    p.fnorm2 = t.fiber_norm2;
    p.gamma0 = gamma0;
    p.f_part = w.f_part;
    p.resid_flag = resid_flag;
    switch (w.RP) {
        case 8: {
            const size_t sm = sizeof(double) * (kFobjThreads / 32) * 8 * 32;
            CPFIT_CUDA(cudaFuncSetAttribute(fobj_slab_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            fobj_slab_kernel<8><<<w.fiber_grid, kFobjThreads, sm, st>>>(p);
            break;
        }
        default: {
            const size_t sm = sizeof(double) * (kFobjThreads / 32) * 16 * 32;
            CPFIT_CUDA(cudaFuncSetAttribute(fobj_slab_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            fobj_slab_kernel<16><<<w.fiber_grid, kFobjThreads, sm, st>>>(p);
            break;
        }
    }
    CPFIT_CUDA(cudaGetLastError());
}

}  // namespace cpfit_gpu
