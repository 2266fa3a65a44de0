// Dense CP kernels for sm_100a (fp64).
//
// The hot path of the reference's objective_and_gradient (kruskal.cpp:127-149) and
// mttkrp (tensor.cpp:206-240) is rebuilt around ONE streaming pass over mode-0 fibers:
//   S(f, :)  = T(:, f)^T A^(0)          (head contraction, per fiber f)        2KR flops
//   M0      += T(:, f) W(f, :)           (tail contraction, W = KR of modes>=1) 2KR flops
//   f_fiber  = ||t_f||^2 - 2 w.s + w^T G0 w                              (per-fiber objective)
// Both contractions run on the fp64 tensor cores (mma.sync m8n8k4 -> SASS DMMA) out of a
// bulk-async-copied shared-memory tile of F fibers. Modes >= 1 are then contracted from
// S (20 MB at 400^3 R=16, L2-resident) by the level kernels, so T is read once per
// evaluation instead of N+1 times.
#include "device.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace cpfit_gpu {

namespace {

int sm_count() {
    static int n = [] {
        int d = 0, c = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, d);
        return c > 0 ? c : 148;
    }();
    return n;
}

// ---------------------------------------------------------------------------------------
// Fiber pass
// ---------------------------------------------------------------------------------------
struct FiberParams {
    const double* T;
    int64_t ldT;
    int I0;
    int64_t J;
    int nchunk;  // warps per CTA; each owns 32 rows of the fiber
    int I0s;     // smem row stride (32*nchunk + 4)
    int do_s, do_m0, do_f;
    int R;
    const double* A0;  // col-major I0 x R
    int order;
    int64_t dims[kMaxOrder];
    const double* fac[kMaxOrder];  // col-major factor of each mode (modes >= 1 used for W)
    double* S_out;                 // J x RP
    double* m0_part;               // grid x RP x (32*nchunk)
    double* f_part;                // grid
    const double* gamma0;          // RP x RP
    const double* fnorm2;          // J
    const int* resid_flag;         // device flag: residual-form objective when nonzero
    int64_t tiles_per_cta;
    int64_t ntiles;
};

#include "fiber.cuh"

#if 0  // first version (CTA-wide barriers per tile), superseded by fiber.cuh
constexpr int kStages = 3;

template <int RP, int F>
__host__ __device__ constexpr int ws_ld() {
    return RP + 4;  // RP + 4 is 4 or 12 mod 16 for RP in {8,16,24,32}: conflict-free frags
}

template <int RP, int F>
size_t fiber_smem_bytes(int nchunk) {
    const int I0s = 32 * nchunk + 4;
    size_t b = 0;
    b += sizeof(double) * (size_t)kStages * F * I0s;          // T tiles
    b += sizeof(double) * (size_t)nchunk * F * RP;             // S partials per warp
    b += sizeof(double) * 2 * (size_t)F * ws_ld<RP, F>();      // W tile (double buffered)
    b += sizeof(double) * (size_t)F * RP;                      // per-fiber objective terms
    b += sizeof(uint64_t) * kStages;
    return b;
}

template <int RP, int F, bool A0REG>
__global__ void __launch_bounds__(512) fiber_kernel(const FiberParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int WLD = ws_ld<RP, F>();
    constexpr int NRT = RP / 8;
    const int I0s = p.I0s;
    double* tiles = reinterpret_cast<double*>(smem_raw);
    double* spart = tiles + (size_t)kStages * F * I0s;
    double* wsb = spart + (size_t)p.nchunk * F * RP;
    double* fterm = wsb + 2 * F * WLD;
    uint64_t* full = reinterpret_cast<uint64_t*>(fterm + F * RP);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthr = blockDim.x;
    const int64_t t_begin = (int64_t)blockIdx.x * p.tiles_per_cta;
    const int64_t t_end = imin64(p.ntiles, t_begin + p.tiles_per_cta);
    const int64_t ntl = t_end > t_begin ? t_end - t_begin : 0;

    // zero tiles once (padding rows beyond ldT must read as 0)
    for (int64_t e = tid; e < (int64_t)kStages * F * I0s; e += nthr) tiles[e] = 0.0;
    if (tid == 0)
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    auto issue = [&](int64_t t, int s) {
        // thread 0 only
        const int64_t f0 = t * F;
        const int nvalid = (int)cpfit_gpu::imin64(F, p.J - f0);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(nvalid * p.ldT * 8));
        for (int f = 0; f < nvalid; ++f)
            bulk_g2s(tiles + ((size_t)s * F + f) * I0s, p.T + (f0 + f) * p.ldT, (uint32_t)(p.ldT * 8), &full[s]);
    };
    auto zero_invalid = [&](int64_t t, int s) {
        const int64_t f0 = t * F;
        const int nvalid = (int)cpfit_gpu::imin64(F, p.J - f0);
        for (int e = tid; e < (F - nvalid) * I0s; e += nthr) tiles[((size_t)s * F + nvalid) * I0s + e] = 0.0;
    };
    if (tid == 0)
        for (int64_t k = 0; k < cpfit_gpu::imin64(kStages, ntl); ++k) issue(t_begin + k, (int)k);
    for (int64_t k = 0; k < cpfit_gpu::imin64(kStages, ntl); ++k) zero_invalid(t_begin + k, (int)k);

    const int c = warp;  // this warp's 32-row chunk
    // A0 fragments (B operand of the S contraction): A0[i][r], i = c*32 + ks*4 + lane%4
    double a0f[A0REG ? 8 : 1][A0REG ? NRT : 1];
    auto a0_at = [&](int ks, int rt) -> double {
        const int i = c * 32 + ks * 4 + (lane & 3);
        const int r = rt * 8 + (lane >> 2);
        return (i < p.I0 && r < p.R) ? p.A0[(int64_t)r * p.I0 + i] : 0.0;
    };
    if (A0REG && p.do_s) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt) a0f[ks][rt] = a0_at(ks, rt);
    }
    double macc[NRT][4][2];
#pragma unroll
    for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) macc[rt][nt][0] = macc[rt][nt][1] = 0.0;
    double facc = 0.0;
    const bool need_w = p.do_m0 || p.do_f;

    for (int64_t k = 0; k < ntl; ++k) {
        const int64_t t = t_begin + k;
        const int s = (int)(k % kStages);
        const uint32_t parity = (uint32_t)((k / kStages) & 1);
        double* wsv = wsb + (k & 1) * F * WLD;
        if (need_w) {
            for (int e = tid; e < F * RP; e += nthr) {
                const int f = e / RP, r = e % RP;
                const int64_t fib = t * F + f;
                double w = 0.0;
                if (fib < p.J && r < p.R) {
                    w = 1.0;
                    int64_t rem = fib;
                    for (int m = 1; m < p.order; ++m) {
                        const int64_t jm = rem % p.dims[m];
                        rem /= p.dims[m];
                        w *= p.fac[m][(int64_t)r * p.dims[m] + jm];
                    }
                }
                wsv[f * WLD + r] = w;
            }
        }
        __syncthreads();
        mbar_wait(&full[s], parity);
        const double* tt = tiles + (size_t)s * F * I0s;
        if (p.do_s) {
            double sacc[F / 8][NRT][2];
#pragma unroll
            for (int ft = 0; ft < F / 8; ++ft)
#pragma unroll
                for (int rt = 0; rt < NRT; ++rt) sacc[ft][rt][0] = sacc[ft][rt][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int i = c * 32 + ks * 4 + (lane & 3);
                double a[F / 8];
#pragma unroll
                for (int ft = 0; ft < F / 8; ++ft) a[ft] = tt[(ft * 8 + (lane >> 2)) * I0s + i];
#pragma unroll
                for (int rt = 0; rt < NRT; ++rt) {
                    const double b = A0REG ? a0f[A0REG ? ks : 0][A0REG ? rt : 0] : a0_at(ks, rt);
#pragma unroll
                    for (int ft = 0; ft < F / 8; ++ft) dmma_8x8x4(sacc[ft][rt][0], sacc[ft][rt][1], a[ft], b);
                }
            }
            double* sp = spart + (size_t)warp * F * RP;
#pragma unroll
            for (int ft = 0; ft < F / 8; ++ft)
#pragma unroll
                for (int rt = 0; rt < NRT; ++rt) {
                    const int f = ft * 8 + (lane >> 2), r = rt * 8 + 2 * (lane & 3);
                    *reinterpret_cast<double2*>(sp + f * RP + r) = make_double2(sacc[ft][rt][0], sacc[ft][rt][1]);
                }
        }
        if (p.do_m0) {
#pragma unroll
            for (int kf = 0; kf < F / 4; ++kf) {
                const int f = kf * 4 + (lane & 3);
                double wa[NRT];
#pragma unroll
                for (int rt = 0; rt < NRT; ++rt) wa[rt] = wsv[f * WLD + rt * 8 + (lane >> 2)];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const double b = tt[f * I0s + c * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
                    for (int rt = 0; rt < NRT; ++rt) dmma_8x8x4(macc[rt][nt][0], macc[rt][nt][1], wa[rt], b);
                }
            }
        }
        __syncthreads();  // stage s and spart complete
        if (k + kStages < ntl) {
            if (tid == 0) issue(t + kStages, s);
            zero_invalid(t + kStages, s);
        }
        if (p.do_s) {
            const int64_t f0 = t * F;
            for (int e = tid; e < F * RP; e += nthr) {
                const int f = e / RP, r = e % RP;
                double v = 0.0;
                for (int ww = 0; ww < p.nchunk; ++ww) v += spart[((size_t)ww * F + f) * RP + r];
                if (f0 + f < p.J) p.S_out[(f0 + f) * RP + r] = v;
                if (p.do_f) {
                    // per-fiber objective term: w_r * ((G0 w)_r - 2 s_r)
                    double q = 0.0;
#pragma unroll 8
                    for (int qq = 0; qq < RP; ++qq) q += p.gamma0[r * RP + qq] * wsv[f * WLD + qq];
                    const double w = wsv[f * WLD + r];
                    fterm[f * RP + r] = w * (q - 2.0 * v);
                }
            }
            if (p.do_f) {
                __syncthreads();
                if (tid < F && f0 + tid < p.J) {
                    double pf = p.fnorm2[f0 + tid];
                    for (int r = 0; r < RP; ++r) pf += fterm[tid * RP + r];
                    facc += pf;
                }
            }
        }
    }
    // write M0 partials: M0^T[r][i] tile fragments
    if (p.do_m0) {
        const int ld = 32 * p.nchunk;
        double* out = p.m0_part + (size_t)blockIdx.x * RP * ld;
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int r = rt * 8 + (lane >> 2);
                const int i = c * 32 + nt * 8 + 2 * (lane & 3);
                out[(size_t)r * ld + i] = macc[rt][nt][0];
                out[(size_t)r * ld + i + 1] = macc[rt][nt][1];
            }
    }
    if (p.do_f) {
        // fixed-order block reduction of the per-fiber sums (threads < F hold them)
        __shared__ double red[32];
        double v = warp_sum(facc);
        if (lane == 0) red[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int ww = 0; ww < (nthr + 31) / 32; ++ww) s += red[ww];
            p.f_part[blockIdx.x] = s;
        }
    }
}

template <int RP>
void launch_fiber(const FiberParams& p, int grid, int nchunk, size_t smem, cudaStream_t st) {
    constexpr int F = 16;
    if (RP <= 16) {
        auto k = fiber_kernel<RP, F, true>;
        CPFIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, 32 * nchunk, smem, st>>>(p);
    } else {
        auto k = fiber_kernel<RP, F, false>;
        CPFIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, 32 * nchunk, smem, st>>>(p);
    }
    CPFIT_CUDA(cudaGetLastError());
}

size_t fiber_smem(int RP, int nchunk) {
    switch (RP) {
        case 8: return fiber_smem_bytes<8, 16>(nchunk);
        case 16: return fiber_smem_bytes<16, 16>(nchunk);
        case 24: return fiber_smem_bytes<24, 16>(nchunk);
        default: return fiber_smem_bytes<32, 16>(nchunk);
    }
}

#endif

// M0 = sum over the fiber-pass CTAs of their [RP][32 NC] partials (fixed order)
void reduce_parts(const double* part, int nparts, int64_t nout, double* out, cudaStream_t st);
void reduce_m0(EvalWork& w, cudaStream_t st) {
    reduce_parts(w.m0_part, w.fiber_grid, (int64_t)w.RP * 32 * w.fiber_nchunk, w.m0, st);
}

void run_fiber(const DevTensor& t, EvalWork& w, const double* u, bool do_s, bool do_m0, bool do_f,
               const double* gamma0, cudaStream_t st, const int* resid_flag = nullptr) {
    FiberParams p{};
    p.T = t.T;
    p.ldT = t.ldT;
    p.I0 = (int)t.dims[0];
    p.J = t.J;
    p.nchunk = w.fiber_nchunk;
    p.I0s = 32 * w.fiber_nchunk + 4;
    p.do_s = do_s;
    p.do_m0 = do_m0;
    p.do_f = do_f;
    p.R = w.R;
    p.A0 = u;
    p.order = t.order;
    for (int m = 0; m < t.order; ++m) {
        p.dims[m] = t.dims[m];
        p.fac[m] = u + w.off[m];
    }
    p.S_out = w.S;
    p.m0_part = w.m0_part;
    p.f_part = w.f_part;
    p.gamma0 = gamma0;
    p.fnorm2 = t.fiber_norm2;
    p.resid_flag = resid_flag;
    p.ntiles = (t.J + w.fiber_F - 1) / w.fiber_F;
    p.tiles_per_cta = (p.ntiles + w.fiber_grid - 1) / w.fiber_grid;
    const int grid = (int)((p.ntiles + p.tiles_per_cta - 1) / p.tiles_per_cta);
    // unused CTA slots of the partial buffers must read as zero
    if (grid < w.fiber_grid) {
        if (do_m0)
            CPFIT_CUDA(cudaMemsetAsync(w.m0_part + (size_t)grid * w.RP * 32 * w.fiber_nchunk, 0,
                                       sizeof(double) * (size_t)(w.fiber_grid - grid) * w.RP * 32 * w.fiber_nchunk, st));
        if (do_f) CPFIT_CUDA(cudaMemsetAsync(w.f_part + grid, 0, sizeof(double) * (w.fiber_grid - grid), st));
    }
    switch (w.RP) {
        case 8: launch_fiber<8>(p, grid, w.fiber_nchunk, w.fiber_smem, st); break;
        case 16: launch_fiber<16>(p, grid, w.fiber_nchunk, w.fiber_smem, st); break;
        default: launch_fiber<32>(p, grid, w.fiber_nchunk, w.fiber_smem, st); break;
    }
}

// ---------------------------------------------------------------------------------------
// Level contraction: Sin viewed as (Ih x Jt x RP) [(jh + Ih*s)*RP + r]
//   Mh(jh, r)   = sum_s Sin(jh, s, r) * Wt(s, r),  Wt = KR of modes h+1..N-1
//   Sout(s, r)  = sum_jh Sin(jh, s, r) * Ah(jh, r)
// Thread t owns pairs p = t + k*B of (jh, r) (B % RP == 0 so r = t % RP is fixed).
// ---------------------------------------------------------------------------------------
struct LevelParams {
    const double* Sin;
    int64_t Ih, Jt;
    int R, RP;
    const double* Ah;  // col-major Ih x R (head factor) or null (no Sout)
    int ntail;
    int64_t tdims[kMaxOrder];
    const double* tfac[kMaxOrder];
    double* mh_part;  // grid x Ih x RP  (null: skip Mh)
    double* Sout;     // Jt x RP (null: skip)
    int64_t slabs_per_cta;
};

constexpr int kLevelThreads = 256;
constexpr int kSlabBatch = 8;

__global__ void __launch_bounds__(kLevelThreads) level_kernel(const LevelParams p) {
    extern __shared__ __align__(16) double lsm[];
    const int tid = threadIdx.x, B = blockDim.x;
    const int RP = p.RP;
    const int64_t npairs = p.Ih * RP;
    const int kmax = (int)((npairs + B - 1) / B);
    double* acc = lsm;                          // kmax * B (private per thread)
    double* ah = acc + (size_t)kmax * B;        // kmax * B
    double* wt = ah + (size_t)kmax * B;         // kSlabBatch * RP
    double* spart = wt + kSlabBatch * RP;       // kSlabBatch * B
    const int64_t s_begin = (int64_t)blockIdx.x * p.slabs_per_cta;
    const int64_t s_end = imin64(p.Jt, s_begin + p.slabs_per_cta);
    const int r = tid % RP;
    for (int k = 0; k < kmax; ++k) {
        const int64_t pr = tid + (int64_t)k * B;
        acc[k * B + tid] = 0.0;
        double a = 0.0;
        if (p.Ah && pr < npairs && r < p.R) a = p.Ah[(int64_t)r * p.Ih + pr / RP];
        ah[k * B + tid] = a;
    }
    for (int64_t s0 = s_begin; s0 < s_end; s0 += kSlabBatch) {
        const int nb = (int)cpfit_gpu::imin64(kSlabBatch, s_end - s0);
        __syncthreads();
        for (int e = tid; e < nb * RP; e += B) {
            const int sl = e / RP, rr = e % RP;
            double w = 0.0;
            if (rr < p.R) {
                w = 1.0;
                int64_t rem = s0 + sl;
                for (int m = 0; m < p.ntail; ++m) {
                    const int64_t jm = rem % p.tdims[m];
                    rem /= p.tdims[m];
                    w *= p.tfac[m][(int64_t)rr * p.tdims[m] + jm];
                }
            }
            wt[sl * RP + rr] = w;
        }
        __syncthreads();
        for (int sl = 0; sl < nb; ++sl) {
            const double* src = p.Sin + (s0 + sl) * p.Ih * RP;
            const double wv = wt[sl * RP + r];
            double sp = 0.0;
            for (int k = 0; k < kmax; ++k) {
                const int64_t pr = tid + (int64_t)k * B;
                if (pr < npairs) {
                    const double v = src[pr];
                    acc[k * B + tid] += v * wv;
                    sp += v * ah[k * B + tid];
                }
            }
            spart[sl * B + tid] = sp;
        }
        __syncthreads();
        if (p.Sout) {
            for (int e = tid; e < nb * RP; e += B) {
                const int sl = e / RP, rr = e % RP;
                double v = 0.0;
                for (int t2 = rr; t2 < B; t2 += RP) v += spart[sl * B + t2];
                p.Sout[(s0 + sl) * RP + rr] = v;
            }
        }
    }
    if (p.mh_part) {
        double* out = p.mh_part + (size_t)blockIdx.x * npairs;
        for (int k = 0; k < kmax; ++k) {
            const int64_t pr = tid + (int64_t)k * B;
            if (pr < npairs) out[pr] = acc[k * B + tid];
        }
    }
}

// Fixed-order reduction of `nparts` contiguous partial vectors: out[o] = sum_c part[c*nout+o].
// Block = 32 outputs x 8 part-slices (coalesced across lanes), slices combined in order.
__global__ void __launch_bounds__(256) reduce_parts_kernel(const double* __restrict__ part, int nparts, int64_t nout,
                                                           double* __restrict__ out) {
    __shared__ double sl[8][33];
    const int lane = threadIdx.x & 31, ws = threadIdx.x >> 5;
    const int64_t o = (int64_t)blockIdx.x * 32 + lane;
    double v = 0.0;
    if (o < nout)
        for (int c = ws; c < nparts; c += 8) v += part[(int64_t)c * nout + o];
    sl[ws][lane] = v;
    __syncthreads();
    if (ws == 0 && o < nout) {
        double s = 0.0;
        for (int k = 0; k < 8; ++k) s += sl[k][lane];
        out[o] = s;
    }
}

void reduce_parts(const double* part, int nparts, int64_t nout, double* out, cudaStream_t st) {
    reduce_parts_kernel<<<(unsigned)((nout + 31) / 32), 256, 0, st>>>(part, nparts, nout, out);
    CPFIT_CUDA(cudaGetLastError());
}

// M_h(jh, r) = sum_s Sin(jh, s, r) Wt(s, r) over a chunk of slabs per CTA: thread (jh, r),
// coalesced over consecutive (jh, r) for each slab; chunk partials -> reduce_parts.
struct LevelMParams {
    const double* Sin;
    int64_t Ih, Jt;
    int R, RP;
    int ntail;
    int64_t tdims[kMaxOrder];
    const double* tfac[kMaxOrder];
    int64_t chunk;  // slabs per chunk
    double* part;   // [chunk][Ih*RP]
};

__global__ void __launch_bounds__(256) level_m_kernel(const LevelMParams p) {
    extern __shared__ double wt[];  // [chunk][RP]
    const int64_t npairs = p.Ih * p.RP;
    const int64_t s0 = (int64_t)blockIdx.y * p.chunk;
    const int64_t s1 = imin64(p.Jt, s0 + p.chunk);
    const int ns = (int)(s1 - s0);
    for (int e = threadIdx.x; e < ns * p.RP; e += blockDim.x) {
        const int sl = e / p.RP, r = e % p.RP;
        double w = 0.0;
        if (r < p.R) {
            w = 1.0;
            int64_t rem = s0 + sl;
            for (int m = 0; m < p.ntail; ++m) {
                const int64_t jm = rem % p.tdims[m];
                rem /= p.tdims[m];
                w *= p.tfac[m][(int64_t)r * p.tdims[m] + jm];
            }
        }
        wt[e] = w;
    }
    __syncthreads();
    const int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= npairs) return;
    const int r = (int)(pr % p.RP);
    const double* src = p.Sin + s0 * npairs + pr;
    double a0 = 0.0, a1 = 0.0;
    int sl = 0;
    for (; sl + 1 < ns; sl += 2) {
        a0 += src[(int64_t)sl * npairs] * wt[sl * p.RP + r];
        a1 += src[(int64_t)(sl + 1) * npairs] * wt[(sl + 1) * p.RP + r];
    }
    if (sl < ns) a0 += src[(int64_t)sl * npairs] * wt[sl * p.RP + r];
    p.part[(int64_t)blockIdx.y * npairs + pr] = a0 + a1;
}

void run_level(const DevTensor& t, EvalWork& w, int h, const double* Sin, const double* u, bool do_m, bool do_s,
               double* Sout, cudaStream_t st) {
    const int64_t Ih = t.dims[h];
    int64_t Jt = 1;
    for (int m = h + 1; m < t.order; ++m) Jt *= t.dims[m];
    const int64_t npairs = Ih * w.RP;
    if (do_m) {
        LevelMParams q{};
        q.Sin = Sin;
        q.Ih = Ih;
        q.Jt = Jt;
        q.R = w.R;
        q.RP = w.RP;
        q.ntail = t.order - h - 1;
        for (int m = h + 1; m < t.order; ++m) {
            q.tdims[m - h - 1] = t.dims[m];
            q.tfac[m - h - 1] = u + w.off[m];
        }
        q.chunk = w.lvl_chunk[h];
        q.part = w.lvl_part[h];
        const int nchunk = (int)((Jt + q.chunk - 1) / q.chunk);
        dim3 grid((unsigned)((npairs + 255) / 256), (unsigned)nchunk);
        level_m_kernel<<<grid, 256, sizeof(double) * q.chunk * w.RP, st>>>(q);
        CPFIT_CUDA(cudaGetLastError());
        reduce_parts(w.lvl_part[h], nchunk, npairs, w.lvl_m[h], st);
    }
    if (!do_s) return;
    LevelParams p{};
    p.Sin = Sin;
    p.Ih = Ih;
    p.Jt = Jt;
    p.R = w.R;
    p.RP = w.RP;
    p.Ah = u + w.off[h];
    p.ntail = t.order - h - 1;
    for (int m = h + 1; m < t.order; ++m) {
        p.tdims[m - h - 1] = t.dims[m];
        p.tfac[m - h - 1] = u + w.off[m];
    }
    p.mh_part = nullptr;
    p.Sout = Sout;
    const int gmax = w.lvl_grid[h];
    p.slabs_per_cta = (p.Jt + gmax - 1) / gmax;
    const int grid = (int)((p.Jt + p.slabs_per_cta - 1) / p.slabs_per_cta);
    const int B = kLevelThreads;
    const int kmax = (int)((npairs + B - 1) / B);
    const size_t smem = sizeof(double) * ((size_t)2 * kmax * B + kSlabBatch * w.RP + (size_t)kSlabBatch * B);
    CPFIT_CUDA(cudaFuncSetAttribute(level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    level_kernel<<<grid, B, smem, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------
// Grams in double-double: G_n(r,q) = sum_i A_n(i,r) A_n(i,q); one warp per (mode, pair,
// row chunk). Then a combine kernel sums chunks in order and rounds.
// ---------------------------------------------------------------------------------------
struct GramParams {
    int order, R, RP;
    int64_t dims[kMaxOrder];
    const double* fac[kMaxOrder];
    int chunks[kMaxOrder];
    int64_t chunk_rows;
    dd* part;    // [mode][chunk][R*R]
    double* out; // [mode][RP*RP]
    int maxchunks;
    int mode0;
};

__global__ void gram_partial_kernel(const GramParams p) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int npair = p.R * (p.R + 1) / 2;
    // decode (mode, chunk, pair)
    int rem = gw;
    for (int n = 0; n < p.order; ++n) {
        const int cnt = p.chunks[n] * npair;
        if (rem < cnt) {
            const int chunk = rem / npair, pr = rem % npair;
            int r = 0, acc = 0;
            while (acc + (p.R - r) <= pr) {
                acc += p.R - r;
                ++r;
            }
            const int q = r + (pr - acc);
            const int64_t i0 = (int64_t)chunk * p.chunk_rows;
            const int64_t i1 = min(p.dims[n], i0 + p.chunk_rows);
            const double* a = p.fac[n] + (int64_t)r * p.dims[n];
            const double* b = p.fac[n] + (int64_t)q * p.dims[n];
            dd s{0.0, 0.0};
            for (int64_t i = i0 + lane; i < i1; i += 32) s = dd_fma(s, a[i], b[i]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                dd t{__shfl_xor_sync(0xffffffffu, s.hi, o), __shfl_xor_sync(0xffffffffu, s.lo, o)};
                s = dd_add(s, t);
            }
            if (lane == 0) {
                dd* dst = p.part + ((size_t)n * p.maxchunks + chunk) * p.R * p.R;
                dst[r * p.R + q] = s;
            }
            return;
        }
        rem -= cnt;
    }
}

__global__ void gram_combine_kernel(const GramParams p) {
    const int n = p.mode0 + blockIdx.x;
    for (int e = threadIdx.x; e < p.RP * p.RP; e += blockDim.x) {
        const int r = e / p.RP, q = e % p.RP;
        double v = 0.0;
        if (r < p.R && q < p.R) {
            const int a = min(r, q), b = max(r, q);
            dd s{0.0, 0.0};
            for (int c = 0; c < p.chunks[n]; ++c) s = dd_add(s, p.part[((size_t)n * p.maxchunks + c) * p.R * p.R + a * p.R + b]);
            v = s.hi + s.lo;
        }
        p.out[(size_t)n * p.RP * p.RP + e] = v;
    }
}

GramParams gram_params(EvalWork& w, const double* u) {
    GramParams p{};
    p.order = w.order;
    p.R = w.R;
    p.RP = w.RP;
    p.chunk_rows = 2048;
    p.maxchunks = 1;
    for (int n = 0; n < w.order; ++n) {
        p.dims[n] = w.dims[n];
        p.fac[n] = u + w.off[n];
        p.chunks[n] = w.gram_chunks[n];
        p.maxchunks = std::max(p.maxchunks, p.chunks[n]);
    }
    p.part = w.gram_part;
    p.out = w.gram;
    return p;
}

// ---------------------------------------------------------------------------------------
// Gradient epilogue: g_n(i,r) = -M_n(i,r) + sum_q A_n(i,q) Gamma_n(q,r)
// M_0 from fiber partials [cta][r][i]; M_h (1..N-2) from level partials [cta][i][r];
// M_{N-1} from the last level's Sout [i][r] (complete).  Also per-block partial
// ||g||^2 and g.d; block 0 of the finalize kernel adds them in order.
// ---------------------------------------------------------------------------------------
struct GradParams {
    int order, R, RP;
    int64_t dims[kMaxOrder];
    int64_t off[kMaxOrder + 1];
    const double* u;
    double* g;
    const double* d;
    const double* gram;  // [mode][RP*RP]
    const double* m0;    // reduced M_0 [r][m0_ld]
    int m0_ld;
    const double* lvl_m[kMaxOrder];  // reduced M_h [i][r], 1 <= h <= N-2
    const double* mlast;   // [i][r] complete M_{N-1} (dense) or null
    const double* sp_out;  // sparse: per-mode complete M_n [mode offset][i][r] (null for dense)
    int64_t sp_off[kMaxOrder];
    double* red;           // gridDim x 3
    int need_grad;
    // finalisation by the last block to finish (fixed-order sums of the block partials)
    const double* f_part;
    int f_grid;
    int sparse;  // three-term objective (kruskal.cpp:146-148)
    double norm_sq;
    EvalScalars* sc;
    int has_d;
    unsigned int* counter;
};

__device__ double gamma_entry(const GradParams& p, int n, int q, int r) {
    double v = 1.0;
    for (int m = 0; m < p.order; ++m)
        if (m != n) v *= p.gram[(size_t)m * p.RP * p.RP + q * p.RP + r];
    return v;  // Grams are exactly symmetric, so the (X+X^T)/2 symmetrisation is the identity
}

__global__ void grad_kernel(const GradParams p) {
    extern __shared__ double gsm[];
    __shared__ double red[3][32];
    const int tid = threadIdx.x;
    const int RR = p.R * p.R;
    for (int e = tid; e < p.order * RR; e += blockDim.x) {
        const int n = e / RR, q = (e / p.R) % p.R, r = e % p.R;
        gsm[e] = gamma_entry(p, n, q, r);
    }
    __syncthreads();
    const int64_t total = p.off[p.order];
    double g2 = 0.0, gd = 0.0, inner = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + tid; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int n = 0;
        while (e >= p.off[n + 1]) ++n;
        const int64_t loc = e - p.off[n];
        const int64_t In = p.dims[n];
        const int r = (int)(loc / In);
        const int64_t i = loc % In;
        double m;
        if (p.sp_out)
            m = p.sp_out[p.sp_off[n] + i * p.RP + r];
        else if (n == 0)
            m = p.m0[(size_t)r * p.m0_ld + i];
        else if (n == p.order - 1)
            m = p.mlast[i * p.RP + r];
        else
            m = p.lvl_m[n][i * p.RP + r];
        if (n == 0) inner += m * p.u[e];
        if (p.need_grad) {
            const double* a = p.u + p.off[n];
            double ag = 0.0;
            for (int q = 0; q < p.R; ++q) ag += a[(int64_t)q * In + i] * gsm[n * RR + q * p.R + r];
            const double gv = -m + ag;
            p.g[e] = gv;
            g2 += gv * gv;
            if (p.d) gd += gv * p.d[e];
        }
    }
    const int lane = tid & 31, warp = tid >> 5;
    g2 = warp_sum(g2);
    gd = warp_sum(gd);
    inner = warp_sum(inner);
    if (lane == 0) {
        red[0][warp] = g2;
        red[1][warp] = gd;
        red[2][warp] = inner;
    }
    __syncthreads();
    __shared__ bool last;
    if (tid == 0) {
        double a = 0, b = 0, c = 0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) {
            a += red[0][w];
            b += red[1][w];
            c += red[2][w];
        }
        p.red[blockIdx.x * 3 + 0] = a;
        p.red[blockIdx.x * 3 + 1] = b;
        p.red[blockIdx.x * 3 + 2] = c;
        __threadfence();
        last = (atomicAdd(p.counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!last || warp != 0) return;
    // last block, one warp: lane-strided partial sums then a fixed shuffle tree (deterministic)
    __threadfence();
    double a = 0.0, b = 0.0, c = 0.0, fs = 0.0;
    for (int k = lane; k < (int)gridDim.x; k += 32) {
        a += p.red[k * 3 + 0];
        b += p.red[k * 3 + 1];
        c += p.red[k * 3 + 2];
    }
    for (int k = lane; k < p.f_grid; k += 32) fs += p.f_part[k];
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    fs = warp_sum(fs);
    double gs = 0.0;
    if (p.sparse) {
        // kruskal.cpp:146-148: 1/2||T||^2 - <M0, A0> + 1/2 1^T Gamma 1, Gamma = gram_hadamard(-1)
        for (int e = lane; e < p.R * p.R; e += 32) {
            const int q = e / p.R, r = e % p.R;
            double v = 1.0;
            for (int m = 0; m < p.order; ++m) v *= p.gram[(size_t)m * p.RP * p.RP + q * p.RP + r];
            gs += v;
        }
        gs = warp_sum(gs);
    }
    if (lane == 0) {
        p.sc->f = p.sparse ? 0.5 * p.norm_sq - c + 0.5 * gs : 0.5 * fs;
        p.sc->gnorm2 = a;
        p.sc->inner = c;
        if (p.has_d) p.sc->gdotd = b;
        *p.counter = 0u;  // ready for the next evaluation (stream order)
    }
}

}  // namespace

// ---------------------------------------------------------------------------------------
// sparse hooks (sparse.cu)
void sparse_all_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st);

// ---------------------------------------------------------------------------------------

EvalWork* work_create(const DevTensor& t, int R) {
    if (R < 1 || R > kMaxRank) throw std::invalid_argument("device path supports 1 <= rank <= 32");
    auto* w = new EvalWork();
    w->R = R;
    w->RP = (R <= 8) ? 8 : (R <= 16 ? 16 : 32);  // power of two: per-fiber lane groups
    w->order = t.order;
    w->off[0] = 0;
    for (int n = 0; n < t.order; ++n) {
        w->dims[n] = t.dims[n];
        w->off[n + 1] = w->off[n] + t.dims[n] * R;
    }
    w->nu = w->off[t.order];
    const int sms = sm_count();
    int maxchunks = 1;
    for (int n = 0; n < t.order; ++n) {
        w->gram_chunks[n] = (int)((t.dims[n] + 2047) / 2048);
        maxchunks = std::max(maxchunks, w->gram_chunks[n]);
    }
    CPFIT_CUDA(cudaMalloc(&w->gram_part, sizeof(dd) * (size_t)t.order * maxchunks * R * R));
    CPFIT_CUDA(cudaMalloc(&w->gram, sizeof(double) * (size_t)t.order * w->RP * w->RP));
    w->red_grid = sms * 2;
    CPFIT_CUDA(cudaMalloc(&w->red, sizeof(double) * 3 * (size_t)w->red_grid));
    CPFIT_CUDA(cudaMalloc(&w->counter, sizeof(unsigned int)));
    CPFIT_CUDA(cudaMemset(w->counter, 0, sizeof(unsigned int)));
    if (!t.sparse) {
        if (t.order < 2) throw std::invalid_argument("device dense path needs order >= 2");
        const int I0 = (int)t.dims[0];
        w->fiber_nchunk = (I0 + 31) / 32;
        if (w->fiber_nchunk > 13) throw std::invalid_argument("device dense path supports I_1 <= 416");
        w->fiber_smem = fiber_smem(w->RP, w->fiber_nchunk);
        if (w->fiber_smem > 227 * 1024) throw std::invalid_argument("fiber tile does not fit shared memory");
        const int64_t ntiles = (t.J + w->fiber_F - 1) / w->fiber_F;
        const int per_sm = std::max(1, std::min(2048 / (32 * (w->fiber_nchunk + 3)),
                                                (int)((228 * 1024) / (w->fiber_smem + 1024))));
        w->fiber_grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
        CPFIT_CUDA(cudaMalloc(&w->S, sizeof(double) * (size_t)t.J * w->RP));
        CPFIT_CUDA(cudaMalloc(&w->m0_part, sizeof(double) * (size_t)w->fiber_grid * w->RP * 32 * w->fiber_nchunk));
        CPFIT_CUDA(cudaMalloc(&w->m0, sizeof(double) * (size_t)w->RP * 32 * w->fiber_nchunk));
        CPFIT_CUDA(cudaMalloc(&w->f_part, sizeof(double) * (size_t)w->fiber_grid));
        for (int h = 1; h < t.order - 1; ++h) {
            int64_t Jt = 1;
            for (int m = h + 1; m < t.order; ++m) Jt *= t.dims[m];
            w->lvl_grid[h] = (int)std::min<int64_t>(Jt, (int64_t)sms);
            const int64_t npairs = t.dims[h] * w->RP;
            const int64_t bx = (npairs + 255) / 256;
            const int64_t want = std::max<int64_t>(1, (2 * sms + bx - 1) / bx);
            w->lvl_chunk[h] = std::max<int64_t>(1, std::min<int64_t>((Jt + want - 1) / want, 6144 / w->RP));
            const int64_t nch = (Jt + w->lvl_chunk[h] - 1) / w->lvl_chunk[h];
            CPFIT_CUDA(cudaMalloc(&w->lvl_part[h], sizeof(double) * (size_t)nch * npairs));
            CPFIT_CUDA(cudaMalloc(&w->lvl_m[h], sizeof(double) * (size_t)npairs));
            CPFIT_CUDA(cudaMalloc(&w->lvl_S[h], sizeof(double) * (size_t)Jt * w->RP));
        }
    } else {
        int64_t tot = 0;
        for (int n = 0; n < t.order; ++n) tot += t.dims[n] * w->RP;
        CPFIT_CUDA(cudaMalloc(&w->sp_part, sizeof(double) * (size_t)tot));
        CPFIT_CUDA(cudaMalloc(&w->frows, sizeof(double) * (size_t)tot));
        CPFIT_CUDA(cudaMalloc(&w->f_part, sizeof(double) * 4));
    }
    return w;
}

void work_destroy(EvalWork* w) {
    if (!w) return;
    cudaFree(w->gram_part);
    cudaFree(w->gram);
    cudaFree(w->red);
    cudaFree(w->S);
    cudaFree(w->m0_part);
    cudaFree(w->m0);
    cudaFree(w->f_part);
    cudaFree(w->sp_part);
    cudaFree(w->frows);
    cudaFree(w->counter);
    for (int h = 0; h < kMaxOrder; ++h) {
        cudaFree(w->lvl_part[h]);
        cudaFree(w->lvl_m[h]);
        cudaFree(w->lvl_S[h]);
    }
    delete w;
}

void grams_device(EvalWork& w, const double* u, cudaStream_t st) {
    GramParams p = gram_params(w, u);
    const int npair = w.R * (w.R + 1) / 2;
    int warps = 0;
    for (int n = 0; n < w.order; ++n) warps += w.gram_chunks[n] * npair;
    gram_partial_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(p);
    gram_combine_kernel<<<w.order, 256, 0, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
}

void gram_mode_device(EvalWork& w, const double* u, int mode, cudaStream_t st) {
    GramParams p = gram_params(w, u);
    const int npair = w.R * (w.R + 1) / 2;
    // restrict to one mode by zeroing the other chunk counts and offsetting pointers
    GramParams q = p;
    for (int n = 0; n < w.order; ++n) q.chunks[n] = (n == mode) ? p.chunks[n] : 0;
    const int warps = p.chunks[mode] * npair;
    q.mode0 = mode;
    gram_partial_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(q);
    gram_combine_kernel<<<1, 256, 0, st>>>(q);
    CPFIT_CUDA(cudaGetLastError());
}

namespace {
void run_grad(const DevTensor& t, EvalWork& w, const double* u, double* g, const double* d, bool need_grad,
              EvalScalars* sc, cudaStream_t st) {
    GradParams p{};
    p.order = t.order;
    p.R = w.R;
    p.RP = w.RP;
    for (int n = 0; n < t.order; ++n) {
        p.dims[n] = t.dims[n];
        p.off[n] = w.off[n];
        p.lvl_m[n] = w.lvl_m[n];
    }
    p.off[t.order] = w.off[t.order];
    p.u = u;
    p.g = g;
    p.d = d;
    p.gram = w.gram;
    p.need_grad = need_grad ? 1 : 0;
    if (t.sparse) {
        p.sp_out = w.sp_part;
        int64_t acc = 0;
        for (int n = 0; n < t.order; ++n) {
            p.sp_off[n] = acc;
            acc += t.dims[n] * w.RP;
        }
    } else {
        p.m0 = w.m0;
        p.m0_ld = 32 * w.fiber_nchunk;
        p.mlast = (t.order == 2) ? w.S : w.lvl_S[t.order - 2];
    }
    p.red = w.red;
    p.f_part = w.f_part;
    p.f_grid = t.sparse ? 0 : w.fiber_grid;
    p.sparse = t.sparse ? 1 : 0;
    p.norm_sq = t.norm_sq;
    p.sc = sc;
    p.has_d = d ? 1 : 0;
    p.counter = w.counter;
    // enough blocks to cover n_u once (latency-bound epilogue, no grid-stride tail)
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(w.red_grid, (w.nu + 255) / 256));
    grad_kernel<<<blocks, 256, sizeof(double) * t.order * w.R * w.R, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
}
}  // namespace

void eval_device(const DevTensor& t, EvalWork& w, const double* u, double* g, EvalScalars* sc, const double* d,
                 int* status, cudaStream_t st, bool need_grad, const int* resid_flag) {
    (void)status;
    grams_device(w, u, st);
    if (!t.sparse) {
        // fused pass: S, M0 partials and per-fiber objective
        run_fiber(t, w, u, true, true, true, w.gram /* mode-0 Gram */, st, resid_flag);
        reduce_m0(w, st);
        // modes 1..N-1 from S
        const double* Sin = w.S;
        for (int h = 1; h < t.order - 1; ++h) {
            run_level(t, w, h, Sin, u, true, true, w.lvl_S[h], st);
            Sin = w.lvl_S[h];
        }
    } else {
        sparse_all_modes(t, w, u, -1, st);
    }
    run_grad(t, w, u, g, d, need_grad, sc, st);
}

namespace {
// out (I_mode x R col-major) from the row-major [i][r] / fiber-partial layouts
__global__ void gather_m_kernel(int64_t In, int R, int RP, const double* part, int grid, int ld, int layout,
                                double* out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < In * R; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / In);
        const int64_t i = e % In;
        double v = 0.0;
        if (layout == 0) {  // [cta][r][i] with ld
            for (int c = 0; c < grid; ++c) v += part[((size_t)c * RP + r) * ld + i];
        } else {  // [cta][i][r]
            for (int c = 0; c < grid; ++c) v += part[((size_t)c * In + i) * RP + r];
        }
        out[e] = v;
    }
}
}  // namespace

void mttkrp_device(const DevTensor& t, EvalWork& w, const double* u, int mode, double* out, cudaStream_t st) {
    const int64_t In = t.dims[mode];
    const int blocks = (int)std::min<int64_t>(1024, (In * w.R + 255) / 256);
    if (t.sparse) {
        sparse_all_modes(t, w, u, mode, st);
        int64_t off = 0;
        for (int n = 0; n < mode; ++n) off += t.dims[n] * w.RP;
        gather_m_kernel<<<blocks, 256, 0, st>>>(In, w.R, w.RP, w.sp_part + off, 1, 0, 1, out);
        CPFIT_CUDA(cudaGetLastError());
        return;
    }
    if (mode == 0) {
        run_fiber(t, w, u, false, true, false, nullptr, st);
        reduce_m0(w, st);
        gather_m_kernel<<<blocks, 256, 0, st>>>(In, w.R, w.RP, w.m0, 1, 32 * w.fiber_nchunk, 0, out);
    } else {
        run_fiber(t, w, u, true, false, false, nullptr, st);
        const double* Sin = w.S;
        for (int h = 1; h <= mode && h < t.order - 1; ++h) {
            const bool last = (h == mode);
            run_level(t, w, h, Sin, u, last, !last, w.lvl_S[h], st);
            Sin = w.lvl_S[h];
        }
        if (mode == t.order - 1)
            gather_m_kernel<<<blocks, 256, 0, st>>>(In, w.R, w.RP, Sin, 1, 0, 1, out);
        else
            gather_m_kernel<<<blocks, 256, 0, st>>>(In, w.R, w.RP, w.lvl_m[mode], 1, 0, 1, out);
    }
    CPFIT_CUDA(cudaGetLastError());
}

// exported for als.cu
void dense_fiber(const DevTensor& t, EvalWork& w, const double* u, bool do_s, bool do_m0, cudaStream_t st) {
    run_fiber(t, w, u, do_s, do_m0, false, nullptr, st);
    if (do_m0) reduce_m0(w, st);  // -> w.m0
}
// the fused evaluation pass alone (S + M0 + per-fiber objective); Grams of u must be current
void dense_fiber_fused(const DevTensor& t, EvalWork& w, const double* u, cudaStream_t st, const int* resid_flag) {
    run_fiber(t, w, u, true, true, true, w.gram, st, resid_flag);
}
void dense_level(const DevTensor& t, EvalWork& w, int h, const double* Sin, const double* u, bool do_m, bool do_s,
                 double* Sout, cudaStream_t st) {
    run_level(t, w, h, Sin, u, do_m, do_s, Sout, st);
}
void gather_m(int64_t In, EvalWork& w, const double* part, int grid, int ld, int layout, double* out,
              cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(1024, (In * w.R + 255) / 256);
    gather_m_kernel<<<blocks, 256, 0, st>>>(In, w.R, w.RP, part, grid, ld, layout, out);
    CPFIT_CUDA(cudaGetLastError());
}

}  // namespace cpfit_gpu
