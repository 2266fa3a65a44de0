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
#include <memory>

namespace cpfit_gpu {

int sm_count() {
    static int n = [] {
        int d = 0, c = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, d);
        return c > 0 ? c : 148;
    }();
    return n;
}

namespace {

// ---------------------------------------------------------------------------------------
// Fiber pass
// ---------------------------------------------------------------------------------------
constexpr int kMaxM0W = 16;  // M0 warps per fiber CTA (fiber.cuh FiberRoles)

struct alignas(64) FiberParams {
    CUtensorMap tmap;  // T as [J][ldT] with a 16 x pitch box (use_tmap)
    int use_tmap;
    const double* T;
    int64_t ldT;
    int I0;
    int64_t J;
    int nchunk;  // 32-row chunks of the fiber (smem stride / M0 ld = 32*nchunk)
    int I0s;     // smem row stride (32*nchunk + 4)
    // M0 warps and their 8-row m-tiles: warp m owns m-tiles [mt_start[m], +mt_cnt[m]),
    // balanced across the SM's four schedulers (fiber_schedule)
    int mt_cnt[kMaxM0W];
    int mt_start[kMaxM0W];
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
    int only_resid;                // exit at once unless *resid_flag (the slab passes did M0 + f)
    int64_t tiles_per_cta;
    int64_t ntiles;
    unsigned long long* prof;  // diagnostic build only (fiber.cuh FIBER_WAIT)
    const double* S_in;        // S given (M0 + per-fiber objective pass): J x RP
    int nst;                   // T ring stages (EvalWork::fiber_nst: kFStages or kDeepFStages)
    int sreg_groups;           // S pass without K split: tile groups (0: K-split mode)
};

#include "fiber.cuh"


}  // namespace

// diagnostic counters of the -DCPFIT_FIBER_PROF build (zeros otherwise)
unsigned long long* fiber_prof_buffer() {
    static unsigned long long* buf = nullptr;
    if (!buf) {
        CPFIT_CUDA(cudaMalloc(&buf, sizeof(unsigned long long) * kProfSlots));
        CPFIT_CUDA(cudaMemset(buf, 0, sizeof(unsigned long long) * kProfSlots));
    }
    return buf;
}

namespace {

// fixed-order reductions of partial vectors, several in one launch (reduce_jobs)
struct RedJob {
    const double* part;
    int nparts;
    int64_t nout;
    double* out;
    // gradient epilogue (reduce_grad): the reduced vector is M_mode, laid out [r][ld] (layout 0,
    // M0) or [i][RP] (layout 1, the levels)
    int mode, layout, ld;
};
struct RedJobs {
    static constexpr int kMax = 2 * kMaxOrder + 1;
    RedJob j[kMax];
    int n = 0;
    void add(const double* part, int nparts, int64_t nout, double* out, int mode = -1, int layout = 1, int ld = 0) {
        j[n++] = RedJob{part, nparts, nout, out, mode, layout, ld};
    }
    int64_t blocks() const {
        int64_t b = 0;
        for (int k = 0; k < n; ++k) b += (j[k].nout + 31) / 32;
        return b;
    }
};
void reduce_jobs(const RedJobs& jobs, cudaStream_t st);
// M0 = sum over the fiber-pass CTAs of their [RP][32 NC] partials (fixed order)
void add_m0_job(EvalWork& w, RedJobs& j) {
    j.add(w.m0_part, w.fiber_grid, (int64_t)w.RP * 32 * w.fiber_nchunk, w.m0, 0, 0, 32 * w.fiber_nchunk);
}
void reduce_m0(EvalWork& w, cudaStream_t st) {
    RedJobs j;
    add_m0_job(w, j);
    reduce_jobs(j, st);
}

void run_fiber(const DevTensor& t, EvalWork& w, const double* u, bool do_s, bool do_m0, bool do_f,
               const double* gamma0, cudaStream_t st, const int* resid_flag = nullptr, double* s_out = nullptr,
               const double* s_in = nullptr) {
    // M0 only, short fibres with 16 | I_1: the slab pass (slab.cu) writes the same partials
    if (do_m0 && !do_s && !do_f && dense_m0_slab(t, w, u, st, nullptr)) return;
    // M0 + per-fibre objective with S given, same shapes: the slab pass and a per-fibre objective
    // kernel (S, the fibre norms and the factor rows; T is not read twice); under the residual form
    // (a device flag) both exit and the fibre kernel below does the pass instead
    const bool slab_f = do_m0 && !do_s && do_f && s_in && m0_slab_applies(t, w);
    FiberParams p{};
    p.only_resid = 0;
    p.T = t.T;
    p.ldT = t.ldT;
    p.I0 = (int)t.dims[0];
    p.J = t.J;
    p.nchunk = w.fiber_nchunk;
    p.I0s = 32 * w.fiber_nchunk + 4;
    p.nst = w.fiber_nst;
    // the S-only pass (sreg_kernel, RP <= 16) has its own row pitch
    const bool sreg = do_s && !do_m0 && !do_f && w.RP <= 16;
    p.use_tmap = w.fiber_tmap ? 1 : 0;
    p.sreg_groups = w.sreg_groups;
    if (w.fiber_tmap) p.tmap = sreg ? w.tmap_sreg : w.tmap_fws;
    fiber_schedule(w.RP, p.I0, do_s, p);
#ifdef CPFIT_FIBER_PROF
    p.prof = fiber_prof_buffer();
#endif
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
    p.S_out = s_out ? s_out : w.S;
    p.S_in = s_in;
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
    if (slab_f) {
        dense_m0_slab(t, w, u, st, resid_flag);
        dense_fobj_slab(t, w, u, s_in, gamma0, st, resid_flag);
        if (!resid_flag) return;  // the per-fibre form always: no residual fallback needed
        p.only_resid = 1;
    }
    if (do_s && !do_m0 && !do_f) {  // S only: every warp on S
        switch (w.RP) {
            case 8: launch_spass<8>(p, grid, st); break;
            case 16: launch_spass<16>(p, grid, st); break;
            default: launch_spass<32>(p, grid, st); break;
        }
        return;
    }
    switch (w.RP) {
        case 8: launch_fiber<8>(p, grid, w.fiber_smem, st); break;
        case 16: launch_fiber<16>(p, grid, w.fiber_smem, st); break;
        default: launch_fiber<32>(p, grid, w.fiber_smem, st); break;
    }
}

// ---------------------------------------------------------------------------------------
// Level contraction: Sin viewed as Jt slabs of (Ih x RP) doubles [(s*Ih + jh)*RP + r]
//   M_h(jh, r) = sum_s Sin(s, jh, r) * Wt(s, r),  Wt = KR rows of modes h+1..N-1
//   Sout(s, r) = sum_jh Sin(s, jh, r) * A_h(jh, r)
// Both from one read of Sin. CTA (x, y) streams slabs [x*spc, (x+1)*spc) over the pair range
// [y*256*KM, (y+1)*256*KM); a thread owns pairs base + tid + 256 k (k < KM; 256 % RP == 0 so
// r = tid % RP) with its M accumulators and A_h entries in registers. M partials per x go
// through reduce_parts (fixed order); Sout per (y, slab) from a shuffle + shared-memory tree.
// ---------------------------------------------------------------------------------------
struct LevelParams {
    const double* Sin;
    int64_t Ih, Jt;
    int R;
    const double* Ah;  // col-major Ih x R (Sout) or null
    int ntail;
    int64_t tdims[kMaxOrder];
    const double* tfac[kMaxOrder];
    double* m_part;  // [gridDim.x][Ih*RP] or null (no M_h)
    double* s_out;   // [gridDim.y][Jt][RP] or null (no Sout)
    int64_t spc;     // slabs per CTA
    // optional: the input is Sin + beta Sd (beta on the device), read on the fly, where Sin
    // itself is given as S' with Sin[s][i][r] = S'[s][i][perm r] sc0[r] when perm is set
    const double* Sd;
    const double* beta;
    const int* perm;
    const double* sc0;
    // optional (bulk kernel, M only): the last slab-range CTA of each pair tile sums the tile's
    // partials in order and writes M_h col-major (I_h x R) here — the MTTKRP's final output
    double* m_final;
    unsigned int* tile_cnt;
};

constexpr int kLevelThreads = 256;
constexpr int kSlabBatch = 8;

// Slabs are processed two at a time (both slabs' loads issue before the FMAs: two rounds of
// L2 latency in flight per thread); the Khatri-Rao tail rows of a batch of slabs are built once
// per batch with 32-bit index math.
template <int RP, int KM, bool DO_M, bool DO_S>
__global__ void __launch_bounds__(kLevelThreads, 2) level_kernel(const LevelParams p) {
    constexpr int B = kLevelThreads, NW = B / 32;
    __shared__ double wt[kSlabBatch][RP];
    __shared__ double sred[kSlabBatch][NW][RP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = tid % RP;
    const int npairs = (int)(p.Ih * RP);
    const int pbase = blockIdx.y * B * KM + tid;
    const int s_begin = (int)(blockIdx.x * p.spc);
    const int s_end = (int)imin64(p.Jt, s_begin + p.spc);
    double acc[KM], ah[KM];
    const double bt = p.Sd ? *p.beta : 0.0;
#pragma unroll
    for (int k = 0; k < KM; ++k) {
        const int pr = pbase + k * B;
        acc[k] = 0.0;
        ah[k] = (DO_S && pr < npairs && r < p.R) ? p.Ah[(int64_t)r * p.Ih + pr / RP] : 0.0;
    }
    for (int s0 = s_begin; s0 < s_end; s0 += kSlabBatch) {
        const int nb = min(kSlabBatch, s_end - s0);
        __syncthreads();  // previous batch's wt / sred consumers are done
        if (DO_M) {
            for (int e = tid; e < nb * RP; e += B) {
                const int sl = e / RP, rr = e % RP;
                double w = 0.0;
                if (rr < p.R) {
                    w = 1.0;
                    int rem = s0 + sl;
                    for (int m = 0; m < p.ntail; ++m) {
                        const int d = (int)p.tdims[m];
                        const int q = rem / d;
                        w *= p.tfac[m][(int64_t)rr * d + (rem - q * d)];
                        rem = q;
                    }
                }
                wt[sl][rr] = w;
            }
            __syncthreads();
        }
        for (int sl = 0; sl < nb; sl += 2) {
            const bool two = sl + 1 < nb;
            const double* src0 = p.Sin + (int64_t)(s0 + sl) * npairs;
            const double* src1 = src0 + npairs;
            double v0[KM], v1[KM];
#pragma unroll
            for (int k = 0; k < KM; ++k) {
                const int pr = pbase + k * B;
                v0[k] = pr < npairs ? __ldg(src0 + pr) : 0.0;
                v1[k] = (two && pr < npairs) ? __ldg(src1 + pr) : 0.0;
            }
            if (p.Sd) {  // S(u_bar + beta d) = S(u_bar) + beta S_d, as the separate axpy would
                const double* d0 = p.Sd + (int64_t)(s0 + sl) * npairs;
                const double* d1 = d0 + npairs;
#pragma unroll
                for (int k = 0; k < KM; ++k) {
                    const int pr = pbase + k * B;
                    if (pr < npairs) v0[k] = fma(bt, __ldg(d0 + pr), v0[k]);
                    if (two && pr < npairs) v1[k] = fma(bt, __ldg(d1 + pr), v1[k]);
                }
            }
            if (DO_M) {
                const double w0 = wt[sl][r], w1 = two ? wt[sl + 1][r] : 0.0;
#pragma unroll
                for (int k = 0; k < KM; ++k) acc[k] = fma(v1[k], w1, fma(v0[k], w0, acc[k]));
            }
            if (DO_S) {
                double sp0 = 0.0, sp1 = 0.0;
#pragma unroll
                for (int k = 0; k < KM; ++k) {
                    sp0 = fma(v0[k], ah[k], sp0);
                    sp1 = fma(v1[k], ah[k], sp1);
                }
#pragma unroll
                for (int o = 16; o >= RP; o >>= 1) {
                    sp0 += __shfl_xor_sync(0xffffffffu, sp0, o);
                    sp1 += __shfl_xor_sync(0xffffffffu, sp1, o);
                }
                if (lane < RP) {
                    sred[sl][warp][lane] = sp0;
                    if (two) sred[sl + 1][warp][lane] = sp1;
                }
            }
        }
        if (DO_S) {
            __syncthreads();
            for (int e = tid; e < nb * RP; e += B) {
                const int sl = e / RP, rr = e % RP;
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < NW; ++w) v += sred[sl][w][rr];
                p.s_out[((int64_t)blockIdx.y * p.Jt + s0 + sl) * RP + rr] = v;
            }
        }
    }
    if (DO_M) {
        double* out = p.m_part + (int64_t)blockIdx.x * npairs;
#pragma unroll
        for (int k = 0; k < KM; ++k) {
            const int pr = pbase + k * B;
            if (pr < npairs) out[pr] = acc[k];
        }
    }
}

// Last level (one Khatri-Rao tail factor, e.g. h = 1 of an order-3 tensor): CTA (x, y) owns the
// pair tile [256 x, 256 (x + 1)) of slabs [kBulkSlabs y, kBulkSlabs (y + 1)). One thread issues
// the tile's slab rows (2 KB each, and those of Sd) as bulk async copies into shared memory while
// the others stage the tail factor's rows; a thread then owns one pair:
//   M partial (per y)   = sum over its slabs of Sin * A_tail[slab][r]
//   Sout partial (per x) = per slab, the sum over the tile's pairs of rank r of Sin * A_h[i][r]
// (lanes of equal r by shuffles, then the warps in order). Partials reduced by reduce_jobs.
constexpr int kBulkSlabs = 16;
constexpr int kBulkPairs = kLevelThreads;

template <int RP, bool DO_M, bool DO_S>
__global__ void __launch_bounds__(kBulkPairs) level_bulk_kernel(const LevelParams p) {
    constexpr int NW = kBulkPairs / 32;
    extern __shared__ __align__(16) double lbuf[];  // [kBulkSlabs][kBulkPairs] Sin, then Sd
    __shared__ double a2s[kBulkSlabs][RP];
    __shared__ __align__(8) uint64_t bar;
    // the per-warp Sout sums reuse the Sin rows once every warp has read them
    static_assert(NW * kBulkSlabs * RP <= kBulkSlabs * kBulkPairs, "sred alias");
    double(*sred)[kBulkSlabs][RP] = reinterpret_cast<double(*)[kBulkSlabs][RP]>(lbuf);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int npairs = (int)(p.Ih * RP);
    const int pr0 = blockIdx.x * kBulkPairs, pr = pr0 + tid;
    const int s0 = blockIdx.y * kBulkSlabs;
    const int nsl = (int)imin64(kBulkSlabs, p.Jt - s0);
    const int npr = min(kBulkPairs, npairs - pr0);
    const bool has_d = p.Sd != nullptr;
    if (warp == 0) {  // lane l < nsl copies slab row l (and lane 16 + l its Sd row)
        const uint32_t row = (uint32_t)npr * 8u;
        if (lane == 0) {
            mbar_init(&bar, 1);
            mbar_fence_init();
            mbar_arrive_expect_tx(&bar, row * (uint32_t)nsl * (has_d ? 2u : 1u));
        }
        __syncwarp();
        const int sl = lane & 15;
        if (sl < nsl && (lane < 16 || has_d)) {
            const int64_t off = (int64_t)(s0 + sl) * npairs + pr0;
            if (lane < 16)
                bulk_g2s(lbuf + sl * kBulkPairs, p.Sin + off, row, &bar);
            else
                bulk_g2s(lbuf + (kBulkSlabs + sl) * kBulkPairs, p.Sd + off, row, &bar);
        }
    }
    const int r = tid % RP;
    const double bt = has_d ? *p.beta : 0.0;
    // Sin column permutation / scale (the normalised iterate's S from the sweep's S')
    const bool pm = p.perm != nullptr && r < p.R;
    const int src = pm ? tid - r + p.perm[r] : tid;
    const double scl = pm ? p.sc0[r] : 1.0;
    const double ah = (DO_S && pr < npairs && r < p.R) ? p.Ah[(int64_t)r * p.Ih + pr / RP] : 0.0;
    if (DO_M)  // kBulkSlabs x RP entries (512 at RP = 32: more than the block's threads)
        for (int e = tid; e < kBulkSlabs * RP; e += kBulkPairs) {
            const int sl = e % kBulkSlabs, rr = e / kBulkSlabs;  // consecutive slabs of a column
            a2s[sl][rr] = (sl < nsl && rr < p.R) ? p.tfac[0][(int64_t)rr * p.tdims[0] + s0 + sl] : 0.0;
        }
    __syncthreads();  // a2s staged; the barrier's init is visible
    mbar_wait(&bar, 0);
    double acc = 0.0, xs[kBulkSlabs];
    const bool live = pr < npairs;
#pragma unroll
    for (int sl = 0; sl < kBulkSlabs; ++sl) {
        xs[sl] = 0.0;
        if (sl < nsl) {
            double v = live ? lbuf[sl * kBulkPairs + src] : 0.0;
            if (pm) v *= scl;
            if (has_d && live) v = fma(bt, lbuf[(kBulkSlabs + sl) * kBulkPairs + tid], v);
            if (DO_M) acc = fma(v, a2s[sl][r], acc);
            if (DO_S) {
                double x = v * ah;
#pragma unroll
                for (int o = 16; o >= RP; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                xs[sl] = x;
            }
        }
    }
    if (DO_M && live) p.m_part[(int64_t)blockIdx.y * npairs + pr] = acc;
    if (DO_M && p.m_final) {
        __shared__ bool last;
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            last = (atomicAdd(p.tile_cnt + blockIdx.x, 1u) == gridDim.y - 1);
            if (last) p.tile_cnt[blockIdx.x] = 0u;
        }
        __syncthreads();
        if (!last) return;
        __threadfence();
        if (live && r < p.R) {
            double v = 0.0;
            for (int c = 0; c < (int)gridDim.y; ++c) v += __ldcg(p.m_part + (int64_t)c * npairs + pr);
            p.m_final[(int64_t)r * p.Ih + pr / RP] = v;
        }
        return;
    }
    if (DO_S) {
        __syncthreads();  // every warp is done with the Sin rows
        if (lane < RP)
#pragma unroll
            for (int sl = 0; sl < kBulkSlabs; ++sl) sred[warp][sl][lane] = xs[sl];
        __syncthreads();
        for (int e = tid; e < nsl * RP; e += kBulkPairs) {
            const int sl = e / RP, rr = e % RP;
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += sred[w][sl][rr];
            p.s_out[((int64_t)blockIdx.x * p.Jt + s0 + sl) * RP + rr] = v;
        }
    }
}

template <int RP>
void launch_level_bulk(const LevelParams& p, dim3 grid, cudaStream_t st) {
    const bool m = p.m_part != nullptr, s = p.s_out != nullptr;
    const size_t smem = sizeof(double) * kBulkSlabs * kBulkPairs * (p.Sd ? 2 : 1);
    static bool attr = [] {  // every variant (the kernels share one function-pointer type)
        const int mx = (int)(sizeof(double) * kBulkSlabs * kBulkPairs * 2);
        cudaFuncSetAttribute(level_bulk_kernel<RP, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(level_bulk_kernel<RP, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(level_bulk_kernel<RP, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        return true;
    }();
    (void)attr;
    if (m && s)
        level_bulk_kernel<RP, true, true><<<grid, kBulkPairs, smem, st>>>(p);
    else if (m)
        level_bulk_kernel<RP, true, false><<<grid, kBulkPairs, smem, st>>>(p);
    else
        level_bulk_kernel<RP, false, true><<<grid, kBulkPairs, smem, st>>>(p);
}

template <int RP, int KM>
void launch_level_km(const LevelParams& p, dim3 grid, cudaStream_t st) {
    const bool m = p.m_part != nullptr, s = p.s_out != nullptr;
    if (m && s)
        level_kernel<RP, KM, true, true><<<grid, kLevelThreads, 0, st>>>(p);
    else if (m)
        level_kernel<RP, KM, true, false><<<grid, kLevelThreads, 0, st>>>(p);
    else
        level_kernel<RP, KM, false, true><<<grid, kLevelThreads, 0, st>>>(p);
}
template <int RP>
void launch_level_rp(const LevelParams& p, dim3 grid, int km, cudaStream_t st) {
    switch (km) {
        case 4: launch_level_km<RP, 4>(p, grid, st); break;
        case 8: launch_level_km<RP, 8>(p, grid, st); break;
        default: launch_level_km<RP, 16>(p, grid, st); break;
    }
}

// Fixed-order reduction of `nparts` contiguous partial vectors: out[o] = sum_c part[c*nout+o],
// for up to RedJobs::kMax jobs in one launch (job k owns blocks [blk0[k], blk0[k+1])).
// Block = 32 outputs x 8 part-slices (coalesced across lanes), slices combined in order.
// With a gradient epilogue (dense evaluation; the jobs then hold M_0 .. M_{N-1}) each reduced
// M_n(i, r) also gives g_n(i, r) = (A_n Gamma_n)(i, r) - M_n(i, r), Gamma_n = Hadamard of the
// other Grams (kruskal.cpp:127-149), and the last block to finish forms ||g||^2, g.d, <M0, A0>
// and the per-fiber objective sum (as grad_kernel does).
struct GradEpi {
    int order, R, RP, need_grad;
    int64_t dims[kMaxOrder];
    int64_t off[kMaxOrder + 1];
    const double* u;
    double* g;
    const double* d;
    const double* gram;  // [mode][RP*RP]
    const double* f_part;
    int f_grid;
    EvalScalars* sc;
    double* red;  // [block][3]
    unsigned int* counter;
};
struct RedLaunch {
    RedJob j[RedJobs::kMax];
    int blk0[RedJobs::kMax + 1];
    int n;
    int grad;  // gradient epilogue on
    GradEpi ge;
};
__global__ void __launch_bounds__(256) reduce_parts_kernel(const RedLaunch L) {
    __shared__ double sl[8][33];
    extern __shared__ double gam[];  // grad: Gamma_n [RP][RP]
    int k = 0;
    while (k + 1 < L.n && (int)blockIdx.x >= L.blk0[k + 1]) ++k;
    const double* __restrict__ part = L.j[k].part;
    const int nparts = L.j[k].nparts;
    const int64_t nout = L.j[k].nout;
    const int lane = threadIdx.x & 31, ws = threadIdx.x >> 5;
    const int64_t o = (int64_t)(blockIdx.x - L.blk0[k]) * 32 + lane;
    const GradEpi& G = L.ge;
    const int n = L.j[k].mode;
    if (L.grad && n >= 0) {  // Gamma_n, alongside the partial loads
        const int RR = G.RP * G.RP;
        for (int e = threadIdx.x; e < RR; e += blockDim.x) {
            double v = 1.0;
            for (int m = 0; m < G.order; ++m)
                if (m != n) v *= G.gram[(size_t)m * RR + e];
            gam[e] = v;
        }
    }
    double v = 0.0;
    if (o < nout)
        for (int c0 = ws; c0 < nparts; c0 += 8 * 8) {
            double x[8];  // loads batched ahead of the in-order adds
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = c0 + 8 * u;
                x[u] = c < nparts ? part[(int64_t)c * nout + o] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) v += x[u];
        }
    sl[ws][lane] = v;
    __syncthreads();
    if (ws != 0) {
        if (!L.grad) return;
    } else {
        double s = 0.0;
        if (o < nout) {
            for (int u = 0; u < 8; ++u) s += sl[u][lane];
            L.j[k].out[o] = s;
        }
        if (L.grad) {
            double g2 = 0.0, gd = 0.0, inner = 0.0;
            if (n >= 0 && o < nout) {
                int64_t i;
                int r;
                if (L.j[k].layout == 0) {
                    r = (int)(o / L.j[k].ld);
                    i = o % L.j[k].ld;
                } else {
                    r = (int)(o % G.RP);
                    i = o / G.RP;
                }
                const int64_t In = G.dims[n];
                if (r < G.R && i < In) {
                    const int64_t e = G.off[n] + (int64_t)r * In + i;
                    if (n == 0) inner = s * G.u[e];
                    if (G.need_grad) {
                        const double* a = G.u + G.off[n];
                        double av[kMaxRank];  // row i of A_n, loaded before the in-order dot product
#pragma unroll
                        for (int q = 0; q < kMaxRank; ++q) av[q] = q < G.R ? a[(int64_t)q * In + i] : 0.0;
                        double ag = 0.0;
#pragma unroll
                        for (int q = 0; q < kMaxRank; ++q)
                            if (q < G.R) ag += av[q] * gam[q * G.RP + r];
                        const double gv = -s + ag;
                        G.g[e] = gv;
                        g2 = gv * gv;
                        if (G.d) gd = gv * G.d[e];
                    }
                }
            }
            g2 = warp_sum(g2);
            gd = warp_sum(gd);
            inner = warp_sum(inner);
            if (lane == 0) {
                G.red[blockIdx.x * 3 + 0] = g2;
                G.red[blockIdx.x * 3 + 1] = gd;
                G.red[blockIdx.x * 3 + 2] = inner;
            }
        }
    }
    if (!L.grad) return;
    if (!last_block_arrives(G.counter)) return;
    // last block, all warps: thread-strided partial sums (loads batched), a fixed shuffle tree
    // per warp, then the warps in order
    double a = 0.0, b = 0.0, c = 0.0, fs = 0.0;
    for (int q0 = threadIdx.x; q0 < (int)gridDim.x; q0 += 256 * 4) {
        double x[4][3];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = q0 + 256 * u;
#pragma unroll
            for (int t = 0; t < 3; ++t) x[u][t] = q < (int)gridDim.x ? G.red[q * 3 + t] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a += x[u][0];
            b += x[u][1];
            c += x[u][2];
        }
    }
    for (int q = threadIdx.x; q < G.f_grid; q += 256) fs += G.f_part[q];
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    fs = warp_sum(fs);
    __shared__ double wr[4][8];
    if (lane == 0) {
        wr[0][ws] = a;
        wr[1][ws] = b;
        wr[2][ws] = c;
        wr[3][ws] = fs;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a = b = c = fs = 0.0;
        for (int w8 = 0; w8 < 8; ++w8) {
            a += wr[0][w8];
            b += wr[1][w8];
            c += wr[2][w8];
            fs += wr[3][w8];
        }
        G.sc->f = 0.5 * fs;
        G.sc->gnorm2 = a;
        G.sc->inner = c;
        if (G.d) G.sc->gdotd = b;
    }
}

void reduce_launch(RedLaunch& L, const RedJobs& jobs, size_t smem, cudaStream_t st) {
    L.n = jobs.n;
    int b = 0;
    for (int k = 0; k < jobs.n; ++k) {
        L.j[k] = jobs.j[k];
        L.blk0[k] = b;
        b += (int)((jobs.j[k].nout + 31) / 32);
    }
    L.blk0[jobs.n] = b;
    reduce_parts_kernel<<<(unsigned)b, 256, smem, st>>>(L);
    CPFIT_CUDA(cudaGetLastError());
}
void reduce_jobs(const RedJobs& jobs, cudaStream_t st) {
    if (jobs.n == 0) return;
    RedLaunch L{};
    reduce_launch(L, jobs, 0, st);
}

// defer_m / defer_s: append the partial reductions of M_h / Sout to a job list instead of
// launching them (reduce_jobs later, together with other reductions)
void run_level(const DevTensor& t, EvalWork& w, int h, const double* Sin, const double* u, bool do_m, bool do_s,
               double* Sout, cudaStream_t st, RedJobs* defer_m = nullptr, RedJobs* defer_s = nullptr,
               const double* Sd = nullptr, const double* beta = nullptr, const int* perm = nullptr,
               const double* sc0 = nullptr, double* m_final = nullptr) {
    if (!do_m && !do_s) return;
    LevelParams p{};
    p.Sin = Sin;
    p.Sd = Sd;
    p.beta = beta;
    p.perm = perm;
    p.sc0 = sc0;
    p.m_final = (m_final && do_m && !do_s && w.lvl_bulk[h]) ? m_final : nullptr;
    p.tile_cnt = w.lvl_cnt;
    p.Ih = t.dims[h];
    p.Jt = 1;
    for (int m = h + 1; m < t.order; ++m) p.Jt *= t.dims[m];
    p.R = w.R;
    p.Ah = do_s ? u + w.off[h] : nullptr;
    p.ntail = t.order - h - 1;
    for (int m = h + 1; m < t.order; ++m) {
        p.tdims[m - h - 1] = t.dims[m];
        p.tfac[m - h - 1] = u + w.off[m];
    }
    const int ny = w.lvl_ny[h];
    p.m_part = do_m ? w.lvl_part[h] : nullptr;
    p.s_out = do_s ? (ny > 1 ? w.lvl_spart[h] : Sout) : nullptr;
    p.spc = w.lvl_spc[h];
    if (w.lvl_bulk[h]) {
        // grid x over pair tiles (the Sout partials), y over slab ranges (the M partials)
        const dim3 grid((unsigned)ny, (unsigned)w.lvl_nx[h]);
        switch (w.RP) {
            case 8: launch_level_bulk<8>(p, grid, st); break;
            case 16: launch_level_bulk<16>(p, grid, st); break;
            default: launch_level_bulk<32>(p, grid, st); break;
        }
    } else {
        if (Sd || perm) throw std::logic_error("level: Sd / perm need the bulk level kernel");
        const dim3 grid((unsigned)w.lvl_nx[h], (unsigned)ny);
        switch (w.RP) {
            case 8: launch_level_rp<8>(p, grid, w.lvl_km[h], st); break;
            case 16: launch_level_rp<16>(p, grid, w.lvl_km[h], st); break;
            default: launch_level_rp<32>(p, grid, w.lvl_km[h], st); break;
        }
    }
    CPFIT_CUDA(cudaGetLastError());
    RedJobs own;
    RedJobs& jm = defer_m ? *defer_m : own;
    RedJobs& js = defer_s ? *defer_s : own;
    // job modes for the gradient epilogue: M_h is mode h; the last level's Sout is mode N-1
    const int smode = (h == t.order - 2) ? t.order - 1 : -1;
    if (do_m) jm.add(w.lvl_part[h], w.lvl_nx[h], p.Ih * w.RP, w.lvl_m[h], h);
    if (do_s && ny > 1) js.add(w.lvl_spart[h], ny, p.Jt * w.RP, Sout, smode);
    if (do_s && ny == 1 && defer_s) js.add(Sout, 1, p.Jt * w.RP, Sout, smode);  // in place: reads it once
    reduce_jobs(own, st);
}

// ---------------------------------------------------------------------------------------
// Grams in double-double (gram.cuh): blocks [blk0[n], blk0[n] + nblk[n]) own mode n's row
// tiles; the last block to finish combines the partials of modes [mode_lo, mode_hi).
// ---------------------------------------------------------------------------------------
struct GramParams {
    int order, R, RP, mode_lo, mode_hi;
    int64_t dims[kMaxOrder];
    const double* fac[kMaxOrder];
    int nchunk[kMaxOrder], chunk0[kMaxOrder];  // chunks per mode, prefix over all modes
    int64_t rows[kMaxOrder];                   // rows per chunk
    dd* part;     // [global chunk][npair]
    double* out;  // [mode][RP*RP]
    unsigned int* counter;
};

__global__ void __launch_bounds__(256) gram_kernel(const GramParams p) {
    const int npair = p.R * (p.R + 1) / 2;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    // tasks of modes [lo, hi) back to back
    int total = 0;
    for (int m = p.mode_lo; m < p.mode_hi; ++m) total += p.nchunk[m] * npair;
    for (int t = warp; t < total; t += nwarps) {
        int m = p.mode_lo, tl = t;
        while (tl >= p.nchunk[m] * npair) {
            tl -= p.nchunk[m] * npair;
            ++m;
        }
        gram_task(p.fac[m], p.dims[m], p.rows[m], p.R, tl, p.part + (size_t)p.chunk0[m] * npair);
    }
    if (!last_block_arrives(p.counter)) return;
    for (int m = p.mode_lo; m < p.mode_hi; ++m) gram_zero_pads(p.R, p.RP, p.out + (size_t)m * p.RP * p.RP);
    for (int f = threadIdx.x; f < (p.mode_hi - p.mode_lo) * npair; f += blockDim.x) {
        const int m = p.mode_lo + f / npair;
        gram_combine_pair(p.part + (size_t)p.chunk0[m] * npair, p.nchunk[m], f % npair, p.R, p.RP,
                          p.out + (size_t)m * p.RP * p.RP);
    }
}

void launch_gram(EvalWork& w, const double* u, int lo, int hi, cudaStream_t st) {
    GramParams p{};
    p.order = w.order;
    p.R = w.R;
    p.RP = w.RP;
    p.mode_lo = lo;
    p.mode_hi = hi;
    for (int n = 0; n < w.order; ++n) {
        p.dims[n] = w.dims[n];
        p.fac[n] = u + w.off[n];
        p.nchunk[n] = w.gram_nchunk[n];
        p.chunk0[n] = w.gram_chunk0[n];
        p.rows[n] = gram_chunk_rows(w.dims[n]);
    }
    p.part = w.gram_part;
    p.out = w.gram;
    p.counter = w.counter + kCounterGram;
    int tasks = 0;
    for (int n = lo; n < hi; ++n) tasks += w.gram_nchunk[n] * (w.R * (w.R + 1) / 2);
    const int grid = std::max(1, std::min((tasks + 7) / 8, 4 * sm_count()));
    gram_kernel<<<grid, 256, 0, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
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
    const double* norm_sq;  // device ||T||^2 (DevTensor::dscal + 1)
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
            for (int q0 = 0; q0 < p.R; q0 += kMaxRank) {  // one chunk for R <= 32, two above
                double av[kMaxRank];  // row i of A_n, loaded before the in-order dot product
#pragma unroll
                for (int q = 0; q < kMaxRank; ++q) av[q] = q0 + q < p.R ? a[(int64_t)(q0 + q) * In + i] : 0.0;
#pragma unroll
                for (int q = 0; q < kMaxRank; ++q)
                    if (q0 + q < p.R) ag += av[q] * gsm[n * RR + (q0 + q) * p.R + r];
            }
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
        p.sc->f = p.sparse ? 0.5 * *p.norm_sq - c + 0.5 * gs : 0.5 * fs;
        p.sc->gnorm2 = a;
        p.sc->inner = c;
        if (p.has_d) p.sc->gdotd = b;
        *p.counter = 0u;  // ready for the next evaluation (stream order)
    }
}

}  // namespace

// ---------------------------------------------------------------------------------------
// sparse hooks (sparse.cu)
void sparse_all_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st,
                      int skip_mode = -1);
// generic dense hooks (generic.cu)
void generic_all_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st,
                       int skip_mode = -1);
void generic_plan(const DevTensor& t, int RP, int n, int* gx, int64_t* cols_per_cta, int* gy);

// every mode's M_n (only_mode < 0) or one mode's into w.sp_part, for a rowwise tensor
void rowwise_modes(const DevTensor& t, EvalWork& w, const double* u, int only_mode, cudaStream_t st,
                   int skip_mode = -1) {
    if (generic_dense(t, w))
        generic_all_modes(t, w, u, only_mode, st, skip_mode);
    else
        sparse_all_modes(t, w, u, only_mode, st, skip_mode);
}

bool fiber_path_fits(int order, int64_t I0) {
    if (order < 2 || I0 < 1) return false;
    const int nchunk = (int)((I0 + 31) / 32);
    if (nchunk > 13) return false;
    for (int rp : {8, 16, 32})
        if (std::max(fiber_smem(rp, nchunk, I0, kFStages), spass_smem(rp, nchunk, I0, kFStages)) > 227 * 1024)
            return false;
    return true;
}

// ---------------------------------------------------------------------------------------

EvalWork* work_create(const DevTensor& t, int R) {
    if (R < 1 || R > kMaxRankWide) throw std::invalid_argument("device path supports 1 <= rank <= 64");
    auto* w = new EvalWork();
    // freed by work_destroy if a later allocation or shape check throws
    std::unique_ptr<EvalWork, void (*)(EvalWork*)> owner(w, work_destroy);
    w->R = R;
    // power of two: per-fiber lane groups; ranks above 32 (RP = 64) run the per-mode path
    w->RP = (R <= 8) ? 8 : (R <= 16 ? 16 : (R <= 32 ? 32 : 64));
    if (sizeof(double) * t.order * R * R > 220 * 1024)  // grad_kernel stages every Gamma_n
        throw std::invalid_argument("device path: order * rank^2 too large for the gradient epilogue");
    w->order = t.order;
    w->off[0] = 0;
    for (int n = 0; n < t.order; ++n) {
        w->dims[n] = t.dims[n];
        w->off[n + 1] = w->off[n] + t.dims[n] * R;
    }
    w->nu = w->off[t.order];
    if (w->nu >= ((int64_t)1 << 31)) throw std::invalid_argument("device path: R * sum(I_n) must be < 2^31");
    const int sms = sm_count();
    int chunks = 0;
    for (int n = 0; n < t.order; ++n) {
        w->gram_nchunk[n] = gram_chunks(t.dims[n]);
        w->gram_chunk0[n] = chunks;
        chunks += w->gram_nchunk[n];
    }
    CPFIT_CUDA(cudaMalloc(&w->gram_part, sizeof(dd) * (size_t)chunks * (R * (R + 1) / 2)));
    CPFIT_CUDA(cudaMalloc(&w->gram, sizeof(double) * (size_t)t.order * w->RP * w->RP));
    w->red_grid = sms * 2;
    CPFIT_CUDA(cudaMalloc(&w->red, sizeof(double) * 3 * (size_t)w->red_grid));
    if (!rowwise(t, *w)) {  // reduce_grad: one block per 32 outputs of M_0 .. M_{N-1}
        int64_t b = (w->RP * 32 * (int64_t)((t.dims[0] + 31) / 32) + 31) / 32;
        for (int n = 1; n < t.order; ++n) b += (t.dims[n] * w->RP + 31) / 32;
        w->rg_blocks = b;
        CPFIT_CUDA(cudaMalloc(&w->rg_red, sizeof(double) * 3 * (size_t)b));
    }
    // ALS solve Gram partials: <= 148 blocks per mode (als.cu solve_blocks)
    w->solve_part_stride = (int64_t)148 * (R * (R + 1) / 2);
    CPFIT_CUDA(cudaMalloc(&w->solve_part, sizeof(dd) * (size_t)t.order * w->solve_part_stride));
    CPFIT_CUDA(cudaMalloc(&w->nperm, sizeof(int) * kMaxRankWide));
    CPFIT_CUDA(cudaMalloc(&w->nscale0, sizeof(double) * kMaxRankWide));
    w->chol_stride = (int64_t)R * R + R + 1;
    CPFIT_CUDA(cudaMalloc(&w->chol, sizeof(double) * (size_t)t.order * w->chol_stride));
    CPFIT_CUDA(cudaStreamCreateWithFlags(&w->side, cudaStreamNonBlocking));
    CPFIT_CUDA(cudaEventCreateWithFlags(&w->ev_fork, cudaEventDisableTiming));
    CPFIT_CUDA(cudaEventCreateWithFlags(&w->ev_join, cudaEventDisableTiming));
    CPFIT_CUDA(cudaEventCreateWithFlags(&w->ev_gram, cudaEventDisableTiming));
    CPFIT_CUDA(cudaMalloc(&w->counter, sizeof(unsigned int) * kCounters));
    CPFIT_CUDA(cudaMemset(w->counter, 0, sizeof(unsigned int) * kCounters));
    CPFIT_CUDA(cudaMalloc(&w->lvl_cnt, sizeof(unsigned int) * kLvlCounters));
    CPFIT_CUDA(cudaMemset(w->lvl_cnt, 0, sizeof(unsigned int) * kLvlCounters));
    if (!rowwise(t, *w)) {
        if (t.order < 2) throw std::invalid_argument("device dense path needs order >= 2");
        const int I0 = (int)t.dims[0];
        w->fiber_nchunk = (I0 + 31) / 32;
        if (w->fiber_nchunk > 13) throw std::invalid_argument("device dense path supports I_1 <= 416");
        // short fibres: a deep T ring (a 16-fibre tile of I0 <= 128 is <= 17 KB; three of them do
        // not cover the HBM latency at one CTA per SM)
        w->fiber_nst = kFStages;
        if (w->fiber_nchunk <= 4 &&
            std::max(fiber_smem(w->RP, w->fiber_nchunk, I0, kDeepFStages),
                     spass_smem(w->RP, w->fiber_nchunk, I0, kDeepFStages)) <= 220 * 1024)
            w->fiber_nst = kDeepFStages;
        w->fiber_smem = fiber_smem(w->RP, w->fiber_nchunk, I0, w->fiber_nst);
        {  // S pass without K split when a warp's register-held A0 fragments cover the whole fibre
            const int nrt = w->RP / 8, kmax = w->RP == 8 ? SRegRoles<8>::KMAX : SRegRoles<16>::KMAX;
            w->sreg_groups = 0;
            if (w->RP <= 16 && t.ldT / 4 <= kmax && w->fiber_nst == kDeepFStages)
                for (int ng = CPFIT_SREG_WARPS / nrt; ng >= 2; --ng)
                    if (w->fiber_nst % ng == 0) {
                        w->sreg_groups = ng;
                        break;
                    }
        }
        {
            const int pitch_fws = 32 * w->fiber_nchunk + 4, pitch_sreg = sreg_pitch(t.ldT);
            if (w->fiber_nst == kDeepFStages && pitch_fws <= 256 && pitch_sreg <= 256 && t.J < ((int64_t)1 << 31)) {
                using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                              CUtensorMapFloatOOBfill);
                void* fn = nullptr;
                cudaDriverEntryPointQueryResult q{};
                if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                    q == cudaDriverEntryPointSuccess && fn) {
                    auto encode = reinterpret_cast<EncodeFn>(fn);
                    const cuuint64_t gdim[2] = {(cuuint64_t)t.ldT, (cuuint64_t)t.J};
                    const cuuint64_t gstride[1] = {(cuuint64_t)t.ldT * sizeof(double)};
                    const cuuint32_t estride[2] = {1, 1};
                    auto make = [&](CUtensorMap* m, int pitch) {
                        const cuuint32_t box[2] = {(cuuint32_t)pitch, (cuuint32_t)w->fiber_F};
                        return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)t.T, gdim, gstride, box, estride,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
                    };
                    w->fiber_tmap = make(&w->tmap_fws, pitch_fws) && make(&w->tmap_sreg, pitch_sreg);
                } else {
                    (void)cudaGetLastError();
                }
            }
        }
        if (std::max(w->fiber_smem, spass_smem(w->RP, w->fiber_nchunk, I0, w->fiber_nst)) > 227 * 1024)
            throw std::invalid_argument("fiber tile does not fit shared memory");
        const int64_t ntiles = (t.J + w->fiber_F - 1) / w->fiber_F;
        // resident CTAs per SM: threads, shared memory and registers (128 per thread)
        const int per_sm = std::max(1, std::min({2048 / fiber_threads(w->RP), 65536 / (128 * fiber_threads(w->RP)),
                                                 (int)((228 * 1024) / (w->fiber_smem + 1024))}));
        w->fiber_grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
        // order 3: room for the line search's S_d right after S
        const size_t sn = (size_t)t.J * w->RP;
        CPFIT_CUDA(cudaMalloc(&w->S, sizeof(double) * sn * (t.order <= 4 ? 2 : 1)));
        if (t.order == 3 || t.order == 4) w->S2 = w->S + sn;
        CPFIT_CUDA(cudaMalloc(&w->m0_part, sizeof(double) * (size_t)w->fiber_grid * w->RP * 32 * w->fiber_nchunk));
        // rows >= 8 ceil(I0 / 8) of the partials are never written: keep them zero
        CPFIT_CUDA(cudaMemset(w->m0_part, 0, sizeof(double) * (size_t)w->fiber_grid * w->RP * 32 * w->fiber_nchunk));
        CPFIT_CUDA(cudaMalloc(&w->m0, sizeof(double) * (size_t)w->RP * 32 * w->fiber_nchunk));
        CPFIT_CUDA(cudaMalloc(&w->f_part, sizeof(double) * (size_t)w->fiber_grid));
        for (int h = 1; h < t.order - 1; ++h) {
            int64_t Jt = 1;
            for (int m = h + 1; m < t.order; ++m) Jt *= t.dims[m];
            const int64_t npairs = t.dims[h] * w->RP;
            if (h == t.order - 2) {  // one tail factor: the bulk-copy kernel
                w->lvl_bulk[h] = true;
                w->lvl_ny[h] = (int)((npairs + kBulkPairs - 1) / kBulkPairs);
                w->lvl_nx[h] = (int)((Jt + kBulkSlabs - 1) / kBulkSlabs);
                w->lvl_spc[h] = kBulkSlabs;
            } else {
                const int64_t need = (npairs + kLevelThreads - 1) / kLevelThreads;
                w->lvl_km[h] = need <= 4 ? 4 : need <= 8 ? 8 : 16;
                w->lvl_ny[h] =
                    (int)((npairs + (int64_t)kLevelThreads * w->lvl_km[h] - 1) / (kLevelThreads * w->lvl_km[h]));
                const int64_t nx_want =
                    std::max<int64_t>(1, std::min<int64_t>(Jt, (2 * sms + w->lvl_ny[h] - 1) / w->lvl_ny[h]));
                w->lvl_spc[h] = (Jt + nx_want - 1) / nx_want;
                w->lvl_nx[h] = (int)((Jt + w->lvl_spc[h] - 1) / w->lvl_spc[h]);
            }
            CPFIT_CUDA(cudaMalloc(&w->lvl_part[h], sizeof(double) * (size_t)w->lvl_nx[h] * npairs));
            CPFIT_CUDA(cudaMalloc(&w->lvl_m[h], sizeof(double) * (size_t)npairs));
            CPFIT_CUDA(cudaMalloc(&w->lvl_S[h], sizeof(double) * (size_t)Jt * w->RP));
            if (w->lvl_ny[h] > 1)
                CPFIT_CUDA(cudaMalloc(&w->lvl_spart[h], sizeof(double) * (size_t)w->lvl_ny[h] * Jt * w->RP));
        }
    } else {
        int64_t tot = 0;
        for (int n = 0; n < t.order; ++n) tot += t.dims[n] * w->RP;
        CPFIT_CUDA(cudaMalloc(&w->sp_part, sizeof(double) * (size_t)tot));
        w->m0_rowwise = true;
        CPFIT_CUDA(cudaMalloc(&w->frows, sizeof(double) * (size_t)tot));
        if (generic_dense(t, *w)) {
            int64_t most = 1;
            for (int n = 0; n < t.order; ++n) {
                int gx, gy;
                int64_t cpc;
                generic_plan(t, w->RP, n, &gx, &cpc, &gy);
                most = std::max<int64_t>(most, (int64_t)gx * t.dims[n] * w->RP);
                if (n == 0) w->gen_fgrid = gx * gy;
            }
            CPFIT_CUDA(cudaMalloc(&w->gen_part, sizeof(double) * (size_t)most));
        }
        CPFIT_CUDA(cudaMalloc(&w->f_part, sizeof(double) * (size_t)std::max(4, w->gen_fgrid)));
    }
    return owner.release();
}

void work_destroy(EvalWork* w) {
    if (!w) return;
    cudaFree(w->gram_part);
    cudaFree(w->gram);
    cudaFree(w->red);
    cudaFree(w->rg_red);
    cudaFree(w->S);
    cudaFree(w->m0_part);
    cudaFree(w->m0);
    cudaFree(w->f_part);
    cudaFree(w->sp_part);
    cudaFree(w->frows);
    cudaFree(w->gen_part);
    cudaFree(w->counter);
    cudaFree(w->lvl_cnt);
    cudaFree(w->chol);
    cudaFree(w->solve_part);
    cudaFree(w->nperm);
    cudaFree(w->nscale0);
    if (w->ev_fork) cudaEventDestroy(w->ev_fork);
    if (w->ev_join) cudaEventDestroy(w->ev_join);
    if (w->ev_gram) cudaEventDestroy(w->ev_gram);
    if (w->side) cudaStreamDestroy(w->side);
    for (int h = 0; h < kMaxOrder; ++h) {
        cudaFree(w->lvl_part[h]);
        cudaFree(w->lvl_m[h]);
        cudaFree(w->lvl_S[h]);
        cudaFree(w->lvl_spart[h]);
    }
    delete w;
}

void grams_device(EvalWork& w, const double* u, cudaStream_t st) { launch_gram(w, u, 0, w.order, st); }

void gram_mode_device(EvalWork& w, const double* u, int mode, cudaStream_t st) {
    launch_gram(w, u, mode, mode + 1, st);
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
    if (rowwise(t, w)) {
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
    p.f_grid = t.sparse ? 0 : (generic_dense(t, w) ? w.gen_fgrid : w.fiber_grid);
    p.sparse = t.sparse ? 1 : 0;
    p.norm_sq = t.dscal + 1;
    p.sc = sc;
    p.has_d = d ? 1 : 0;
    p.counter = w.counter + kCounterGrad;
    // enough blocks to cover n_u once (latency-bound epilogue, no grid-stride tail)
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(w.red_grid, (w.nu + 255) / 256));
    const size_t gsmem = sizeof(double) * t.order * w.R * w.R;  // > 48 KB only for ranks above 32
    if (gsmem > 48 * 1024)
        CPFIT_CUDA(cudaFuncSetAttribute(grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
    grad_kernel<<<blocks, 256, gsmem, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
}
}  // namespace

namespace {
// the deferred reductions of a dense evaluation (M_0 .. M_{N-1}) with the gradient epilogue
void reduce_grad(const DevTensor& t, EvalWork& w, const RedJobs& jobs, const double* u, double* g,
                 const double* d, bool need_grad, EvalScalars* sc, cudaStream_t st) {
    if (jobs.blocks() > w.rg_blocks) throw std::logic_error("reduce_grad: block partial buffer too small");
    RedLaunch L{};
    L.grad = 1;
    GradEpi& G = L.ge;
    G.order = t.order;
    G.R = w.R;
    G.RP = w.RP;
    G.need_grad = need_grad ? 1 : 0;
    for (int n = 0; n < t.order; ++n) {
        G.dims[n] = t.dims[n];
        G.off[n] = w.off[n];
    }
    G.off[t.order] = w.off[t.order];
    G.u = u;
    G.g = g;
    G.d = d;
    G.gram = w.gram;
    G.f_part = w.f_part;
    G.f_grid = w.fiber_grid;
    G.sc = sc;
    G.red = w.rg_red;
    G.counter = w.counter + kCounterGrad;
    reduce_launch(L, jobs, sizeof(double) * w.RP * w.RP, st);
}
}  // namespace

void eval_device(const DevTensor& t, EvalWork& w, const double* u, double* g, EvalScalars* sc, const double* d,
                 int* status, cudaStream_t st, bool need_grad, const int* resid_flag, bool s_given, bool grams_given,
                 cudaEvent_t grad_dep, int rowwise_skip) {
    (void)status;
    if (!grams_given) grams_device(w, u, st);
    if (!rowwise(t, w)) {
        // fused pass: S, M0 partials and per-fiber objective — or, when w.S already holds
        // T x_1 A0(u), M0 and the objective only (no S contraction)
        if (s_given)
            run_fiber(t, w, u, false, true, true, w.gram, st, resid_flag, nullptr, w.S);
        else
            run_fiber(t, w, u, true, true, true, w.gram /* mode-0 Gram */, st, resid_flag);
        // modes 1..N-1 from S; the partial sums of M0, the M_h and the last level's Sout in one
        // reduction launch
        RedJobs jobs;
        add_m0_job(w, jobs);
        const double* Sin = w.S;
        for (int h = 1; h < t.order - 1; ++h) {
            run_level(t, w, h, Sin, u, true, true, w.lvl_S[h], st, &jobs, h == t.order - 2 ? &jobs : nullptr);
            Sin = w.lvl_S[h];
        }
        if (t.order >= 3) {
            if (grad_dep) CPFIT_CUDA(cudaStreamWaitEvent(st, grad_dep, 0));
            reduce_grad(t, w, jobs, u, g, d, need_grad, sc, st);
            return;
        }
        reduce_jobs(jobs, st);
    } else {
        // s_given for a rowwise tensor: M_{N-1} at u is already in w.sp_part (the deferred ALS
        // sweep's last mode, computed from the same factors of modes 0 .. N-2)
        rowwise_modes(t, w, u, -1, st, rowwise_skip >= 0 ? rowwise_skip : (s_given ? t.order - 1 : -1));
        if (grad_dep) CPFIT_CUDA(cudaStreamWaitEvent(st, grad_dep, 0));
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

namespace {
// Order-3 MTTKRP of the last mode from S = T x_1 A0 ([J][RP] row-major, fibre f = j + I1 k):
//   M2[k][r] = sum_j S[j + I1 k][r] A1[j][r]: one CTA per k (its slab of S is contiguous), the
//     256 / RP j-lanes of each r combined in order, written straight to the col-major output
//     (one kernel instead of the bulk level kernel + gather; mode 1 keeps the level kernel,
//     whose bulk copies hide the S latency better than a second kernel of this form did)
constexpr int kM3Threads = 512, kM3Batch = 16;
// A1 is staged in shared memory as [j][RP + 1] from a coalesced read of the col-major factor: a
// direct load of A1[j][r] by lane (r, j) touches RP separate 128-byte lines per instruction and
// the L1 wavefronts, not the bytes, then bound the kernel
template <int RP>
__global__ void __launch_bounds__(kM3Threads) mttkrp3_last_kernel(const double* __restrict__ S,
                                                                  const double* __restrict__ A1, int I1, int I2, int R,
                                                                  double* out) {
    constexpr int JL = kM3Threads / RP, LD = RP + 1;
    extern __shared__ double a_s[];
    __shared__ double red[kM3Threads];
    const int tid = threadIdx.x, r = tid % RP, jl = tid / RP;
    const int k = blockIdx.x;
    const double* Sk = S + (int64_t)k * I1 * RP;
    // the slab's first batch of S loads goes out before the staging
    double x[kM3Batch];
#pragma unroll
    for (int q = 0; q < kM3Batch; ++q) {
        const int j = jl + q * JL;
        x[q] = j < I1 ? Sk[j * RP + r] : 0.0;
    }
    for (int e = tid; e < I1 * RP; e += kM3Threads) {
        const int rr = e / I1, j = e - rr * I1;
        a_s[j * LD + rr] = rr < R ? A1[e] : 0.0;
    }
    __syncthreads();
    double acc0 = 0.0, acc1 = 0.0;
    for (int j0 = jl;;) {
#pragma unroll
        for (int q = 0; q < kM3Batch; q += 2) {
            const int j = j0 + q * JL;
            if (j < I1) acc0 = fma(x[q], a_s[j * LD + r], acc0);
            if (j + JL < I1) acc1 = fma(x[q + 1], a_s[(j + JL) * LD + r], acc1);
        }
        j0 += kM3Batch * JL;
        if (j0 >= I1) break;
#pragma unroll
        for (int q = 0; q < kM3Batch; ++q) {
            const int j = j0 + q * JL;
            x[q] = j < I1 ? Sk[j * RP + r] : 0.0;
        }
    }
    red[tid] = acc0 + acc1;
    __syncthreads();
    if (tid < R) {
        double v = 0.0;
#pragma unroll 8
        for (int q = 0; q < JL; ++q) v += red[q * RP + tid];
        out[(int64_t)tid * I2 + k] = v;
    }
}

// the kernel's A1 copy fits shared memory (and the slab index math 32 bits)
inline bool mttkrp3_fits(int64_t I1, int64_t I2, int RP) {
    return (size_t)I1 * (RP + 1) * sizeof(double) <= 160 * 1024 && I1 * I2 * RP < (int64_t)1 << 31;
}

template <int RP>
void launch_mttkrp3_last(const EvalWork& w, const double* u, double* out, cudaStream_t st) {
    static bool attr = [] {
        cudaFuncSetAttribute(mttkrp3_last_kernel<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        return true;
    }();
    (void)attr;
    const size_t smem = sizeof(double) * (size_t)w.dims[1] * (RP + 1);
    mttkrp3_last_kernel<RP><<<(unsigned)w.dims[2], kM3Threads, smem, st>>>(w.S, u + w.off[1], (int)w.dims[1],
                                                                           (int)w.dims[2], w.R, out);
    CPFIT_CUDA(cudaGetLastError());
}
}  // namespace

// measurement hook: the last-mode contraction alone, from the S left by the previous pass
void mttkrp3_last_only(EvalWork& w, const double* u, double* out, cudaStream_t st) {
    switch (w.RP) {
        case 8: launch_mttkrp3_last<8>(w, u, out, st); break;
        case 16: launch_mttkrp3_last<16>(w, u, out, st); break;
        default: launch_mttkrp3_last<32>(w, u, out, st); break;
    }
}

void mttkrp_device(const DevTensor& t, EvalWork& w, const double* u, int mode, double* out, cudaStream_t st) {
    const int64_t In = t.dims[mode];
    const int blocks = (int)std::min<int64_t>(1024, (In * w.R + 255) / 256);
    if (rowwise(t, w)) {
        rowwise_modes(t, w, u, mode, st);
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
        if (t.order == 3 && mode == 2 && mttkrp3_fits(t.dims[1], t.dims[2], w.RP)) {
            switch (w.RP) {
                case 8: launch_mttkrp3_last<8>(w, u, out, st); break;
                case 16: launch_mttkrp3_last<16>(w, u, out, st); break;
                default: launch_mttkrp3_last<32>(w, u, out, st); break;
            }
            return;
        }
        const double* Sin = w.S;
        // the level that produces M_mode leaves its per-CTA partials to the gather (one launch
        // fewer): M_h partials [slab range][i][r] at h = mode < N-1, the last level's Sout
        // partials [pair tile][slab][r] for mode N-1
        RedJobs skip;
        const double* part = w.S;  // order 2: M_1 = S
        int nparts = 1;
        for (int h = 1; h <= mode && h < t.order - 1; ++h) {
            const bool last = (h == mode);
            const bool final = last || h == t.order - 2;
            // the bulk last level can finish M_mode itself (no gather launch)
            const bool fin = last && w.lvl_bulk[h] && w.lvl_ny[h] <= kLvlCounters;
            run_level(t, w, h, Sin, u, last, !last, w.lvl_S[h], st, final ? &skip : nullptr, final ? &skip : nullptr,
                      nullptr, nullptr, nullptr, nullptr, fin ? out : nullptr);
            if (fin) return;
            Sin = w.lvl_S[h];
            if (final) {
                if (last) {
                    part = w.lvl_part[h];
                    nparts = w.lvl_nx[h];
                } else {
                    part = w.lvl_ny[h] > 1 ? w.lvl_spart[h] : w.lvl_S[h];
                    nparts = w.lvl_ny[h];
                }
            }
        }
        gather_m_kernel<<<blocks, 256, 0, st>>>(In, w.R, w.RP, part, nparts, 0, 1, out);
    }
    CPFIT_CUDA(cudaGetLastError());
}

// exported for poly.cu
void dense_s_pass(const DevTensor& t, EvalWork& w, const double* u, double* S_out, cudaStream_t st) {
    run_fiber(t, w, u, true, false, false, nullptr, st, nullptr, S_out);
}
void eval_given_s_device(const DevTensor& t, EvalWork& w, const double* u, double* g, EvalScalars* sc,
                         cudaStream_t st, const double* Sd, const double* beta, bool grams_given, const int* perm,
                         const double* sc0) {
    if (!grams_given) grams_device(w, u, st);
    run_fiber(t, w, u, false, true, false, nullptr, st);  // M0 only
    RedJobs jobs;
    add_m0_job(w, jobs);
    const double* Sin = w.S;
    for (int h = 1; h < t.order - 1; ++h) {
        run_level(t, w, h, Sin, u, true, true, w.lvl_S[h], st, &jobs, h == t.order - 2 ? &jobs : nullptr,
                  h == 1 ? Sd : nullptr, beta, h == 1 ? perm : nullptr, sc0);
        Sin = w.lvl_S[h];
    }
    reduce_grad(t, w, jobs, u, g, nullptr, true, sc, st);
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
// defer: leave the partial sums to the caller (the ALS solves read them directly)
void dense_level(const DevTensor& t, EvalWork& w, int h, const double* Sin, const double* u, bool do_m, bool do_s,
                 double* Sout, cudaStream_t st, bool defer) {
    RedJobs discard;
    run_level(t, w, h, Sin, u, do_m, do_s, Sout, st, defer ? &discard : nullptr, defer ? &discard : nullptr);
}
void gather_m(int64_t In, EvalWork& w, const double* part, int grid, int ld, int layout, double* out,
              cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(1024, (In * w.R + 255) / 256);
    gather_m_kernel<<<blocks, 256, 0, st>>>(In, w.R, w.RP, part, grid, ld, layout, out);
    CPFIT_CUDA(cudaGetLastError());
}

}  // namespace cpfit_gpu
