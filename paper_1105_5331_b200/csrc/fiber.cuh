// Warp-specialized fiber pass (included by dense.cu inside cpfit_gpu::(anonymous)).
//
// One CTA per SM streams a contiguous range of F-fiber tiles of T (mode-0 fibers, padded to
// ldT doubles) through a kFStages-deep shared-memory ring. Roles:
//   warp 0                 producer: one bulk async copy per fiber into the ring (mbarrier
//                          complete_tx), and the W tile (Khatri-Rao rows of modes >= 1,
//                          never materialised in HBM) into a double-buffered smem tile — the
//                          factor gathers are independent and issued back to back, and run
//                          ahead of the consumers instead of on their critical path;
//   warps 1 .. NC          compute: each owns 32 rows i of the fiber; per tile it runs
//                            S^T partial (F x RP)  = T(rows, F)^T A0(rows, :)   DMMA m8n8k4
//                            M0^T      (RP x 32)  += W(F, :)^T T(rows, F)^T     DMMA m8n8k4
//                          (+ model(rows, F) = A0 W^T and the squared residual in the
//                          residual-objective mode), with the M0 accumulators held in
//                          registers for the whole pass;
//   warps NC+1, NC+2       epilogue: sum the NC per-warp S partials (fixed order), store S,
//                          and fold the per-fiber objective ||t||^2 - 2 w.s + w^T G0 w
//                          (G0 w on DMMA, per-fiber sums by lane shuffles).
// Hand-offs are mbarrier phases only; there is no CTA-wide barrier in the steady state.
// Shared-memory fragment layouts: T rows padded to I0s = 32 NC + 4 doubles and W rows to
// RP + 4 doubles (both 4 or 12 mod 16), which makes every DMMA operand load conflict free.
#pragma once

constexpr int kFStages = 3;
constexpr int kEpiWarps = 2;
constexpr int kFiberF = 16;  // fibers per tile (2 DMMA m-tiles; one per epilogue warp)

template <int RP>
__host__ __device__ constexpr int w_ld() {
    return RP + 4;
}

struct FiberSmem {
    size_t tiles, spart, wbuf, gam, bars, total;
};

template <int RP, int F>
__host__ __device__ FiberSmem fiber_layout(int nchunk) {
    const int I0s = 32 * nchunk + 4;
    FiberSmem s{};
    size_t off = 0;
    s.tiles = off;
    off += sizeof(double) * (size_t)kFStages * F * I0s;
    s.spart = off;
    off += sizeof(double) * 2 * (size_t)nchunk * F * RP;
    s.wbuf = off;
    off += sizeof(double) * 2 * (size_t)F * w_ld<RP>();
    s.gam = off;
    off += sizeof(double) * (size_t)RP * RP;
    s.bars = off;
    off += sizeof(uint64_t) * 16;
    s.total = off;
    return s;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Multi-index (modes >= 1) of fiber `fib`, as offsets into each mode's factor column.
// ORD is the tensor order when specialised (2, 3, 4), 0 for the generic path; all loops over
// modes run to a compile-time bound so the index lives in registers and the factor gathers
// issue back to back.
template <int ORD>
struct FiberIndex {
    int j[ORD > 0 ? ORD : kMaxOrder];
    bool valid;
};
template <int ORD>
__device__ __forceinline__ bool mode_active(const FiberParams& p, int m) {
    return ORD > 0 ? true : (m < p.order);
}
// full decode (64-bit divisions): once per CTA
template <int ORD>
__device__ __forceinline__ FiberIndex<ORD> decode_fiber(const FiberParams& p, int64_t fib) {
    FiberIndex<ORD> x;
    x.valid = fib < p.J;
    int64_t rem = x.valid ? fib : 0;
#pragma unroll
    for (int m = 1; m < (ORD > 0 ? ORD : kMaxOrder); ++m) {
        x.j[m] = 0;
        if (mode_active<ORD>(p, m)) {
            const int64_t d = p.dims[m];
            const int64_t q = rem / d;
            x.j[m] = (int)(rem - q * d);
            rem = q;
        }
    }
    return x;
}
// x advanced by delta fibers (first mode >= 1 fastest), carries without 64-bit division
template <int ORD>
__device__ __forceinline__ FiberIndex<ORD> advance_fiber(const FiberParams& p, FiberIndex<ORD> x, int delta,
                                                         int64_t fib) {
    x.valid = fib < p.J;
    int carry = delta;
#pragma unroll
    for (int m = 1; m < (ORD > 0 ? ORD : kMaxOrder); ++m) {
        if (mode_active<ORD>(p, m)) {
            const int d = (int)p.dims[m];
            int v = x.j[m] + carry;
            carry = 0;
            if (v >= d) {
                carry = v / d;
                v -= carry * d;
            }
            x.j[m] = v;
        }
    }
    return x;
}

template <int RP, int F, bool A0REG, int ORD>
__global__ void __launch_bounds__(512) fiber_ws_kernel(const FiberParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int NRT = RP / 8;
    constexpr int WLD = w_ld<RP>();
    static_assert(F == 16, "two epilogue warps cover two 8-fiber m-tiles");
    const FiberSmem L = fiber_layout<RP, F>(p.nchunk);
    const int NC = p.nchunk;
    const int I0s = p.I0s;
    double* tiles = reinterpret_cast<double*>(smem_raw + L.tiles);
    double* spart = reinterpret_cast<double*>(smem_raw + L.spart);  // [2][NC][F][RP]
    double* wbuf = reinterpret_cast<double*>(smem_raw + L.wbuf);    // [2][F][WLD]
    double* gam = reinterpret_cast<double*>(smem_raw + L.gam);      // [RP][RP]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bars);
    uint64_t* tfull = bars;        // [kFStages] tx bytes
    uint64_t* tempty = bars + 3;   // [kFStages] NC arrivals
    uint64_t* sfull = bars + 6;    // [2] NC
    uint64_t* sempty = bars + 8;   // [2] kEpiWarps
    uint64_t* wfull = bars + 10;   // [2] producer
    uint64_t* wempty = bars + 12;  // [2] NC (+ kEpiWarps for the per-fiber objective)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t_begin = (int64_t)blockIdx.x * p.tiles_per_cta;
    const int64_t t_end = imin64(p.ntiles, t_begin + p.tiles_per_cta);
    const int64_t ntl = t_end > t_begin ? t_end - t_begin : 0;
    // objective form: residual 1/2 sum (T - model)^2 (kruskal.cpp:83-102) when requested,
    // else the per-fiber three-term form folded by the epilogue
    const bool resid = p.do_f && p.resid_flag && *p.resid_flag;
    const bool need_w = p.do_m0 || p.do_f;
    const bool epi_w = p.do_f && !resid;  // epilogue reads W
    dd racc{0.0, 0.0};

    for (int64_t e = tid; e < (int64_t)kFStages * F * I0s; e += blockDim.x) tiles[e] = 0.0;
    if (p.do_f)
        for (int e = tid; e < RP * RP; e += blockDim.x) gam[e] = p.gamma0[e];
    if (tid == 0) {
        for (int s = 0; s < kFStages; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], NC);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sfull[b], NC);
            mbar_init(&sempty[b], kEpiWarps);
            mbar_init(&wfull[b], 1);
            mbar_init(&wempty[b], NC + (epi_w ? kEpiWarps : 0));
        }
    }
    mbar_fence_init();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    double facc = 0.0;
    if (warp == 0) {
        // ---------------- producer ----------------
        // W lane mapping: fiber f = lane % F, r-slice h = lane / F (RS = RP / 2 values)
        constexpr int RS = RP * F / 32;
        const int fw = lane % F, hw = lane / F;
        FiberIndex<ORD> xw = decode_fiber<ORD>(p, t_begin * F + fw);
        for (int64_t k = 0; k < ntl; ++k) {
            const int64_t t = t_begin + k;
            const int s = (int)(k % kFStages);
            const int64_t f0 = t * F;
            if (k >= kFStages) mbar_wait(&tempty[s], (uint32_t)(((k / kFStages) - 1) & 1));
            const int nvalid = (int)imin64(F, p.J - f0);
            double* st = tiles + (size_t)s * F * I0s;
            if (nvalid < F)
                for (int e = lane; e < (F - nvalid) * I0s; e += 32) st[(size_t)nvalid * I0s + e] = 0.0;
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_expect_tx(&tfull[s], (uint32_t)(nvalid * p.ldT * 8));
                for (int f = 0; f < nvalid; ++f)
                    bulk_g2s(st + (size_t)f * I0s, p.T + (f0 + f) * p.ldT, (uint32_t)(p.ldT * 8), &tfull[s]);
            }
            if (need_w) {
                const int b = (int)(k & 1);
                if (k > 0) xw = advance_fiber<ORD>(p, xw, F, f0 + fw);
                // gathers first (independent), then wait for the buffer
                double w[RS];
#pragma unroll
                for (int j = 0; j < RS; ++j) {
                    const int r = hw * RS + j;
                    const bool ok = xw.valid && r < p.R;
                    double v = ok ? 1.0 : 0.0;
#pragma unroll
                    for (int m = 1; m < (ORD > 0 ? ORD : kMaxOrder); ++m)
                        if (ok && mode_active<ORD>(p, m)) v *= __ldg(p.fac[m] + (int64_t)r * p.dims[m] + xw.j[m]);
                    w[j] = v;
                }
                if (k >= 2) mbar_wait(&wempty[b], (uint32_t)(((k / 2) - 1) & 1));
                double* wv = wbuf + (size_t)b * F * WLD;
#pragma unroll
                for (int j = 0; j < RS; ++j) wv[fw * WLD + hw * RS + j] = w[j];
                __syncwarp();
                if (lane == 0) mbar_arrive(&wfull[b]);
            }
        }
    } else if (warp <= NC) {
        // ---------------- compute ----------------
        const int c = warp - 1;
        double a0f[A0REG ? 8 : 1][A0REG ? NRT : 1];
        auto a0_at = [&](int ks, int rt) -> double {
            const int i = c * 32 + ks * 4 + (lane & 3);
            const int r = rt * 8 + (lane >> 2);
            return (i < p.I0 && r < p.R) ? __ldg(p.A0 + (int64_t)r * p.I0 + i) : 0.0;
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
        for (int64_t k = 0; k < ntl; ++k) {
            const int s = (int)(k % kFStages);
            const int b = (int)(k & 1);
            mbar_wait(&tfull[s], (uint32_t)((k / kFStages) & 1));
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
                        const double bb = A0REG ? a0f[A0REG ? ks : 0][A0REG ? rt : 0] : a0_at(ks, rt);
#pragma unroll
                        for (int ft = 0; ft < F / 8; ++ft) dmma_8x8x4(sacc[ft][rt][0], sacc[ft][rt][1], a[ft], bb);
                    }
                }
                if (k >= 2) mbar_wait(&sempty[b], (uint32_t)(((k / 2) - 1) & 1));
                double* sp = spart + ((size_t)b * NC + c) * F * RP;
#pragma unroll
                for (int ft = 0; ft < F / 8; ++ft)
#pragma unroll
                    for (int rt = 0; rt < NRT; ++rt) {
                        const int f = ft * 8 + (lane >> 2), r = rt * 8 + 2 * (lane & 3);
                        *reinterpret_cast<double2*>(sp + f * RP + r) = make_double2(sacc[ft][rt][0], sacc[ft][rt][1]);
                    }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sfull[b]);
            }
            if (need_w) {
                mbar_wait(&wfull[b], (uint32_t)((k / 2) & 1));
                const double* wv = wbuf + (size_t)b * F * WLD;
                if (p.do_m0) {
#pragma unroll
                    for (int kf = 0; kf < F / 4; ++kf) {
                        const int f = kf * 4 + (lane & 3);
                        double wa[NRT];
#pragma unroll
                        for (int rt = 0; rt < NRT; ++rt) wa[rt] = wv[f * WLD + rt * 8 + (lane >> 2)];
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) {
                            const double bb = tt[f * I0s + c * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
                            for (int rt = 0; rt < NRT; ++rt) dmma_8x8x4(macc[rt][nt][0], macc[rt][nt][1], wa[rt], bb);
                        }
                    }
                }
                if (resid) {
                    // model(i, f) = sum_r A0(i, r) W(f, r) for this warp's 32 rows on DMMA,
                    // then the squared residual against the tile (padding is 0 - 0)
                    double tsum = 0.0;
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) {
                        const int i = c * 32 + mt * 8 + (lane >> 2);
                        double a0r[RP / 4];
#pragma unroll
                        for (int kr = 0; kr < RP / 4; ++kr) {
                            const int r = kr * 4 + (lane & 3);
                            a0r[kr] = (i < p.I0 && r < p.R) ? __ldg(p.A0 + (int64_t)r * p.I0 + i) : 0.0;
                        }
#pragma unroll
                        for (int nt = 0; nt < F / 8; ++nt) {
                            double d0 = 0.0, d1 = 0.0;
#pragma unroll
                            for (int kr = 0; kr < RP / 4; ++kr)
                                dmma_8x8x4(d0, d1, a0r[kr], wv[(nt * 8 + (lane >> 2)) * WLD + kr * 4 + (lane & 3)]);
                            const int f = nt * 8 + 2 * (lane & 3);
                            const double r0 = tt[f * I0s + i] - d0;
                            const double r1 = tt[(f + 1) * I0s + i] - d1;
                            tsum += r0 * r0 + r1 * r1;
                        }
                    }
                    racc = dd_add(racc, dd{tsum, 0.0});
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&tempty[s]);
                if (need_w) mbar_arrive(&wempty[b]);
            }
        }
        if (p.do_m0) {
            const int ld = 32 * NC;
            double* out = p.m0_part + (size_t)blockIdx.x * RP * ld;
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const int r = rt * 8 + (lane >> 2);
                    const int i = c * 32 + nt * 8 + 2 * (lane & 3);
                    *reinterpret_cast<double2*>(out + (size_t)r * ld + i) =
                        make_double2(macc[rt][nt][0], macc[rt][nt][1]);
                }
        }
    } else if (p.do_s) {
        // ---------------- epilogue ----------------
        // warp ew owns fibers m0 = 8 ew .. 8 ew + 7; lane holds the (f, r) items of a DMMA
        // D fragment: f = m0 + lane/4, r = 8 nt + 2 (lane%4) + {0, 1}
        const int m0 = (warp - NC - 1) * 8;
        const int fl = m0 + (lane >> 2);
        for (int64_t k = 0; k < ntl; ++k) {
            const int b = (int)(k & 1);
            const int64_t f0 = (t_begin + k) * F;
            mbar_wait(&sfull[b], (uint32_t)((k / 2) & 1));
            if (epi_w) mbar_wait(&wfull[b], (uint32_t)((k / 2) & 1));
            const double* sp = spart + (size_t)b * NC * F * RP;
            const double* wv = wbuf + (size_t)b * F * WLD;
            double term = 0.0;
#pragma unroll
            for (int nt = 0; nt < NRT; ++nt) {
                const int r = nt * 8 + 2 * (lane & 3);
                double2 sv = make_double2(0.0, 0.0);
                for (int ww = 0; ww < NC; ++ww) {
                    const double2 v = *reinterpret_cast<const double2*>(sp + ((size_t)ww * F + fl) * RP + r);
                    sv.x += v.x;
                    sv.y += v.y;
                }
                if (f0 + fl < p.J) *reinterpret_cast<double2*>(p.S_out + (f0 + fl) * RP + r) = sv;
                if (epi_w) {
                    // Q = W G0 for this n-tile (DMMA over k = r')
                    double q0 = 0.0, q1 = 0.0;
#pragma unroll
                    for (int ks = 0; ks < RP / 4; ++ks) {
                        const double gb = gam[(ks * 4 + (lane & 3)) * RP + nt * 8 + (lane >> 2)];
                        dmma_8x8x4(q0, q1, wv[fl * WLD + ks * 4 + (lane & 3)], gb);
                    }
                    const double2 wd = *reinterpret_cast<const double2*>(wv + fl * WLD + r);
                    term += wd.x * (q0 - 2.0 * sv.x) + wd.y * (q1 - 2.0 * sv.y);
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sempty[b]);
                if (epi_w) mbar_arrive(&wempty[b]);
            }
            if (epi_w) {
                term += __shfl_xor_sync(0xffffffffu, term, 1);
                term += __shfl_xor_sync(0xffffffffu, term, 2);
                if ((lane & 3) == 0 && f0 + fl < p.J) facc += p.fnorm2[f0 + fl] + term;
            }
        }
    }
    if (resid) facc = racc.hi + racc.lo;
    if (p.do_f) {
        __shared__ double red[32];
        double v = warp_sum(facc);
        if (lane == 0) red[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) s += red[ww];
            p.f_part[blockIdx.x] = s;
        }
    }
}

template <int RP, int ORD>
void launch_fiber_ord(const FiberParams& p, int grid, int threads, size_t smem, cudaStream_t st) {
    auto k = fiber_ws_kernel<RP, kFiberF, (RP <= 16), ORD>;
    CPFIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, threads, smem, st>>>(p);
}

template <int RP>
void launch_fiber(const FiberParams& p, int grid, int nchunk, size_t smem, cudaStream_t st) {
    const int threads = 32 * (1 + nchunk + (p.do_s ? kEpiWarps : 0));
    switch (p.order) {
        case 2: launch_fiber_ord<RP, 2>(p, grid, threads, smem, st); break;
        case 3: launch_fiber_ord<RP, 3>(p, grid, threads, smem, st); break;
        case 4: launch_fiber_ord<RP, 4>(p, grid, threads, smem, st); break;
        default: launch_fiber_ord<RP, 0>(p, grid, threads, smem, st); break;
    }
    CPFIT_CUDA(cudaGetLastError());
}

size_t fiber_smem(int RP, int nchunk) {
    switch (RP) {
        case 8: return fiber_layout<8, kFiberF>(nchunk).total;
        case 16: return fiber_layout<16, kFiberF>(nchunk).total;
        default: return fiber_layout<32, kFiberF>(nchunk).total;
    }
}
