// Warp-specialized fiber pass (included by dense.cu inside cpfit_gpu::(anonymous)).
//
// One CTA per SM streams a contiguous range of F = 16-fiber tiles of T (mode-0 fibers, padded
// to ldT doubles) through a kFStages-deep (short fibres: kDeepFStages) shared-memory ring. Roles:
//   T producer (warp 0)    one bulk async copy per fiber into the ring, issued by 16 lanes at
//                          once (mbarrier complete_tx);
//   W producers (warps 1-2) the W tile — Khatri-Rao rows of modes >= 1, never materialised in
//                          HBM — into a double-buffered smem tile (independent gathers; two
//                          warps, since their multiplies queue behind DMMAs on the fp64 pipe);
//   S warps                warp s owns 8 x 8 sub-tile(s) (m-tile ft of fibers x r-tile rt) of
//                            S(F x RP) = T(:, F)^T A0    DMMA m8n8k4 over the FULL fiber length,
//                          four interleaved accumulator chains, A0 fragments from a shared-memory
//                          copy of A0 staged once per CTA; then the epilogue of its sub-tile:
//                          store S, Q = W G0 (DMMA) and the per-fiber objective
//                          ||t||^2 - 2 w.s + w^T G0 w folded into a per-warp sum;
//   M0 warps               warp m owns a run of 8-row m-tiles of the fiber:
//                            M0^T (RP x rows) += W(F, :)^T T(rows, F)^T   DMMA m8n8k4,
//                          accumulators in registers for the whole pass (+ the squared
//                          residual against A0 W^T in the residual-objective mode).
// S needs no cross-warp partial sums, so no scalar fp64 reduction competes with the DMMAs for
// the fp64 pipe. The M0 m-tiles are spread so each SM scheduler (warp w issues on w % 4) gets
// the same DMMA work (fiber_schedule). Hand-offs are mbarrier phases only.
// Shared-memory layouts: T rows padded to I0s = 32 NC + 4 doubles (4 mod 16) and W rows to
// RP + 4 doubles; A0 rows of RP doubles with an XOR column swizzle (a0s_index) — every DMMA
// fragment load is conflict free (two wavefronts per 32 doubles).
#pragma once

#include <type_traits>

constexpr int kFStages = 3;      // T ring depth for long fibres (a tile is ~54 KB at I0 = 400)
constexpr int kDeepFStages = 8;  // short fibres (I0 <= 128): ~70 KB of T in flight per SM
constexpr int kFiberF = 16;
constexpr int kWStages = 4;  // W (Khatri-Rao row) ring: the gathers of a tile take about a tile's time
// W ring depth of a T ring depth: the deep (short-fibre) ring runs M0 tile groups, where warp m
// consumes tiles m, m + 8, ... — with 8 slots every warp owns one W slot, so each warp's waits on
// it are in phase order (an mbarrier wait on phase parity 1 passes before phase 0 has completed)
__host__ __device__ constexpr int wstages(int nst) { return nst == kDeepFStages ? 8 : kWStages; }
constexpr int kMaxKSteps = 104;  // ldT / 4 for I_0 <= 416 (work_create checks)
#ifndef CPFIT_SREG_CHAINS
#define CPFIT_SREG_CHAINS 1
#endif
constexpr int kSRegChains = CPFIT_SREG_CHAINS;
#ifndef CPFIT_FUSED_CHAINS
#define CPFIT_FUSED_CHAINS 2
#endif
#ifndef CPFIT_FUSED_SREG
#define CPFIT_FUSED_SREG 1  // 0: S warps with both DMMA operands from shared memory (A/B builds)
#endif

template <int RP>
__host__ __device__ constexpr int w_ld() {
    return RP + 4;
}

// role counts per padded rank
template <int RP>
struct FiberRoles {
    static constexpr int NRT = RP / 8;
    static constexpr int NWP = RP <= 16 ? 2 : 0;            // W producer warps (0: the T producer)
    static constexpr bool SEPW = NWP > 0;
    static constexpr int NQ = 2 * NRT;                      // 8x8 S sub-tiles per tile
    // RP = 8 (SREG): S warp q owns K quarter q for BOTH 8-fibre groups with its A0 B-fragments in
    // registers (one shared-memory fragment load per DMMA; four S warps instead of two, so the S
    // work no longer sits on two sub-partitions); warps 0 / 1 sum the four quarters of fibre
    // group 0 / 1 and run its epilogue. (At RP = 16 the same scheme needs 19 warps, i.e. 96
    // registers and spills, or fewer W-producer / M0 warps, which slows the M0 pass of the solve
    // loop; measured in DESIGN.md §5, the 15-warp layout stays.)
    static constexpr bool SREG = CPFIT_FUSED_SREG && RP == 8;
    static constexpr int KQ = SREG ? 4 : 1;                 // K parts of the SREG S warps
    static constexpr int NS = SREG ? NRT * KQ : (RP == 32 ? 4 : NQ);  // S warps
    static constexpr int SPW = SREG ? 1 : NQ / NS;          // sub-tiles per S warp (S-given path)
    static constexpr int NEPI = SREG ? NQ : NS;             // S warps that consume W (epilogues)
    static constexpr int NM = RP == 32 ? 11 : 8;            // M0 warps
    static constexpr int MAXMT = RP == 8 ? 14 : (RP == 16 ? 7 : 5);  // m-tiles per M0 warp
    // short fibres (deep ring, ceil(I0 / 8) <= TGMT m-tiles): M0 tile groups — warp m takes whole
    // tiles m, m + NM, ... (every m-tile of the fibre: NRT x TGMT independent accumulators, one
    // barrier round trip per 4 NRT TGMT DMMAs) instead of its own rows of every tile
    static constexpr int TGMT = RP == 32 ? 4 : 16 / NRT;
    static constexpr bool A0SMEM = RP <= 16;                // A0 staged in shared memory
    static constexpr int S0 = 1 + NWP;                      // first S warp
    static constexpr int M0W = S0 + NS;                     // first M0 warp
    static constexpr int WARPS = M0W + NM;
    // registers per thread with one CTA of WARPS warps per SM: the register file is split over
    // the block's warps rounded up to a multiple of 4 (one per sub-partition), in units of 8
    static constexpr int WARPS4 = (WARPS + 3) / 4 * 4;
    static constexpr int MAXNREG = (65536 / (32 * WARPS4)) / 8 * 8 > 128 ? 128 : (65536 / (32 * WARPS4)) / 8 * 8;
};
static_assert(FiberRoles<32>::WARPS <= 16 && FiberRoles<16>::WARPS <= 16 && FiberRoles<8>::WARPS <= 16,
              "<= 512 threads (128 registers)");

struct FiberSmem {
    size_t tiles, a0, wbuf, gam, spart, bars, total;
};

// A0 rows staged in shared memory: every row an M0 warp's m-tiles touch (8 ceil(I0 / 8) >= ldT)
__host__ __device__ inline int64_t a0_rows(int64_t I0) { return (I0 + 7) / 8 * 8; }

template <int RP, int F>
__host__ __device__ FiberSmem fiber_layout(int nchunk, int64_t I0, int nst) {
    const int I0s = 32 * nchunk + 4;
    FiberSmem s{};
    size_t off = 0;
    s.tiles = off;
    off += sizeof(double) * (size_t)nst * F * I0s;
    s.a0 = off;
    if (FiberRoles<RP>::A0SMEM) off += sizeof(double) * (size_t)a0_rows(I0) * RP;
    s.wbuf = off;
    off += sizeof(double) * wstages(nst) * (size_t)F * w_ld<RP>();
    s.gam = off;
    off += sizeof(double) * (size_t)RP * RP;
    s.spart = off;  // SREG K-quarter exchange [NRT][6 slots][64] (the three other quarters of each group)
    if (FiberRoles<RP>::SREG) off += sizeof(double) * (size_t)FiberRoles<RP>::NRT * 6 * 64;
    s.bars = off;
    off += sizeof(uint64_t) * (2 * nst + 2 * wstages(nst));
    s.total = off;
    return s;
}

// Spread the ceil(I0 / 8) m-tiles over the M0 warps so the DMMA work per SM scheduler is as even
// as possible (the S warps' k-steps and the producers count as loads), at most MAXMT per warp.
template <int RP>
inline void fiber_schedule_rp(int I0, bool do_s, FiberParams& p) {
    using Ro = FiberRoles<RP>;
    const int MT = (I0 + 7) / 8;
    const int KS = (I0 + 3) / 4;
    double load[4] = {0.0, 0.0, 0.0, 0.0};
    load[0] += 2.0;
    for (int w = 0; w < Ro::NWP; ++w) load[(1 + w) % 4] += 2.0;
    if (do_s)
        for (int s = 0; s < Ro::NS; ++s)
            load[(Ro::S0 + s) % 4] += Ro::SREG ? 2.0 * KS / Ro::KQ + (s / Ro::NRT < 2 ? 6.0 : 0.0)
                                               : (double)KS * Ro::SPW + 6.0 * Ro::SPW;
    const double mt_w = 4.0 * Ro::NRT;  // DMMAs per m-tile per tile
    int cnt[16] = {};
    for (int t = 0; t < MT; ++t) {
        int best = -1;
        for (int m = 0; m < Ro::NM; ++m) {
            if (cnt[m] >= Ro::MAXMT) continue;
            if (best < 0 || load[(Ro::M0W + m) % 4] < load[(Ro::M0W + best) % 4] ||
                (load[(Ro::M0W + m) % 4] == load[(Ro::M0W + best) % 4] && cnt[m] < cnt[best]))
                best = m;
        }
        if (best < 0) throw std::invalid_argument("fiber pass: I_1 too large for the M0 warps");
        ++cnt[best];
        load[(Ro::M0W + best) % 4] += mt_w;
    }
    int acc = 0;
    for (int m = 0; m < Ro::NM; ++m) {
        p.mt_cnt[m] = cnt[m];
        p.mt_start[m] = acc;
        acc += cnt[m];
    }
}
inline void fiber_schedule(int RP, int I0, bool do_s, FiberParams& p) {
    switch (RP) {
        case 8: fiber_schedule_rp<8>(I0, do_s, p); break;
        case 16: fiber_schedule_rp<16>(I0, do_s, p); break;
        default: fiber_schedule_rp<32>(I0, do_s, p); break;
    }
}
inline int fiber_threads(int RP) {
    switch (RP) {
        case 8: return 32 * FiberRoles<8>::WARPS;
        case 16: return 32 * FiberRoles<16>::WARPS;
        default: return 32 * FiberRoles<32>::WARPS;
    }
}

// Diagnostic build (-DCPFIT_FIBER_PROF): cycles each warp role spends in every barrier wait,
// accumulated into FiberParams::prof[kProfSlots] (tools/fiber_prof.py).
constexpr int kProfSlots = 12;
#ifdef CPFIT_FIBER_PROF
#define FIBER_WAIT(slot, bar, par)                      \
    do {                                                \
        const long long t0_ = clock64();                \
        mbar_wait(bar, par);                            \
        prof_acc[slot] += clock64() - t0_;              \
    } while (0)
#else
#define FIBER_WAIT(slot, bar, par) mbar_wait(bar, par)
#endif

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

// shared-memory A0 position of (i, r): rows of RP doubles, column XOR-swizzled so the 16 lanes of
// each half-warp of a DMMA fragment load (rows i = 4k + lane%4, columns r = 8t + lane/4, or the
// transposed pattern) hit 16 distinct 8-byte bank pairs
template <int RP>
__device__ __forceinline__ int a0s_index(int i, int r) {
    if (RP == 16) return i * 16 + (r ^ ((i & 3) << 2));
    if (RP == 8) return i * 8 + (r ^ ((i & 2) << 1));
    return i * RP + r;
}

template <int RP, int F, int ORD, int NST>
__global__ void __maxnreg__(FiberRoles<RP>::MAXNREG) fiber_ws_kernel(const __grid_constant__ FiberParams p) {
    if (p.only_resid && !*p.resid_flag) return;  // the slab passes did this evaluation (slab.cu)
    using Ro = FiberRoles<RP>;
    constexpr int WST = wstages(NST);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int NRT = Ro::NRT;
    constexpr int WLD = w_ld<RP>();
    constexpr int NW = Ro::NWP > 0 ? Ro::NWP : 1;  // warps building W
    static_assert(F == 16, "two 8-fiber m-tiles per tile");
    const FiberSmem L = fiber_layout<RP, F>(p.nchunk, p.I0, NST);
    const int I0s = p.I0s;
    const int KS = (int)(p.ldT / 4);  // k-steps of 4 rows (ldT = I0 rounded up to 4; pad rows are 0)
    double* tiles = reinterpret_cast<double*>(smem_raw + L.tiles);
    double* a0s = reinterpret_cast<double*>(smem_raw + L.a0);    // [a0_rows][RP] swizzled
    double* wbuf = reinterpret_cast<double*>(smem_raw + L.wbuf);  // [WST][F][WLD]
    double* gam = reinterpret_cast<double*>(smem_raw + L.gam);    // [RP][RP]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bars);
    uint64_t* tfull = bars;          // [NST] tx bytes
    uint64_t* tempty = bars + NST;   // [NST] T consumers
    uint64_t* wfull = bars + 2 * NST;               // [WST] W producer
    uint64_t* wempty = bars + 2 * NST + WST;   // [WST] W consumers

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef CPFIT_FIBER_PROF
    long long prof_acc[kProfSlots] = {};
    const long long prof_t0 = clock64();
#endif
    const int64_t t_begin = (int64_t)blockIdx.x * p.tiles_per_cta;
    const int64_t t_end = imin64(p.ntiles, t_begin + p.tiles_per_cta);
    const int64_t ntl = t_end > t_begin ? t_end - t_begin : 0;
    // objective form: residual 1/2 sum (T - model)^2 (kruskal.cpp:83-102) when requested,
    // else the per-fiber three-term form folded by the S warps
    const bool resid = p.do_f && p.resid_flag && *p.resid_flag;
    const bool need_w = p.do_m0 || p.do_f;
    const bool m0w_on = p.do_m0 || resid;  // M0 warps consume T (and W)
    const bool epi_w = p.do_f && !resid;   // S warps consume W
    const bool need_a0 = (p.do_s && !Ro::SREG) || resid;  // SREG S warps hold A0 in registers
    dd racc{0.0, 0.0};

    for (int64_t e = tid; e < (int64_t)NST * F * I0s; e += blockDim.x) tiles[e] = 0.0;
    if (Ro::A0SMEM && need_a0)
        for (int64_t e = tid; e < a0_rows(p.I0) * RP; e += blockDim.x) {
            const int i = (int)(e / RP), r = (int)(e % RP);
            a0s[a0s_index<RP>(i, r)] = (i < p.I0 && r < p.R) ? p.A0[(int64_t)r * p.I0 + i] : 0.0;
        }
    if (p.do_f)
        for (int e = tid; e < RP * RP; e += blockDim.x) gam[e] = p.gamma0[e];
    // M0 tile groups (short fibres): one M0 consumer per T stage / W slot
    const bool m0tg = NST == kDeepFStages && (p.I0 + 7) / 8 <= Ro::TGMT &&
                      Ro::NM * RP * 32 * p.nchunk <= NST * F * I0s;  // the final sums reuse the T ring
    const int m0_cons = m0w_on ? (m0tg ? 1 : Ro::NM) : 0;
    if (tid == 0) {
        const int t_cons = (p.do_s ? Ro::NS : 0) + m0_cons;
        const int w_cons = m0_cons + (epi_w ? Ro::NEPI : 0);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], t_cons);
        }
        for (int b = 0; b < WST; ++b) {
            mbar_init(&wfull[b], NW);
            mbar_init(&wempty[b], w_cons);
        }
    }
    mbar_fence_init();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    auto a0_at = [&](int i, int r) -> double {  // fragment operand A0(i, r)
        if (Ro::A0SMEM) return a0s[a0s_index<RP>(i, r)];
        return (i < p.I0 && r < p.R) ? __ldg(p.A0 + (int64_t)r * p.I0 + i) : 0.0;
    };

    double facc = 0.0;
    double tacc[NRT][Ro::TGMT][2];  // M0 tile-group accumulators (short fibres, M0 warps)
    // W tile k: lane = (fiber fw, r-slice hw) of one of the NW producer warps; gathers first
    // (independent), then the buffer
    constexpr int RS = RP * F / (32 * NW);
    auto w_gather = [&](int64_t k, FiberIndex<ORD>& xw, int fw, int hw, double (&w)[RS]) {
        const int64_t f0 = (t_begin + k) * F;
        if (k > 0) xw = advance_fiber<ORD>(p, xw, F, f0 + fw);
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
    };
    auto w_store = [&](int64_t k, int fw, int hw, const double (&w)[RS]) {
        const int b = (int)(k % WST);
        if (k >= WST) FIBER_WAIT(1, &wempty[b], (uint32_t)(((k / WST) - 1) & 1));
        double* wv = wbuf + (size_t)b * F * WLD;
#pragma unroll
        for (int j = 0; j < RS; ++j) wv[fw * WLD + hw * RS + j] = w[j];
        __syncwarp();
        if (lane == 0) mbar_arrive(&wfull[b]);
    };
    auto w_producer = [&](int64_t k, FiberIndex<ORD>& xw, int fw, int hw) {
        double w[RS];
        w_gather(k, xw, fw, hw, w);
        w_store(k, fw, hw, w);
    };

    if (warp == 0) {
        // ---------------- T producer (+ W when RP = 32) ----------------
        const int fw = lane % F, hw = lane / F;
        FiberIndex<ORD> xw;
        if (!Ro::SEPW && need_w) xw = decode_fiber<ORD>(p, t_begin * F + fw);
        for (int64_t k = 0; k < ntl; ++k) {
            const int s = (int)(k % NST);
            const int64_t f0 = (t_begin + k) * F;
            if (k >= NST) FIBER_WAIT(0, &tempty[s], (uint32_t)(((k / NST) - 1) & 1));
            const int nvalid = (int)imin64(F, p.J - f0);
            double* st = tiles + (size_t)s * F * I0s;
            if (NST == kDeepFStages && p.use_tmap) {  // one box of F rows x pitch (pads / rows past J arrive as 0)
                if (lane == 0) {
                    mbar_arrive_expect_tx(&tfull[s], (uint32_t)(F * I0s * 8));
                    tma_2d_g2s_hint(st, &p.tmap, 0, (int)f0, &tfull[s], l2_evict_first());
                }
            } else {
                if (nvalid < F)
                    for (int e = lane; e < (F - nvalid) * I0s; e += 32) st[(size_t)nvalid * I0s + e] = 0.0;
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&tfull[s], (uint32_t)(nvalid * p.ldT * 8));
                __syncwarp();
                if (lane < nvalid)
                    bulk_g2s_hint(st + (size_t)lane * I0s, p.T + (f0 + lane) * p.ldT, (uint32_t)(p.ldT * 8), &tfull[s],
                                  l2_evict_first());
            }
            if (!Ro::SEPW && need_w) w_producer(k, xw, fw, hw);
        }
    } else if (Ro::SEPW && warp <= Ro::NWP) {
        // ---------------- W producers ----------------
        if (need_w) {
            const int fw = lane % F, hw = (warp - 1) * (32 / F) + lane / F;
            FiberIndex<ORD> xw = decode_fiber<ORD>(p, t_begin * F + fw);
            // short fibres: one tile ahead — the next tile's gathers are in flight while this one
            // waits for its ring slot (the producers are latency bound there)
            if (NST == kDeepFStages && ORD >= 3 && p.dims[1] % F == 0) {
                // I1 % 16 == 0: a tile's fibres share their modes >= 2 and take 16 consecutive
                // j1, so the multi-index is a tile-uniform counter advanced without divisions or
                // per-lane carries (the branchy per-lane advance made these warps the M0 pass's
                // bottleneck at 64^4), and W(f, r) = A1(j1, r) * prod_{m >= 2} A_m(j_m, r)
                // The tail product changes only when j1 wraps (every I1 / 16 tiles): it is kept in
                // registers, the next group's factor values are loaded one wrap ahead, and a tile
                // costs one A1 load per (fibre, r), issued a tile before the multiply that uses it.
                FiberIndex<ORD> xn = decode_fiber<ORD>(p, t_begin * F);
                const int I1 = (int)p.dims[1];
                constexpr int NT = (ORD > 2 ? ORD : kMaxOrder) - 2;  // tail modes (this branch: ORD >= 3)
                const double* a1p[RS];
                double tail[RS], nxt[NT][RS];
                auto next_group = [&]() {
#pragma unroll
                    for (int m = 2; m < (ORD > 0 ? ORD : kMaxOrder); ++m) {
                        if (++xn.j[m] < (int)p.dims[m]) break;
                        xn.j[m] = 0;
                    }
                };
                auto load_group = [&]() {  // factor values of group xn (indices wrap: always in range)
#pragma unroll
                    for (int j = 0; j < RS; ++j) {
                        const int r = hw * RS + j < p.R ? hw * RS + j : 0;
#pragma unroll
                        for (int m = 2; m < (ORD > 0 ? ORD : kMaxOrder); ++m)
                            nxt[m - 2][j] = mode_active<ORD>(p, m) ? __ldg(p.fac[m] + (int64_t)r * p.dims[m] + xn.j[m]) : 1.0;
                    }
                };
                auto take_group = [&]() {
#pragma unroll
                    for (int j = 0; j < RS; ++j) {
                        double v = 1.0;
#pragma unroll
                        for (int m = 0; m < NT; ++m) v *= nxt[m][j];
                        tail[j] = hw * RS + j < p.R ? v : 0.0;
                    }
                };
#pragma unroll
                for (int j = 0; j < RS; ++j) {
                    const int r = hw * RS + j;
                    a1p[j] = p.fac[1] + (int64_t)(r < p.R ? r : 0) * I1 + fw;
                }
                int j1 = xn.j[1];
                load_group();
                take_group();
                next_group();
                load_group();
                // gather tile k (raw A1 values + the tail of its group)
                auto ugather = [&](int64_t k, double (&a)[RS], double (&tl)[RS]) {
                    const bool valid = (t_begin + k) * F + fw < p.J;
#pragma unroll
                    for (int j = 0; j < RS; ++j) {
                        a[j] = valid && hw * RS + j < p.R ? __ldg(a1p[j] + j1) : 0.0;
                        tl[j] = tail[j];
                    }
                    j1 += F;  // next tile
                    if (j1 >= I1) {
                        j1 = 0;
                        take_group();
                        next_group();
                        load_group();
                    }
                };
                double ac[RS], tc[RS], an[RS], tn[RS];
                if (ntl > 0) ugather(0, ac, tc);
                for (int64_t k = 0; k < ntl; ++k) {
                    if (k + 1 < ntl) ugather(k + 1, an, tn);
                    double w[RS];
#pragma unroll
                    for (int j = 0; j < RS; ++j) w[j] = ac[j] * tc[j];
                    w_store(k, fw, hw, w);
#pragma unroll
                    for (int j = 0; j < RS; ++j) {
                        ac[j] = an[j];
                        tc[j] = tn[j];
                    }
                }
            } else if (NST == kDeepFStages) {
                double wc[RS], wn[RS];
                if (ntl > 0) w_gather(0, xw, fw, hw, wc);
                for (int64_t k = 0; k < ntl; ++k) {
                    if (k + 1 < ntl) w_gather(k + 1, xw, fw, hw, wn);
                    w_store(k, fw, hw, wc);
#pragma unroll
                    for (int j = 0; j < RS; ++j) wc[j] = wn[j];
                }
            } else {
                for (int64_t k = 0; k < ntl; ++k) w_producer(k, xw, fw, hw);
            }
        }
    } else if (warp < Ro::M0W) {
        // ---------------- S warps ----------------
        if (!p.do_s && epi_w && p.S_in) {
            // S is given (the ALS sweep's S' rescaled to u_bar): only the per-fiber objective
            const int sw = warp - Ro::S0;
            for (int64_t k = 0; k < (sw < Ro::NEPI ? ntl : 0); ++k) {
                const int b = (int)(k % WST);
                const int64_t f0 = (t_begin + k) * F;
                double sv[Ro::SPW][2], fn[Ro::SPW];
#pragma unroll
                for (int j = 0; j < Ro::SPW; ++j) {
                    const int q = sw * Ro::SPW + j, ft = q / NRT, nt = q % NRT;
                    const int64_t f = f0 + ft * 8 + (lane >> 2);
                    const int r = nt * 8 + 2 * (lane & 3);
                    fn[j] = (nt == 0 && f < p.J) ? p.fnorm2[f] : 0.0;
                    const double2 v = f < p.J ? *reinterpret_cast<const double2*>(p.S_in + f * RP + r) : make_double2(0.0, 0.0);
                    sv[j][0] = v.x;
                    sv[j][1] = v.y;
                }
                FIBER_WAIT(6, &wfull[b], (uint32_t)((k / WST) & 1));
                const double* wv = wbuf + (size_t)b * F * WLD;
#pragma unroll
                for (int j = 0; j < Ro::SPW; ++j) {
                    const int q = sw * Ro::SPW + j, ft = q / NRT, nt = q % NRT;
                    const int fl = ft * 8 + (lane >> 2);
                    const int r = nt * 8 + 2 * (lane & 3);
                    double q0 = 0.0, q1 = 0.0;
#pragma unroll
                    for (int kr = 0; kr < RP / 4; ++kr) {
                        const double gb = gam[(kr * 4 + (lane & 3)) * RP + nt * 8 + (lane >> 2)];
                        dmma_8x8x4(q0, q1, wv[fl * WLD + kr * 4 + (lane & 3)], gb);
                    }
                    const double2 wd = *reinterpret_cast<const double2*>(wv + fl * WLD + r);
                    double term = wd.x * (q0 - 2.0 * sv[j][0]) + wd.y * (q1 - 2.0 * sv[j][1]);
                    term += __shfl_xor_sync(0xffffffffu, term, 1);
                    term += __shfl_xor_sync(0xffffffffu, term, 2);
                    if ((lane & 3) == 0 && f0 + fl < p.J) facc += fn[j] + term;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&wempty[b]);
            }
        } else if (p.do_s && Ro::SREG) {
            constexpr int KM = (NST == kDeepFStages) ? 8 : (kMaxKSteps + 3) / 4;  // k-steps per quarter
            constexpr int CH = CPFIT_FUSED_CHAINS;  // accumulator chains per fibre group
            const int sw = warp - Ro::S0;
            const int nt = sw % NRT, q = sw / NRT;
            const int rr = nt * 8 + (lane >> 2);
            const int k_lo = (KS * q) / 4, nk = (KS * (q + 1)) / 4 - k_lo;
            double breg[KM];
#pragma unroll
            for (int kk = 0; kk < KM; ++kk) {
                const int i = 4 * (k_lo + kk) + (lane & 3);
                breg[kk] = (kk < nk && i < p.I0 && rr < p.R) ? __ldg(p.A0 + (int64_t)rr * p.I0 + i) : 0.0;
            }
            // exchange slots of column group nt: [group g][3 other quarters][64]
            double* xch = reinterpret_cast<double*>(smem_raw + L.spart) + (size_t)nt * 6 * 64;
            auto slot = [&](int g, int from) -> double* {  // quarter `from`'s partial of group g (from != g)
                return xch + ((size_t)g * 3 + (from < g ? from : from - 1)) * 64;
            };
            for (int64_t k = 0; k < ntl; ++k) {
                const int s = (int)(k % NST);
                const int b = (int)(k % WST);
                const int64_t f0 = (t_begin + k) * F;
                const bool fin = q < 2;             // finishes fibre group q
                const int fl = q * 8 + (lane >> 2);
                const double fnv = (fin && epi_w && nt == 0 && f0 + fl < p.J) ? p.fnorm2[f0 + fl] : 0.0;
                FIBER_WAIT(2, &tfull[s], (uint32_t)((k / NST) & 1));
                const double* ta0 = tiles + (size_t)s * F * I0s + (lane >> 2) * I0s + (lane & 3) + 4 * k_lo;
                const double* ta1 = ta0 + 8 * I0s;
                double acc[2][CH][2];
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int c = 0; c < CH; ++c) acc[g][c][0] = acc[g][c][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < KM; kk += CH) {
                    if (kk >= nk) break;  // warp-uniform exit: no predicated-off DMMAs past the quarter
                    double x0[CH], x1[CH];
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        x0[c] = (kk + c < nk) ? ta0[(kk + c) * 4] : 0.0;
                        x1[c] = (kk + c < nk) ? ta1[(kk + c) * 4] : 0.0;
                    }
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        dmma_8x8x4(acc[0][c][0], acc[0][c][1], x0[c], breg[kk + c < KM ? kk + c : KM - 1]);
                        dmma_8x8x4(acc[1][c][0], acc[1][c][1], x1[c], breg[kk + c < KM ? kk + c : KM - 1]);
                    }
                }
                double sv[2][2];
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double t = acc[g][0][e];
#pragma unroll
                        for (int c = 1; c < CH; ++c) t += acc[g][c][e];
                        sv[g][e] = t;
                    }
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[s]);
                // partials of the groups this warp does not finish go to their finishers
#pragma unroll
                for (int g = 0; g < 2; ++g)
                    if (g != q) {
                        double* d = slot(g, q);
                        d[2 * lane] = sv[g][0];
                        d[2 * lane + 1] = sv[g][1];
                    }
                asm volatile("bar.sync %0, %1;" ::"r"(1 + nt), "r"(32 * Ro::KQ) : "memory");
                double s0 = 0.0, s1 = 0.0;
                if (fin) {  // quarters in order 0, 1, 2, 3
#pragma unroll
                    for (int qq = 0; qq < Ro::KQ; ++qq) {
                        const double* o = qq == q ? nullptr : slot(q, qq);
                        s0 += o ? o[2 * lane] : sv[q][0];
                        s1 += o ? o[2 * lane + 1] : sv[q][1];
                    }
                }
                // the slots are rewritten only after every finisher has read them
                asm volatile("bar.sync %0, %1;" ::"r"(1 + NRT + nt), "r"(32 * Ro::KQ) : "memory");
                if (!fin) continue;
                if (epi_w) FIBER_WAIT(6, &wfull[b], (uint32_t)((k / WST) & 1));
                const double* wv = wbuf + (size_t)b * F * WLD;
                const int r = nt * 8 + 2 * (lane & 3);
                if (f0 + fl < p.J) *reinterpret_cast<double2*>(p.S_out + (f0 + fl) * RP + r) = make_double2(s0, s1);
                if (epi_w) {
                    double q0 = 0.0, q1 = 0.0;
#pragma unroll
                    for (int kr = 0; kr < RP / 4; ++kr) {
                        const double gb = gam[(kr * 4 + (lane & 3)) * RP + nt * 8 + (lane >> 2)];
                        dmma_8x8x4(q0, q1, wv[fl * WLD + kr * 4 + (lane & 3)], gb);
                    }
                    const double2 wd = *reinterpret_cast<const double2*>(wv + fl * WLD + r);
                    double term = wd.x * (q0 - 2.0 * s0) + wd.y * (q1 - 2.0 * s1);
                    term += __shfl_xor_sync(0xffffffffu, term, 1);
                    term += __shfl_xor_sync(0xffffffffu, term, 2);
                    if ((lane & 3) == 0 && f0 + fl < p.J) facc += fnv + term;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wempty[b]);
                }
            }
        } else if (p.do_s) {
            const int sw = warp - Ro::S0;
            for (int64_t k = 0; k < ntl; ++k) {
                const int s = (int)(k % NST);
                const int b = (int)(k % WST);
                const int64_t f0 = (t_begin + k) * F;
                double fn[Ro::SPW];  // ||t_f||^2 of this lane's fiber, prefetched (r-tile 0 only)
#pragma unroll
                for (int j = 0; j < Ro::SPW; ++j) {
                    const int q = sw * Ro::SPW + j, ft = q / NRT, nt = q % NRT;
                    const int64_t f = f0 + ft * 8 + (lane >> 2);
                    fn[j] = (epi_w && nt == 0 && f < p.J) ? p.fnorm2[f] : 0.0;
                }
                FIBER_WAIT(2, &tfull[s], (uint32_t)((k / NST) & 1));
                const double* tt = tiles + (size_t)s * F * I0s;
                double sv[Ro::SPW][2];
#pragma unroll
                for (int j = 0; j < Ro::SPW; ++j) {
                    const int q = sw * Ro::SPW + j, ft = q / NRT, nt = q % NRT;
                    const double* ta = tt + (ft * 8 + (lane >> 2)) * I0s + (lane & 3);
                    const int rr = nt * 8 + (lane >> 2);
                    // eight interleaved accumulator chains over the k-steps; each group's 16
                    // fragment loads issue before its 8 DMMAs
                    constexpr int U = 8;
                    double acc[U][2];
#pragma unroll
                    for (int u = 0; u < U; ++u) acc[u][0] = acc[u][1] = 0.0;
                    int ks = 0;
                    for (; ks + U <= KS; ks += U) {
                        double a[U], bb[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            a[u] = ta[(ks + u) * 4];
                            bb[u] = a0_at((ks + u) * 4 + (lane & 3), rr);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) dmma_8x8x4(acc[u][0], acc[u][1], a[u], bb[u]);
                    }
                    {
                        double a[U - 1], bb[U - 1];
#pragma unroll
                        for (int u = 0; u < U - 1; ++u) {
                            a[u] = ks + u < KS ? ta[(ks + u) * 4] : 0.0;
                            bb[u] = ks + u < KS ? a0_at((ks + u) * 4 + (lane & 3), rr) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < U - 1; ++u)
                            if (ks + u < KS) dmma_8x8x4(acc[u][0], acc[u][1], a[u], bb[u]);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        acc[u][0] += acc[u + 4][0];
                        acc[u][1] += acc[u + 4][1];
                    }
                    sv[j][0] = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
                    sv[j][1] = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[s]);
                // epilogue of the sub-tile(s): lane holds D fragment items f = 8 ft + lane/4,
                // r = 8 nt + 2 (lane%4) + {0, 1}
                // epilogue of the sub-tile(s): lane holds D fragment items f = 8 ft + lane/4,
                // r = 8 nt + 2 (lane%4) + {0, 1}
                if (epi_w) FIBER_WAIT(6, &wfull[b], (uint32_t)((k / WST) & 1));
                const double* wv = wbuf + (size_t)b * F * WLD;
#pragma unroll
                for (int j = 0; j < Ro::SPW; ++j) {
                    const int q = sw * Ro::SPW + j, ft = q / NRT, nt = q % NRT;
                    const int fl = ft * 8 + (lane >> 2);
                    const int r = nt * 8 + 2 * (lane & 3);
                    if (f0 + fl < p.J)
                        *reinterpret_cast<double2*>(p.S_out + (f0 + fl) * RP + r) = make_double2(sv[j][0], sv[j][1]);
                    if (epi_w) {
                        // Q = W G0 for this r-tile (DMMA over k = r')
                        double q0 = 0.0, q1 = 0.0;
#pragma unroll
                        for (int kr = 0; kr < RP / 4; ++kr) {
                            const double gb = gam[(kr * 4 + (lane & 3)) * RP + nt * 8 + (lane >> 2)];
                            dmma_8x8x4(q0, q1, wv[fl * WLD + kr * 4 + (lane & 3)], gb);
                        }
                        const double2 wd = *reinterpret_cast<const double2*>(wv + fl * WLD + r);
                        double term = wd.x * (q0 - 2.0 * sv[j][0]) + wd.y * (q1 - 2.0 * sv[j][1]);
                        term += __shfl_xor_sync(0xffffffffu, term, 1);
                        term += __shfl_xor_sync(0xffffffffu, term, 2);
                        if ((lane & 3) == 0 && f0 + fl < p.J) facc += fn[j] + term;
                    }
                }
                if (epi_w) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wempty[b]);
                }
            }
        }
    } else {
        // ---------------- M0 warps ----------------
        if (NST == kDeepFStages && m0tg) {
            // tile groups: warp m runs tiles m, m + NM, ... over every m-tile of the fibre
            const int m = warp - Ro::M0W;
            const int mt = (p.I0 + 7) / 8;
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
                for (int nt = 0; nt < Ro::TGMT; ++nt) tacc[rt][nt][0] = tacc[rt][nt][1] = 0.0;
            if (m0w_on) {
                for (int64_t k = m; k < ntl; k += Ro::NM) {
                    const int s = (int)(k % NST);
                    const int b = (int)(k % WST);
                    FIBER_WAIT(3, &tfull[s], (uint32_t)((k / NST) & 1));
                    FIBER_WAIT(4, &wfull[b], (uint32_t)((k / WST) & 1));
                    const double* tt = tiles + (size_t)s * F * I0s;
                    const double* wv = wbuf + (size_t)b * F * WLD;
                    if (p.do_m0) {
#pragma unroll
                        for (int kf = 0; kf < F / 4; ++kf) {
                            const int f = kf * 4 + (lane & 3);
                            double wa[NRT];
#pragma unroll
                            for (int rt = 0; rt < NRT; ++rt) wa[rt] = wv[f * WLD + rt * 8 + (lane >> 2)];
                            double bb[Ro::TGMT];
#pragma unroll
                            for (int nt = 0; nt < Ro::TGMT; ++nt)
                                bb[nt] = nt < mt ? tt[f * I0s + nt * 8 + (lane >> 2)] : 0.0;
#pragma unroll
                            for (int nt = 0; nt < Ro::TGMT; ++nt) {
                                if (nt >= mt) break;
#pragma unroll
                                for (int rt = 0; rt < NRT; ++rt)
                                    dmma_8x8x4(tacc[rt][nt][0], tacc[rt][nt][1], wa[rt], bb[nt]);
                            }
                        }
                    }
                    if (resid) {
                        double tsum = 0.0;
#pragma unroll
                        for (int nt2 = 0; nt2 < Ro::TGMT; ++nt2) {
                            if (nt2 >= mt) break;
                            const int i = nt2 * 8 + (lane >> 2);
                            double a0r[RP / 4];
#pragma unroll
                            for (int kr = 0; kr < RP / 4; ++kr) a0r[kr] = a0_at(i, kr * 4 + (lane & 3));
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
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&tempty[s]);
                        mbar_arrive(&wempty[b]);
                    }
                }
            }
        } else {
        // rows [rb, rb + 8 cnt) of the fiber (cnt <= MAXMT m-tiles)
        const int m = warp - Ro::M0W;
        const int cnt = p.mt_cnt[m];
        const int rb = 8 * p.mt_start[m];
        double macc[NRT][Ro::MAXMT][2];
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
            for (int nt = 0; nt < Ro::MAXMT; ++nt) macc[rt][nt][0] = macc[rt][nt][1] = 0.0;
        if (m0w_on) {
            for (int64_t k = 0; k < ntl; ++k) {
                const int s = (int)(k % NST);
                const int b = (int)(k % WST);
                FIBER_WAIT(3, &tfull[s], (uint32_t)((k / NST) & 1));
                FIBER_WAIT(4, &wfull[b], (uint32_t)((k / WST) & 1));
                const double* tt = tiles + (size_t)s * F * I0s;
                const double* wv = wbuf + (size_t)b * F * WLD;
                if (p.do_m0) {
                    // few m-tiles per warp (short fibres): warp-uniform exit, no predicated-off
                    // DMMAs; otherwise the predicated form, which schedules better
                    const bool few = NST == kDeepFStages && 2 * cnt <= Ro::MAXMT;
#pragma unroll
                    for (int kf = 0; kf < F / 4; ++kf) {
                        const int f = kf * 4 + (lane & 3);
                        double wa[NRT];
#pragma unroll
                        for (int rt = 0; rt < NRT; ++rt) wa[rt] = wv[f * WLD + rt * 8 + (lane >> 2)];
                        if (few) {
#pragma unroll
                            for (int nt = 0; nt < Ro::MAXMT; ++nt) {
                                if (nt >= cnt) break;
                                const double bb = tt[f * I0s + rb + nt * 8 + (lane >> 2)];
#pragma unroll
                                for (int rt = 0; rt < NRT; ++rt)
                                    dmma_8x8x4(macc[rt][nt][0], macc[rt][nt][1], wa[rt], bb);
                            }
                        } else {
#pragma unroll
                            for (int nt = 0; nt < Ro::MAXMT; ++nt) {
                                if (nt < cnt) {
                                    const double bb = tt[f * I0s + rb + nt * 8 + (lane >> 2)];
#pragma unroll
                                    for (int rt = 0; rt < NRT; ++rt)
                                        dmma_8x8x4(macc[rt][nt][0], macc[rt][nt][1], wa[rt], bb);
                                }
                            }
                        }
                    }
                }
                if (resid) {
                    // model(i, f) = sum_r A0(i, r) W(f, r) for this warp's rows on DMMA, then the
                    // squared residual against the tile (padding is 0 - 0)
                    double tsum = 0.0;
#pragma unroll
                    for (int mt = 0; mt < Ro::MAXMT; ++mt) {
                        if (mt >= cnt) break;
                        {
                            const int i = rb + mt * 8 + (lane >> 2);
                            double a0r[RP / 4];
#pragma unroll
                            for (int kr = 0; kr < RP / 4; ++kr) a0r[kr] = a0_at(i, kr * 4 + (lane & 3));
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
                    }
                    racc = dd_add(racc, dd{tsum, 0.0});
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&tempty[s]);
                    mbar_arrive(&wempty[b]);
                }
            }
        }
        if (p.do_m0) {
            const int ld = 32 * p.nchunk;
            double* out = p.m0_part + (size_t)blockIdx.x * RP * ld;
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
                for (int nt = 0; nt < Ro::MAXMT; ++nt) {
                    if (nt < cnt) {
                        const int r = rt * 8 + (lane >> 2);
                        const int i = rb + nt * 8 + 2 * (lane & 3);
                        *reinterpret_cast<double2*>(out + (size_t)r * ld + i) =
                            make_double2(macc[rt][nt][0], macc[rt][nt][1]);
                    }
                }
        }
        }  // M0 rows per warp
    }
#ifdef CPFIT_FIBER_PROF
    {
        // slot 7/8/9: producer / S-warp / M0-warp lifetime
        const int role = warp < Ro::S0 ? 7 : (warp < Ro::M0W ? 8 : 9);
        prof_acc[role] = clock64() - prof_t0;
        if (lane == 0 && p.prof)
            for (int q = 0; q < kProfSlots; ++q)
                if (prof_acc[q]) atomicAdd(p.prof + q, (unsigned long long)prof_acc[q]);
    }
#endif
    if (NST == kDeepFStages && m0tg && p.do_m0) {
        // the NM tile-group partials of every m-tile, summed in warp order through shared memory
        // (the T ring is free once every warp has left its role loop)
        const int ld = 32 * p.nchunk;
        const int mt = (p.I0 + 7) / 8;
        double* red = tiles;  // [NM][RP][ld]
        __syncthreads();
        if (warp >= Ro::M0W) {
            const int m = warp - Ro::M0W;
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt)
#pragma unroll
                for (int nt = 0; nt < Ro::TGMT; ++nt) {
                    if (nt < mt) {
                        const int r = rt * 8 + (lane >> 2);
                        const int i = nt * 8 + 2 * (lane & 3);
                        *reinterpret_cast<double2*>(red + ((size_t)m * RP + r) * ld + i) =
                            make_double2(tacc[rt][nt][0], tacc[rt][nt][1]);
                    }
                }
        }
        __syncthreads();
        double* out = p.m0_part + (size_t)blockIdx.x * RP * ld;
        for (int e = tid; e < RP * 8 * mt; e += blockDim.x) {
            const int r = e / (8 * mt), i = e % (8 * mt);
            double v = 0.0;
            for (int w2 = 0; w2 < Ro::NM; ++w2) v += red[((size_t)w2 * RP + r) * ld + i];
            out[(size_t)r * ld + i] = v;
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
void launch_fiber_ord(const FiberParams& p, int grid, size_t smem, cudaStream_t st) {
    auto k = p.nst == kDeepFStages ? fiber_ws_kernel<RP, kFiberF, ORD, kDeepFStages>
                                   : fiber_ws_kernel<RP, kFiberF, ORD, kFStages>;
    CPFIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 32 * FiberRoles<RP>::WARPS, smem, st>>>(p);
}

template <int RP>
void launch_fiber(const FiberParams& p, int grid, size_t smem, cudaStream_t st) {
    switch (p.order) {
        case 2: launch_fiber_ord<RP, 2>(p, grid, smem, st); break;
        case 3: launch_fiber_ord<RP, 3>(p, grid, smem, st); break;
        case 4: launch_fiber_ord<RP, 4>(p, grid, smem, st); break;
        default: launch_fiber_ord<RP, 0>(p, grid, smem, st); break;
    }
    CPFIT_CUDA(cudaGetLastError());
}

size_t fiber_smem(int RP, int nchunk, int64_t I0, int nst) {
    switch (RP) {
        case 8: return fiber_layout<8, kFiberF>(nchunk, I0, nst).total;
        case 16: return fiber_layout<16, kFiberF>(nchunk, I0, nst).total;
        default: return fiber_layout<32, kFiberF>(nchunk, I0, nst).total;
    }
}

// ---------------------------------------------------------------------------------------
// S-only pass (the ALS S' = T x_1 A0' and the MTTKRP of modes >= 1): no W, no M0 — every
// compute warp takes a K-part of one 8 x 8 sub-tile, so the whole SM issues DMMAs instead of
// the fused kernel's four S warps; part 0 adds the other parts (in part order) and stores S.
// ---------------------------------------------------------------------------------------
template <int RP>
struct SPassRoles {
    static constexpr int NRT = RP / 8;
    static constexpr int NQ = 2 * NRT;                       // 8x8 sub-tiles per tile
    static constexpr int KSPLIT = RP == 8 ? 6 : (RP == 16 ? 3 : 1);
    static constexpr int NCW = NQ * KSPLIT;                  // compute warps (12, 12, 8)
    static constexpr int NPART = NQ * (KSPLIT - 1);
    static constexpr int WARPS = 1 + NCW;
};

template <int RP, int F>
__host__ __device__ FiberSmem spass_layout(int nchunk, int64_t I0, int nst) {
    const int I0s = 32 * nchunk + 4;
    FiberSmem s{};
    size_t off = 0;
    s.tiles = off;
    off += sizeof(double) * (size_t)nst * F * I0s;
    s.a0 = off;
    if (FiberRoles<RP>::A0SMEM) off += sizeof(double) * (size_t)a0_rows(I0) * RP;
    s.spart = off;
    off += sizeof(double) * (size_t)nst * SPassRoles<RP>::NPART * 64;
    s.wbuf = s.gam = off;
    s.bars = off;
    off += sizeof(uint64_t) * (2 + SPassRoles<RP>::NQ) * nst;
    s.total = off;
    return s;
}

template <int RP, int F, int NST>
__global__ void __launch_bounds__(32 * SPassRoles<RP>::WARPS, 1) spass_kernel(const __grid_constant__ FiberParams p) {
    using Ro = SPassRoles<RP>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int NRT = Ro::NRT;
    const FiberSmem L = spass_layout<RP, F>(p.nchunk, p.I0, NST);
    const int I0s = p.I0s;
    const int KS = (int)(p.ldT / 4);
    double* tiles = reinterpret_cast<double*>(smem_raw + L.tiles);
    double* a0s = reinterpret_cast<double*>(smem_raw + L.a0);
    double* spart = reinterpret_cast<double*>(smem_raw + L.spart);  // [stage][NPART][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bars);
    uint64_t* tfull = bars;            // [NST]
    uint64_t* tempty = bars + NST;     // [NST] compute warps
    uint64_t* pfull = bars + 2 * NST;  // [NST][NQ] the other K-parts of a sub-tile

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t_begin = (int64_t)blockIdx.x * p.tiles_per_cta;
    const int64_t t_end = imin64(p.ntiles, t_begin + p.tiles_per_cta);
    const int64_t ntl = t_end > t_begin ? t_end - t_begin : 0;

    for (int64_t e = tid; e < (int64_t)NST * F * I0s; e += blockDim.x) tiles[e] = 0.0;
    if (FiberRoles<RP>::A0SMEM)
        for (int64_t e = tid; e < a0_rows(p.I0) * RP; e += blockDim.x) {
            const int i = (int)(e / RP), r = (int)(e % RP);
            a0s[a0s_index<RP>(i, r)] = (i < p.I0 && r < p.R) ? p.A0[(int64_t)r * p.I0 + i] : 0.0;
        }
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], Ro::NCW);
            for (int q = 0; q < Ro::NQ; ++q) mbar_init(&pfull[s * Ro::NQ + q], Ro::KSPLIT > 1 ? Ro::KSPLIT - 1 : 1);
        }
    }
    mbar_fence_init();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    auto a0_at = [&](int i, int r) -> double {
        if (FiberRoles<RP>::A0SMEM) return a0s[a0s_index<RP>(i, r)];
        return (i < p.I0 && r < p.R) ? __ldg(p.A0 + (int64_t)r * p.I0 + i) : 0.0;
    };

    if (warp == 0) {
        for (int64_t k = 0; k < ntl; ++k) {
            const int s = (int)(k % NST);
            const int64_t f0 = (t_begin + k) * F;
            if (k >= NST) mbar_wait(&tempty[s], (uint32_t)(((k / NST) - 1) & 1));
            const int nvalid = (int)imin64(F, p.J - f0);
            double* st = tiles + (size_t)s * F * I0s;
            if (NST == kDeepFStages && p.use_tmap) {  // one box of F rows x pitch (pads / rows past J arrive as 0)
                if (lane == 0) {
                    mbar_arrive_expect_tx(&tfull[s], (uint32_t)(F * I0s * 8));
                    tma_2d_g2s_hint(st, &p.tmap, 0, (int)f0, &tfull[s], l2_evict_first());
                }
            } else {
                if (nvalid < F)
                    for (int e = lane; e < (F - nvalid) * I0s; e += 32) st[(size_t)nvalid * I0s + e] = 0.0;
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&tfull[s], (uint32_t)(nvalid * p.ldT * 8));
                __syncwarp();
                if (lane < nvalid)
                    bulk_g2s_hint(st + (size_t)lane * I0s, p.T + (f0 + lane) * p.ldT, (uint32_t)(p.ldT * 8), &tfull[s],
                                  l2_evict_first());
            }
        }
        return;
    }
    const int c = warp - 1;
    const int q = c % Ro::NQ, h = c / Ro::NQ;
    const int ft = q / NRT, nt = q % NRT;
    const int fl = ft * 8 + (lane >> 2);
    const int rr = nt * 8 + (lane >> 2);
    const int k_lo = (int)((int64_t)KS * h / Ro::KSPLIT), k_hi = (int)((int64_t)KS * (h + 1) / Ro::KSPLIT);
    for (int64_t k = 0; k < ntl; ++k) {
        const int s = (int)(k % NST);
        const int64_t f0 = (t_begin + k) * F;
        mbar_wait(&tfull[s], (uint32_t)((k / NST) & 1));
        const double* ta = tiles + (size_t)s * F * I0s + fl * I0s + (lane & 3);
        constexpr int U = 8;
        double acc[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u][0] = acc[u][1] = 0.0;
        int ks = k_lo;
        for (; ks + U <= k_hi; ks += U) {
            double a[U], bb[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                a[u] = ta[(ks + u) * 4];
                bb[u] = a0_at((ks + u) * 4 + (lane & 3), rr);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) dmma_8x8x4(acc[u][0], acc[u][1], a[u], bb[u]);
        }
#pragma unroll
        for (int u = 0; u < U - 1; ++u)
            if (ks + u < k_hi)
                dmma_8x8x4(acc[u][0], acc[u][1], ta[(ks + u) * 4], a0_at((ks + u) * 4 + (lane & 3), rr));
        double sv0 = ((acc[0][0] + acc[4][0]) + (acc[1][0] + acc[5][0])) + ((acc[2][0] + acc[6][0]) + (acc[3][0] + acc[7][0]));
        double sv1 = ((acc[0][1] + acc[4][1]) + (acc[1][1] + acc[5][1])) + ((acc[2][1] + acc[6][1]) + (acc[3][1] + acc[7][1]));
        if (h > 0) {
            // this stage's slot is refilled only after part 0 has read it (it releases the T
            // stage after the read)
            double* sp = spart + ((size_t)s * Ro::NPART + q * (Ro::KSPLIT - 1) + (h - 1)) * 64 + 2 * lane;
            sp[0] = sv0;
            sp[1] = sv1;
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&pfull[s * Ro::NQ + q]);
                mbar_arrive(&tempty[s]);
            }
            continue;
        }
        if (Ro::KSPLIT > 1) {
            mbar_wait(&pfull[s * Ro::NQ + q], (uint32_t)((k / NST) & 1));
#pragma unroll
            for (int hh = 1; hh < Ro::KSPLIT; ++hh) {
                const double* sp = spart + ((size_t)s * Ro::NPART + q * (Ro::KSPLIT - 1) + (hh - 1)) * 64 + 2 * lane;
                sv0 += sp[0];
                sv1 += sp[1];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[s]);
        const int r = nt * 8 + 2 * (lane & 3);
        if (f0 + fl < p.J) *reinterpret_cast<double2*>(p.S_out + (f0 + fl) * RP + r) = make_double2(sv0, sv1);
    }
}

// ---------------------------------------------------------------------------------------
// S-only pass for RP <= 16 with the A0 operand in registers. With both DMMA operands read from
// shared memory (spass_kernel) the pass is bound by shared-memory bandwidth and the DMMA pipe
// together (~63% of each: two 256-byte fragment loads per 8x8x4 DMMA). Here compute warp c owns
// column group nt = c % NRT over K part h = c / NRT for BOTH 8-fibre groups of the tile: its B
// fragments (A0 rows of its K range, one column group) stay in registers for the whole pass, so
// each DMMA needs one shared-memory fragment load (of T). Parts h > 0 leave their sums in shared
// memory for part 0, which writes the S rows.
// ---------------------------------------------------------------------------------------
#ifndef CPFIT_SREG_WARPS
#define CPFIT_SREG_WARPS 12
#endif
template <int RP>
struct SRegRoles {
    static constexpr int NRT = RP / 8;             // column groups
    static constexpr int KSPLIT = CPFIT_SREG_WARPS / NRT;  // K parts
    static constexpr int NCW = NRT * KSPLIT;       // compute warps
    static constexpr int WARPS = 1 + NCW;          // + the T producer
    static constexpr int KMAX = (kMaxKSteps + KSPLIT - 1) / KSPLIT;  // k-steps per warp (9, 18)
    static constexpr int CH = kSRegChains;         // accumulator chains per fibre group
    static constexpr int NPART = NRT * (KSPLIT - 1);
};

// T rows at a pitch of ldT + 4 rounded to 4 mod 16 doubles (conflict-free fragment loads)
__host__ __device__ inline int sreg_pitch(int64_t ldT) { return (int)(((ldT + 15) / 16) * 16 + 4); }

template <int RP, int F>
__host__ __device__ FiberSmem sreg_layout(int64_t ldT, int nst) {
    using Ro = SRegRoles<RP>;
    const int I0s = sreg_pitch(ldT);
    FiberSmem s{};
    size_t off = 0;
    s.tiles = off;
    off += sizeof(double) * (size_t)nst * F * I0s;
    s.spart = off;  // [stage][NPART][2 fibre groups][64]
    off += sizeof(double) * (size_t)nst * Ro::NPART * 128;
    s.a0 = s.wbuf = s.gam = off;
    s.bars = off;
    off += sizeof(uint64_t) * (2 * nst + nst * Ro::NRT);
    s.total = off;
    return s;
}

template <int RP, int F, int NSTG>
__global__ void __launch_bounds__(32 * SRegRoles<RP>::WARPS, 1) sreg_kernel(const __grid_constant__ FiberParams p) {
    static_assert(F == 16, "two 8-fibre groups per tile");
    using Ro = SRegRoles<RP>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int NS = NSTG;
    const FiberSmem L = sreg_layout<RP, F>(p.ldT, NS);
    const int I0s = sreg_pitch(p.ldT);
    const int KS = (int)(p.ldT / 4);
    double* tiles = reinterpret_cast<double*>(smem_raw + L.tiles);
    double* spart = reinterpret_cast<double*>(smem_raw + L.spart);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bars);
    uint64_t* tfull = bars;           // [NS] tx bytes
    uint64_t* tempty = bars + NS;     // [NS] compute warps
    uint64_t* pfull = bars + 2 * NS;  // [NS][NRT] the other K parts of a column group

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t_begin = (int64_t)blockIdx.x * p.tiles_per_cta;
    const int64_t t_end = imin64(p.ntiles, t_begin + p.tiles_per_cta);
    const int64_t ntl = t_end > t_begin ? t_end - t_begin : 0;

    for (int64_t e = tid; e < (int64_t)NS * F * I0s; e += blockDim.x) tiles[e] = 0.0;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], p.sreg_groups ? Ro::NRT : Ro::NCW);
            for (int q = 0; q < Ro::NRT; ++q) mbar_init(&pfull[s * Ro::NRT + q], Ro::KSPLIT - 1);
        }
    }
    mbar_fence_init();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    if (warp == 0) {  // T producer
        for (int64_t k = 0; k < ntl; ++k) {
            const int s = (int)(k % NS);
            const int64_t f0 = (t_begin + k) * F;
            if (k >= NS) mbar_wait(&tempty[s], (uint32_t)(((k / NS) - 1) & 1));
            const int nvalid = (int)imin64(F, p.J - f0);
            double* st = tiles + (size_t)s * F * I0s;
            if (NS == kDeepFStages && p.use_tmap) {  // one box of F rows x pitch (pads / rows past J arrive as 0)
                if (lane == 0) {
                    mbar_arrive_expect_tx(&tfull[s], (uint32_t)(F * I0s * 8));
                    tma_2d_g2s_hint(st, &p.tmap, 0, (int)f0, &tfull[s], l2_evict_first());
                }
            } else {
                if (nvalid < F)
                    for (int e = lane; e < (F - nvalid) * I0s; e += 32) st[(size_t)nvalid * I0s + e] = 0.0;
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&tfull[s], (uint32_t)(nvalid * p.ldT * 8));
                __syncwarp();
                if (lane < nvalid)
                    bulk_g2s_hint(st + (size_t)lane * I0s, p.T + (f0 + lane) * p.ldT, (uint32_t)(p.ldT * 8), &tfull[s],
                                  l2_evict_first());
            }
        }
        return;
    }
    const int c = warp - 1;
    // short fibres (KS <= KMAX, p.sreg_groups = NG > 0): no K split — NG groups of NRT warps take
    // whole tiles in turn (NG divides the ring depth, so every stage has one consumer group)
    constexpr bool SHORT = NSTG == kDeepFStages;  // short-fibre features compiled in
    const int NG = SHORT ? p.sreg_groups : 0;
    const int nt = c % Ro::NRT, h = NG ? 0 : c / Ro::NRT, grp = NG ? c / Ro::NRT : 0;
    if (NG && grp >= NG) return;
    const int rr = nt * 8 + (lane >> 2);
    const int k_lo = NG ? 0 : (int)((int64_t)KS * h / Ro::KSPLIT);
    const int k_hi = NG ? KS : (int)((int64_t)KS * (h + 1) / Ro::KSPLIT);
    double bq[Ro::KMAX];  // B fragments A0[4 ks + lane % 4][rr], ks in [k_lo, k_hi)
#pragma unroll
    for (int u = 0; u < Ro::KMAX; ++u) {
        const int i = (k_lo + u) * 4 + (lane & 3);
        bq[u] = (k_lo + u < k_hi && i < p.I0 && rr < p.R) ? __ldg(p.A0 + (int64_t)rr * p.I0 + i) : 0.0;
    }
    for (int64_t k = grp; k < ntl; k += (NG ? NG : 1)) {
        const int s = (int)(k % NS);
        const int64_t f0 = (t_begin + k) * F;
        mbar_wait(&tfull[s], (uint32_t)((k / NS) & 1));
        // fibre group g's A fragments: T[g * 8 + lane / 4][4 ks + lane % 4]
        const double* ta0 = tiles + (size_t)s * F * I0s + (lane >> 2) * I0s + (lane & 3);
        const double* ta1 = ta0 + 8 * I0s;
        double acc[2][Ro::CH][2];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int j = 0; j < Ro::CH; ++j) acc[g][j][0] = acc[g][j][1] = 0.0;
        // short K ranges (short fibres: k_hi - k_lo << KMAX) take a warp-uniform exit so the
        // predicated-off DMMAs of the remaining unrolled steps are not issued; long ones keep the
        // predicated form, which schedules better
        auto kloop = [&](auto few_tag) {
            constexpr bool FEW = decltype(few_tag)::value;
#pragma unroll
            for (int u0 = 0; u0 < Ro::KMAX; u0 += Ro::CH) {
                if (FEW && u0 >= k_hi - k_lo) break;
                double a0[Ro::CH], a1[Ro::CH];
#pragma unroll
                for (int j = 0; j < Ro::CH; ++j) {
                    const int ks = k_lo + u0 + j;
                    const bool ok = u0 + j < Ro::KMAX && ks < k_hi;
                    a0[j] = ok ? ta0[ks * 4] : 0.0;
                    a1[j] = ok ? ta1[ks * 4] : 0.0;
                }
#pragma unroll
                for (int j = 0; j < Ro::CH; ++j)
                    if (u0 + j < Ro::KMAX && k_lo + u0 + j < k_hi) {
                        dmma_8x8x4(acc[0][j][0], acc[0][j][1], a0[j], bq[u0 + j]);
                        dmma_8x8x4(acc[1][j][0], acc[1][j][1], a1[j], bq[u0 + j]);
                    }
            }
        };
        if (SHORT && 2 * (k_hi - k_lo) <= Ro::KMAX)
            kloop(std::true_type{});
        else
            kloop(std::false_type{});
        double sv[2][2];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                // chain sums: scalar fp64 shares the DMMA pipe, so few chains
                double v = acc[g][0][e];
#pragma unroll
                for (int j = 1; j < Ro::CH; ++j) v += acc[g][j][e];
                sv[g][e] = v;
            }
        if (h > 0) {
            double* sp = spart + ((size_t)s * Ro::NPART + nt * (Ro::KSPLIT - 1) + (h - 1)) * 128 + 2 * lane;
            sp[0] = sv[0][0];
            sp[1] = sv[0][1];
            sp[64] = sv[1][0];
            sp[65] = sv[1][1];
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&pfull[s * Ro::NRT + nt]);
                mbar_arrive(&tempty[s]);
            }
            continue;
        }
        if (!NG) mbar_wait(&pfull[s * Ro::NRT + nt], (uint32_t)((k / NS) & 1));
#pragma unroll
        for (int hh = 1; hh < Ro::KSPLIT; ++hh) {
            if (NG) break;
            const double* sp = spart + ((size_t)s * Ro::NPART + nt * (Ro::KSPLIT - 1) + (hh - 1)) * 128 + 2 * lane;
            sv[0][0] += sp[0];
            sv[0][1] += sp[1];
            sv[1][0] += sp[64];
            sv[1][1] += sp[65];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[s]);
        const int r = nt * 8 + 2 * (lane & 3);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int64_t f = f0 + g * 8 + (lane >> 2);
            if (f < p.J) *reinterpret_cast<double2*>(p.S_out + f * RP + r) = make_double2(sv[g][0], sv[g][1]);
        }
    }
}

template <int RP>
void launch_spass(const FiberParams& p, int grid, cudaStream_t st) {
    const bool deep = p.nst == kDeepFStages;
    if constexpr (RP <= 16) {
        const size_t smem = sreg_layout<RP, kFiberF>(p.ldT, p.nst).total;
        auto k = deep ? sreg_kernel<RP, kFiberF, kDeepFStages> : sreg_kernel<RP, kFiberF, kFStages>;
        CPFIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, 32 * SRegRoles<RP>::WARPS, smem, st>>>(p);
        CPFIT_CUDA(cudaGetLastError());
        return;
    }
    const size_t smem = spass_layout<RP, kFiberF>(p.nchunk, p.I0, p.nst).total;
    auto k = deep ? spass_kernel<RP, kFiberF, kDeepFStages> : spass_kernel<RP, kFiberF, kFStages>;
    CPFIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 32 * SPassRoles<RP>::WARPS, smem, st>>>(p);
    CPFIT_CUDA(cudaGetLastError());
}

size_t spass_smem(int RP, int nchunk, int64_t I0, int nst) {
    switch (RP) {
        case 8: return sreg_layout<8, kFiberF>(4 * ((I0 + 3) / 4), nst).total;
        case 16: return sreg_layout<16, kFiberF>(4 * ((I0 + 3) / 4), nst).total;
        default: return spass_layout<32, kFiberF>(nchunk, I0, nst).total;
    }
}
