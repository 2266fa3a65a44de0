// Shared device helpers for the cpfit B200 path: error plumbing, double-double arithmetic,
// and the sm_100a PTX wrappers (fp64 tensor-core DMMA, mbarrier, bulk async copy).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

// Guard-band build (-DCPFIT_GUARD, `make guard`): every device allocation of the library gets
// 4 KB guard bands of a fixed byte pattern on both sides; frees and cpfit_debug_guard_check()
// verify them, so an out-of-bounds write past either end of any buffer is reported (guard.cu).
// compute-sanitizer is closed on the GPU pool this was built on; this is the substitute check.
namespace cpfit_gpu {
cudaError_t guard_malloc(void** p, size_t bytes);
cudaError_t guard_free(void* p);
}  // namespace cpfit_gpu
#if defined(CPFIT_GUARD) && !defined(CPFIT_GUARD_IMPL)
#define cudaMalloc(p, n) ::cpfit_gpu::guard_malloc(reinterpret_cast<void**>(p), (n))
#define cudaFree(p) ::cpfit_gpu::guard_free((void*)(p))
#endif

namespace cpfit_gpu {

constexpr int kMaxOrder = 8;   // tensor order supported on device
constexpr int kMaxRank = 32;   // the fibre-tile / level / polynomial kernels: R <= 32 (RP = R rounded up to 8)
constexpr int kMaxRankWide = 64;  // ranks 33..64 (RP = 64) run the per-mode ("rowwise") path
constexpr int kMaxWindow = 112;  // N-GMRES window: the 2m x m damped system of accelerate in shared memory

struct cuda_error : std::runtime_error {
    explicit cuda_error(const std::string& w) : std::runtime_error(w) {}
};
// Mirrors cpfit::numerical_error (errors.hpp:9-12).
struct numerical_error : std::runtime_error {
    explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};

#define CPFIT_CUDA(x)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            throw ::cpfit_gpu::cuda_error(std::string(#x) + ": " + cudaGetErrorString(e_) +    \
                                          " @" __FILE__ ":" + std::to_string(__LINE__));       \
    } while (0)

__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
inline int64_t round_up64(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---- double-double (error-free transforms; used for Grams and the window Gram) --------
struct dd {
    double hi, lo;
};
__host__ __device__ inline dd dd_two_sum(double a, double b) {
    double s = a + b;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    return {s, e};
}
__host__ __device__ inline dd dd_add(dd a, dd b) {
    dd s = dd_two_sum(a.hi, b.hi);
    dd t = dd_two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = dd_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return dd_two_sum(s.hi, s.lo);
}
// a += x*y exactly-ish (TwoProd via fma)
__host__ __device__ inline dd dd_fma(dd a, double x, double y) {
    double p = x * y;
    double pe = fma(x, y, -p);
    dd s = dd_two_sum(a.hi, p);
    s.lo += a.lo + pe;
    return dd_two_sum(s.hi, s.lo);
}
__host__ __device__ inline dd dd_mul(dd a, dd b) {
    double p = a.hi * b.hi;
    double e = fma(a.hi, b.hi, -p);
    e += a.hi * b.lo + a.lo * b.hi;
    return dd_two_sum(p, e);
}
__host__ __device__ inline dd dd_sub(dd a, dd b) { return dd_add(a, dd{-b.hi, -b.lo}); }
__host__ __device__ inline dd dd_div(dd a, dd b) {
    double q1 = a.hi / b.hi;
    dd r = dd_sub(a, dd_mul(b, dd{q1, 0.0}));
    double q2 = r.hi / b.hi;
    r = dd_sub(r, dd_mul(b, dd{q2, 0.0}));
    double q3 = r.hi / b.hi;
    dd q = dd_two_sum(q1, q2);
    return dd_add(q, dd{q3, 0.0});
}
__host__ __device__ inline dd dd_sqrt(dd a) {
    if (a.hi <= 0.0) return {0.0, 0.0};
    double x = sqrt(a.hi);
    dd xx = dd_mul(dd{x, 0.0}, dd{x, 0.0});
    double corr = (dd_sub(a, xx).hi) / (2.0 * x);
    return dd_two_sum(x, corr);
}

#ifdef __CUDACC__
// ---- fp64 tensor core: D(8x8) += A(8x4, row) * B(4x8, col) -----------------------------
// Fragment ownership (lane l): A[l/4][l%4], B[l%4][l/4], D[l/4][2*(l%4) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ---- mbarrier + bulk async copy (global -> shared, completes tx bytes on the mbarrier) --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// L2 eviction-priority policies for cache hints (createpolicy): the tensor is streamed once per
// pass and must not displace the L2-resident working set (S, S_d, partial sums, factors)
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// bulk_g2s with an L2 cache hint
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// 2D tensor-map copy (TMA): box at (x = column, y = row) of the map into shared memory,
// completing tx bytes on bar; out-of-bounds elements of the box arrive as zeros
__device__ __forceinline__ void tma_2d_g2s_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                                uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
        "[%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
#endif

}  // namespace cpfit_gpu
