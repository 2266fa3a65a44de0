// Grams in double-double, shared by the Gram pass (dense.cu) and the fused ALS solve + Gram
// update (als.cu).
//
// G_n(r, q) = sum_i A_n(i, r) A_n(i, q) over the upper-triangle pairs r <= q. Mode n's rows
// are cut into gram_chunks(I_n) chunks; one warp owns a (chunk, pair) task: lanes stride the
// chunk's rows with a dd accumulator each, then a shuffle tree adds the 32 lanes. The task
// partials are summed in chunk order and rounded once by the last block of the grid to finish
// (atomic counter) — so a Gram is the dd sum rounded, independent of the launch shape up to
// dd rounding (~1e-32 relative). Many short warp tasks keep the serial dd chains short: the
// fp64 add latency, not the flop count, bounds these R x R reductions.
#pragma once

#include "common.cuh"

namespace cpfit_gpu {

constexpr int kGramChunkRows = 128;  // 4 rows per lane
constexpr int kGramMaxChunks = 16;   // bounds the serial combine

inline int gram_chunks(int64_t In) { return (int)imin64((In + kGramChunkRows - 1) / kGramChunkRows, kGramMaxChunks); }
inline int64_t gram_chunk_rows(int64_t In) {
    const int c = gram_chunks(In);
    return (In + c - 1) / c;
}

// upper-triangle pair index p -> (r, q), r <= q < R
__device__ __forceinline__ void pair_rq(int p, int R, int& r, int& q) {
    int a = 0, start = 0;
    while (start + (R - a) <= p) {
        start += R - a;
        ++a;
    }
    r = a;
    q = a + (p - start);
}

// dd sum over rows [i0, i1) of a[i] * b[i] by one warp (lane-strided, then a fixed xor tree);
// every lane returns the total
__device__ __forceinline__ dd warp_dot_dd(const double* a, const double* b, int64_t i0, int64_t i1) {
    const int lane = threadIdx.x & 31;
    dd s{0.0, 0.0};
    // loads batched ahead of the serial dd chain (an L2 round trip per row otherwise)
    for (int64_t ib = i0 + lane; ib < i1; ib += 4 * 32) {
        double x[4], y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = ib + 32 * k;
            x[k] = i < i1 ? a[i] : 0.0;
            y[k] = i < i1 ? b[i] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (ib + 32 * k < i1) s = dd_fma(s, x[k], y[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const dd t{__shfl_xor_sync(0xffffffffu, s.hi, o), __shfl_xor_sync(0xffffffffu, s.lo, o)};
        s = dd_add(s, t);
    }
    return s;
}

// Warp task t of a mode (t = chunk * npair + pair) -> part[t] (dd partial of one chunk).
__device__ __forceinline__ void gram_task(const double* A, int64_t In, int64_t rows, int R, int t, dd* part) {
    const int npair = R * (R + 1) / 2;
    const int c = t / npair, p = t % npair;
    int r, q;
    pair_rq(p, R, r, q);
    const int64_t i0 = (int64_t)c * rows;
    const dd s = warp_dot_dd(A + (int64_t)r * In, A + (int64_t)q * In, i0, imin64(In, i0 + rows));
    if ((threadIdx.x & 31) == 0) part[t] = s;
}

// All threads call; returns true in the last block of the grid to arrive (its reads of the
// other blocks' partials are ordered after their writes). Resets the counter for reuse.
__device__ __forceinline__ bool last_block_arrives(unsigned int* counter) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        last = (atomicAdd(counter, 1u) == gridDim.x - 1);
        if (last) *counter = 0u;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// Zero the padding entries (r or q >= R) of an RP x RP Gram.
__device__ __forceinline__ void gram_zero_pads(int R, int RP, double* out) {
    for (int e = threadIdx.x; e < RP * RP; e += blockDim.x)
        if (e / RP >= R || e % RP >= R) out[e] = 0.0;
}
// Gram pair p <- rounded sum over chunks c < nchunk (in order) of part[c*npair + p]
__device__ __forceinline__ void gram_combine_pair(const dd* part, int nchunk, int p, int R, int RP, double* out) {
    const int npair = R * (R + 1) / 2;
    dd v[kGramMaxChunks];
#pragma unroll
    for (int c = 0; c < kGramMaxChunks; ++c) v[c] = (c < nchunk) ? part[(size_t)c * npair + p] : dd{0.0, 0.0};
    dd s = v[0];
#pragma unroll
    for (int c = 1; c < kGramMaxChunks; ++c)
        if (c < nchunk) s = dd_add(s, v[c]);
    int r, q;
    pair_rq(p, R, r, q);
    const double g = s.hi + s.lo;
    out[r * RP + q] = g;
    out[q * RP + r] = g;
}

}  // namespace cpfit_gpu
