// Device mirror of cpfit::DataTensor (tensor.hpp:129-148): upload once, cache the norm.
//
// Dense: fibers padded to ldT = round_up(I_0, 4) so each mode-0 fiber is a 32-byte aligned
// bulk copy; ||T||^2 and the per-fiber ||t_f||^2 (used by the per-fiber objective) are
// accumulated on device in double-double.
// Sparse: the COO is canonicalised exactly like SparseTensor's constructor
// (tensor.cpp:56-103: stable lexicographic sort, duplicates summed, zeros dropped), then
// for every mode n a mode-n-sorted copy (counting sort, stable) is stored as CSR-like
// rows: rowptr (I_n+1), the other modes' indices (int32 SoA) and values. Each sparse
// MTTKRP then streams one copy with no atomics ("CSF copies per mode").
#include "device.cuh"
#include "sparse.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <memory>
#include <numeric>
#include <vector>

namespace cpfit_gpu {

namespace {

// one pass over T: per-fibre ||t_f||^2 and block partials of ||T||^2 in double-double, and the
// finite check (DenseTensor's all_finite, tensor.cpp:44-54)
__global__ void fiber_norm_kernel(const double* T, int64_t ldT, int I0, int64_t J, double* fn2, dd* block_part,
                                  int* bad) {
    __shared__ dd red[32];
    dd acc{0.0, 0.0};
    bool finite = true;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t f = gw; f < J; f += nw) {
        dd s{0.0, 0.0};
        for (int i = lane; i < I0; i += 32) {
            const double v = T[f * ldT + i];
            finite = finite && isfinite(v);
            s = dd_fma(s, v, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            dd t{__shfl_xor_sync(0xffffffffu, s.hi, o), __shfl_xor_sync(0xffffffffu, s.lo, o)};
            s = dd_add(s, t);
        }
        if (lane == 0) {
            fn2[f] = s.hi + s.lo;
            acc = dd_add(acc, s);
        }
    }
    if (!finite) atomicOr(bad, 1);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        dd t{0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = dd_add(t, red[w]);
        block_part[blockIdx.x] = t;
    }
}

void set_device_norms(DevTensor& t, cudaStream_t st) {
    const double h[3] = {t.norm, t.norm_sq, t.norm_sq_lo};
    CPFIT_CUDA(cudaMemcpyAsync(t.dscal, h, sizeof(h), cudaMemcpyHostToDevice, st));
    CPFIT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

DevTensor* tensor_create_dense(int order, const int64_t* dims, const double* host_vals, cudaStream_t st) {
    if (order < 1 || order > kMaxOrder) throw std::invalid_argument("Shape: order must be in [1, 8] on device");
    auto* t = new DevTensor();
    std::unique_ptr<DevTensor, void (*)(DevTensor*)> owner(t, tensor_destroy);  // freed if a check throws
    t->order = order;
    t->K = 1;
    for (int n = 0; n < order; ++n) {
        if (dims[n] < 1) throw std::invalid_argument("Shape: every mode size must be >= 1");
        if (t->K > std::numeric_limits<int64_t>::max() / dims[n])
            throw std::invalid_argument("Shape: element count overflows the index range");
        t->dims[n] = dims[n];
        t->K *= dims[n];
    }
    t->sparse = false;
    // shapes the fibre tiles do not take run the generic per-mode kernels (generic.cu);
    // CPFIT_FORCE_GENERIC=1 at creation selects them for any shape (tests)
    const char* fg = std::getenv("CPFIT_FORCE_GENERIC");
    t->generic = !fiber_path_fits(order, dims[0]) || (fg && fg[0] == '1');
    t->ldT = round_up64(dims[0], 4);
    t->J = t->K / dims[0];
    const size_t bytes = sizeof(double) * (size_t)t->ldT * t->J;
    CPFIT_CUDA(cudaMalloc(&t->T, bytes));
    CPFIT_CUDA(cudaMalloc(&t->fiber_norm2, sizeof(double) * t->J));
    CPFIT_CUDA(cudaMalloc(&t->dscal, sizeof(double) * 3));
    if (t->ldT != dims[0]) CPFIT_CUDA(cudaMemsetAsync(t->T, 0, bytes, st));  // pads stay zero
    tensor_fill_dense(*t, host_vals, st);
    return owner.release();
}

void tensor_fill_dense(DevTensor& t, const double* host_vals, cudaStream_t st) {
    const int64_t I0 = t.dims[0];
    if (t.ldT == I0)  // unpadded fibres: one linear copy (a pitched 2D copy runs below the link rate)
        CPFIT_CUDA(cudaMemcpyAsync(t.T, host_vals, sizeof(double) * (size_t)(I0 * t.J), cudaMemcpyHostToDevice, st));
    else
        CPFIT_CUDA(cudaMemcpy2DAsync(t.T, sizeof(double) * t.ldT, host_vals, sizeof(double) * I0, sizeof(double) * I0,
                                     t.J, cudaMemcpyHostToDevice, st));
    const int blocks = 592;
    struct Scratch {
        dd* part = nullptr;
        int* bad = nullptr;
        ~Scratch() {
            cudaFree(part);
            cudaFree(bad);
        }
    } sc;
    CPFIT_CUDA(cudaMalloc(&sc.part, sizeof(dd) * blocks));
    CPFIT_CUDA(cudaMalloc(&sc.bad, sizeof(int)));
    CPFIT_CUDA(cudaMemsetAsync(sc.bad, 0, sizeof(int), st));
    fiber_norm_kernel<<<blocks, 256, 0, st>>>(t.T, t.ldT, (int)I0, t.J, t.fiber_norm2, sc.part, sc.bad);
    CPFIT_CUDA(cudaGetLastError());
    std::vector<dd> hp(blocks);
    int hbad = 0;
    CPFIT_CUDA(cudaMemcpyAsync(hp.data(), sc.part, sizeof(dd) * blocks, cudaMemcpyDeviceToHost, st));
    CPFIT_CUDA(cudaMemcpyAsync(&hbad, sc.bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CPFIT_CUDA(cudaStreamSynchronize(st));
    if (hbad) throw std::invalid_argument("DenseTensor: entries must be finite");
    dd s{0.0, 0.0};
    for (const dd& x : hp) s = dd_add(s, x);
    t.norm_sq = s.hi + s.lo;
    t.norm_sq_lo = (s.hi - t.norm_sq) + s.lo;  // ||T||^2 = norm_sq + norm_sq_lo in double-double
    t.norm = std::sqrt(t.norm_sq);
    set_device_norms(t, st);
}

DevTensor* tensor_create_coo(int order, const int64_t* dims, int64_t nnz_in, const int64_t* coords,
                             const double* vals, cudaStream_t st) {
    if (order < 1 || order > kMaxOrder) throw std::invalid_argument("Shape: order must be in [1, 8] on device");
    auto* t = new DevTensor();
    std::unique_ptr<DevTensor, void (*)(DevTensor*)> owner(t, tensor_destroy);  // freed if a check throws
    t->order = order;
    t->sparse = true;
    t->K = 1;
    for (int n = 0; n < order; ++n) {
        if (dims[n] < 1) throw std::invalid_argument("Shape: every mode size must be >= 1");
        if (dims[n] > std::numeric_limits<int32_t>::max())
            throw std::invalid_argument("device sparse path needs mode sizes < 2^31");
        if (t->K > std::numeric_limits<int64_t>::max() / dims[n])
            throw std::invalid_argument("Shape: element count overflows the index range");
        t->dims[n] = dims[n];
        t->K *= dims[n];
    }
    const size_t N = (size_t)order;
    for (int64_t i = 0; i < nnz_in; ++i) {
        if (!std::isfinite(vals[i])) throw std::invalid_argument("SparseTensor: entries must be finite");
        for (size_t k = 0; k < N; ++k)
            if (coords[i * N + k] < 0 || coords[i * N + k] >= dims[k])
                throw std::invalid_argument("SparseTensor: coordinate out of bounds");
    }
    // canonicalise (tensor.cpp:74-102): stable lexicographic sort, sum duplicates, drop zeros.
    // Input already strictly increasing (the generators' and write_tns' output, any canonical
    // tensor read back) needs neither the sort nor the duplicate pass: one O(nnz) check.
    std::vector<int64_t> cc;
    std::vector<double> vv;
    cc.reserve((size_t)nnz_in * N);
    vv.reserve((size_t)nnz_in);
    bool increasing = true;
    for (int64_t i = 1; i < nnz_in && increasing; ++i)
        increasing = std::lexicographical_compare(coords + (i - 1) * N, coords + i * N, coords + i * N,
                                                  coords + (i + 1) * N);
    std::vector<int64_t> ord;
    if (increasing) {
        for (int64_t i = 0; i < nnz_in; ++i)
            if (vals[i] != 0.0) {
                cc.insert(cc.end(), coords + i * N, coords + i * N + N);
                vv.push_back(vals[i]);
            }
    } else {
        ord.resize((size_t)nnz_in);
        std::iota(ord.begin(), ord.end(), int64_t{0});
        std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
            return std::lexicographical_compare(coords + a * N, coords + a * N + N, coords + b * N, coords + b * N + N);
        });
    }
    for (size_t i = 0; !increasing && i < (size_t)nnz_in;) {
        double sum = vals[ord[i]];
        size_t j = i + 1;
        while (j < (size_t)nnz_in && std::equal(coords + ord[i] * N, coords + ord[i] * N + N, coords + ord[j] * N))
            sum += vals[ord[j++]];
        if (sum != 0.0) {
            cc.insert(cc.end(), coords + ord[i] * N, coords + ord[i] * N + N);
            vv.push_back(sum);
        }
        i = j;
    }
    t->nnz = (int64_t)vv.size();
    double s2 = 0.0;
    for (double v : vv) s2 += v * v;  // Eigen norm(): sqrt(squaredNorm())
    t->norm = std::sqrt(s2);
    t->norm_sq = t->norm * t->norm;
    CPFIT_CUDA(cudaMalloc(&t->dscal, sizeof(double) * 3));
    set_device_norms(*t, st);
    upload_sparse_modes(*t, cc, vv, st);
    return owner.release();
}

void tensor_destroy(DevTensor* t) {
    if (!t) return;
    cudaFree(t->T);
    cudaFree(t->fiber_norm2);
    cudaFree(t->dscal);
    free_sparse_modes(*t);
    delete t;
}

}  // namespace cpfit_gpu
