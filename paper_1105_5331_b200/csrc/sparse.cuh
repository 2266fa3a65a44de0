#pragma once

#include "device.cuh"

#include <vector>

namespace cpfit_gpu {

// Per-mode sorted copies of a canonical COO tensor.
struct SparseModes {
    int64_t* rowptr[kMaxOrder] = {};
    int32_t* oidx[kMaxOrder] = {};  // (N-1) x nnz, other modes in increasing order
    double* vals[kMaxOrder] = {};
    // order 3 with both other mode sizes <= 65536: the two other indices packed (lo | hi << 16)
    uint32_t* pidx[kMaxOrder] = {};
};


void upload_sparse_modes(DevTensor& t, const std::vector<int64_t>& coords, const std::vector<double>& vals,
                         cudaStream_t st);
void free_sparse_modes(DevTensor& t);
SparseModes* sparse_modes(const DevTensor& t);

}  // namespace cpfit_gpu
