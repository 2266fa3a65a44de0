// DMMA m8n8k4 issue rate per SM vs warps per scheduler: one CTA of W warps on one SM, each warp
// issuing N DMMAs round-robin over C independent accumulators. Prints cycles per DMMA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_issue tools/dmma_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 2048;

template <int C>
__global__ void issue(double* out, double a, double b, long long* cyc) {
    double acc[C][2];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; i += C) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1])
                         : "d"(a), "d"(b));
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int warps) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
        issue<C><<<1, 32 * warps>>>(out, 1e-3, 1e-3, cyc);
        cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    }
    const double total = (double)N * warps;
    printf("warps %2d (%.2f per scheduler) chains %2d: %6.2f cycles per DMMA per SM, %6.1f cycles per DMMA per warp\n",
           warps, warps / 4.0, C, (double)h / total, (double)h / N);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 2, 4, 8, 12, 16}) {
        run<4>(w);
        run<8>(w);
        run<16>(w);
    }
    return 0;
}
