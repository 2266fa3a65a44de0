// DMMA m8n8k4 issue rate vs independent accumulator chains per warp and warps per SM sub-partition
// (how much ILP one warp needs to keep the fp64 tensor pipe busy).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_chains tools/dmma_chains.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, double a, double b, int iters) {
    double x[C][2];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c][0] = x[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(x[c][0]), "+d"(x[c][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c][0] + x[c][1];
    if (s == 1.2345) out[0] = s;
}

template <int C>
void run(int warps_per_cta, double* d) {
    const int iters = 4096 / C * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<C><<<148, 32 * warps_per_cta>>>(d, 1.0, 1e-9, iters);
    cudaEventRecord(e0);
    chains<C><<<148, 32 * warps_per_cta>>>(d, 1.0, 1e-9, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * warps_per_cta * iters * C * 512.0;
    printf("chains %2d  warps/SMSP %d : %.2f TFLOP/s\n", C, warps_per_cta / 4, flops / (ms * 1e-3) / 1e12);
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    for (int w : {4, 8, 16}) {
        run<1>(w, d);
        run<2>(w, d);
        run<4>(w, d);
        run<8>(w, d);
        run<16>(w, d);
    }
    return 0;
}
