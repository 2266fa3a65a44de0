// DMMA m8n8k4 throughput when its fragments come from shared memory (as in the fibre passes):
// per DMMA 0, 1 or 2 fragment loads (LDS.64, conflict-free pattern), W warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_smem tools/dmma_smem.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int LOADS, int CH>
__global__ void k(double* out, int iters) {
    __shared__ double sm[6144];
    for (int i = threadIdx.x; i < 6144; i += blockDim.x) sm[i] = 1e-3 * (i & 15);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* pa = sm + (warp * 256 + (lane >> 2) * 20 + (lane & 3)) % 3000;
    const double* pb = sm + 4096 + (lane >> 2) + 8 * (lane & 3);
    double acc[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
    double ra = 1.0, rb = 0.5;
    for (int it = 0; it < iters; ++it) {
        double a[CH], b[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int o = ((it * CH + c) * 4) & 255;
            a[c] = LOADS >= 1 ? pa[o] : ra;
            b[c] = LOADS >= 2 ? pb[o * 8 & 1023] : rb;
        }
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1])
                         : "d"(a[c]), "d"(b[c]));
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
    if (s == 1.2345) out[0] = s;
}

template <int LOADS, int CH>
void run(int warps, double* d) {
    const int iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<LOADS, CH><<<148, 32 * warps>>>(d, iters);
    cudaEventRecord(e0);
    k<LOADS, CH><<<148, 32 * warps>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * warps * iters * CH * 512.0;
    printf("loads/DMMA %d  chains %d  warps/SM %2d : %.2f TFLOP/s\n", LOADS, CH, warps, flops / (ms * 1e-3) / 1e12);
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    for (int w : {4, 8, 12, 16}) {
        run<0, 8>(w, d);
        run<1, 8>(w, d);
        run<2, 8>(w, d);
    }
    return 0;
}
