// DMMA m8n8k4 f64 rate per SM when each DMMA's A fragment comes from shared memory (one
// LDS.64 per DMMA, as in the register-B S pass) vs all operands in registers; W warps per CTA,
// one CTA on one SM. Prints cycles per DMMA per SM (peak: 4, i.e. 16 cycles per SMSP).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_mix tools/dmma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;  // DMMAs per warp

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int MODE>  // 0: registers only; 1: A from smem (2 groups, 4 chains each)
__global__ void run(double* out, long long* cyc) {
    __shared__ double t[16 * 372];
    for (int e = threadIdx.x; e < 16 * 372; e += blockDim.x) t[e] = 1e-3 * (e % 7);
    double b[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) b[u] = 1e-3 * (threadIdx.x + u);
    double acc[2][4][2] = {};
    const int lane = threadIdx.x & 31;
    const double* ta0 = t + (lane >> 2) * 372 + (lane & 3);
    const double* ta1 = ta0 + 8 * 372;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N / 32; ++it) {
#pragma unroll
        for (int u0 = 0; u0 < 16; u0 += 4) {
            double a0[4], a1[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (MODE == 1) {
                    a0[j] = ta0[((u0 + j + it) & 63) * 4 % 368];
                    a1[j] = ta1[((u0 + j + it) & 63) * 4 % 368];
                } else {
                    a0[j] = b[(u0 + j + 1) & 15];
                    a1[j] = b[(u0 + j + 2) & 15];
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                dmma(acc[0][j][0], acc[0][j][1], a0[j], b[u0 + j]);
                dmma(acc[1][j][0], acc[1][j][1], a1[j], b[u0 + j]);
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += acc[g][j][0] + acc[g][j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void go(int warps) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
        run<MODE><<<1, 32 * warps>>>(out, cyc);
        cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    }
    printf("mode %d warps %2d: %6.2f cycles per DMMA per SM\n", MODE, warps, (double)h / ((double)N * warps));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {4, 8, 12, 16}) {
        go<0>(w);
        go<1>(w);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
