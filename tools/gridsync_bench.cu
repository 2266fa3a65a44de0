// Cost of a grid-wide barrier on B200: cooperative_groups grid.sync() vs a hand-rolled
// arrive/spin barrier (one atomic per CTA, release/acquire), 148..592 CTAs of 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridsync_bench tools/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int K = 200;

__global__ void cg_sync(double* x) {
    cg::grid_group g = cg::this_grid();
    double v = x[blockIdx.x * blockDim.x + threadIdx.x];
    for (int k = 0; k < K; ++k) {
        v = v * 0.5 + 1.0;
        g.sync();
    }
    x[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

// generation barrier: bar[0] arrivals, bar[1] generation
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int gen;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1));
        const unsigned int arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) {
            atomicExch(bar, 0u);
            asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1));
        } else {
            unsigned int now;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(now) : "l"(bar + 1));
            } while (now == gen);
        }
    }
    __syncthreads();
}

__global__ void my_sync(double* x, unsigned int* bar) {
    double v = x[blockIdx.x * blockDim.x + threadIdx.x];
    for (int k = 0; k < K; ++k) {
        v = v * 0.5 + 1.0;
        grid_barrier(bar, gridDim.x);
    }
    x[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

int main() {
    double* x;
    unsigned int* bar;
    cudaMalloc(&x, sizeof(double) * 592 * 256);
    cudaMalloc(&bar, 8);
    cudaMemset(bar, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid : {148, 296, 592}) {
        void* args[] = {&x};
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void*)cg_sync, dim3(grid), dim3(256), args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %d cg grid.sync: %.3f us per barrier (%s)\n", grid, 1e3 * ms / K, cudaGetErrorString(cudaGetLastError()));
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            my_sync<<<grid, 256>>>(x, bar);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %d arrive/spin: %.3f us per barrier (%s)\n", grid, 1e3 * ms / K, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
