// Per-boundary cost of a chain of small dependent kernels captured in a CUDA graph, with and
// without programmatic dependent launch (PDL: griddepcontrol.launch_dependents at kernel start,
// griddepcontrol.wait before the first dependent read).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_bench tools/pdl_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(double* x, int n, int pdl) {
    if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (i < n) x[i] = x[i] * 0.999 + 1.0;
}

int main() {
    const int n = 148 * 256, chain = 64;
    double* x;
    cudaMalloc(&x, sizeof(double) * n);
    cudaMemset(x, 0, sizeof(double) * n);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int grid : {1, 148, 592}) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaGraph_t g;
            cudaGraphExec_t gx;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
            for (int k = 0; k < chain; ++k) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl ? 1 : 0;
                cudaLaunchKernelEx(&cfg, step, x, grid * 256 < n ? grid * 256 : n, pdl);
            }
            cudaStreamEndCapture(st, &g);
            if (cudaGraphInstantiate(&gx, g, 0) != cudaSuccess) {
                printf("instantiate failed\n");
                return 1;
            }
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int w = 0; w < 3; ++w) cudaGraphLaunch(gx, st);
            cudaEventRecord(e0, st);
            const int reps = 20;
            for (int w = 0; w < reps; ++w) cudaGraphLaunch(gx, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("grid %4d pdl %d: %.2f us per kernel\n", grid, pdl, 1e3 * ms / reps / chain);
            cudaGraphExecDestroy(gx);
            cudaGraphDestroy(g);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
