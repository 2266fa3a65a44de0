// fp64 peak probes for the roofline denominators: DFMA loop, DMMA (mma.sync m8n8k4 f64)
// loop, both interleaved, and an fp64 streaming read. MEASURED_PEAKS.json carries no fp64
// figure, so these numbers are measured on the box.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void dmma_loop(double* out, int iters, double a, double b) {
    double d[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
    }
    double s = 0; for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.678) out[0] = s;
}

// interleave: per iteration CH dmma + CH2 dfma chains
template <int CH, int CH2>
__global__ void mixed_loop(double* out, int iters, double a, double b) {
    double d[CH][2]; double acc[CH2];
#pragma unroll
    for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
#pragma unroll
    for (int c = 0; c < CH2; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
#pragma unroll
        for (int c = 0; c < CH2; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0; for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
    for (int c = 0; c < CH2; ++c) s += acc[c];
    if (s == 12345.678) out[0] = s;
}

__global__ void stream_read(const double2* __restrict__ x, size_t n2, double* out) {
    double s = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
        double2 v = __ldcs(x + i); s += v.x + v.y;
    }
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out; CK(cudaMalloc(&out, 64));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto launch, double flops, const char* name) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        printf("%-28s %8.3f ms  %8.2f TFLOP/s\n", name, ms, flops / (ms * 1e-3) / 1e12);
    };
    const int iters = 4096;
    for (int bpsm : {1, 2, 4}) {
        int blocks = sms * bpsm, thr = 256;
        char nm[64];
        snprintf(nm, 64, "dfma x8 %dblk/sm", bpsm);
        timeit([&] { dfma_loop<8><<<blocks, thr>>>(out, iters, 1.0000001, 1e-9); },
               2.0 * 8 * iters * (double)blocks * thr, nm);
        snprintf(nm, 64, "dmma x8 %dblk/sm", bpsm);
        timeit([&] { dmma_loop<8><<<blocks, thr>>>(out, iters, 1.0000001, 1e-9); },
               2.0 * 256 * 8 * iters * (double)blocks * (thr / 32), nm);
        snprintf(nm, 64, "mixed 4dmma+8dfma %dblk/sm", bpsm);
        timeit([&] { mixed_loop<4, 8><<<blocks, thr>>>(out, iters, 1.0000001, 1e-9); },
               2.0 * 256 * 4 * iters * (double)blocks * (thr / 32) + 2.0 * 8 * iters * (double)blocks * thr, nm);
        snprintf(nm, 64, "mixed 8dmma+8dfma %dblk/sm", bpsm);
        timeit([&] { mixed_loop<8, 8><<<blocks, thr>>>(out, iters, 1.0000001, 1e-9); },
               2.0 * 256 * 8 * iters * (double)blocks * (thr / 32) + 2.0 * 8 * iters * (double)blocks * thr, nm);
    }
    size_t n = 64ull << 20;  // 64M doubles = 512 MB, the 400^3 tensor
    double2* x; CK(cudaMalloc(&x, n * 8)); CK(cudaMemset(x, 0, n * 8));
    for (int bpsm : {2, 4, 8}) {
        char nm[64]; snprintf(nm, 64, "stream read %dblk/sm", bpsm);
        for (int w = 0; w < 3; ++w) stream_read<<<sms * bpsm, 512>>>(x, n / 2, out);
        cudaEventRecord(e0); for (int r = 0; r < 10; ++r) stream_read<<<sms * bpsm, 512>>>(x, n / 2, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
        printf("%-28s %8.3f ms  %8.1f GB/s\n", nm, ms, n * 8.0 / (ms * 1e-3) / 1e9);
    }
    CK(cudaGetLastError());
    return 0;
}
