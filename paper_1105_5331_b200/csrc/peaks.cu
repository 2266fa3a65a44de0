// fp64 roofline denominators measured live (MEASURED_PEAKS.json carries only HBM and bf16):
// a DMMA (mma.sync m8n8k4 f64, the fp64 tensor-core path the fiber pass uses) issue loop and
// a DFMA loop, both over 148 x 4 CTAs.
#include "../../include/cpfit_gpu.h"
#include "common.cuh"

namespace {

__global__ void dmma_peak_kernel(double* out, int iters, double a, double b) {
    double d[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) cpfit_gpu::dmma_8x8x4(d[c][0], d[c][1], a, b);
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
    if (s == 1234.5678) out[0] = s;
}

__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == 1234.5678) out[0] = s;
}

}  // namespace

extern "C" int cpfit_measure_fp64_peak(double* dmma_tflops, double* dfma_tflops) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 3;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    if (cudaMalloc(&out, 64) != cudaSuccess) return 3;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, thr = 256, iters = 8192;
    auto run = [&](auto launch) {
        for (int w = 0; w < 2; ++w) launch();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / 5.0;
    };
    const double ms_m = run([&] { dmma_peak_kernel<<<blocks, thr>>>(out, iters, 1.0000001, 1e-9); });
    const double ms_f = run([&] { dfma_peak_kernel<<<blocks, thr>>>(out, iters, 1.0000001, 1e-9); });
    *dmma_tflops = 2.0 * 256 * 8 * (double)iters * blocks * (thr / 32) / (ms_m * 1e-3) / 1e12;
    *dfma_tflops = 2.0 * 8 * (double)iters * blocks * thr / (ms_f * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

extern "C" int cpfit_host_register(void* p, int64_t bytes) {
    return cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault) == cudaSuccess ? 0 : 3;
}
extern "C" int cpfit_host_unregister(void* p) { return cudaHostUnregister(p) == cudaSuccess ? 0 : 3; }
