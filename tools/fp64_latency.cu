// Dependent-chain latency (cycles per op) of fp64 arithmetic on the current GPU, one thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

template <int OP>
__global__ void chain(double* out, double a, double b, long long* cyc) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        if (OP == 0) x = fma(x, b, a);        // DFMA
        if (OP == 1) x = x + b;               // DADD
        if (OP == 2) x = x * b;               // DMUL
        if (OP == 3) x = sqrt(x) + a;         // sqrt (+ add)
        if (OP == 4) x = rsqrt(x) + a;        // rsqrt (+ add)
        if (OP == 5) x = b / x + a;           // IEEE division (+ add)
        if (OP == 6) x = __drcp_rn(x) + a;    // reciprocal (+ add)
        if (OP == 7) x = __shfl_sync(0xffffffffu, x, 0) + b;  // shuffle (+ add)
        if (OP == 8) {                                         // DMMA m8n8k4 accumulator chain
            double d1 = 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(x), "+d"(d1)
                         : "d"(a), "d"(b));
            x += d1 * 0.0;
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const char* names[] = {"dfma", "dadd", "dmul", "sqrt+add", "rsqrt+add", "div+add", "rcp+add", "shfl+add",
                           "dmma+dfma"};
    for (int op = 0; op < 9; ++op) {
        long long h = 0;
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: chain<0><<<1, 32>>>(out, 1e-3, 0.999, cyc); break;
                case 1: chain<1><<<1, 32>>>(out, 1e-3, 1e-9, cyc); break;
                case 2: chain<2><<<1, 32>>>(out, 1.0, 1.0000001, cyc); break;
                case 3: chain<3><<<1, 32>>>(out, 2.0, 1.0, cyc); break;
                case 4: chain<4><<<1, 32>>>(out, 2.0, 1.0, cyc); break;
                case 5: chain<5><<<1, 32>>>(out, 1.5, 3.0, cyc); break;
                case 6: chain<6><<<1, 32>>>(out, 1.5, 3.0, cyc); break;
                case 7: chain<7><<<1, 32>>>(out, 1.5, 1e-9, cyc); break;
                case 8: chain<8><<<1, 32>>>(out, 1e-3, 1e-3, cyc); break;
            }
            cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        }
        printf("%-10s %7.1f cycles/op\n", names[op], (double)h / N);
    }
    return 0;
}
