// Microbenchmark: fp64 FMA pipe (DFMA) vs fp64 tensor pipe (DMMA.8x8x4) peak on
// this GPU, alone and interleaved (are the pipes separate?). Prints TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MODE>  // 0 = DFMA only, 1 = DMMA only, 2 = both
__global__ void bench(double* out, int iters, double seed) {
    double a = seed + threadIdx.x * 1e-9, b = 1.0000001;
    double f[16];
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = a + i;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = a * i;
    for (int it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 16; ++i) f[i] = fma(f[i], b, 1e-12);
        }
        if (MODE != 0) {
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;
}

template <int MODE>
double run(int blocks, int threads, int iters) {
    double* out;
    cudaMalloc(&out, 8);
    bench<MODE><<<blocks, threads>>>(out, 10, 1.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<MODE><<<blocks, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    const double warps = (double)blocks * threads / 32;
    double flops = 0;
    if (MODE != 1) flops += (double)blocks * threads * iters * 64 * 2;   // 64 DFMA per thread-iter
    if (MODE != 0) flops += warps * iters * 16 * 512;                    // 16 DMMA (8x8x4 = 256 FMA) per warp-iter
    return flops / (ms * 1e-3) / 1e12;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = nsm * 4, threads = 256, iters = 20000;
    const double t0 = run<0>(blocks, threads, iters);
    const double t1 = run<1>(blocks, threads, iters);
    const double t2 = run<2>(blocks, threads, iters);
    printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"both_tflops\": %.2f, \"sms\": %d}\n", t0, t1, t2, nsm);
    return 0;
}
