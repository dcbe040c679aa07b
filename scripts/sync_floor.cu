// Host<->device round-trip floor on this box: launch + sync variants for a
// tiny kernel (what every host-API oracle call pays once).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a scripts/sync_floor.cu -o scripts/_bin/sync_floor
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(double* out, unsigned long long* flag, unsigned long long seq) {
    if (threadIdx.x == 0) {
        out[0] = (double)seq;
        __threadfence_system();
        *(volatile unsigned long long*)flag = seq;
    }
}
__global__ void k_dev(double* out, unsigned long long seq) {
    if (threadIdx.x == 0) out[0] = (double)seq;
}

int main() {
    cudaSetDeviceFlags(cudaDeviceMapHost);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double *hout, *dout;
    unsigned long long* hflag;
    cudaHostAlloc(&hout, 64, cudaHostAllocMapped);
    cudaHostAlloc(&hflag, 64, cudaHostAllocMapped);
    double* dmap;
    unsigned long long* dflag;
    cudaHostGetDevicePointer(&dmap, hout, 0);
    cudaHostGetDevicePointer(&dflag, hflag, 0);
    cudaMalloc(&dout, 64);
    *hflag = 0;
    auto bench = [&](const char* name, auto&& fn) {
        for (int i = 0; i < 200; ++i) fn(i);
        const int R = 5000;
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < R; ++i) fn(1000 + i);
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / R;
        std::printf("%-44s %8.2f us/call\n", name, us);
    };
    unsigned long long seq = 1;
    bench("kernel + cudaStreamSynchronize", [&](int) { k_dev<<<1, 32, 0, s>>>(dout, seq++); cudaStreamSynchronize(s); });
    bench("kernel + D2H 8B + cudaStreamSynchronize", [&](int) {
        k_dev<<<1, 32, 0, s>>>(dout, seq++);
        cudaMemcpyAsync(hout, dout, 8, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
    });
    bench("kernel -> mapped pinned, host spin on flag", [&](int) {
        const unsigned long long my = ++seq;
        k_write<<<1, 32, 0, s>>>(dmap, dflag, my);
        while (*(volatile unsigned long long*)hflag != my) {
        }
    });
    // graph of (kernel, D2H)
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_dev<<<1, 32, 0, s>>>(dout, 7);
    cudaMemcpyAsync(hout, dout, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    bench("graph(kernel, D2H) + cudaStreamSynchronize", [&](int) { cudaGraphLaunch(ge, s); cudaStreamSynchronize(s); });
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_write<<<1, 32, 0, s>>>(dmap, dflag, 0);
    cudaStreamEndCapture(s, &g2);
    cudaGraphInstantiate(&ge2, g2, 0);
    bench("graph(kernel->mapped) + cudaStreamSynchronize", [&](int) { cudaGraphLaunch(ge2, s); cudaStreamSynchronize(s); });
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    bench("kernel + event record + spin on cudaEventQuery", [&](int) {
        k_dev<<<1, 32, 0, s>>>(dout, seq++);
        cudaEventRecord(ev, s);
        while (cudaEventQuery(ev) == cudaErrorNotReady) {
        }
    });
    return 0;
}
