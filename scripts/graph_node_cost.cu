// Host-visible latency of small CUDA-graph shapes (what a host-API oracle op
// pays around its kernels): memcpy nodes vs mapped pinned memory.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a scripts/graph_node_cost.cu -o scripts/_bin/graph_node_cost
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(const double* in, double* out, int n) {
    int i = threadIdx.x;
    if (i < n) out[i] = in[i] * 2.0;
}
__global__ void tiny_flag(const double* in, double* out, int n, volatile int* flag, int v) {
    int i = threadIdx.x;
    if (i < n) out[i] = in[i] * 2.0;
    __syncthreads();
    if (i == 0) {
        __threadfence_system();
        *flag = v;
    }
}

// every CTA reads the same n-vector (the op's input row) and writes one value
__global__ void readers(const double* in, double* out, int n) {
    double s = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += in[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out + blockIdx.x % 8, s);
}
__global__ void writer(const double* in, double* out, int n) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) out[i] = in[i];
}

int main() {
    const int n = 128;
    double *h_in, *h_out, *d_in, *d_out, *m_in, *m_out;
    int* m_flag;
    cudaHostAlloc(&h_in, 4096, cudaHostAllocDefault);
    cudaHostAlloc(&h_out, 4096, cudaHostAllocDefault);
    cudaHostAlloc(&m_in, 4096, cudaHostAllocMapped);
    cudaHostAlloc(&m_out, 4096, cudaHostAllocMapped);
    cudaHostAlloc(&m_flag, 64, cudaHostAllocMapped);
    double *dm_in, *dm_out;
    int* dm_flag;
    cudaHostGetDevicePointer(&dm_in, m_in, 0);
    cudaHostGetDevicePointer(&dm_out, m_out, 0);
    cudaHostGetDevicePointer(&dm_flag, m_flag, 0);
    cudaMalloc(&d_in, 4096);
    cudaMalloc(&d_out, 4096);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto capture = [&](auto&& body) {
        cudaGraph_t g;
        cudaGraphExec_t e;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        body();
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&e, g, 0);
        return e;
    };
    auto bench = [&](const char* name, auto&& fn) {
        for (int i = 0; i < 200; ++i) fn(i);
        const int R = 5000;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < R; ++i) fn(i);
        double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / R;
        std::printf("%-58s %7.2f us\n", name, us);
    };
    cudaGraphExec_t g1 = capture([&] { tiny<<<1, 128, 0, s>>>(d_in, d_out, n); });
    cudaGraphExec_t g2 = capture([&] {
        cudaMemcpyAsync(d_in, h_in, n * 8, cudaMemcpyHostToDevice, s);
        tiny<<<1, 128, 0, s>>>(d_in, d_out, n);
        cudaMemcpyAsync(h_out, d_out, 40, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(h_out + 8, d_out, n * 8, cudaMemcpyDeviceToHost, s);
    });
    cudaGraphExec_t g3 = capture([&] {
        cudaMemcpyAsync(d_in, h_in, n * 8, cudaMemcpyHostToDevice, s);
        tiny<<<1, 128, 0, s>>>(d_in, d_out, n);
        cudaMemcpyAsync(h_out, d_out, n * 8, cudaMemcpyDeviceToHost, s);
    });
    cudaGraphExec_t g4 = capture([&] { tiny<<<1, 128, 0, s>>>(dm_in, dm_out, n); });
    cudaGraphExec_t g5 = capture([&] {
        tiny<<<1, 128, 0, s>>>(dm_in, d_out, n);
        tiny<<<1, 128, 0, s>>>(d_out, d_in, n);
        tiny<<<1, 128, 0, s>>>(d_in, dm_out, n);
    });
    cudaGraphExec_t g6 = capture([&] {
        tiny<<<1, 128, 0, s>>>(d_in, d_out, n);
        tiny<<<1, 128, 0, s>>>(d_out, d_in, n);
        tiny<<<1, 128, 0, s>>>(d_in, d_out, n);
    });
    bench("graph(kernel) + sync", [&](int) { cudaGraphLaunch(g1, s); cudaStreamSynchronize(s); });
    bench("graph(H2D, kernel, D2H 40B, D2H 1KB) + sync", [&](int) { cudaGraphLaunch(g2, s); cudaStreamSynchronize(s); });
    bench("graph(H2D, kernel, D2H 1KB) + sync", [&](int) { cudaGraphLaunch(g3, s); cudaStreamSynchronize(s); });
    bench("graph(kernel mapped in/out) + sync", [&](int) { cudaGraphLaunch(g4, s); cudaStreamSynchronize(s); });
    bench("graph(3 kernels, mapped in/out) + sync", [&](int) { cudaGraphLaunch(g5, s); cudaStreamSynchronize(s); });
    bench("graph(3 kernels) + sync", [&](int) { cudaGraphLaunch(g6, s); cudaStreamSynchronize(s); });
    bench("kernel launch (no graph) mapped + sync", [&](int) { tiny<<<1, 128, 0, s>>>(dm_in, dm_out, n); cudaStreamSynchronize(s); });
    bench("kernel mapped + host spin on mapped flag", [&](int i) {
        tiny_flag<<<1, 128, 0, s>>>(dm_in, dm_out, n, dm_flag, i + 1);
        while (*(volatile int*)m_flag != i + 1) {
        }
    });
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    bench("graph(kernel mapped) + event record + spin query", [&](int) {
        cudaGraphLaunch(g4, s);
        cudaEventRecord(ev, s);
        while (cudaEventQuery(ev) != cudaSuccess) {
        }
    });
    {
        double *mbig, *dmbig, *dbig, *dacc;
        cudaHostAlloc(&mbig, 1 << 20, cudaHostAllocMapped);
        cudaHostGetDevicePointer(&dmbig, mbig, 0);
        cudaMalloc(&dbig, 1 << 20);
        cudaMalloc(&dacc, 64);
        for (int nn : {20, 128, 1024, 5000}) {
            for (int grid : {32, 148}) {
                cudaGraphExec_t a = capture([&] { readers<<<grid, 128, 0, s>>>(dmbig, dacc, nn); });
                cudaGraphExec_t b = capture([&] {
                    cudaMemcpyAsync(dbig, mbig, nn * 8, cudaMemcpyHostToDevice, s);
                    readers<<<grid, 128, 0, s>>>(dbig, dacc, nn);
                });
                char name[128];
                std::snprintf(name, sizeof name, "n=%d grid=%d: kernel reads mapped", nn, grid);
                bench(name, [&](int) { cudaGraphLaunch(a, s); cudaStreamSynchronize(s); });
                std::snprintf(name, sizeof name, "n=%d grid=%d: H2D node + kernel reads device", nn, grid);
                bench(name, [&](int) { cudaGraphLaunch(b, s); cudaStreamSynchronize(s); });
            }
            cudaGraphExec_t c = capture([&] { writer<<<8, 256, 0, s>>>(dbig, dmbig, nn); });
            cudaGraphExec_t d = capture([&] {
                writer<<<8, 256, 0, s>>>(dbig, dbig + 65536, nn);
                cudaMemcpyAsync(mbig, dbig + 65536, nn * 8, cudaMemcpyDeviceToHost, s);
            });
            char name[128];
            std::snprintf(name, sizeof name, "n=%d: kernel writes mapped", nn);
            bench(name, [&](int) { cudaGraphLaunch(c, s); cudaStreamSynchronize(s); });
            std::snprintf(name, sizeof name, "n=%d: kernel writes device + D2H node", nn);
            bench(name, [&](int) { cudaGraphLaunch(d, s); cudaStreamSynchronize(s); });
        }
    }
    cudaStream_t s2;
    cudaStreamCreate(&s2);  // blocking stream
    bench("kernel (default-flag stream) + sync", [&](int) { tiny<<<1, 128, 0, s2>>>(d_in, d_out, n); cudaStreamSynchronize(s2); });
    return 0;
}
