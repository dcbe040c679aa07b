// Per-call latency of the host-pointer C-ABI on a small panel (C1 shape):
// make_cache, gradient, hvp, line_model; compare with a bare stream sync.
//   nvcc -O2 -I include scripts/latency_bench.cpp -Lpaper_2604_25378_b200/_build -lmvsk_b200 -o scripts/_bin/latency_bench
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#include "mvsk_gpu.h"

int main(int argc, char** argv) {
    const long long T = argc > 1 ? atoll(argv[1]) : 500, n = argc > 2 ? atoll(argv[2]) : 20;
    std::mt19937_64 rng(1);
    std::normal_distribution<double> N(0.0, 0.01);
    std::vector<double> A((size_t)(T * n)), mu((size_t)n, 0.0);
    for (auto& a : A) a = N(rng);
    for (long long t = 0; t < T; ++t)
        for (long long j = 0; j < n; ++j) mu[(size_t)j] += A[(size_t)(t * n + j)] / (double)T;
    for (long long t = 0; t < T; ++t)
        for (long long j = 0; j < n; ++j) A[(size_t)(t * n + j)] -= mu[(size_t)j];
    mvsk_coeffs c{1.0, 5.0, 18.333333333333332, 55.0};
    mvsk_gpu_ctx* ctx = nullptr;
    if (mvsk_gpu_create(A.data(), T, n, mu.data(), &c, 0, &ctx)) {
        std::printf("create failed: %s\n", mvsk_gpu_last_error(nullptr));
        return 1;
    }
    std::vector<double> x((size_t)n, 1.0 / (double)n), g((size_t)n), v((size_t)n), hv((size_t)n), lm(14);
    for (long long j = 0; j < n; ++j) v[(size_t)j] = (j % 2 ? 1.0 : -1.0) / (double)n;
    double f = 0;
    auto bench = [&](const char* name, auto&& fn) {
        for (int i = 0; i < 20; ++i) fn();
        const int R = 2000;
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < R; ++i) fn();
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / R;
        std::printf("%-28s %8.2f us/call\n", name, us);
    };
    cudaStream_t s;
    cudaStreamCreate(&s);
    bench("cudaStreamSynchronize", [&] { cudaStreamSynchronize(s); });
    bench("empty kernel-less memcpy", [&] { cudaMemcpyAsync(hv.data(), hv.data(), 8, cudaMemcpyHostToHost, s); cudaStreamSynchronize(s); });
    bench("make_cache", [&] { mvsk_gpu_make_cache(ctx, 0, x.data(), &f); });
    bench("make_cache + gradient", [&] {
        mvsk_gpu_make_cache(ctx, 0, x.data(), &f);
        mvsk_gpu_gradient(ctx, 0, g.data());
    });
    bench("hvp", [&] { mvsk_gpu_hvp(ctx, 0, v.data(), 1, hv.data()); });
    bench("line_model", [&] { mvsk_gpu_line_model(ctx, 0, v.data(), 1.0, lm.data()); });
    mvsk_gpu_destroy(ctx);
    return 0;
}
