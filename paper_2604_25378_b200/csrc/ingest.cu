// Panel ingest straight into (row-sharded) device memory: the reference's
// binary panel format (panel_io.hpp:121-141: magic "MVSK", u32 T, u32 n,
// T*n little-endian f64 row-major raw returns R) read block-wise through pinned
// staging into this rank's rows, then centred on the device with the GLOBAL
// column means (center_panel, panel.hpp:32-44; the column sums are allreduced
// over the row-shard group), with the reference's non-finite check.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>

#include "host_ops.hpp"

namespace mvsk_b200 {
namespace {

// column sums of a T x ld block (one thread per column, rows in order) and a
// non-finite flag
__global__ void colsum_kernel(const double* X, long long T, int ld, int n, double* sums, int* bad) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double s = 0.0;
    int nf = 0;
    for (long long t = 0; t < T; ++t) {
        const double v = X[t * ld + c];
        s += v;
        nf |= !isfinite(v);
    }
    sums[c] = s;
    if (nf) atomicOr(bad, 1);
}

__global__ void center_kernel(double* X, long long T, int ld, int n, const double* mu) {
    const long long tot = T * (long long)ld;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % ld);
        if (c < n) X[i] -= mu[c];
    }
}

struct FileCloser {
    void operator()(FILE* f) const {
        if (f) std::fclose(f);
    }
};

}  // namespace

struct BinaryHeader {
    long long T = 0, n = 0;
};

// panel_io.hpp:123-134 (header checks) — host side, no device needed
BinaryHeader read_binary_header(const char* path) {
    std::unique_ptr<FILE, FileCloser> f(std::fopen(path, "rb"));
    if (!f) throw ApiError(MVSK_DATA_ERROR, std::string("cannot open returns file: ") + path);
    char magic[4];
    if (std::fread(magic, 1, 4, f.get()) != 4 || std::memcmp(magic, "MVSK", 4) != 0)
        throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": bad magic, not a binary panel file");
    uint32_t T = 0, n = 0;
    if (std::fread(&T, 4, 1, f.get()) != 1 || std::fread(&n, 4, 1, f.get()) != 1)
        throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": truncated header");
    if (T < 2 || n < 1) throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": degenerate dimensions in header");
    std::fseek(f.get(), 0, SEEK_END);
    const long long size = std::ftell(f.get());
    if (size < 12 + 8LL * T * n) throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": truncated payload");
    BinaryHeader h;
    h.T = T;
    h.n = n;
    return h;
}

// Reads rows [row0, row0 + T_local) of the file into ctx->X (ld-padded) and
// centres them with the global column means; fills ctx->mu / mu_dev.
void ingest_binary(mvsk_gpu_ctx* ctx, const char* path) {
    std::unique_ptr<FILE, FileCloser> f(std::fopen(path, "rb"));
    if (!f) throw ApiError(MVSK_DATA_ERROR, std::string("cannot open returns file: ") + path);
    const long long n = ctx->n, ld = ctx->ld, T_loc = ctx->T_local;
    const size_t row_bytes = (size_t)n * sizeof(double);
    // pinned double buffer of ~16 MB row blocks
    const long long rows_per = std::max<long long>(1, (16LL << 20) / (long long)row_bytes);
    double* pin[2] = {nullptr, nullptr};
    cudaEvent_t ev[2];
    MVSK_CUDA(cudaMallocHost(&pin[0], rows_per * row_bytes));
    MVSK_CUDA(cudaMallocHost(&pin[1], rows_per * row_bytes));
    MVSK_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    MVSK_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    bool ok = true;
    std::string err;
    try {
        if (ld != n) MVSK_CUDA(cudaMemsetAsync(ctx->X, 0, (size_t)std::max<long long>(1, T_loc) * ld * sizeof(double), ctx->stream));
        if (std::fseek(f.get(), 12 + (long)(ctx->row0 * (long long)row_bytes), SEEK_SET) != 0)
            throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": truncated payload");
        int b = 0;
        for (long long r = 0; r < T_loc; r += rows_per, b ^= 1) {
            const long long rows = std::min(rows_per, T_loc - r);
            MVSK_CUDA(cudaEventSynchronize(ev[b]));  // the H2D that last used this buffer is done
            if (std::fread(pin[b], row_bytes, (size_t)rows, f.get()) != (size_t)rows)
                throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": truncated payload");
            MVSK_CUDA(cudaMemcpy2DAsync(ctx->X + r * ld, ld * sizeof(double), pin[b], row_bytes, row_bytes, rows,
                                        cudaMemcpyHostToDevice, ctx->stream));
            MVSK_CUDA(cudaEventRecord(ev[b], ctx->stream));
        }
        // global column means (allreduce of the per-shard column sums)
        double* sums = nullptr;
        int* bad = nullptr;
        MVSK_CUDA(cudaMalloc(&sums, (n + 1) * sizeof(double)));
        MVSK_CUDA(cudaMalloc(&bad, sizeof(int)));
        MVSK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
        ++ctx->launches;
        colsum_kernel<<<(int)((n + 127) / 128), 128, 0, ctx->stream>>>(ctx->X, T_loc, (int)ld, (int)n, sums, bad);
        MVSK_CUDA(cudaGetLastError());
        int hbad = 0;
        std::vector<double> hs((size_t)n + 1, 0.0);
        // append the flag as a double so one allreduce carries both
        MVSK_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
        const double flag = hbad ? 1.0 : 0.0;
        MVSK_CUDA(cudaMemcpyAsync(sums + n, &flag, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        allreduce_sum(ctx, sums, (size_t)n + 1);
        MVSK_CUDA(cudaMemcpyAsync(hs.data(), sums, (n + 1) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
        if (hs[(size_t)n] != 0.0) {
            cudaFree(sums);
            cudaFree(bad);
            throw ApiError(MVSK_DATA_ERROR, "center_panel: non-finite return entry");
        }
        ctx->mu.resize((size_t)n);
        for (long long j = 0; j < n; ++j) ctx->mu[(size_t)j] = hs[(size_t)j] / (double)ctx->T_global;
        MVSK_CUDA(cudaMemcpyAsync(sums, ctx->mu.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        ++ctx->launches;
        center_kernel<<<4 * ctx->nsm, 256, 0, ctx->stream>>>(ctx->X, T_loc, (int)ld, (int)n, sums);
        MVSK_CUDA(cudaGetLastError());
        MVSK_CUDA(cudaMemcpyAsync(ctx->mu_dev, ctx->mu.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
        cudaFree(sums);
        cudaFree(bad);
    } catch (const std::exception& e) {
        ok = false;
        err = e.what();
        cudaStreamSynchronize(ctx->stream);
        cudaFreeHost(pin[0]);
        cudaFreeHost(pin[1]);
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        throw;
    }
    cudaFreeHost(pin[0]);
    cudaFreeHost(pin[1]);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    (void)ok;
}

}  // namespace mvsk_b200
