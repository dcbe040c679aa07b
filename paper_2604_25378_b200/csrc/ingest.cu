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

// column sums of a T x ld block in two fixed-order stages (deterministic): each
// block sums one row chunk for a slice of columns (coalesced rows), then the
// chunk partials are summed in chunk order; plus a non-finite flag
__global__ void colsum_part_kernel(const double* X, long long T, int ld, int n, long long rows_per, double* part,
                                   int* bad) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const long long t0 = (long long)blockIdx.y * rows_per, t1 = min(T, t0 + rows_per);
    if (c >= n) return;
    double s = 0.0;
    int nf = 0;
    for (long long t = t0; t < t1; ++t) {
        const double v = X[t * ld + c];
        s += v;
        nf |= !isfinite(v);
    }
    part[(size_t)blockIdx.y * n + c] = s;
    if (nf) atomicOr(bad, 1);
}
__global__ void colsum_finish_kernel(const double* part, int nsplit, int n, double* sums) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double s = 0.0;
    for (int k = 0; k < nsplit; ++k) s += part[(size_t)k * n + c];
    sums[c] = s;
}

// RAII holders for the ingest's temporaries (freed on every exit path)
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};
struct PinBuf {
    void* p = nullptr;
    ~PinBuf() {
        if (p) cudaFreeHost(p);
    }
};
struct Event {
    cudaEvent_t e = nullptr;
    ~Event() {
        if (e) cudaEventDestroy(e);
    }
};

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
    PinBuf pin[2];
    Event ev[2];
    // the stream may hold this rank's earlier work; every exit path below
    // drains it before the RAII holders free what it may still touch
    struct Drain {
        cudaStream_t s;
        ~Drain() { cudaStreamSynchronize(s); }
    } drain{ctx->stream};
    for (int i = 0; i < 2; ++i) {
        MVSK_CUDA(cudaMallocHost(&pin[i].p, rows_per * row_bytes));
        MVSK_CUDA(cudaEventCreateWithFlags(&ev[i].e, cudaEventDisableTiming));
    }
    if (ld != n) MVSK_CUDA(cudaMemsetAsync(ctx->X, 0, (size_t)std::max<long long>(1, T_loc) * ld * sizeof(double), ctx->stream));
    if (std::fseek(f.get(), 12 + (long)(ctx->row0 * (long long)row_bytes), SEEK_SET) != 0)
        throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": truncated payload");
    int b = 0;
    for (long long r = 0; r < T_loc; r += rows_per, b ^= 1) {
        const long long rows = std::min(rows_per, T_loc - r);
        MVSK_CUDA(cudaEventSynchronize(ev[b].e));  // the H2D that last used this buffer is done
        if (std::fread(pin[b].p, row_bytes, (size_t)rows, f.get()) != (size_t)rows)
            throw ApiError(MVSK_DATA_ERROR, std::string(path) + ": truncated payload");
        MVSK_CUDA(cudaMemcpy2DAsync(ctx->X + r * ld, ld * sizeof(double), pin[b].p, row_bytes, row_bytes, rows,
                                    cudaMemcpyHostToDevice, ctx->stream));
        MVSK_CUDA(cudaEventRecord(ev[b].e, ctx->stream));
    }
    // global column means (allreduce of the per-shard column sums)
    const int cb = (int)((n + 127) / 128);
    const long long rows_chunk = std::max<long long>(64, (T_loc + 4LL * ctx->nsm / cb) / std::max(1, 4 * ctx->nsm / cb));
    const int nsplit = (int)std::max<long long>(1, (T_loc + rows_chunk - 1) / rows_chunk);
    DevBuf part, sums, bad;
    MVSK_CUDA(cudaMalloc(&part.p, (size_t)nsplit * n * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&sums.p, (n + 1) * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&bad.p, sizeof(int)));
    double* sp = static_cast<double*>(sums.p);
    MVSK_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
    ctx->launches += 2;
    colsum_part_kernel<<<dim3(cb, nsplit), 128, 0, ctx->stream>>>(ctx->X, T_loc, (int)ld, (int)n, rows_chunk,
                                                                  static_cast<double*>(part.p), static_cast<int*>(bad.p));
    MVSK_CUDA(cudaGetLastError());
    colsum_finish_kernel<<<cb, 128, 0, ctx->stream>>>(static_cast<double*>(part.p), nsplit, (int)n, sp);
    MVSK_CUDA(cudaGetLastError());
    int hbad = 0;
    std::vector<double> hs((size_t)n + 1, 0.0);
    // append the flag as a double so one allreduce carries both
    MVSK_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
    const double flag = hbad ? 1.0 : 0.0;
    MVSK_CUDA(cudaMemcpyAsync(sp + n, &flag, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    allreduce_sum(ctx, sp, (size_t)n + 1);
    MVSK_CUDA(cudaMemcpyAsync(hs.data(), sp, (n + 1) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hs[(size_t)n] != 0.0) throw ApiError(MVSK_DATA_ERROR, "center_panel: non-finite return entry");
    ctx->mu.resize((size_t)n);
    for (long long j = 0; j < n; ++j) ctx->mu[(size_t)j] = hs[(size_t)j] / (double)ctx->T_global;
    MVSK_CUDA(cudaMemcpyAsync(sp, ctx->mu.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ++ctx->launches;
    center_kernel<<<4 * ctx->nsm, 256, 0, ctx->stream>>>(ctx->X, T_loc, (int)ld, (int)n, sp);
    MVSK_CUDA(cudaGetLastError());
    MVSK_CUDA(cudaMemcpyAsync(ctx->mu_dev, ctx->mu.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace mvsk_b200
