// C-ABI implementation (include/mvsk_gpu.h): lifecycle, row sharding, the
// oracle method set of mvsk::Oracle (oracle.hpp:29-149) and line_model
// (linesearch.hpp:62-81). Host vectors cross the boundary; caches stay in HBM.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "collective.cuh"
#include "host_ops.hpp"
#include "pcg_device.hpp"

using namespace mvsk_b200;

namespace {

thread_local std::string g_err;

template <class F>
int32_t guard(mvsk_gpu_ctx* ctx, F&& f) {
    try {
        f();
        return MVSK_OK;
    } catch (const ApiError& e) {
        if (ctx) ctx->err = e.what();
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        g_err = e.what();
        return MVSK_INTERNAL_ERROR;
    }
}

void set_device(mvsk_gpu_ctx* ctx) { MVSK_CUDA(cudaSetDevice(ctx->device)); }

bool finite(const double* v, long long n) {
    for (long long i = 0; i < n; ++i)
        if (!std::isfinite(v[i])) return false;
    return true;
}

mvsk_gpu_ctx* make_ctx(long long T_local, long long row0, long long T_global, long long n, const double* mu,
                       const mvsk_coeffs* c, int device, int nranks, int rank, const void* id) {
    if (n < 1) throw ApiError(MVSK_DIMENSION_ERROR, "oracle: need at least one asset");
    // the row ring and the per-thread column accumulators of the streaming kernels hold whole rows
    if (n > MVSK_GPU_MAX_ASSETS)
        throw ApiError(MVSK_DIMENSION_ERROR, "oracle: this build supports at most " + std::to_string(MVSK_GPU_MAX_ASSETS) +
                                                 " assets (n = " + std::to_string(n) + ")");
    if (T_global < 1 || T_local < 0 || row0 < 0 || row0 + T_local > T_global)
        throw ApiError(MVSK_DIMENSION_ERROR, "oracle: bad row block");
    if (!mu || !c) throw ApiError(MVSK_DIMENSION_ERROR, "oracle: mu length does not match panel columns");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw ApiError(MVSK_DOMAIN_ERROR, "bad rank / nranks");
    int ndev = 0;
    MVSK_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ApiError(MVSK_CUDA_ERROR, "no such CUDA device");
    auto* ctx = new mvsk_gpu_ctx();
    try {
        ctx->device = device;
        MVSK_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        MVSK_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw ApiError(MVSK_CUDA_ERROR, "device is not Blackwell (sm_100a build)");
        ctx->nsm = prop.multiProcessorCount;
        ctx->max_smem = prop.sharedMemPerBlockOptin;
        MVSK_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream;
        ctx->T_local = T_local;
        ctx->T_global = T_global;
        ctx->row0 = row0;
        ctx->n = n;
        // row pitch: 16-byte rows for the bulk-copy engine; for n >= 512 a
        // multiple of 16 doubles so the tensor-core multi-RHS kernel can split
        // rows over 8-CTA clusters (<= 3 % padding, zero-filled)
        ctx->ld = n >= 512 ? (n + 15) / 16 * 16 : (n + 1) / 2 * 2;
        ctx->pub_face.m = n;
        ctx->mu.assign(mu, mu + n);
        ctx->c = *c;
        ctx->nranks = nranks;
        ctx->rank = rank;
        // a communicator is created whenever an id is given (also for a 1-rank
        // group, which runs the same allreduce path on one GPU)
        if (nranks > 1 || id) {
            if (!id) throw ApiError(MVSK_DOMAIN_ERROR, "nccl unique id required for nranks > 1");
            ncclUniqueId uid;
            std::memcpy(&uid, id, sizeof(uid));
            MVSK_NCCL(ncclCommInitRank(&ctx->comm, nranks, uid, rank));
        }
        return ctx;
    } catch (...) {
        ctx_free(ctx);
        throw;
    }
}

void upload_panel(mvsk_gpu_ctx* ctx, const double* A_rows) {
    const size_t bytes = (size_t)std::max<long long>(1, ctx->T_local) * ctx->ld * sizeof(double);
    MVSK_CUDA(cudaMalloc(&ctx->X, bytes));
    ctx->owns_X = true;
    if (ctx->T_local == 0) return;
    if (ctx->ld == ctx->n) {
        MVSK_CUDA(cudaMemcpy(ctx->X, A_rows, (size_t)ctx->T_local * ctx->n * sizeof(double), cudaMemcpyHostToDevice));
    } else {
        MVSK_CUDA(cudaMemset(ctx->X, 0, bytes));
        MVSK_CUDA(cudaMemcpy2D(ctx->X, ctx->ld * sizeof(double), A_rows, ctx->n * sizeof(double),
                               ctx->n * sizeof(double), ctx->T_local, cudaMemcpyHostToDevice));
    }
}

}  // namespace

// ============================================================================
extern "C" {

int32_t mvsk_gpu_abi_version(void) { return MVSK_GPU_ABI_VERSION; }

const char* mvsk_gpu_status_string(int32_t s) {
    switch (s) {
    case MVSK_OK: return "ok";
    case MVSK_DIMENSION_ERROR: return "dimension_error";
    case MVSK_DOMAIN_ERROR: return "domain_error";
    case MVSK_DATA_ERROR: return "data_error";
    case MVSK_NUMERIC_ERROR: return "numeric_error";
    case MVSK_CUDA_ERROR: return "cuda_error";
    case MVSK_NCCL_ERROR: return "nccl_error";
    default: return "internal_error";
    }
}

int32_t mvsk_gpu_nccl_unique_id(void* out) {
    return guard(nullptr, [&] {
        ncclUniqueId id;
        MVSK_NCCL(ncclGetUniqueId(&id));
        static_assert(sizeof(id) == MVSK_NCCL_UNIQUE_ID_BYTES, "nccl id size");
        std::memcpy(out, &id, sizeof(id));
    });
}

int32_t mvsk_gpu_create(const double* A, int64_t T, int64_t n, const double* mu, const mvsk_coeffs* c,
                        int32_t device, mvsk_gpu_ctx** out) {
    return mvsk_gpu_create_sharded(A, T, 0, T, n, mu, c, device, 1, 0, nullptr, out);
}

int32_t mvsk_gpu_create_sharded(const double* A_rows, int64_t T_local, int64_t row0, int64_t T_global, int64_t n,
                                const double* mu, const mvsk_coeffs* c, int32_t device, int32_t nranks,
                                int32_t rank, const void* nccl_unique_id, mvsk_gpu_ctx** out) {
    return guard(nullptr, [&] {
        if (!out) throw ApiError(MVSK_DOMAIN_ERROR, "null out");
        *out = nullptr;
        mvsk_gpu_ctx* ctx = make_ctx(T_local, row0, T_global, n, mu, c, device, nranks, rank, nccl_unique_id);
        try {
            upload_panel(ctx, A_rows);
            ctx_alloc_workspaces(ctx);
        } catch (...) {
            ctx_free(ctx);
            throw;
        }
        *out = ctx;
    });
}

namespace {
__global__ void padding_check_kernel(const double* X, long long T, long long ld, long long n, int* flag) {
    const long long w = ld - n, cells = T * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cells; e += (long long)gridDim.x * blockDim.x) {
        const long long t = e / w, j = n + (e - t * w);
        if (!isfinite(X[t * ld + j])) *flag = 1;
    }
}
}  // namespace

struct mvsk_gpu_group {
    mvsk_b200::LocalGroup* g = nullptr;
};

int32_t mvsk_gpu_group_create(int32_t nranks, mvsk_gpu_group** out) {
    return guard(nullptr, [&] {
        if (!out) throw ApiError(MVSK_DOMAIN_ERROR, "null out");
        *out = nullptr;
        auto* grp = new mvsk_gpu_group();
        grp->g = group_new(nranks);
        *out = grp;
    });
}

int32_t mvsk_gpu_group_destroy(mvsk_gpu_group* group) {
    return guard(nullptr, [&] {
        if (!group) return;
        if (group_live(group->g) != 0)
            throw ApiError(MVSK_DOMAIN_ERROR, "group_destroy: member contexts are still alive");
        group_delete(group->g);
        delete group;
    });
}

int32_t mvsk_gpu_create_sharded_in_group(const double* A_rows, int64_t T_local, int64_t row0, int64_t T_global,
                                         int64_t n, const double* mu, const mvsk_coeffs* c, int32_t device,
                                         mvsk_gpu_group* group, int32_t rank, mvsk_gpu_ctx** out) {
    return guard(nullptr, [&] {
        if (!out) throw ApiError(MVSK_DOMAIN_ERROR, "null out");
        *out = nullptr;
        if (!group) throw ApiError(MVSK_DOMAIN_ERROR, "null group");
        mvsk_gpu_ctx* ctx = make_ctx(T_local, row0, T_global, n, mu, c, device, 1, 0, nullptr);
        try {
            upload_panel(ctx, A_rows);
            ctx_alloc_workspaces(ctx);
            group_join(group->g, ctx, rank);
        } catch (...) {
            ctx_free(ctx);
            throw;
        }
        *out = ctx;
    });
}

int32_t mvsk_gpu_create_from_device(const double* A_dev, int64_t ld, int64_t T_local, int64_t row0,
                                    int64_t T_global, int64_t n, const double* mu, const mvsk_coeffs* c,
                                    int32_t device, int32_t nranks, int32_t rank, const void* nccl_unique_id,
                                    mvsk_gpu_ctx** out) {
    return guard(nullptr, [&] {
        if (!out) throw ApiError(MVSK_DOMAIN_ERROR, "null out");
        *out = nullptr;
        if (ld < n || (ld & 1) || (reinterpret_cast<uintptr_t>(A_dev) & 15))
            throw ApiError(MVSK_DIMENSION_ERROR, "device panel needs even ld >= n and a 16-byte aligned base");
        mvsk_gpu_ctx* ctx = make_ctx(T_local, row0, T_global, n, mu, c, device, nranks, rank, nccl_unique_id);
        try {
            ctx->ld = ld;
            ctx->X = const_cast<double*>(A_dev);
            ctx->owns_X = false;
            ctx_alloc_workspaces(ctx);
            // the streaming kernels read whole ld-wide rows and multiply the
            // padding columns [n, ld) by zero weights: 0 * NaN would poison
            // every result, so non-finite padding is rejected up front
            if (ld > n && T_local > 0) {
                int* flag = nullptr;
                MVSK_CUDA(cudaMalloc(&flag, sizeof(int)));
                MVSK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
                const long long cells = (long long)T_local * (ld - n);
                const int nb = (int)std::min<long long>(4LL * ctx->nsm, (cells + 255) / 256);
                padding_check_kernel<<<nb, 256, 0, ctx->stream>>>(A_dev, T_local, ld, n, flag);
                int h = 0;
                const cudaError_t e1 = cudaGetLastError();
                const cudaError_t e2 = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
                const cudaError_t e3 = cudaStreamSynchronize(ctx->stream);
                cudaFree(flag);
                MVSK_CUDA(e1);
                MVSK_CUDA(e2);
                MVSK_CUDA(e3);
                if (h) throw ApiError(MVSK_DATA_ERROR, "device panel: non-finite values in the padding columns [n, ld)");
            }
        } catch (...) {
            ctx_free(ctx);
            throw;
        }
        *out = ctx;
    });
}

}  // extern "C"

namespace mvsk_b200 {
struct BinaryHeader {
    long long T = 0, n = 0;
};
BinaryHeader read_binary_header(const char* path);
void ingest_binary(mvsk_gpu_ctx* ctx, const char* path);
}  // namespace mvsk_b200

extern "C" {

int32_t mvsk_gpu_binary_dims(const char* path, int64_t* T, int64_t* n) {
    return guard(nullptr, [&] {
        const auto h = read_binary_header(path);
        if (T) *T = h.T;
        if (n) *n = h.n;
    });
}

int32_t mvsk_gpu_create_from_binary(const char* path, const mvsk_coeffs* c, int32_t device, int32_t nranks,
                                    int32_t rank, const void* nccl_unique_id, mvsk_gpu_ctx** out) {
    return guard(nullptr, [&] {
        if (!out) throw ApiError(MVSK_DOMAIN_ERROR, "null out");
        *out = nullptr;
        const auto h = read_binary_header(path);
        if (nranks < 1 || rank < 0 || rank >= nranks) throw ApiError(MVSK_DOMAIN_ERROR, "bad rank / nranks");
        const long long row0 = h.T * rank / nranks, T_loc = h.T * (rank + 1) / nranks - row0;
        std::vector<double> mu0((size_t)h.n, 0.0);
        mvsk_gpu_ctx* ctx = make_ctx(T_loc, row0, h.T, h.n, mu0.data(), c, device, nranks, rank, nccl_unique_id);
        try {
            const size_t bytes = (size_t)std::max<long long>(1, ctx->T_local) * ctx->ld * sizeof(double);
            MVSK_CUDA(cudaMalloc(&ctx->X, bytes));
            ctx->owns_X = true;
            ctx_alloc_workspaces(ctx);
            ingest_binary(ctx, path);
        } catch (...) {
            ctx_free(ctx);
            throw;
        }
        *out = ctx;
    });
}

int32_t mvsk_gpu_mu(const mvsk_gpu_ctx* ctx, double* mu_out) {
    std::memcpy(mu_out, ctx->mu.data(), ctx->mu.size() * sizeof(double));
    return MVSK_OK;
}

int32_t mvsk_gpu_launch_count(const mvsk_gpu_ctx* ctx, uint64_t* launches) {
    if (!ctx || !launches) return MVSK_DOMAIN_ERROR;
    *launches = ctx->launches;
    return MVSK_OK;
}

int32_t mvsk_gpu_destroy(mvsk_gpu_ctx* ctx) {
    ctx_free(ctx);
    return MVSK_OK;
}

const char* mvsk_gpu_last_error(const mvsk_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int32_t mvsk_gpu_set_stream(mvsk_gpu_ctx* ctx, void* stream) {
    return guard(ctx, [&] {
        set_device(ctx);
        MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    });
}

int32_t mvsk_gpu_synchronize(mvsk_gpu_ctx* ctx) {
    return guard(ctx, [&] { MVSK_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int32_t mvsk_gpu_dims(const mvsk_gpu_ctx* ctx, int64_t* T_global, int64_t* T_local, int64_t* n) {
    if (T_global) *T_global = ctx->T_global;
    if (T_local) *T_local = ctx->T_local;
    if (n) *n = ctx->n;
    return MVSK_OK;
}

int32_t mvsk_gpu_set_offset(mvsk_gpu_ctx* ctx, const double* zoff, double value_offset) {
    return guard(ctx, [&] {
        set_device(ctx);
        // *_device ops return without a host sync: a pass still in flight on
        // ctx->stream may be reading zoff_dev, so drain the stream first
        MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
        if (zoff) {
            if (!ctx->zoff_dev)
                MVSK_CUDA(cudaMalloc(&ctx->zoff_dev, (size_t)std::max<long long>(1, ctx->T_local) * sizeof(double)));
            MVSK_CUDA(cudaMemcpy(ctx->zoff_dev, zoff, ctx->T_local * sizeof(double), cudaMemcpyHostToDevice));
        } else if (ctx->zoff_dev) {
            MVSK_CUDA(cudaFree(ctx->zoff_dev));
            ctx->zoff_dev = nullptr;
        }
        ctx->value_offset = value_offset;
        ++ctx->epoch;  // the z offset pointer / value offset are baked into captured passes
        for (auto& s : ctx->slots) s.valid = false;
    });
}

int32_t mvsk_gpu_set_face(mvsk_gpu_ctx* ctx, const int64_t* free_idx, int64_t nf, double tau) {
    return guard(ctx, [&] {
        if (nf < 1 || nf > ctx->n) throw ApiError(MVSK_DOMAIN_ERROR, "degenerate face, all coordinates pinned");
        FaceMap f;
        f.tau = tau;
        f.m = nf;
        if (nf == ctx->n && !free_idx) {
            f.active = false;
        } else {
            if (!free_idx) throw ApiError(MVSK_DOMAIN_ERROR, "face needs free indices");
            f.idx.assign(free_idx, free_idx + nf);
            for (long long j = 0; j < nf; ++j)
                if (f.idx[j] < 0 || f.idx[j] >= ctx->n || (j && f.idx[j] <= f.idx[j - 1]))
                    throw ApiError(MVSK_DOMAIN_ERROR, "free indices must be increasing and in range");
            f.active = nf != ctx->n;
        }
        ctx->pub_face = f;
        for (auto& s : ctx->slots) s.valid = false;
    });
}

int32_t mvsk_gpu_make_cache(mvsk_gpu_ctx* ctx, int32_t slot, const double* x, double* f_out) {
    return guard(ctx, [&] {
        set_device(ctx);
        const double f = op_make_cache(ctx, slot, ctx->pub_face, x);
        if (f_out) *f_out = f;
    });
}

int32_t mvsk_gpu_value(mvsk_gpu_ctx* ctx, int32_t slot, double* f_out) {
    return guard(ctx, [&] {
        *f_out = op_value(ctx, slot);
    });
}

int32_t mvsk_gpu_moments(mvsk_gpu_ctx* ctx, int32_t slot, double out[4]) {
    return guard(ctx, [&] { op_moments(ctx, slot, out); });
}

int32_t mvsk_gpu_gradient(mvsk_gpu_ctx* ctx, int32_t slot, double* g_out) {
    return guard(ctx, [&] {
        set_device(ctx);
        op_gradient(ctx, slot, ctx->pub_face, g_out);
    });
}

int32_t mvsk_gpu_hvp(mvsk_gpu_ctx* ctx, int32_t slot, const double* V, int32_t k, double* HV) {
    return guard(ctx, [&] {
        set_device(ctx);
        op_hvp(ctx, slot, ctx->pub_face, V, k, HV);
    });
}

int32_t mvsk_gpu_third_action(mvsk_gpu_ctx* ctx, int32_t slot, const double* U, const double* V, int32_t k,
                              double* out) {
    return guard(ctx, [&] {
        set_device(ctx);
        op_third(ctx, slot, ctx->pub_face, U, V, k, out);
    });
}

int32_t mvsk_gpu_hessian_diag_weights(mvsk_gpu_ctx* ctx, int32_t slot, double* out) {
    return guard(ctx, [&] {
        set_device(ctx);
        op_psi2(ctx, slot, out);
    });
}

int32_t mvsk_gpu_sample_direction(mvsk_gpu_ctx* ctx, const double* d, double* out) {
    return guard(ctx, [&] {
        set_device(ctx);
        op_sample_direction(ctx, ctx->pub_face, d, out);
    });
}

int32_t mvsk_gpu_line_model(mvsk_gpu_ctx* ctx, int32_t slot, const double* d, double cap, double out[14]) {
    (void)cap;  // alpha_cap only parameterises the host-side minimisation
    return guard(ctx, [&] {
        set_device(ctx);
        op_line_model(ctx, slot, ctx->pub_face, d, out);
    });
}

int32_t mvsk_gpu_line_models(mvsk_gpu_ctx* ctx, int32_t slot, const double* D, int32_t k, double* out) {
    return guard(ctx, [&] {
        set_device(ctx);
        op_line_models(ctx, slot, ctx->pub_face, D, k, out);
        ctx->fwd += (uint64_t)k;
    });
}

int32_t mvsk_gpu_weighted_gram(mvsk_gpu_ctx* ctx, int32_t slot, double* G_out) {
    return guard(ctx, [&] {
        set_device(ctx);
        op_weighted_gram(ctx, slot, ctx->pub_face, G_out);
    });
}

int32_t mvsk_gpu_weighted_gram_device(mvsk_gpu_ctx* ctx, int32_t slot, double* G_dev) {
    return guard(ctx, [&] {
        set_device(ctx);
        check_slot(ctx, slot);
        run_weighted_gram(ctx, nullptr, G_dev, 1.0 / (double)ctx->T_global, ctx->slots[slot].z);
        ctx->fwd += 1;
    });
}

int32_t mvsk_gpu_passes(const mvsk_gpu_ctx* ctx, uint64_t* forward, uint64_t* transpose, uint64_t* physical) {
    if (forward) *forward = ctx->fwd;
    if (transpose) *transpose = ctx->tr;
    if (physical) *physical = ctx->phys;
    return MVSK_OK;
}

int32_t mvsk_gpu_reset_passes(mvsk_gpu_ctx* ctx) {
    ctx->fwd = ctx->tr = ctx->phys = 0;
    return MVSK_OK;
}

// ---- device-resident fast path ---------------------------------------------
int32_t mvsk_gpu_make_cache_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* x_dev) {
    return guard(ctx, [&] {
        set_device(ctx);
        check_slot(ctx, slot, false);
        if (ctx->pub_face.active) throw ApiError(MVSK_DOMAIN_ERROR, "device path works on the full problem (no face)");
        MVSK_CUDA(cudaMemcpyAsync(ctx->vin, x_dev, ctx->n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        PassIO io;
        io.vin = ctx->vin;
        io.slot = slot;
        io.x_for_mux = ctx->vin;
        run_pass(ctx, Op::FGRAD, 1, io);
        ctx->fwd += 1;
        ctx->slots[slot].valid = true;  // scalars stay on device (slot sc)
        ctx->slots[slot].g_host_valid = false;
        ctx->slots[slot].scalars_host_valid = false;
        ctx->slots[slot].grad_counted = false;
    });
}

int32_t mvsk_gpu_hvp_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* V_dev, int32_t k, double* HV_dev) {
    return guard(ctx, [&] {
        set_device(ctx);
        check_slot(ctx, slot);
        if (k < 1 || k > MVSK_GPU_MAX_RHS) throw ApiError(MVSK_DIMENSION_ERROR, "hvp: k out of range");
        const double* vin = V_dev;
        if (ctx->ld != ctx->n) {
            MVSK_CUDA(cudaMemcpy2DAsync(ctx->vin, ctx->ld * sizeof(double), V_dev, ctx->n * sizeof(double),
                                        ctx->n * sizeof(double), k, cudaMemcpyDeviceToDevice, ctx->stream));
            vin = ctx->vin;
        }
        PassIO io;
        io.vin = vin;
        io.z = ctx->slots[slot].z;
        io.out = HV_dev;
        io.ldo = ctx->n;
        run_pass(ctx, Op::HVP, k, io);
        ctx->fwd += k;
        ctx->tr += k;
    });
}

int32_t mvsk_gpu_third_action_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* U_dev, const double* V_dev,
                                     int32_t k, double* out_dev) {
    return guard(ctx, [&] {
        set_device(ctx);
        check_slot(ctx, slot);
        if (k < 1 || k > MVSK_GPU_MAX_RHS) throw ApiError(MVSK_DIMENSION_ERROR, "third_action: k out of range");
        const double* u = U_dev;
        const double* v = V_dev;
        if (ctx->ld != ctx->n) {
            MVSK_CUDA(cudaMemcpy2DAsync(ctx->vin, ctx->ld * sizeof(double), U_dev, ctx->n * sizeof(double),
                                        ctx->n * sizeof(double), k, cudaMemcpyDeviceToDevice, ctx->stream));
            MVSK_CUDA(cudaMemcpy2DAsync(ctx->vin + (size_t)MVSK_GPU_MAX_RHS * ctx->ld, ctx->ld * sizeof(double), V_dev,
                                        ctx->n * sizeof(double), ctx->n * sizeof(double), k, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
            u = ctx->vin;
            v = ctx->vin + (size_t)MVSK_GPU_MAX_RHS * ctx->ld;
        }
        PassIO io;
        io.vin = u;
        io.vin2 = v;
        io.z = ctx->slots[slot].z;
        io.out = out_dev;
        io.ldo = ctx->n;
        run_pass(ctx, Op::THIRD, k, io);
        ctx->fwd += 2 * k;
        ctx->tr += k;
    });
}

int32_t mvsk_gpu_line_sums_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* d_dev, double* sums_dev) {
    return guard(ctx, [&] {
        set_device(ctx);
        check_slot(ctx, slot);
        const double* d = d_dev;
        if (ctx->ld != ctx->n) {
            MVSK_CUDA(cudaMemcpyAsync(ctx->vin, d_dev, ctx->n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
            d = ctx->vin;
        }
        PassIO io;
        io.vin = d;
        io.z = ctx->slots[slot].z;
        io.out = sums_dev;
        run_pass(ctx, Op::LINESUMS, 1, io);
        ctx->fwd += 1;
    });
}

int32_t mvsk_gpu_slot_pointers(mvsk_gpu_ctx* ctx, int32_t slot, double** z, double** grad, double** scalars) {
    return guard(ctx, [&] {
        check_slot(ctx, slot, false);
        if (z) *z = ctx->slots[slot].z;
        if (grad) *grad = ctx->slots[slot].g;
        if (scalars) *scalars = ctx->slots[slot].sc;
    });
}

}  // extern "C"
