// Device context behind the C-ABI: resident panel shard, per-slot caches,
// workspaces, stream and the NCCL communicator of the row-shard group.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mvsk_gpu.h"
#include "stream_kernels.cuh"

namespace mvsk_b200 {

struct PcgWorkspace;
struct SpgWorkspace;
struct LocalGroup;  // in-process row-shard group (collective.cu)
struct GramPcgWs;   // Gram-PCG direction workspace (gram_pcg.cu)

struct ApiError : std::runtime_error {
    int code;
    ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MVSK_CUDA(call)                                                                             \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            throw ::mvsk_b200::ApiError(MVSK_CUDA_ERROR, std::string(#call " failed: ") +           \
                                                             cudaGetErrorString(e_));               \
    } while (0)

#define MVSK_NCCL(call)                                                                              \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess)                                                                       \
            throw ::mvsk_b200::ApiError(MVSK_NCCL_ERROR, std::string(#call " failed: ") +            \
                                                             ncclGetErrorString(r_));                \
    } while (0)

struct Slot {
    double* z = nullptr;   // T_local
    double* g = nullptr;   // ld (gradient, full coordinates)
    double* sc = nullptr;  // [f, mu'x, Ez2, Ez3, Ez4, ...] (8)
    bool valid = false;
    bool grad_counted = false;
    double f = 0.0;
    double mom[4] = {0, 0, 0, 0};
    std::vector<double> x_full;  // host copy of the cached point (full coordinates)
    std::vector<double> g_host;  // host copy of the gradient (full coordinates, ld)
    bool g_host_valid = false;
    bool scalars_host_valid = false;  // f / mom mirror the device scalars
};

// Face view over the resident panel (replaces the column-gathered face panel of
// solver.hpp:343-363): vectors in face coordinates map to full coordinates with
// the pinned entries fixed (tau for iterates, 0 for directions).
struct FaceMap {
    bool active = false;
    std::vector<int64_t> idx;  // free coordinates, increasing
    double tau = 0.0;
    long long m = 0;           // vector length in face coordinates
};

}  // namespace mvsk_b200

struct mvsk_gpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    int nsm = 148;
    size_t max_smem = 227 * 1024;

    long long T_global = 0, T_local = 0, row0 = 0;
    long long n = 0, ld = 0;
    double* X = nullptr;
    bool owns_X = false;
    double* mu_dev = nullptr;  // ld, zero padded
    std::vector<double> mu;    // n
    mvsk_coeffs c{};
    double* zoff_dev = nullptr;  // T_local or null
    double value_offset = 0.0;
    double* value_offset_dev = nullptr;  // compact face contexts: the offset lives on the device

    // face selected through the C-ABI (mvsk_gpu_set_face)
    mvsk_b200::FaceMap pub_face;

    mvsk_b200::Slot slots[MVSK_GPU_MAX_SLOTS];

    // workspaces (device)
    double* vin = nullptr;  // MVSK_GPU_MAX_RHS * 2 * ld input staging
    double* part_acc = nullptr;
    size_t part_acc_elems = 0;
    double* part_sc = nullptr;
    double* red = nullptr;   // MVSK_GPU_MAX_RHS * ld + kNumScalars
    double* outd = nullptr;  // MVSK_GPU_MAX_RHS * ld output staging
    double* tvec = nullptr;  // T_local scratch (sample directions / weights)
    double* gram = nullptr;  // n x n (lazy)
    double* tvec2 = nullptr; // T_local scratch (lazy)
    double* pmat = nullptr;  // ld x ld (lazy)
    mvsk_b200::PcgWorkspace* pcg = nullptr;  // device-resident PCG buffers (lazy)
    mvsk_b200::SpgWorkspace* spg = nullptr;  // device-resident SPG preamble (lazy)
    mvsk_b200::GramPcgWs* gpcg = nullptr;     // reduced-Hessian PCG directions (lazy)
    double* gram_part = nullptr;
    size_t gram_part_elems = 0;
    // pinned host staging
    double* h_in = nullptr;
    double* h_out = nullptr;
    double* h_out_dev = nullptr;  // device alias of h_out (mapped)
    size_t h_elems = 0;
    double* h_mat = nullptr;  // pinned n x n staging (direct branch: Gram out, P in), mapped
    double* h_mat_dev = nullptr;  // device alias of h_mat
    size_t h_mat_elems = 0;

    ncclComm_t comm = nullptr;
    bool owns_comm = true;  // false for a compact face context (it borrows the parent's comm / group)
    // in-process group (mvsk_gpu_group): collective.cu's peer-memory allreduce
    // instead of NCCL; its member ops never run as captured CUDA graphs
    mvsk_b200::LocalGroup* group = nullptr;
    bool no_capture = false;
    double* ar_scratch = nullptr;
    size_t ar_scratch_elems = 0;
    cudaEvent_t ar_ev[2] = {nullptr, nullptr};
    int nranks = 1, rank = 0;
    long long ld_alloc = 0;  // row length the ld-sized workspaces were allocated for
    // compact face contexts of a solve (face.cu): the reference's face panel
    // A[:, free] with its pinned offset, gathered once per face when it pays;
    // one per power-of-two width class, kept across solves
    std::vector<mvsk_gpu_ctx*> face_pool;
    unsigned char* face_scratch = nullptr;       // child: device staging of a rebuild
    unsigned char* face_scratch_host = nullptr;  // child: pinned staging of a rebuild
    size_t face_scratch_bytes = 0;

    uint64_t fwd = 0, tr = 0, phys = 0;
    uint64_t launches = 0;  // kernels this context enqueued (graph replays included)
    std::string err;

    // host-API ops replayed as CUDA graphs (host_ops.cu); entries are dropped
    // whenever a captured device/pinned buffer may have moved (epoch)
    struct GraphEntry {
        int op, k, slot;
        uint64_t epoch;
        cudaGraphExec_t exec;
        uint64_t phys;  // physical passes one replay performs
        uint64_t launches;  // kernels one replay launches
        bool ok;
    };
    std::vector<GraphEntry> graphs;
    uint64_t epoch = 0;
};
