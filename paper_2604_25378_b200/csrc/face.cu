// Compact face panels for the solve driver (solver.hpp:343-370).
//
// The reference rebuilds, at every pin/release event, a face oracle over the
// gathered panel Af = A[:, free] with the pinned contribution folded into a
// per-sample offset zoff = tau * sum_{pinned i} A[:, i] and the value offset
// -c1 * mu_pin (here: zoff = A d with d = tau on the pinned columns, one
// streaming pass, summed in the pass's fixed order). On the device the face can instead stay an index map over
// the resident panel (host_ops.cu FaceMap): no gather, but every face pass then
// streams all n columns. Once most assets are pinned (C4: 53 of 5000 free after
// the identification pass) that is ~100x the bytes the face needs, so the
// driver switches to a compact face context when the face is small enough:
// one gather of the free columns + one pass for zoff per rebuild, after which
// every face pass streams T x nf. The child context shares the parent's device,
// stream and communicator (row-sharded groups gather their own rows) and has
// its own slots, workspaces and graphs; it is reused while the face fits.
#include <algorithm>
#include <cstring>
#include <vector>

#include "host_ops.hpp"
#include "oracle_ops.cuh"
#include "pcg_device.hpp"

namespace mvsk_b200 {
namespace {

// Xf[t, j] = X[t, idx[j]] (j < nf), zero padding up to ldf
__global__ void face_gather_kernel(const double* __restrict__ X, long long T, long long ld,
                                   const long long* __restrict__ idx, int nf, int ldf, double* __restrict__ Xf) {
    const long long tot = T * (long long)ldf;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
         e += (long long)gridDim.x * blockDim.x) {
        const long long t = e / ldf;
        const int j = (int)(e - t * ldf);
        Xf[e] = j < nf ? X[t * ld + idx[j]] : 0.0;
    }
}

long long face_ld(long long n) { return n >= 512 ? (n + 15) / 16 * 16 : (n + 1) / 2 * 2; }

// a child context (no panel yet) with the parent's device / stream / group
mvsk_gpu_ctx* make_child(mvsk_gpu_ctx* p, long long n_cap) {
    auto* c = new mvsk_gpu_ctx();
    try {
        c->device = p->device;
        c->stream = p->stream;
        c->own_stream = nullptr;
        c->nsm = p->nsm;
        c->max_smem = p->max_smem;
        c->T_global = p->T_global;
        c->T_local = p->T_local;
        c->row0 = p->row0;
        c->n = n_cap;
        c->ld = face_ld(n_cap);
        c->mu.assign((size_t)n_cap, 0.0);
        c->c = p->c;
        c->comm = p->comm;
        c->group = p->group;
        c->no_capture = p->no_capture;
        c->owns_comm = false;
        c->nranks = p->nranks;
        c->rank = p->rank;
        c->pub_face.m = n_cap;
        const size_t bytes = (size_t)std::max<long long>(1, c->T_local) * c->ld * sizeof(double);
        MVSK_CUDA(cudaMalloc(&c->X, bytes));
        c->owns_X = true;
        MVSK_CUDA(cudaMalloc(&c->zoff_dev, (size_t)std::max<long long>(1, c->T_local) * sizeof(double)));
        ctx_alloc_workspaces(c);
        return c;
    } catch (...) {
        ctx_free(c);
        throw;
    }
}

}  // namespace

mvsk_gpu_ctx* face_context(mvsk_gpu_ctx* p, const std::vector<int64_t>& free_idx, const std::vector<char>& pinned,
                           double tau) {
    const long long nf = (long long)free_idx.size();
    const long long n0 = p->n;
    // The child has a fixed width n_cap >= nf (zero columns past nf, zero mu):
    // its shapes, buffers and therefore its captured graphs survive face
    // rebuilds; only the panel data, zoff and the device-side value offset
    // change. Widths are power-of-two classes (<= 2x the face), one child per
    // class, kept in the parent's pool across faces and solves.
    long long cap = 64;
    while (cap < nf) cap <<= 1;
    cap = std::min(cap, n0);
    mvsk_gpu_ctx* c = nullptr;
    for (mvsk_gpu_ctx* q : p->face_pool)
        if (q->n == cap) c = q;
    if (!c) {
        c = make_child(p, cap);
        MVSK_CUDA(cudaMalloc(&c->value_offset_dev, sizeof(double)));
        p->face_pool.push_back(c);
    }
    const long long ncap = c->n;
    // follow the parent's stream and coefficients; coefficients are baked into
    // the child's captured graphs, so a change makes them stale (epoch)
    c->stream = p->stream;
    if (std::memcmp(&c->c, &p->c, sizeof(mvsk_coeffs)) != 0) {
        c->c = p->c;
        ++c->epoch;
    }
    std::fill(c->mu.begin(), c->mu.end(), 0.0);
    double mu_pin = 0.0;
    for (long long i = 0, j = 0; i < n0; ++i) {
        if (!pinned[(size_t)i]) {
            c->mu[(size_t)j++] = p->mu[(size_t)i];
        } else {
            mu_pin += tau * p->mu[(size_t)i];  // solver.hpp:360
        }
    }
    c->value_offset = -p->c.c1 * mu_pin;  // solver.hpp:363
    for (auto& s : c->slots) {
        s.valid = false;
        s.g_host_valid = false;
        s.scalars_host_valid = false;
    }

    // device work on the shared stream: idx / mask / mu / offset upload, gather, zoff
    const size_t b_idx = ((size_t)nf * sizeof(long long) + 15) / 16 * 16, b_mu = (size_t)c->ld * sizeof(double);
    const size_t b_d = (size_t)p->ld * sizeof(double);
    const size_t need = b_idx + b_mu + 16 + b_d;
    std::vector<unsigned char> host(need, 0);
    std::memcpy(host.data(), free_idx.data(), (size_t)nf * sizeof(long long));
    std::memcpy(host.data() + b_idx, c->mu.data(), (size_t)ncap * sizeof(double));
    std::memcpy(host.data() + b_idx + b_mu, &c->value_offset, sizeof(double));
    // d = tau on the pinned columns: zoff = A d is tau * sum_{pinned} A[:, i]
    // (solver.hpp:359), one streaming pass over the panel
    double* dh = reinterpret_cast<double*>(host.data() + b_idx + b_mu + 16);
    for (long long i = 0; i < n0; ++i) dh[i] = pinned[(size_t)i] ? tau : 0.0;
    // persistent device / pinned staging in the child (sized for the widest face
    // it can hold against this parent): no allocation per rebuild
    if (c->face_scratch_bytes < need) {
        if (c->face_scratch) MVSK_CUDA(cudaFree(c->face_scratch));
        if (c->face_scratch_host) MVSK_CUDA(cudaFreeHost(c->face_scratch_host));
        c->face_scratch = nullptr;
        c->face_scratch_host = nullptr;
        c->face_scratch_bytes = 0;
        MVSK_CUDA(cudaMalloc(&c->face_scratch, need));
        MVSK_CUDA(cudaMallocHost(&c->face_scratch_host, need));
        c->face_scratch_bytes = need;
    }
    std::memcpy(c->face_scratch_host, host.data(), need);
    unsigned char* dbuf = c->face_scratch;
    MVSK_CUDA(cudaMemcpyAsync(dbuf, c->face_scratch_host, need, cudaMemcpyHostToDevice, p->stream));
    const long long* didx = reinterpret_cast<const long long*>(dbuf);
    MVSK_CUDA(cudaMemcpyAsync(c->mu_dev, dbuf + b_idx, b_mu, cudaMemcpyDeviceToDevice, p->stream));
    MVSK_CUDA(cudaMemcpyAsync(c->value_offset_dev, dbuf + b_idx + b_mu, sizeof(double), cudaMemcpyDeviceToDevice,
                              p->stream));
    const double* d_dev = reinterpret_cast<const double*>(dbuf + b_idx + b_mu + 16);
    if (p->T_local > 0) {
        const int nb = 4 * p->nsm;
        ++p->launches;
        face_gather_kernel<<<nb, 256, 0, p->stream>>>(p->X, p->T_local, p->ld, didx, (int)nf, (int)c->ld, c->X);
        MVSK_CUDA(cudaGetLastError());
        // the fused line-sums pass writes A d per sample (its nine power sums,
        // against a zeroed z, are discarded)
        MVSK_CUDA(cudaMemsetAsync(p->tvec, 0, (size_t)p->T_local * sizeof(double), p->stream));
        PassIO io;
        io.vin = d_dev;
        io.z = p->tvec;
        io.zout = c->zoff_dev;
        io.out = p->outd;
        run_pass(p, Op::LINESUMS, 1, io);
    }
    MVSK_CUDA(cudaStreamSynchronize(p->stream));  // the pinned staging is reused by the next rebuild
    return c;
}

FaceMap face_child_map(const mvsk_gpu_ctx* c, long long nf) {
    // the face's nf coordinates are the child's first nf columns; the padding
    // columns are zero (panel and mu), so their fill value never matters
    FaceMap fm;
    fm.m = nf;
    fm.tau = 0.0;
    fm.active = nf != c->n;
    if (fm.active)
        for (long long j = 0; j < nf; ++j) fm.idx.push_back(j);
    return fm;
}

void fold_face_counters(mvsk_gpu_ctx* p) {
    for (mvsk_gpu_ctx* c : p->face_pool) {
        p->fwd += c->fwd;
        p->tr += c->tr;
        p->phys += c->phys;
        p->launches += c->launches;
        c->fwd = c->tr = c->phys = c->launches = 0;
    }
}

}  // namespace mvsk_b200
