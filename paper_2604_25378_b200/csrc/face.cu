// Compact face panels for the solve driver (solver.hpp:343-370).
//
// The reference rebuilds, at every pin/release event, a face oracle over the
// gathered panel Af = A[:, free] with the pinned contribution folded into a
// per-sample offset zoff = tau * sum_{pinned i, ascending} A[:, i] and the value
// offset -c1 * mu_pin. On the device the face can instead stay an index map over
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

// zoff[t] = sum over pinned columns in ascending order of tau * X[t, i]: the
// reference's `zoff += tau * A.col(i)` (solver.hpp:359), a separately rounded
// product and sum per column (no contraction). One warp per row: lanes load 32
// consecutive columns, the running sum walks them in column order.
__global__ void face_zoff_kernel(const double* __restrict__ X, long long T, long long ld, int n0,
                                 const unsigned char* __restrict__ pinned, double tau, double* __restrict__ zoff) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long t = warp; t < T; t += nwarps) {
        const double* row = X + t * ld;
        double acc = 0.0;
        for (int c0 = 0; c0 < n0; c0 += 32) {
            const int c = c0 + lane;
            const double v = c < n0 ? row[c] : 0.0;
            const unsigned pm = __ballot_sync(0xffffffffu, c < n0 && pinned[c]);
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const double vj = __shfl_sync(0xffffffffu, v, j);
                if (pm & (1u << j)) acc = __dadd_rn(acc, __dmul_rn(tau, vj));
            }
        }
        if (lane == 0) zoff[t] = acc;
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
    mvsk_gpu_ctx* c = p->face_child;
    // The child keeps a fixed width n_cap >= nf (zero columns past nf, zero mu):
    // its shapes, buffers and therefore its captured graphs survive face
    // rebuilds; only the panel data, zoff and the device-side value offset
    // change. A new child is made when the face outgrows it or shrinks to less
    // than half of it (passes would stream mostly zero columns).
    if (c && (nf > c->n || 2 * (nf + 32) < c->n)) {
        fold_face_counters(p);
        ctx_free(c);
        c = p->face_child = nullptr;
    }
    if (!c) {
        const long long cap = std::min<long long>(n0, nf + nf / 4 + 16);
        c = p->face_child = make_child(p, cap);
        MVSK_CUDA(cudaMalloc(&c->value_offset_dev, sizeof(double)));
    }
    const long long ncap = c->n;
    c->c = p->c;
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
    const size_t b_idx = (size_t)nf * sizeof(long long), b_mu = (size_t)c->ld * sizeof(double);
    const size_t need = b_idx + b_mu + sizeof(double) + (size_t)n0 + 64;
    std::vector<unsigned char> host(need, 0);
    std::memcpy(host.data(), free_idx.data(), b_idx);
    std::memcpy(host.data() + b_idx, c->mu.data(), (size_t)ncap * sizeof(double));
    std::memcpy(host.data() + b_idx + b_mu, &c->value_offset, sizeof(double));
    unsigned char* mask = host.data() + b_idx + b_mu + sizeof(double);
    for (long long i = 0; i < n0; ++i) mask[i] = pinned[(size_t)i] ? 1 : 0;
    unsigned char* dbuf = nullptr;
    MVSK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dbuf), need, p->stream));
    MVSK_CUDA(cudaMemcpyAsync(dbuf, host.data(), need, cudaMemcpyHostToDevice, p->stream));
    const long long* didx = reinterpret_cast<const long long*>(dbuf);
    MVSK_CUDA(cudaMemcpyAsync(c->mu_dev, dbuf + b_idx, b_mu, cudaMemcpyDeviceToDevice, p->stream));
    MVSK_CUDA(cudaMemcpyAsync(c->value_offset_dev, dbuf + b_idx + b_mu, sizeof(double), cudaMemcpyDeviceToDevice,
                              p->stream));
    const unsigned char* dmask = dbuf + b_idx + b_mu + sizeof(double);
    if (p->T_local > 0) {
        const int nb = 4 * p->nsm;
        ++p->launches;
        face_gather_kernel<<<nb, 256, 0, p->stream>>>(p->X, p->T_local, p->ld, didx, (int)nf, (int)c->ld, c->X);
        MVSK_CUDA(cudaGetLastError());
        ++p->launches;
        face_zoff_kernel<<<nb, 256, 0, p->stream>>>(p->X, p->T_local, p->ld, (int)n0, dmask, tau, c->zoff_dev);
        MVSK_CUDA(cudaGetLastError());
        p->phys += 1;  // the zoff sweep streams the whole panel once
    }
    MVSK_CUDA(cudaFreeAsync(dbuf, p->stream));
    MVSK_CUDA(cudaStreamSynchronize(p->stream));  // `host` is stack-local
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
    mvsk_gpu_ctx* c = p->face_child;
    if (!c) return;
    p->fwd += c->fwd;
    p->tr += c->tr;
    p->phys += c->phys;
    p->launches += c->launches;
    c->fwd = c->tr = c->phys = c->launches = 0;
}

}  // namespace mvsk_b200
