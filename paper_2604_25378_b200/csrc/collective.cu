// The row-shard group's one collective: an fp64 sum-allreduce of a device
// buffer (every oracle op is "local pass + one allreduce").
//
// Two transports behind one call:
//  * NCCL (one process per GPU, the SPMD production layout): ncclAllReduce on
//    the context's stream;
//  * an in-process group (mvsk_gpu_group): nranks contexts driven by nranks
//    host threads of ONE process, on one or several devices. Every rank reads
//    every member's buffer directly (same-device memory or NVLink peer
//    access) and sums them in rank order into its own scratch, so all ranks
//    hold identical bits, then copies the sum back. Ordering is by CUDA events
//    exchanged at two host rendezvous per call — no kernel ever waits on
//    another rank's kernel, so ranks sharing one GPU cannot deadlock. This is
//    what lets the N > 1 code paths (do_epi = 0 passes, split finish, packed
//    Gram exchange, SPMD solve driver) run and be checked on a single GPU.
#include <chrono>
#include <condition_variable>
#include <mutex>

#include "collective.cuh"

namespace mvsk_b200 {

struct LocalGroup {
    explicit LocalGroup(int n) : nranks(n), members((size_t)n), joined((size_t)n, 0) {}
    const int nranks;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t phase = 0;
    struct Member {
        const double* buf = nullptr;
        cudaEvent_t ready = nullptr, done = nullptr;
        int device = 0;
    };
    std::vector<Member> members;
    std::vector<char> joined;
    int live = 0;

    // host rendezvous of all ranks; a rank that never arrives (it failed)
    // turns into an error instead of a hang
    void rendezvous() {
        std::unique_lock<std::mutex> l(mu);
        const uint64_t ph = phase;
        if (++arrived == nranks) {
            arrived = 0;
            ++phase;
            cv.notify_all();
            return;
        }
        if (!cv.wait_for(l, std::chrono::seconds(300), [&] { return phase != ph; }))
            throw ApiError(MVSK_INTERNAL_ERROR, "in-process group: a rank did not reach the collective");
    }
};

namespace {
constexpr int kMaxGroup = 8;
struct PeerBufs {
    const double* p[kMaxGroup];
};

// out[i] = sum over ranks, in rank order (identical bits on every rank)
__global__ void group_sum_kernel(PeerBufs b, int nr, double* __restrict__ out, long long cnt) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
        double s = b.p[0][i];
        for (int r = 1; r < nr; ++r) s += b.p[r][i];
        out[i] = s;
    }
}

void group_allreduce(mvsk_gpu_ctx* ctx, double* buf, size_t cnt) {
    LocalGroup& g = *ctx->group;
    const int r = ctx->rank;
    if (ctx->ar_scratch_elems < cnt) {
        if (ctx->ar_scratch) MVSK_CUDA(cudaFree(ctx->ar_scratch));
        ctx->ar_scratch = nullptr;
        MVSK_CUDA(cudaMalloc(&ctx->ar_scratch, cnt * sizeof(double)));
        ctx->ar_scratch_elems = cnt;
    }
    for (auto& e : ctx->ar_ev)
        if (!e) MVSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MVSK_CUDA(cudaEventRecord(ctx->ar_ev[0], ctx->stream));
    {
        std::lock_guard<std::mutex> l(g.mu);
        g.members[(size_t)r] = {buf, ctx->ar_ev[0], ctx->ar_ev[1], ctx->device};
    }
    g.rendezvous();  // every member's buffer pointer and ready event are published
    PeerBufs pb{};
    for (int q = 0; q < g.nranks; ++q) {
        pb.p[q] = g.members[(size_t)q].buf;
        if (q != r) MVSK_CUDA(cudaStreamWaitEvent(ctx->stream, g.members[(size_t)q].ready, 0));
    }
    const int nb = (int)std::min<long long>((long long)ctx->nsm * 4, ((long long)cnt + 255) / 256);
    ++ctx->launches;
    group_sum_kernel<<<std::max(nb, 1), 256, 0, ctx->stream>>>(pb, g.nranks, ctx->ar_scratch, (long long)cnt);
    MVSK_CUDA(cudaGetLastError());
    MVSK_CUDA(cudaEventRecord(ctx->ar_ev[1], ctx->stream));
    g.rendezvous();  // every member has enqueued its read of all buffers
    for (int q = 0; q < g.nranks; ++q)
        if (q != r) MVSK_CUDA(cudaStreamWaitEvent(ctx->stream, g.members[(size_t)q].done, 0));
    MVSK_CUDA(cudaMemcpyAsync(buf, ctx->ar_scratch, cnt * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
}
}  // namespace

bool is_sharded(const mvsk_gpu_ctx* ctx) { return ctx->comm != nullptr || ctx->group != nullptr; }

void allreduce_sum(mvsk_gpu_ctx* ctx, double* buf, size_t cnt) {
    if (cnt == 0) return;
    if (ctx->comm) {
        MVSK_NCCL(ncclAllReduce(buf, buf, cnt, ncclFloat64, ncclSum, ctx->comm, ctx->stream));
    } else if (ctx->group) {
        group_allreduce(ctx, buf, cnt);
    }
}

LocalGroup* group_new(int nranks) {
    if (nranks < 1 || nranks > kMaxGroup) throw ApiError(MVSK_DOMAIN_ERROR, "in-process group: 1 <= nranks <= 8");
    return new LocalGroup(nranks);
}

void group_join(LocalGroup* g, mvsk_gpu_ctx* ctx, int rank) {
    if (rank < 0 || rank >= g->nranks) throw ApiError(MVSK_DOMAIN_ERROR, "in-process group: bad rank");
    std::lock_guard<std::mutex> l(g->mu);
    if (g->joined[(size_t)rank]) throw ApiError(MVSK_DOMAIN_ERROR, "in-process group: rank already joined");
    // peer access to every member on another device (NVLink / P2P reads)
    for (int q = 0; q < g->nranks; ++q) {
        if (!g->joined[(size_t)q] || g->members[(size_t)q].device == ctx->device) continue;
        const int other = g->members[(size_t)q].device;
        int can = 0;
        MVSK_CUDA(cudaDeviceCanAccessPeer(&can, ctx->device, other));
        if (!can) throw ApiError(MVSK_CUDA_ERROR, "in-process group: no peer access between member devices");
        for (auto [a, b] : {std::make_pair(ctx->device, other), std::make_pair(other, ctx->device)}) {
            MVSK_CUDA(cudaSetDevice(a));
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) MVSK_CUDA(e);
            cudaGetLastError();
        }
        MVSK_CUDA(cudaSetDevice(ctx->device));
    }
    g->joined[(size_t)rank] = 1;
    g->members[(size_t)rank].device = ctx->device;
    ++g->live;
    ctx->group = g;
    ctx->rank = rank;
    ctx->nranks = g->nranks;
    // the collective synchronises host threads, which a captured CUDA graph
    // cannot replay: ops of group members always launch eagerly
    ctx->no_capture = true;
}

void group_leave(mvsk_gpu_ctx* ctx) {
    if (!ctx->group) return;
    for (auto& e : ctx->ar_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->ar_scratch) cudaFree(ctx->ar_scratch);
    ctx->ar_scratch = nullptr;
    ctx->ar_scratch_elems = 0;
    ctx->ar_ev[0] = ctx->ar_ev[1] = nullptr;
    if (ctx->owns_comm) {
        std::lock_guard<std::mutex> l(ctx->group->mu);
        ctx->group->joined[(size_t)ctx->rank] = 0;
        --ctx->group->live;
    }
    ctx->group = nullptr;
}

int group_live(const LocalGroup* g) { return g->live; }
void group_delete(LocalGroup* g) { delete g; }

}  // namespace mvsk_b200
