// Device-resident PCG for the YAND direction (affine_normal.hpp:189-242).
//
// The reduced tangent operator H e = Q^T U^T grad2 f (U Q e) + lambda e is
// applied without leaving the device: a "lift" kernel applies the two
// Householder reflectors (U: simplex.hpp:63-70, Q: affine_normal.hpp:28-33) to
// every CG column and scatters it into the HVP input rows (face -> full
// coordinates), one fused k-RHS HVP pass runs, and an "update" kernel gathers,
// applies Q^T U^T (:36-39, simplex.hpp:73-78) and performs the capped-CG step
// of every column (cg_capped, affine_normal.hpp:85-113: per-column alpha/beta,
// nonpositive curvature -> breakdown, ||r|| <= tol ||rhs|| or the cap -> stop).
// The host only reads back a k-int activity mask per CG step (and the
// solution at the end); no n-vector crosses PCIe inside the Krylov loops.
// One CTA owns one CG column; every reduction has a fixed order.
#include <algorithm>
#include <cmath>
#include <vector>

#include "host_ops.hpp"
#include "pcg_device.hpp"

namespace mvsk_b200 {
namespace {

constexpr int kPT = 512;  // threads per column CTA
constexpr int kMaxDeferred = 64;  // Krylov loops per direction (probe blocks + main)

__device__ double block_sum(double v, double* sh) {
    // fixed-order tree: warp shuffles then a 16-way smem combine
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
    return s;
}

struct Geo {
    const double* vU;  // m
    double bU;
    const double* vQ;  // m - 1
    double bQ;
    const long long* idx;  // m face -> full index (null: identity)
    int m;
    int ld;
};

// q = Q e (e: m-2) in smem (m-1), then y = U q (m) scattered to a full row
__device__ void lift_col(const Geo& g, const double* e, bool apply_q, double* row, double* q, double* sh) {
    const int m = g.m, m1 = m - 1;
    // q: pad (0, e) and reflect with Q, or take e (length m-1) as is
    double part = 0.0;
    for (int i = threadIdx.x; i < m1; i += blockDim.x) {
        const double v = apply_q ? (i == 0 ? 0.0 : e[i - 1]) : e[i];
        q[i] = v;
        part += g.vQ[i] * v;
    }
    if (apply_q) {
        const double s = g.bQ * block_sum(part, sh);
        for (int i = threadIdx.x; i < m1; i += blockDim.x) q[i] -= s * g.vQ[i];
    }
    __syncthreads();
    double part2 = 0.0;
    for (int i = threadIdx.x + 1; i < m; i += blockDim.x) part2 += g.vU[i] * q[i - 1];
    const double s2 = g.bU * block_sum(part2, sh);
    for (int i = threadIdx.x; i < g.ld; i += blockDim.x) row[i] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double y = (i == 0 ? 0.0 : q[i - 1]) - s2 * g.vU[i];
        row[g.idx ? (int)g.idx[i] : i] = y;
    }
}

// Q^T U^T h (h gathered from a full row): returns a pointer into `t` (2m doubles
// of smem) holding m-2 values (apply_q) or m-1 values (U^T only)
__device__ const double* reduce_col(const Geo& g, const double* row, bool apply_q, double* t, double* sh) {
    const int m = g.m, m1 = m - 1;
    double part = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) part += g.vU[i] * row[g.idx ? (int)g.idx[i] : i];
    const double s = g.bU * block_sum(part, sh);
    double part2 = 0.0;
    for (int i = threadIdx.x; i < m1; i += blockDim.x) {
        const int fi = g.idx ? (int)g.idx[i + 1] : i + 1;
        const double v = row[fi] - s * g.vU[i + 1];
        t[i] = v;
        part2 += g.vQ[i] * v;
    }
    if (!apply_q) {
        __syncthreads();
        return t;
    }
    const double s2 = g.bQ * block_sum(part2, sh);  // (its barriers also publish t)
    double* r = t + m;
    for (int i = threadIdx.x; i < m1 - 1; i += blockDim.x) r[i] = t[i + 1] - s2 * g.vQ[i + 1];
    __syncthreads();
    return r;
}

struct CGState {
    double* X;  // [k][mm]
    double* R;
    double* Z;
    double* P;
    double* rz;      // [k]
    double* target;  // [k]
    int* active;     // [k]
    int* iters;      // [k]
    int* breakdown;  // [k]
    const double* jd;  // mm or null
    int mm;
    int cap;
    double tol;
};

__global__ void __launch_bounds__(kPT) cg_init_kernel(Geo g, CGState s, const double* rhs, double* vin) {
    extern __shared__ double q[];
    __shared__ double sh[32];
    const int c = blockIdx.x, mm = s.mm;
    const double* b = rhs + (size_t)c * mm;
    double* X = s.X + (size_t)c * mm;
    double* R = s.R + (size_t)c * mm;
    double* Z = s.Z + (size_t)c * mm;
    double* P = s.P + (size_t)c * mm;
    double prz = 0.0, pbb = 0.0;
    for (int i = threadIdx.x; i < mm; i += blockDim.x) {
        const double r = b[i];
        const double z = s.jd ? r / s.jd[i] : r;
        X[i] = 0.0;
        R[i] = r;
        Z[i] = z;
        P[i] = z;
        prz += r * z;
        pbb += r * r;
    }
    const double rz = block_sum(prz, sh);
    const double bb = block_sum(pbb, sh);
    if (threadIdx.x == 0) {
        s.rz[c] = rz;
        s.target[c] = s.tol * sqrt(bb);
        s.iters[c] = 0;
        s.breakdown[c] = 0;
        s.active[c] = (s.cap > 0 && sqrt(bb) > s.target[c]) ? 1 : 0;  // :94 loop test at it = 0
    }
    // lift the first search direction into the HVP input row (fused lift_kernel)
    __syncthreads();
    lift_col(g, P, true, vin + (size_t)c * g.ld, q, sh);
}

// lift P (or an arbitrary source block) of the active columns into HVP input rows
__global__ void __launch_bounds__(kPT) lift_kernel(Geo g, const double* E, int ldE, bool apply_q, const int* active,
                                                   double* vin) {
    extern __shared__ double q[];
    __shared__ double sh[32];
    const int c = blockIdx.x;
    double* row = vin + (size_t)c * g.ld;
    if (active && !active[c]) {
        for (int i = threadIdx.x; i < g.ld; i += blockDim.x) row[i] = 0.0;
        return;
    }
    lift_col(g, E + (size_t)c * ldE, apply_q, row, q, sh);
}

// step parameters live in device memory so one instantiated Krylov graph serves
// every direction (the reflector scalars, face size, cap and tolerance change)
struct StepParams {
    Geo g;
    CGState s;
    double lambda;
};

// one capped-CG step per active column, from the HVP rows H (full coordinates)
__device__ __forceinline__ void cg_step_col(const Geo& g, const CGState& s, double lambda, const double* H,
                                            double* vin, double* t, double* sh) {
    const int c = blockIdx.x, mm = s.mm;
    if (!s.active[c]) return;
    // thread 0 rewrites rz only after every thread passed the barriers below
    const double rz_old = s.rz[c];
    double* hp_ = const_cast<double*>(reduce_col(g, H + (size_t)c * g.ld, true, t, sh));  // Q^T U^T H p
    double* X = s.X + (size_t)c * mm;
    double* R = s.R + (size_t)c * mm;
    double* Z = s.Z + (size_t)c * mm;
    double* P = s.P + (size_t)c * mm;
    double pp = 0.0;
    for (int i = threadIdx.x; i < mm; i += blockDim.x) {
        const double hp = hp_[i] + lambda * P[i];  // Hop: red + lambda e (:194)
        hp_[i] = hp;
        pp += P[i] * hp;
    }
    const double pHp = block_sum(pp, sh);
    if (pHp <= 0.0) {  // :97-100
        if (threadIdx.x == 0) {
            s.breakdown[c] = 1;
            s.active[c] = 0;
        }
        return;
    }
    const double alpha = rz_old / pHp;
    double prz = 0.0, prr = 0.0;
    for (int i = threadIdx.x; i < mm; i += blockDim.x) {
        X[i] += alpha * P[i];
        const double r = R[i] - alpha * hp_[i];
        R[i] = r;
        const double z = s.jd ? r / s.jd[i] : r;
        Z[i] = z;
        prz += r * z;
        prr += r * r;
    }
    const double rz2 = block_sum(prz, sh);
    const double rr = block_sum(prr, sh);
    const double beta = rz2 / rz_old;
    for (int i = threadIdx.x; i < mm; i += blockDim.x) P[i] = Z[i] + beta * P[i];
    const int it = s.iters[c] + 1;
    const bool still = it < s.cap && sqrt(rr) > s.target[c];  // :94
    __syncthreads();  // every thread has read iters/target and written its P slice
    if (threadIdx.x == 0) {
        s.rz[c] = rz2;
        s.iters[c] = it;
        s.active[c] = still ? 1 : 0;
    }
    // lift the next search direction into the HVP input row (fused lift_kernel;
    // t's reduced-H values are dead here, so it holds q)
    if (still) lift_col(g, P, true, vin + (size_t)c * g.ld, t, sh);
}

// set_cond (inside the Krylov graph): the last column CTA to finish sets the
// while-loop condition from every column's activity flag, so a CG step is two
// kernels (the HVP pass and this one)
__global__ void __launch_bounds__(kPT) cg_step_kernel(const StepParams* sp, const double* H, double* vin,
                                                      unsigned* arrive, cudaGraphConditionalHandle h, int set_cond) {
    extern __shared__ double t[];
    __shared__ double sh[32];
    const Geo g = sp->g;
    const CGState s = sp->s;
    cg_step_col(g, s, sp->lambda, H, vin, t, sh);
    if (!set_cond) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this column's activity flag before the arrival
        if (atomicAdd(arrive, 1u) == gridDim.x - 1) {
            __threadfence();
            int any = 0;
            for (int col = 0; col < (int)gridDim.x; ++col) any |= ((volatile const int*)s.active)[col];
            *arrive = 0u;
            cudaGraphSetConditional(h, any ? 1u : 0u);
        }
    }
}

// out = Q^T U^T H (+ lambda e) per column, or a += sum_c Q^T U^T H_c (in column order)
__global__ void __launch_bounds__(kPT) reduce_kernel(Geo g, const double* H, int k, bool apply_q, double* out,
                                                     int ldo) {
    extern __shared__ double t[];
    __shared__ double sh[32];
    const int c = blockIdx.x;
    const double* r = reduce_col(g, H + (size_t)c * g.ld, apply_q, t, sh);
    const int len = apply_q ? g.m - 2 : g.m - 1;
    for (int i = threadIdx.x; i < len; i += blockDim.x) out[(size_t)c * ldo + i] = r[i];
}

// Jacobi diagonal from the probe responses (:197-209): mean over probes of
// r o (Qt Ut H U Q r + lambda r), floored at max(1e-12, lambda); probe order fixed
__global__ void jacobi_diag_kernel(const double* probes, const double* rows, int k, int mm, double lambda, double fl,
                                   double* jd) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mm; i += gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int p = 0; p < k; ++p) {
            const double r = probes[(size_t)p * mm + i];
            v += r * (rows[(size_t)p * mm + i] + lambda * r);
        }
        v /= (double)k;
        jd[i] = v > fl ? v : fl;
    }
}

// exact-trace probes e_{b0}..e_{b0+k-1} (:217-226)
__global__ void unit_probe_kernel(double* src, int k, int mm, int b0) {
    const size_t tot = (size_t)k * mm;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        const int p = (int)(e / mm), i = (int)(e - (size_t)p * mm);
        src[e] = (i == b0 + p) ? 1.0 : 0.0;
    }
}

// a += sum of the block's third-action rows, in probe order (:225, :235)
__global__ void accum_rows_kernel(const double* rows, int k, int mm, double* a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mm; i += gridDim.x * blockDim.x) {
        double v = a[i];
        for (int p = 0; p < k; ++p) v += rows[(size_t)p * mm + i];
        a[i] = v;
    }
}

// rhs = h - (||gbar|| / n) a, a averaged over the Hutchinson probes (:236, :239)
__global__ void rhs_kernel(const double* h, const double* a, int mm, double adiv, double coef, double* rhs) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mm; i += gridDim.x * blockDim.x) {
        const double ai = adiv > 0 ? a[i] / adiv : a[i];
        rhs[i] = h[i] - coef * ai;
    }
}

// while-loop condition of the device Krylov graph: another step iff any column
// is still active (each column's own test already includes the cap, :94)
__global__ void cg_decide_kernel(const int* active, int k, cudaGraphConditionalHandle h) {
    if (threadIdx.x == 0) {
        int any = 0;
        for (int c = 0; c < k; ++c) any |= active[c];
        cudaGraphSetConditional(h, any ? 1u : 0u);
    }
}

template <class T>
T* carve(unsigned char*& cur, size_t count) {
    T* p = reinterpret_cast<T*>(cur);
    cur += ((count * sizeof(T) + 255) / 256) * 256;
    return p;
}

}  // namespace

struct PcgWorkspace {
    size_t bytes = 0;
    unsigned char* dev = nullptr;
    int* host_flags = nullptr;  // pinned [4 * kPcgMaxCols]
    StepParams* host_params = nullptr;  // pinned staging of the device StepParams [kMaxDeferred]
    int* host_counts = nullptr;         // pinned [kMaxDeferred][2][K] iters / breakdown snapshots
    double* host_stage = nullptr;       // pinned probe staging
    size_t host_stage_elems = 0;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // device-resident Krylov loops: a conditional-while graph per (k, slot)
    struct LoopGraph {
        int k, slot;
        uint64_t epoch;
        cudaGraphExec_t exec;
        uint64_t phys_per_step, launches_per_step;
    };
    std::vector<LoopGraph> graphs;
    std::vector<std::pair<int, int>> seen;  // (k, slot) keys that ran once at seen_epoch
    uint64_t seen_epoch = ~0ull;
    bool graphs_broken = false;
};

void pcg_workspace_free(mvsk_gpu_ctx* ctx) {
    if (!ctx->pcg) return;
    for (auto& lg : ctx->pcg->graphs)
        if (lg.exec) cudaGraphExecDestroy(lg.exec);
    if (ctx->pcg->host_params) cudaFreeHost(ctx->pcg->host_params);
    if (ctx->pcg->host_counts) cudaFreeHost(ctx->pcg->host_counts);
    if (ctx->pcg->host_stage) cudaFreeHost(ctx->pcg->host_stage);
    if (ctx->pcg->dev) cudaFree(ctx->pcg->dev);
    if (ctx->pcg->host_flags) cudaFreeHost(ctx->pcg->host_flags);
    for (cudaEvent_t e : ctx->pcg->ev)
        if (e) cudaEventDestroy(e);
    delete ctx->pcg;
    ctx->pcg = nullptr;
}

PcgOutput pcg_direction_device(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const PcgInput& in) {
    const int m = (int)in.m, m1 = m - 1, mm = m - 2;
    const int K = kPcgMaxCols;
    const size_t ld = (size_t)ctx->ld;
    // ---- workspace, carved for the full n so its pointers do not move with the
    // face size (they are baked into the instantiated Krylov graphs)
    const long long N = ctx->n;
    const size_t need = 256 * 32 + sizeof(double) * ((size_t)N + N + N + 6 * (size_t)K * N + 4 * N + 4 * K) +
                        sizeof(long long) * N + sizeof(int) * 4 * K + sizeof(StepParams) + 512;
    if (!ctx->pcg) ctx->pcg = new PcgWorkspace();
    PcgWorkspace& ws = *ctx->pcg;
    if (ws.bytes < need) {
        if (ws.dev) MVSK_CUDA(cudaFree(ws.dev));
        ws.dev = nullptr;
        MVSK_CUDA(cudaMalloc(&ws.dev, need));
        ws.bytes = need;
        ++ctx->epoch;
    }
    if (!ws.host_flags) MVSK_CUDA(cudaMallocHost(&ws.host_flags, sizeof(int) * 4 * K));
    // one pinned StepParams per Krylov loop of the direction: the H2D copies are
    // asynchronous, so a later loop must not overwrite an earlier loop's staging
    if (!ws.host_params) MVSK_CUDA(cudaMallocHost(&ws.host_params, sizeof(StepParams) * kMaxDeferred));
    if (!ws.host_counts) MVSK_CUDA(cudaMallocHost(&ws.host_counts, sizeof(int) * kMaxDeferred * 2 * K));
    // pinned probe staging: the Jacobi probes and every Hutchinson probe of this
    // direction, copied asynchronously (no host round trip inside the direction)
    const size_t stage_need = (in.jacobi_probes.size() + in.probes.size()) * (size_t)std::max(mm, 1);
    if (ws.host_stage_elems < stage_need) {
        if (ws.host_stage) MVSK_CUDA(cudaFreeHost(ws.host_stage));
        ws.host_stage = nullptr;
        ws.host_stage_elems = 0;
        MVSK_CUDA(cudaMallocHost(&ws.host_stage, stage_need * sizeof(double)));
        ws.host_stage_elems = stage_need;
    }
    for (cudaEvent_t& e : ws.ev)
        if (!e) MVSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    unsigned char* cur = ws.dev;
    double* vU = carve<double>(cur, N);
    double* vQ = carve<double>(cur, N);
    double* nu = carve<double>(cur, N);
    double* X = carve<double>(cur, (size_t)K * N);  // [k][mm] blocks
    double* Rm = carve<double>(cur, (size_t)K * N);
    double* Z = carve<double>(cur, (size_t)K * N);
    double* P = carve<double>(cur, (size_t)K * N);
    double* src = carve<double>(cur, (size_t)K * N);  // rhs / probes
    double* rows = carve<double>(cur, (size_t)K * N);  // reduced outputs
    double* jd = carve<double>(cur, N);
    double* hvec = carve<double>(cur, N);
    double* avec = carve<double>(cur, N);
    double* rz = carve<double>(cur, K);
    double* target = carve<double>(cur, K);
    long long* idx = carve<long long>(cur, N);
    int* active = carve<int>(cur, K);
    int* iters = carve<int>(cur, K);
    int* bdown = carve<int>(cur, K);
    StepParams* sp_dev = carve<StepParams>(cur, 1);
    unsigned* arrive = carve<unsigned>(cur, 1);
    cudaStream_t st = ctx->stream;

    MVSK_CUDA(cudaMemcpyAsync(vU, in.vU.data(), m * sizeof(double), cudaMemcpyHostToDevice, st));
    MVSK_CUDA(cudaMemcpyAsync(vQ, in.vQ.data(), m1 * sizeof(double), cudaMemcpyHostToDevice, st));
    MVSK_CUDA(cudaMemcpyAsync(nu, in.nu.data(), m1 * sizeof(double), cudaMemcpyHostToDevice, st));
    if (fm.active) MVSK_CUDA(cudaMemcpyAsync(idx, fm.idx.data(), m * sizeof(long long), cudaMemcpyHostToDevice, st));
    Geo g{vU, in.bU, vQ, in.bQ, fm.active ? idx : nullptr, m, (int)ld};
    const size_t dsm = (size_t)2 * std::max(m, 1) * sizeof(double);
    const size_t dsm_max = (size_t)2 * std::max<long long>(N, 1) * sizeof(double);  // cg_step (graph-baked)
    for (const void* fn : {(const void*)lift_kernel, (const void*)cg_step_kernel, (const void*)reduce_kernel,
                           (const void*)cg_init_kernel})
        set_smem_attr(fn, dsm_max);
    const Slot& sl = ctx->slots[slot];
    double* vin = ctx->vin;
    double* vin2 = ctx->vin + (size_t)MVSK_GPU_MAX_RHS * ld;
    double* H = ctx->outd;

    PcgOutput out;
    auto hvp_rows = [&](int k, int logical) {
        PassIO io;
        io.vin = vin;
        io.z = sl.z;
        io.out = H;
        io.ldo = (long long)ld;
        run_pass(ctx, Op::HVP, k, io);
        ctx->fwd += logical;  // reference contract: 2 passes per (active) HVP
        ctx->tr += logical;
    };
    // capped CG on k columns in lock-step (the columns' arithmetic is
    // cg_capped's). Steps are enqueued one ahead of the host's look at the
    // activity flags: step s+1 is already queued while the host reads the flags
    // that gate step s, and a step whose flags are all 0 is a device-side no-op
    // (every kernel of the step, including the HVP pass, exits on entry). So
    // the GPU never idles on a host round trip inside the Krylov loop.
    // Capped CG on k columns in lock-step (the columns' arithmetic is
    // cg_capped's). Preferred: the whole loop is ONE conditional-while CUDA graph
    // (body = the k-RHS HVP pass, cg_step, and a 1-thread kernel that sets the
    // loop condition from the columns' activity flags), so no host round trip
    // happens inside the Krylov loop; the graph is instantiated once per
    // (k, slot) and reused for every direction (its parameters live in device
    // memory). Fallback: a host-driven loop that enqueues step s+1 before
    // reading the flags that gate step s (a step whose flags are all 0 is a
    // device-side no-op), so the GPU does not idle on the round trip either.
    // per-cg-call bookkeeping, settled after the direction's single final sync
    struct Deferred {
        int k;
        int slot;  // pinned row of [iters | breakdown] snapshots
        uint64_t pps, lps;  // passes / launches per step (graph loops); 0: counted already
        bool graph;
    };
    std::vector<Deferred> deferred;
    auto defer_counts = [&](int k, bool graph, uint64_t pps, uint64_t lps) {
        const int row = (int)deferred.size();
        if (row >= kMaxDeferred) throw ApiError(MVSK_INTERNAL_ERROR, "pcg: too many Krylov loops per direction");
        int* hc = ws.host_counts + (size_t)row * 2 * K;
        MVSK_CUDA(cudaMemcpyAsync(hc, iters, k * sizeof(int), cudaMemcpyDeviceToHost, st));
        MVSK_CUDA(cudaMemcpyAsync(hc + K, bdown, k * sizeof(int), cudaMemcpyDeviceToHost, st));
        deferred.push_back({k, row, pps, lps, graph});
    };
    auto settle_counts = [&]() {
        for (const Deferred& d : deferred) {
            const int* hc = ws.host_counts + (size_t)d.slot * 2 * K;
            int steps = 0;
            for (int c = 0; c < d.k; ++c) {
                const int col_steps = hc[c] + (hc[K + c] ? 1 : 0);  // HVPs column c consumed
                out.iters += hc[c];
                if (hc[K + c]) out.breakdown = true;
                steps = std::max(steps, col_steps);
                ctx->fwd += col_steps;  // reference contract: 2 passes per (active) HVP
                ctx->tr += col_steps;
            }
            if (d.graph) {
                ctx->phys += (uint64_t)steps * d.pps;
                ctx->launches += 1 + (uint64_t)steps * d.lps;
            }
        }
        deferred.clear();
    };
    static const bool no_graph = std::getenv("MVSK_NO_CG_GRAPH") != nullptr;
    auto cg_graph = [&](int k) -> PcgWorkspace::LoopGraph* {
        if (no_graph || ws.graphs_broken) return nullptr;
        // the first loop of a key runs host-driven: it sizes the pass workspaces,
        // which must not be (re)allocated while a graph is being captured
        if (ws.seen_epoch != ctx->epoch) {  // buffers may have been resized: size them eagerly again
            ws.seen.clear();
            ws.seen_epoch = ctx->epoch;
        }
        if (std::find(ws.seen.begin(), ws.seen.end(), std::make_pair(k, slot)) == ws.seen.end()) {
            ws.seen.emplace_back(k, slot);
            return nullptr;
        }
        for (auto& lg : ws.graphs)
            if (lg.k == k && lg.slot == slot) {
                if (lg.epoch == ctx->epoch && lg.exec) return &lg;
                if (lg.exec) cudaGraphExecDestroy(lg.exec);
                lg.exec = nullptr;
            }
        cudaGraph_t gr = nullptr;
        cudaGraphExec_t exec = nullptr;
        const uint64_t p0 = ctx->phys, l0 = ctx->launches;
        bool ok = cudaGraphCreate(&gr, 0) == cudaSuccess;
        cudaGraphConditionalHandle h{};
        cudaGraphNode_t n0 = nullptr, wn = nullptr;
        if (ok) ok = cudaGraphConditionalHandleCreate(&h, gr, 0, 0) == cudaSuccess;
        if (ok) {  // initial condition: any column active after cg_init
            int kk = k;
            void* args[] = {&active, &kk, &h};
            cudaKernelNodeParams kp{};
            kp.func = reinterpret_cast<void*>(&cg_decide_kernel);
            kp.gridDim = dim3(1);
            kp.blockDim = dim3(32);
            kp.kernelParams = args;
            ok = cudaGraphAddKernelNode(&n0, gr, nullptr, 0, &kp) == cudaSuccess;
        }
        cudaGraph_t body = nullptr;
        if (ok) {
            cudaGraphNodeParams cp{};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            ok = cudaGraphAddNode(&wn, gr, &n0, 1, &cp) == cudaSuccess;
            if (ok) body = cp.conditional.phGraph_out[0];
        }
        if (ok) ok = cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
                     cudaSuccess;
        if (ok) {
            bool threw = false;
            try {
                PassIO io;
                io.vin = vin;
                io.z = sl.z;
                io.out = H;
                io.ldo = (long long)ld;
                run_pass(ctx, Op::HVP, k, io);
                ++ctx->launches;
                cg_step_kernel<<<k, kPT, dsm_max, st>>>(sp_dev, H, vin, arrive, h, 1);
            } catch (...) {
                threw = true;
            }
            cudaGraph_t captured = nullptr;
            ok = cudaStreamEndCapture(st, &captured) == cudaSuccess && !threw;
        }
        if (ok) ok = cudaGraphInstantiate(&exec, gr, 0) == cudaSuccess;
        const uint64_t dp = ctx->phys - p0, dl = ctx->launches - l0;
        ctx->phys = p0;
        ctx->launches = l0;
        if (gr) cudaGraphDestroy(gr);
        cudaGetLastError();
        if (!ok) {
            if (exec) cudaGraphExecDestroy(exec);
            ws.graphs_broken = true;  // e.g. a launch kind the conditional body rejects: host loop
            return nullptr;
        }
        ws.graphs.push_back({k, slot, ctx->epoch, exec, dp, dl});
        return &ws.graphs.back();
    };
    auto cg = [&](int k, int cap, const double* jdp) {
        CGState s{X, Rm, Z, P, rz, target, active, iters, bdown, jdp, mm, cap, in.tol};
        if (deferred.size() >= (size_t)kMaxDeferred) throw ApiError(MVSK_INTERNAL_ERROR, "pcg: too many Krylov loops");
        StepParams* hp = ws.host_params + deferred.size();
        *hp = StepParams{g, s, in.lambda};
        MVSK_CUDA(cudaMemcpyAsync(sp_dev, hp, sizeof(StepParams), cudaMemcpyHostToDevice, st));
        MVSK_CUDA(cudaMemsetAsync(arrive, 0, sizeof(unsigned), st));
        ++ctx->launches;
        cg_init_kernel<<<k, kPT, dsm, st>>>(g, s, src, vin);
        MVSK_CUDA(cudaGetLastError());
        if (PcgWorkspace::LoopGraph* lg = cg_graph(k)) {
            MVSK_CUDA(cudaGraphLaunch(lg->exec, st));
            defer_counts(k, true, lg->phys_per_step, lg->launches_per_step);
            return;
        }
        int* hf = ws.host_flags;  // [2][K] flag snapshots + [2K..) iters / breakdown
        MVSK_CUDA(cudaMemcpyAsync(hf, active, k * sizeof(int), cudaMemcpyDeviceToHost, st));
        MVSK_CUDA(cudaEventRecord(ws.ev[0], st));
        for (int step = 0; step < cap; ++step) {
            // vin holds the lifted direction of every active column (cg_init /
            // the previous cg_step); inactive columns' rows are stale but finite
            // and their HVP results are ignored
            PassIO io;
            io.vin = vin;
            io.z = sl.z;
            io.out = H;
            io.ldo = (long long)ld;
            io.skip = active;
            io.nskip = k;
            run_pass(ctx, Op::HVP, k, io);
            ++ctx->launches;
            cg_step_kernel<<<k, kPT, dsm_max, st>>>(sp_dev, H, vin, arrive, cudaGraphConditionalHandle{}, 0);
            MVSK_CUDA(cudaGetLastError());
            const int nb = (step + 1) & 1;
            MVSK_CUDA(cudaMemcpyAsync(hf + nb * K, active, k * sizeof(int), cudaMemcpyDeviceToHost, st));
            MVSK_CUDA(cudaEventRecord(ws.ev[nb], st));
            // flags that gated this step
            MVSK_CUDA(cudaEventSynchronize(ws.ev[step & 1]));
            int nact = 0;
            for (int c = 0; c < k; ++c) nact += hf[(step & 1) * K + c];
            if (!nact) {
                ctx->phys -= 1;  // the step ran as a no-op
                break;
            }
        }
        defer_counts(k, false, 0, 0);
    };

    // ---- Jacobi diagonal (:197-209): 8 probes through Hop in one batch
    const double* jdp = nullptr;
    double* stage = ws.host_stage;
    const int nb1 = (int)std::min<long long>(4LL * ctx->nsm, (mm + 255) / 256 + 1);
    if (!in.jacobi_probes.empty()) {
        const int k = (int)in.jacobi_probes.size();
        for (int p = 0; p < k; ++p) std::copy(in.jacobi_probes[p].begin(), in.jacobi_probes[p].end(), stage + (size_t)p * mm);
        MVSK_CUDA(cudaMemcpyAsync(src, stage, (size_t)k * mm * sizeof(double), cudaMemcpyHostToDevice, st));
        stage += (size_t)k * mm;
        ++ctx->launches;
        lift_kernel<<<k, kPT, dsm, st>>>(g, src, mm, true, nullptr, vin);
        MVSK_CUDA(cudaGetLastError());
        hvp_rows(k, k);
        ++ctx->launches;
        reduce_kernel<<<k, kPT, dsm, st>>>(g, H, k, true, rows, mm);
        ++ctx->launches;
        jacobi_diag_kernel<<<nb1, 256, 0, st>>>(src, rows, k, mm, in.lambda, std::max(1e-12, in.lambda), jd);
        MVSK_CUDA(cudaGetLastError());
        jdp = jd;
    }

    // ---- h = Q^T U^T grad2 f (U nu)  (:212-213)
    ++ctx->launches;
    lift_kernel<<<1, kPT, dsm, st>>>(g, nu, m1, false, nullptr, vin);
    MVSK_CUDA(cudaGetLastError());
    hvp_rows(1, 1);
    ++ctx->launches;
    reduce_kernel<<<1, kPT, dsm, st>>>(g, H, 1, true, hvec, mm);
    MVSK_CUDA(cudaGetLastError());

    // ---- a: Hutchinson probes or exact trace (:215-237), blocks of K columns,
    // accumulated on the device in probe order
    MVSK_CUDA(cudaMemsetAsync(avec, 0, mm * sizeof(double), st));
    if (in.has_third) {
        const int P_all = in.unit_probes ? mm : (int)in.probes.size();
        for (int b0 = 0; b0 < P_all; b0 += K) {
            const int k = std::min(K, P_all - b0);
            if (in.unit_probes) {
                ++ctx->launches;
                unit_probe_kernel<<<nb1, 256, 0, st>>>(src, k, mm, b0);
            } else {
                for (int p = 0; p < k; ++p)
                    std::copy(in.probes[b0 + p].begin(), in.probes[b0 + p].end(), stage + (size_t)p * mm);
                MVSK_CUDA(cudaMemcpyAsync(src, stage, (size_t)k * mm * sizeof(double), cudaMemcpyHostToDevice, st));
                stage += (size_t)k * mm;
            }
            cg(k, in.probe_cap, jdp);
            // third_action(U Q s_p, U Q r_p) for the block, one fused pass
            ++ctx->launches;
            lift_kernel<<<k, kPT, dsm, st>>>(g, X, mm, true, nullptr, vin);
            ++ctx->launches;
            lift_kernel<<<k, kPT, dsm, st>>>(g, src, mm, true, nullptr, vin2);
            MVSK_CUDA(cudaGetLastError());
            PassIO io;
            io.vin = vin;
            io.vin2 = vin2;
            io.z = sl.z;
            io.out = H;
            io.ldo = (long long)ld;
            run_pass(ctx, Op::THIRD, k, io);
            ctx->fwd += 2 * k;
            ctx->tr += k;
            ++ctx->launches;
            reduce_kernel<<<k, kPT, dsm, st>>>(g, H, k, true, rows, mm);
            ++ctx->launches;
            accum_rows_kernel<<<nb1, 256, 0, st>>>(rows, k, mm, avec);
            MVSK_CUDA(cudaGetLastError());
            if (in.unit_probes && deferred.size() + 2 >= (size_t)kMaxDeferred) {
                // long exact-trace sweeps: settle the loop counts every few blocks
                MVSK_CUDA(cudaStreamSynchronize(st));
                settle_counts();
            }
        }
    }
    // rhs = h - (||gbar|| / n) a  (:239); a averaged over the Hutchinson probes (:236)
    ++ctx->launches;
    rhs_kernel<<<nb1, 256, 0, st>>>(hvec, avec, mm, (in.has_third && !in.unit_probes) ? (double)in.hutchinson_probes : 0.0,
                                    in.gn / (double)m, src);
    MVSK_CUDA(cudaGetLastError());
    // main CG (:240-241)
    cg(1, in.maxit, jdp);
    out.u.resize((size_t)mm);
    MVSK_CUDA(cudaMemcpyAsync(out.u.data(), X, mm * sizeof(double), cudaMemcpyDeviceToHost, st));
    MVSK_CUDA(cudaStreamSynchronize(st));
    settle_counts();
    return out;
}

}  // namespace mvsk_b200
