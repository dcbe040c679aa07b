// Device-resident SPG identification preamble (solver.hpp:116-185).
//
// The reference's preamble is a projected-gradient loop with Barzilai-Borwein
// steps and doubling backtracking; every trial costs one oracle pass at the
// projected point, and the host-driven version pays a host round trip per
// trial (C2 kappa = 1000: 343 trials, ~10 ms of a 14 ms solve). Here one trial
// is a body of a conditional-while CUDA graph (opt-in, see spg_identify_device:
// on B200 the three kernel boundaries of a trial cost as much as the host round
// trip they replace):
//
//   spg_prep   (1 CTA)  L0 from the BB pair, y = x - g / Lk, projection onto the
//                       tau-slice, dp = xp - x, gdp = g'dp, and the pass flag
//   FGRAD pass          f and the gradient at xp (skipped when gdp >= 0)
//   spg_accept (1 CTA)  Armijo test, BB pair / iterate update or Lk doubling,
//                       active-set patience, the every-10-steps residual test,
//                       and the loop condition
//
// Every host-side reduction of the preamble (the dots of the BB step and of
// gdp, the projection's running sums, the residual) is sequential in the
// reference's order, so the device loop is bitwise the host loop: the same
// sequential sums in the same order, with products and sums rounded
// separately (the host code has no FMA contraction), and the same oracle
// kernels for f and the gradient.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "host_ops.hpp"
#include "oracle_ops.cuh"
#include "spg_device.hpp"

namespace mvsk_b200 {
namespace {

constexpr int kSpgThreads = 1024;
constexpr int kSpgMaxN = 8192;  // sort buffer in shared memory (64 KB)

struct SpgState {
    // loop state
    double f, L, Lk, gdp;
    int have_bb, k, bt, steps, last_change, done, stepped, eval_flag;
    int evals, accepts, trials;
    // parameters
    int n, ld, max_steps, patience;
    double tau, eps_stop;
};

__device__ __forceinline__ double sdot(const double* a, const double* b, int n) {
    double s = 0.0;  // driver.cu dot(): sequential, separately rounded
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
    return s;
}

// block-wide descending bitonic sort of u[0, m) (m a power of two, pad -inf)
__device__ void bitonic_desc(double* u, int m) {
    for (int size = 2; size <= m; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    const double a = u[i], b = u[j];
                    if (desc ? (a < b) : (a > b)) {
                        u[i] = b;
                        u[j] = a;
                    }
                }
            }
        }
    }
    __syncthreads();
}

// project_slice (driver.cu / simplex.hpp:93-117): out = max(v - tau - theta, 0)
// + tau with theta from the running sums of the sorted v - tau. u: smem scratch
// of the next power of two >= n. Every thread returns with out written.
__device__ void project_slice_dev(const double* v, int n, double tau, double mass, double* out, double* u,
                                  double* bcast) {
    int m = 1;
    while (m < n) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) u[i] = i < n ? v[i] - tau : -INFINITY;
    bitonic_desc(u, m);
    if (threadIdx.x == 0) {
        const double s = __dsub_rn(mass, __dmul_rn((double)n, tau));
        double css = 0.0, theta = 0.0;
        for (int k = 0; k < n; ++k) {
            css += u[k];
            const double cand = (css - s) / (double)(k + 1);
            if (u[k] > cand) theta = cand;
        }
        *bcast = theta;
    }
    __syncthreads();
    const double theta = *bcast;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = fmax(v[i] - tau - theta, 0.0) + tau;
    __syncthreads();
}

struct SpgBufs {
    double* x;    // n, current iterate
    double* g;    // n, gradient at x
    double* xp;   // ld, trial point (the FGRAD input row, zero padding)
    double* dp;   // n
    double* bbs;  // n
    double* bby;  // n
    double* y;    // n scratch
    unsigned char* act;  // n
};

__global__ void __launch_bounds__(kSpgThreads) spg_prep_kernel(SpgState* st, SpgBufs b) {
    extern __shared__ double u[];
    __shared__ double bc[2];
    const int n = st->n;
    if (threadIdx.x == 0) ++st->trials;
    if (st->bt == 0 && threadIdx.x == 0) {  // L0 from the BB pair (solver.hpp:131-135)
        double L0 = st->L;
        if (st->have_bb) {
            const double sy = sdot(b.bbs, b.bby, n), ss = sdot(b.bbs, b.bbs, n);
            L0 = (ss > 0 && sy > 0) ? sy / ss : st->L;
            L0 = fmin(fmax(L0, 1e-2), 1e12);
        }
        st->Lk = L0;
    }
    __syncthreads();
    const double Lk = st->Lk;
    for (int i = threadIdx.x; i < n; i += blockDim.x) b.y[i] = b.x[i] - b.g[i] / Lk;
    __syncthreads();
    project_slice_dev(b.y, n, st->tau, 1.0, b.xp, u, &bc[0]);
    for (int i = threadIdx.x; i < n; i += blockDim.x) b.dp[i] = b.xp[i] - b.x[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        const double gdp = sdot(b.g, b.dp, n);
        st->gdp = gdp;
        st->eval_flag = gdp < 0 ? 1 : 0;
        if (gdp < 0) ++st->evals;
    }
}

__global__ void __launch_bounds__(kSpgThreads) spg_accept_kernel(SpgState* st, SpgBufs b, const double* gp,
                                                                 const double* fp_sc, cudaGraphConditionalHandle h,
                                                                 int set_cond) {
    extern __shared__ double u[];
    __shared__ int s_acc, s_change, s_any, s_done;
    __shared__ double bc[2];
    const int n = st->n;
    if (threadIdx.x == 0) {
        int acc = 0;
        if (st->eval_flag) {
            const double fp = fp_sc[0];
            if (fp <= __dadd_rn(st->f, __dmul_rn(1e-4, st->gdp))) {  // Armijo (solver.hpp:146)
                acc = 1;
                st->f = fp;
                st->L = st->Lk;
                st->have_bb = 1;
                ++st->accepts;
            }
        }
        s_acc = acc;
        if (!acc) {
            if (st->Lk > 1e13 || st->bt + 1 >= 40) {  // no step: the preamble ends (:159-160)
                st->done = 1;
            } else {
                st->Lk *= 2.0;
                ++st->bt;
            }
        }
    }
    __syncthreads();
    if (s_acc) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            b.bbs[i] = b.dp[i];
            b.bby[i] = gp[i] - b.g[i];
            b.x[i] = b.xp[i];
            b.g[i] = gp[i];
        }
        if (threadIdx.x == 0) {
            s_change = 0;
            s_any = 0;
        }
        __syncthreads();
        // active set (<= tau + 1e-12) and patience (:163-172)
        const double thr = st->tau + 1e-12;
        int chg = 0, any = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned char a = b.x[i] <= thr ? 1 : 0;
            if (a != b.act[i]) chg = 1;
            if (a) any = 1;
            b.act[i] = a;
        }
        if (chg) atomicOr(&s_change, 1);
        if (any) atomicOr(&s_any, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            const int steps = ++st->steps;
            st->bt = 0;
            ++st->k;
            int done = 0;
            if (s_change) {
                st->last_change = steps;
            } else if (s_any && steps - st->last_change >= st->patience) {
                done = 1;
            }
            if (st->k >= st->max_steps) done = 1;
            s_done = done;
            st->done = done;
        }
        __syncthreads();
        // every 10 steps: gradient-mapping residual ||x - P(x - g)|| (:173-174)
        if (!s_done && st->eps_stop > 0 && st->steps % 10 == 0) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) b.y[i] = b.x[i] - b.g[i];
            __syncthreads();
            project_slice_dev(b.y, n, st->tau, 1.0, b.dp, u, &bc[0]);
            if (threadIdx.x == 0) {
                double s = 0.0;
                for (int i = 0; i < n; ++i) {
                    const double d = b.x[i] - b.dp[i];
                    s = __dadd_rn(s, __dmul_rn(d, d));
                }
                if (sqrt(s) <= st->eps_stop) st->done = 1;
            }
        }
    }
    __syncthreads();
    if (set_cond && threadIdx.x == 0) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

__global__ void spg_cond_kernel(const SpgState* st, cudaGraphConditionalHandle h) {
    if (threadIdx.x == 0) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

size_t carve_off(size_t& off, size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
}

}  // namespace

struct SpgWorkspace {
    size_t bytes = 0;
    unsigned char* dev = nullptr;
    SpgState* host_state = nullptr;  // pinned
    cudaGraphExec_t exec = nullptr;
    uint64_t epoch = ~0ull;
    int slot = -1;
    uint64_t phys_per_trial = 0, launches_per_trial = 0;
    bool broken = false;
};

void spg_workspace_free(mvsk_gpu_ctx* ctx) {
    if (!ctx->spg) return;
    if (ctx->spg->exec) cudaGraphExecDestroy(ctx->spg->exec);
    if (ctx->spg->dev) cudaFree(ctx->spg->dev);
    if (ctx->spg->host_state) cudaFreeHost(ctx->spg->host_state);
    delete ctx->spg;
    ctx->spg = nullptr;
}

bool spg_identify_device(mvsk_gpu_ctx* ctx, int slot, std::vector<double>& x, double f0,
                         const std::vector<double>& g0, double tau, int max_steps, int patience, double eps_stop,
                         int& steps_out) {
    // opt-in (MVSK_SPG_GRAPH=1): measured no faster than the host loop on B200 —
    // a trial is three kernel boundaries (~30 us on a C2 panel, the same as the
    // host round trip) and the bitwise-faithful sequential reductions make
    // n = 5000 trials slower (C4: 9 ms vs ~5 ms)
    static const bool enabled = std::getenv("MVSK_SPG_GRAPH") != nullptr;
    const int n = (int)ctx->n;
    if (!enabled || n > kSpgMaxN || n < 2 || ctx->zoff_dev) return false;
    if (!ctx->spg) ctx->spg = new SpgWorkspace();
    SpgWorkspace& ws = *ctx->spg;
    if (ws.broken) return false;
    const size_t ld = (size_t)ctx->ld;
    size_t off = 0;
    const size_t o_st = carve_off(off, sizeof(SpgState));
    const size_t o_x = carve_off(off, n * sizeof(double)), o_g = carve_off(off, n * sizeof(double));
    const size_t o_xp = carve_off(off, ld * sizeof(double)), o_dp = carve_off(off, n * sizeof(double));
    const size_t o_bs = carve_off(off, n * sizeof(double)), o_by = carve_off(off, n * sizeof(double));
    const size_t o_y = carve_off(off, n * sizeof(double)), o_act = carve_off(off, (size_t)n);
    if (ws.bytes < off) {
        if (ws.dev) MVSK_CUDA(cudaFree(ws.dev));
        ws.dev = nullptr;
        MVSK_CUDA(cudaMalloc(&ws.dev, off));
        MVSK_CUDA(cudaMemset(ws.dev, 0, off));
        ws.bytes = off;
        ++ctx->epoch;
    }
    if (!ws.host_state) MVSK_CUDA(cudaMallocHost(&ws.host_state, sizeof(SpgState)));
    unsigned char* d = ws.dev;
    SpgState* st = reinterpret_cast<SpgState*>(d + o_st);
    SpgBufs b{reinterpret_cast<double*>(d + o_x), reinterpret_cast<double*>(d + o_g),
              reinterpret_cast<double*>(d + o_xp), reinterpret_cast<double*>(d + o_dp),
              reinterpret_cast<double*>(d + o_bs), reinterpret_cast<double*>(d + o_by),
              reinterpret_cast<double*>(d + o_y), d + o_act};
    cudaStream_t sm = ctx->stream;
    int m2 = 1;
    while (m2 < n) m2 <<= 1;
    const size_t smem = (size_t)m2 * sizeof(double);
    set_smem_attr(reinterpret_cast<const void*>(&spg_prep_kernel), smem);
    set_smem_attr(reinterpret_cast<const void*>(&spg_accept_kernel), smem);

    // initial state (solver.hpp:116-129): x, g, f; active set of x
    SpgState& hs = *ws.host_state;
    std::memset(&hs, 0, sizeof(hs));
    hs.f = f0;
    hs.L = 10.0;
    hs.n = n;
    hs.ld = (int)ld;
    hs.max_steps = max_steps;
    hs.patience = patience;
    hs.tau = tau;
    hs.eps_stop = eps_stop;
    hs.done = max_steps <= 0 ? 1 : 0;
    std::vector<unsigned char> act0((size_t)n);
    for (int i = 0; i < n; ++i) act0[(size_t)i] = x[(size_t)i] <= tau + 1e-12 ? 1 : 0;
    MVSK_CUDA(cudaMemcpyAsync(st, &hs, sizeof(SpgState), cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemcpyAsync(b.x, x.data(), n * sizeof(double), cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemcpyAsync(b.g, g0.data(), n * sizeof(double), cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemcpyAsync(b.act, act0.data(), (size_t)n, cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemsetAsync(b.xp, 0, ld * sizeof(double), sm));  // zero padding of the FGRAD row

    Slot& sl = ctx->slots[slot];
    PassIO io;
    io.vin = b.xp;
    io.slot = slot;
    io.x_for_mux = b.xp;
    io.skip = &st->eval_flag;
    io.nskip = 1;

    if (!ws.exec || ws.epoch != ctx->epoch || ws.slot != slot) {
        if (ws.exec) cudaGraphExecDestroy(ws.exec);
        ws.exec = nullptr;
        cudaGraph_t gr = nullptr;
        cudaGraphExec_t exec = nullptr;
        const uint64_t p0 = ctx->phys, l0 = ctx->launches;
        bool ok = cudaGraphCreate(&gr, 0) == cudaSuccess;
        cudaGraphConditionalHandle h{};
        cudaGraphNode_t n0 = nullptr, wn = nullptr;
        if (ok) ok = cudaGraphConditionalHandleCreate(&h, gr, 0, 0) == cudaSuccess;
        if (ok) {
            const SpgState* cst = st;
            void* args[] = {&cst, &h};
            cudaKernelNodeParams kp{};
            kp.func = reinterpret_cast<void*>(&spg_cond_kernel);
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
        if (ok) ok = cudaStreamBeginCaptureToGraph(sm, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
                     cudaSuccess;
        if (ok) {
            bool threw = false;
            try {
                ++ctx->launches;
                spg_prep_kernel<<<1, kSpgThreads, smem, sm>>>(st, b);
                run_pass(ctx, Op::FGRAD, 1, io);
                ++ctx->launches;
                spg_accept_kernel<<<1, kSpgThreads, smem, sm>>>(st, b, sl.g, sl.sc, h, 1);
            } catch (...) {
                threw = true;
            }
            cudaGraph_t captured = nullptr;
            ok = cudaStreamEndCapture(sm, &captured) == cudaSuccess && !threw;
        }
        if (ok) ok = cudaGraphInstantiate(&exec, gr, 0) == cudaSuccess;
        const uint64_t dp = ctx->phys - p0, dl = ctx->launches - l0;
        ctx->phys = p0;
        ctx->launches = l0;
        if (gr) cudaGraphDestroy(gr);
        cudaGetLastError();
        if (!ok) {
            if (exec) cudaGraphExecDestroy(exec);
            ws.broken = true;
            MVSK_CUDA(cudaStreamSynchronize(sm));
            return false;
        }
        ws.exec = exec;
        ws.epoch = ctx->epoch;
        ws.slot = slot;
        ws.phys_per_trial = dp;
        ws.launches_per_trial = dl;
    }
    MVSK_CUDA(cudaGraphLaunch(ws.exec, sm));
    MVSK_CUDA(cudaMemcpyAsync(&hs, st, sizeof(SpgState), cudaMemcpyDeviceToHost, sm));
    MVSK_CUDA(cudaMemcpyAsync(x.data(), b.x, n * sizeof(double), cudaMemcpyDeviceToHost, sm));
    MVSK_CUDA(cudaStreamSynchronize(sm));
    // counters: every trial ran prep + accept; the pass ran (and counts) only for
    // the trials with gdp < 0 (a forward pass each; the gradient of an accepted
    // point is the memoised transpose pass, oracle.hpp:79-90, as on the host path)
    ctx->fwd += (uint64_t)hs.evals;
    ctx->tr += (uint64_t)hs.accepts;
    ctx->phys += (uint64_t)hs.evals * ws.phys_per_trial;
    // the condition kernel, prep + accept per trial, the pass's kernels per evaluated trial
    ctx->launches += 1 + 2 * (uint64_t)hs.trials + (uint64_t)hs.evals * (ws.launches_per_trial - 2);
    // the slot's cached point is the last trial, not x: force a fresh make_cache
    sl.valid = false;
    sl.g_host_valid = false;
    sl.scalars_host_valid = false;
    steps_out = hs.steps;
    return true;
}

}  // namespace mvsk_b200
