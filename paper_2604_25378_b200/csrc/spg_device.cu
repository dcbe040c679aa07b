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
#include <cstdio>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "host_ops.hpp"
#include "oracle_ops.cuh"
#include "ptx.cuh"
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
    // device-side timing of the graph variant's prep / accept kernels (cycles)
    long long cyc_prep, cyc_acc;
    // PAR switches: sort = 1 keeps the sorting projection (MVSK_SPG_SORT);
    // prof = 1 adds the phase cycle sums below (MVSK_PROFILE)
    int sort, prof, rounds_max, sort_fallbacks;
    long long cyc_ph[8];
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

// ---- order-free variants for the cluster-resident preamble (n <= 128): the
// dots as warp-0 reductions and the projection's running sums as a warp scan
// (fixed orders, so every CTA of the cluster gets the same bits; not the host
// loop's sequential order)
__device__ __forceinline__ double wdot(const double* a, const double* b, int n) {  // warp 0; lane 0's value
    double s = 0.0;
    for (int i = threadIdx.x & 31; i < n; i += 32) s += a[i] * b[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// the projection of project_slice_dev for n <= 128, in warp 0: the 128 padded
// values sorted in registers (bitonic network, four per lane: in-lane swaps
// for strides < 4, shuffles above), the running sums as a warp scan
__device__ void project_slice_fast(const double* v, int n, double tau, double mass, double* out, double* u,
                                   double* bcast) {
    (void)u;
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        double e[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = 4 * l + j;
            e[j] = k < n ? v[k] - tau : -INFINITY;
        }
#pragma unroll
        for (int size = 2; size <= 128; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                if (stride >= 4) {
                    const bool lower = (l & (stride >> 2)) == 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool desc = ((4 * l + j) & size) == 0;
                        const double w = __shfl_xor_sync(0xffffffffu, e[j], stride >> 2);
                        // the lower index keeps the larger value in a descending block
                        e[j] = (lower == desc) ? fmax(e[j], w) : fmin(e[j], w);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if ((j & stride) == 0) {
                            const int jj = j ^ stride;
                            const bool desc = ((4 * l + j) & size) == 0;
                            const double a0 = e[j], a1 = e[jj];
                            if (desc ? (a0 < a1) : (a0 > a1)) {
                                e[j] = a1;
                                e[jj] = a0;
                            }
                        }
                    }
                }
            }
        }
        const double s = mass - (double)n * tau;
        double p[4];
        double run = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            run += (4 * l + j) < n ? e[j] : 0.0;
            p[j] = run;
        }
        double inc = run;  // inclusive scan of the lane totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, inc, o);
            if (l >= o) inc += t;
        }
        const double excl = inc - run;
        int kb = -1;
        double cb = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = 4 * l + j;
            if (k < n) {
                const double cand = (excl + p[j] - s) / (double)(k + 1);
                if (e[j] > cand) {
                    kb = k;
                    cb = cand;
                }
            }
        }
        int kmax = kb;  // the last support index: theta is its candidate
#pragma unroll
        for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
        if (kmax < 0) {
            if (l == 0) *bcast = 0.0;
        } else if (kb == kmax) {
            *bcast = cb;
        }
    }
    __syncthreads();
    const double theta = *bcast;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = fmax(v[i] - tau - theta, 0.0) + tau;
    __syncthreads();
}

// ---- block-parallel variants for wide panels (PAR): deterministic tree
// reductions and a block scan instead of the host loop's sequential sums
// (n up to kSpgMaxN; the trajectory matches the host loop to rounding)
__device__ double bsum(double v, double* red) {  // every thread returns the block total
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}
__device__ double bdot(const double* a, const double* b, int n, double* red) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i], b[i], s);
    return bsum(s, red);
}

// project_slice with the sorted running sums as a block scan: each thread
// owns a contiguous chunk of the sorted values; theta is the candidate of the
// last index k with u[k] > (css_k - s) / (k + 1) (simplex.hpp:106-113)
__device__ void project_slice_par(const double* v, int n, double tau, double mass, double* out, double* u,
                                  double* bcast, double* red) {
    int m = 1;
    while (m < n) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) u[i] = i < n ? v[i] - tau : -INFINITY;
    bitonic_desc(u, m);
    const int nt = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chunk = (n + nt - 1) / nt;
    const int k0 = min(n, tid * chunk), k1 = min(n, k0 + chunk);
    double tot = 0.0;
    for (int k = k0; k < k1; ++k) tot += u[k];
    // exclusive prefix of the thread totals: warp scans, then the warp totals
    double inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) red[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int nw = (nt + 31) >> 5;
        double w = lane < nw ? red[lane] : 0.0;
        double wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        red[64 + lane] = wi - w;  // exclusive warp offsets
    }
    __syncthreads();
    double css = red[64 + warp] + (inc - tot);
    const double s = mass - (double)n * tau;
    int kb = -1;
    double cb = 0.0;
    for (int k = k0; k < k1; ++k) {
        css += u[k];
        const double cand = (css - s) / (double)(k + 1);
        if (u[k] > cand) {
            kb = k;
            cb = cand;
        }
    }
    // the largest such k over the block (its thread publishes theta)
    int kmax = kb;
#pragma unroll
    for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    __syncthreads();
    if (lane == 0) reinterpret_cast<int*>(red + 96)[warp] = kmax;
    __syncthreads();
    if (tid == 0) {
        int best = -1;
        const int nw = (nt + 31) >> 5;
        for (int w = 0; w < nw; ++w) best = max(best, reinterpret_cast<int*>(red + 96)[w]);
        reinterpret_cast<int*>(red + 96)[40] = best;
        if (best < 0) *bcast = 0.0;
    }
    __syncthreads();
    if (kb >= 0 && kb == reinterpret_cast<int*>(red + 96)[40]) *bcast = cb;
    __syncthreads();
    const double theta = *bcast;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = fmax(v[i] - tau - theta, 0.0) + tau;
    __syncthreads();
}

// ---- register-blocked PAR bodies (wide panels, the graph variant): each of the
// kSpgThreads threads owns the kSpgE entries i = tid + j * kSpgThreads, so every
// n-vector is read with all of a thread's loads in flight at once (the loops
// above serialise one global round trip per entry), and the projection's
// threshold comes without the sort (spg_theta_fixed_point)
constexpr int kSpgE = kSpgMaxN / kSpgThreads;

// block-wide sums of two values (every thread returns both totals)
__device__ __forceinline__ void bsum2(double& a, double& b, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    __syncthreads();
    if (lane == 0) {
        red[warp] = a;
        red[32 + warp] = b;
    }
    __syncthreads();
    if (warp == 0) {
        double t = lane < nw ? red[lane] : 0.0, t2 = lane < nw ? red[32 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            t += __shfl_xor_sync(0xffffffffu, t, o);
            t2 += __shfl_xor_sync(0xffffffffu, t2, o);
        }
        if (lane == 0) {
            red[64] = t;
            red[65] = t2;
        }
    }
    __syncthreads();
    a = red[64];
    b = red[65];
}

// theta of project_slice (simplex.hpp:93-117) without sorting. The reference
// takes theta = (css_k - s) / (k + 1) at the last k of the descending order with
// u[k] > (css_k - s) / (k + 1): the support is S = {u > theta} and theta =
// (sum_S u - s) / |S|. That fixed point is reached from S = all by iterating
// theta <- (sum_{u > theta} u - s) / |{u > theta}| (theta nondecreasing, S
// shrinking; Michelot's algorithm), a few block reductions instead of a
// log^2(n)-stage sorting network. Returns false if S has not settled within
// kRounds rounds (the caller then sorts); rounds: the count used.
__device__ bool spg_theta_fixed_point(const double (&e)[kSpgE], double s, double& theta, int& rounds, double* red) {
    constexpr int kRounds = 48;
    double th = -INFINITY, cprev = -1.0;
    for (int it = 0; it < kRounds; ++it) {
        double sum = 0.0, cnt = 0.0;
#pragma unroll
        for (int j = 0; j < kSpgE; ++j)
            if (e[j] > th) {
                sum += e[j];
                cnt += 1.0;
            }
        bsum2(sum, cnt, red);
        if (cnt == cprev) {
            theta = th;
            rounds = it;
            return true;
        }
        th = (sum - s) / cnt;
        cprev = cnt;
    }
    rounds = kRounds;
    return false;
}

__device__ __forceinline__ void spg_phase(SpgState* st, int k, long long& t) {
    if (st->prof) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const long long now = clock64();
            st->cyc_ph[k] += now - t;
            t = now;
        }
    }
}

struct SpgBufs;
__device__ void spg_prep_par(SpgState* st, const SpgBufs& b, double* u, double* bc);
__device__ void spg_accept_par(SpgState* st, const SpgBufs& b, const double* gp, const double* fp_sc, double* u,
                               double* bc);

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

// one trial's step (solver.hpp:131-145): every thread of the block calls it;
// u: sort scratch (next power of two >= n), bc: 2 broadcast doubles. FAST: the
// order-free reductions above (cluster preamble, n <= 128)
template <bool FAST, bool PAR = false>
__device__ void spg_prep_body(SpgState* st, const SpgBufs& b, double* u, double* bc) {
    __shared__ double red[160];
    const int n = st->n;
    if (threadIdx.x == 0) ++st->trials;
    if constexpr (PAR) {
        if (st->bt == 0) {  // L0 from the BB pair (solver.hpp:131-135)
            double L0 = st->L;
            if (st->have_bb) {
                const double sy = bdot(b.bbs, b.bby, n, red), ss = bdot(b.bbs, b.bbs, n, red);
                L0 = (ss > 0 && sy > 0) ? sy / ss : st->L;
                L0 = fmin(fmax(L0, 1e-2), 1e12);
            }
            __syncthreads();
            if (threadIdx.x == 0) st->Lk = L0;
        }
    } else if constexpr (FAST) {
        if (st->bt == 0 && threadIdx.x < 32) {  // L0 from the BB pair (solver.hpp:131-135)
            double L0 = st->L;
            if (st->have_bb) {
                const double sy = wdot(b.bbs, b.bby, n), ss = wdot(b.bbs, b.bbs, n);
                L0 = (ss > 0 && sy > 0) ? sy / ss : st->L;
                L0 = fmin(fmax(L0, 1e-2), 1e12);
            }
            __syncwarp();
            if (threadIdx.x == 0) st->Lk = L0;
        }
    } else if (st->bt == 0 && threadIdx.x == 0) {  // L0 from the BB pair (solver.hpp:131-135)
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
    if constexpr (PAR)
        project_slice_par(b.y, n, st->tau, 1.0, b.xp, u, &bc[0], red);
    else if constexpr (FAST)
        project_slice_fast(b.y, n, st->tau, 1.0, b.xp, u, &bc[0]);
    else
        project_slice_dev(b.y, n, st->tau, 1.0, b.xp, u, &bc[0]);
    for (int i = threadIdx.x; i < n; i += blockDim.x) b.dp[i] = b.xp[i] - b.x[i];
    __syncthreads();
    if constexpr (PAR) {
        const double gdp = bdot(b.g, b.dp, n, red);
        if (threadIdx.x == 0) {
            st->gdp = gdp;
            st->eval_flag = gdp < 0 ? 1 : 0;
            if (gdp < 0) ++st->evals;
        }
    } else if (FAST ? threadIdx.x < 32 : threadIdx.x == 0) {
        const double gdp = FAST ? wdot(b.g, b.dp, n) : sdot(b.g, b.dp, n);
        if (threadIdx.x == 0) {
            st->gdp = gdp;
            st->eval_flag = gdp < 0 ? 1 : 0;
            if (gdp < 0) ++st->evals;
        }
    }
}

template <bool PAR>
__global__ void __launch_bounds__(kSpgThreads) spg_prep_kernel(SpgState* st, SpgBufs b) {
    extern __shared__ double u[];
    __shared__ double bc[2];
    const long long t0 = clock64();
    if (PAR && !st->sort)
        spg_prep_par(st, b, u, bc);
    else
        spg_prep_body<false, PAR>(st, b, u, bc);
    __syncthreads();
    if (threadIdx.x == 0) st->cyc_prep += clock64() - t0;
}

// Armijo test and the state update of one trial (solver.hpp:146-174): every
// thread of the block calls it; fp is the trial value, gp its gradient
template <bool FAST, bool PAR = false>
__device__ void spg_accept_body(SpgState* st, const SpgBufs& b, const double* gp, double fp, double* u, double* bc) {
    __shared__ int s_acc, s_change, s_any, s_done;
    __shared__ double red[160];
    const int n = st->n;
    if (threadIdx.x == 0) {
        int acc = 0;
        if (st->eval_flag) {
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
            if constexpr (PAR) {
                project_slice_par(b.y, n, st->tau, 1.0, b.dp, u, &bc[0], red);
                double s = 0.0;
                for (int i = threadIdx.x; i < n; i += blockDim.x) {
                    const double d = b.x[i] - b.dp[i];
                    s = fma(d, d, s);
                }
                s = bsum(s, red);
                if (threadIdx.x == 0 && sqrt(s) <= st->eps_stop) st->done = 1;
            } else if constexpr (FAST) {
                project_slice_fast(b.y, n, st->tau, 1.0, b.dp, u, &bc[0]);
                if (threadIdx.x < 32) {
                    double s = 0.0;
                    for (int i = threadIdx.x; i < n; i += 32) {
                        const double d = b.x[i] - b.dp[i];
                        s += d * d;
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    if (threadIdx.x == 0 && sqrt(s) <= st->eps_stop) st->done = 1;
                }
            } else {
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
    }
    __syncthreads();
}

// PAR trial step (spg_prep_body's PAR branch, register-blocked)
__device__ void spg_prep_par(SpgState* st, const SpgBufs& b, double* u, double* bc) {
    __shared__ double red[160];
    const int n = st->n, tid = threadIdx.x;
    long long t = clock64();
    if (tid == 0) ++st->trials;
    const int bt = st->bt;
    double Lk;
    if (bt == 0) {  // L0 from the BB pair (solver.hpp:131-135)
        double L0 = st->L;
        if (st->have_bb) {
            double sy = 0.0, ss = 0.0;
            double bs[kSpgE], by[kSpgE];
#pragma unroll
            for (int j = 0; j < kSpgE; ++j) {
                const int i = tid + j * kSpgThreads;
                bs[j] = i < n ? b.bbs[i] : 0.0;
                by[j] = i < n ? b.bby[i] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < kSpgE; ++j) {
                sy = fma(bs[j], by[j], sy);
                ss = fma(bs[j], bs[j], ss);
            }
            bsum2(sy, ss, red);
            L0 = (ss > 0 && sy > 0) ? sy / ss : st->L;
            L0 = fmin(fmax(L0, 1e-2), 1e12);
        }
        Lk = L0;
        if (tid == 0) st->Lk = L0;
    } else {
        Lk = st->Lk;
    }
    spg_phase(st, 0, t);
    // u = y - tau with y = x - g / Lk (the values project_slice sorts)
    const double tau = st->tau;
    double e[kSpgE];
    {
        double xr[kSpgE], gr[kSpgE];
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            xr[j] = i < n ? b.x[i] : 0.0;
            gr[j] = i < n ? b.g[i] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) e[j] = tid + j * kSpgThreads < n ? (xr[j] - gr[j] / Lk) - tau : -INFINITY;
    }
    spg_phase(st, 1, t);
    const double s = 1.0 - (double)n * tau;
    double theta = 0.0;
    int rounds = 0;
    const bool fixed = spg_theta_fixed_point(e, s, theta, rounds, red);
    spg_phase(st, 2, t);
    double xp[kSpgE];
    if (fixed) {
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            xp[j] = fmax(e[j] - theta, 0.0) + tau;
            if (i < n) b.xp[i] = xp[j];
        }
    } else {  // S did not settle: the sorting projection
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            if (i < n) b.y[i] = b.x[i] - b.g[i] / Lk;
        }
        __syncthreads();
        project_slice_par(b.y, n, tau, 1.0, b.xp, u, &bc[0], red);
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            xp[j] = i < n ? b.xp[i] : 0.0;
        }
    }
    if (tid == 0) {
        st->rounds_max = max(st->rounds_max, rounds);
        if (!fixed) ++st->sort_fallbacks;
    }
    // dp = xp - x and gdp = g'dp
    double gdp = 0.0, zero = 0.0;
    {
        double xr[kSpgE], gr[kSpgE];
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            xr[j] = i < n ? b.x[i] : 0.0;
            gr[j] = i < n ? b.g[i] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            const double d = xp[j] - xr[j];
            if (i < n) {
                b.dp[i] = d;
                gdp = fma(gr[j], d, gdp);
            }
        }
    }
    bsum2(gdp, zero, red);
    if (tid == 0) {
        st->gdp = gdp;
        st->eval_flag = gdp < 0 ? 1 : 0;
        if (gdp < 0) ++st->evals;
    }
    spg_phase(st, 3, t);
}

// PAR Armijo test and state update (spg_accept_body's PAR branch,
// register-blocked; solver.hpp:146-174)
__device__ void spg_accept_par(SpgState* st, const SpgBufs& b, const double* gp, const double* fp_sc, double* u,
                               double* bc) {
    __shared__ int s_acc, s_change, s_any, s_done;
    __shared__ double red[160];
    const int n = st->n, tid = threadIdx.x;
    long long t = clock64();
    if (tid == 0) {
        const double fp = fp_sc[0];  // read unconditionally: only used when the pass ran
        int acc = 0;
        if (st->eval_flag) {
            if (fp <= __dadd_rn(st->f, __dmul_rn(1e-4, st->gdp))) {  // Armijo (solver.hpp:146)
                acc = 1;
                st->f = fp;
                st->L = st->Lk;
                st->have_bb = 1;
                ++st->accepts;
            }
        }
        s_acc = acc;
        s_change = 0;
        s_any = 0;
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
    if (!s_acc) {
        spg_phase(st, 4, t);
        return;
    }
    // BB pair, iterate and gradient; active set (<= tau + 1e-12) and patience (:163-172)
    const double thr = st->tau + 1e-12;
    int chg = 0, any = 0;
    {
        double dp[kSpgE], gold[kSpgE], xn[kSpgE], gn[kSpgE];
        unsigned char a0[kSpgE];
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            const bool in = i < n;
            dp[j] = in ? b.dp[i] : 0.0;
            gn[j] = in ? gp[i] : 0.0;
            gold[j] = in ? b.g[i] : 0.0;
            xn[j] = in ? b.xp[i] : 0.0;
            a0[j] = in ? b.act[i] : 0;
        }
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            if (i < n) {
                b.bbs[i] = dp[j];
                b.bby[i] = gn[j] - gold[j];
                b.x[i] = xn[j];
                b.g[i] = gn[j];
                const unsigned char a = xn[j] <= thr ? 1 : 0;
                if (a != a0[j]) chg = 1;
                if (a) any = 1;
                b.act[i] = a;
            }
        }
    }
    chg = __syncthreads_or(chg);
    any = __syncthreads_or(any);
    if (tid == 0) {
        const int steps = ++st->steps;
        st->bt = 0;
        ++st->k;
        int done = 0;
        if (chg) {
            st->last_change = steps;
        } else if (any && steps - st->last_change >= st->patience) {
            done = 1;
        }
        if (st->k >= st->max_steps) done = 1;
        s_done = done;
        st->done = done;
    }
    __syncthreads();
    spg_phase(st, 5, t);
    // every 10 steps: gradient-mapping residual ||x - P(x - g)|| (:173-174)
    if (!s_done && st->eps_stop > 0 && st->steps % 10 == 0) {
        const double tau = st->tau;
        double e[kSpgE], xn[kSpgE];
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) {
            const int i = tid + j * kSpgThreads;
            xn[j] = i < n ? b.x[i] : 0.0;
            e[j] = i < n ? b.g[i] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kSpgE; ++j) e[j] = tid + j * kSpgThreads < n ? (xn[j] - e[j]) - tau : -INFINITY;
        const double s = 1.0 - (double)n * tau;
        double theta = 0.0, r2 = 0.0, zero = 0.0;
        int rounds = 0;
        if (spg_theta_fixed_point(e, s, theta, rounds, red)) {
#pragma unroll
            for (int j = 0; j < kSpgE; ++j)
                if (tid + j * kSpgThreads < n) {
                    const double d = xn[j] - (fmax(e[j] - theta, 0.0) + tau);
                    r2 = fma(d, d, r2);
                }
        } else {
#pragma unroll
            for (int j = 0; j < kSpgE; ++j) {
                const int i = tid + j * kSpgThreads;
                if (i < n) b.y[i] = xn[j] - b.g[i];
            }
            __syncthreads();
            project_slice_par(b.y, n, tau, 1.0, b.dp, u, &bc[0], red);
#pragma unroll
            for (int j = 0; j < kSpgE; ++j) {
                const int i = tid + j * kSpgThreads;
                if (i < n) {
                    const double d = xn[j] - b.dp[i];
                    r2 = fma(d, d, r2);
                }
            }
            if (tid == 0) ++st->sort_fallbacks;
        }
        bsum2(r2, zero, red);
        if (tid == 0) {
            st->rounds_max = max(st->rounds_max, rounds);
            if (sqrt(r2) <= st->eps_stop) st->done = 1;
        }
        spg_phase(st, 6, t);
    }
    __syncthreads();
}

template <bool PAR>
__global__ void __launch_bounds__(kSpgThreads) spg_accept_kernel(SpgState* st, SpgBufs b, const double* gp,
                                                                 const double* fp_sc, cudaGraphConditionalHandle h,
                                                                 int set_cond) {
    extern __shared__ double u[];
    __shared__ double bc[2];
    const long long t0 = clock64();
    if (PAR && !st->sort)
        spg_accept_par(st, b, gp, fp_sc, u, bc);
    else
        spg_accept_body<false, PAR>(st, b, gp, st->eval_flag ? fp_sc[0] : 0.0, u, bc);
    if (threadIdx.x == 0) st->cyc_acc += clock64() - t0;
    if (set_cond && threadIdx.x == 0) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

// ---------------------------------------------------------------------------
// Cluster-resident preamble for narrow, short panels (ld <= 128 and each
// 16th of the rows fits a CTA's shared memory: C1 / C2). The whole loop runs
// in ONE launch of one 16-CTA cluster: every CTA stages its row block once
// (bulk copies issued by all warps), then per trial
//   prep (spg_prep_body)     redundantly in every CTA on identical bits
//   FGRAD at xp              each CTA over its rows: z = <x_t, xp>, the power
//                            sums and A^T psi'(z) partials; combined through
//                            distributed shared memory in rank order behind
//                            one cluster barrier (double-buffered partials)
//   accept (spg_accept_body) redundantly, so every CTA takes the same branches
// A trial costs a cluster barrier instead of three kernel boundaries (or a
// host round trip). f and the gradient are the oracle's (oracle.hpp:58-64,
// 82-84) with a different summation order than the streaming pass, so the
// trajectory matches the host loop to rounding, not bitwise.
// ---------------------------------------------------------------------------
constexpr int kSpgCS = 16;     // CTAs per cluster (non-portable size)
constexpr int kSpgCW = 8;      // warps per CTA
constexpr int kSpgCM = 128;    // max ld
constexpr int kSpgCP = kSpgCM + 4;  // partial row: ld gradient entries + 3 power sums

struct SpgClusterArgs {
    SpgState* st;   // global state: initial in, final out (CTA 0)
    SpgBufs gb;     // global x (in / out), g, act (in)
    const double* X;
    const double* mu;
    long long T;
    int ld;
    double c1, c2, c3, c4, Tg, vo;
    unsigned long long* prof;  // timing studies (MVSK_SPG_PROF): prep / pass / accept cycle sums of CTA 0
};

constexpr size_t spg_cluster_smem_fixed() {
    return (size_t)(10 * kSpgCM + 2 * kSpgCP + kSpgCW * kSpgCP) * sizeof(double) + kSpgCM + 64;
}

template <int LPR, int CPL>
__global__ void __launch_bounds__(kSpgCW * 32, 1) spg_cluster_kernel(const SpgClusterArgs a) {
    namespace cgs = cooperative_groups;
    static_assert(LPR * CPL <= kSpgCM && CPL % 2 == 0 && 32 % LPR == 0, "row layout");
    constexpr int M = kSpgCM, MP = kSpgCP, CS = kSpgCS;
    cgs::cluster_group cluster = cgs::this_cluster();
    const int crank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ld = a.ld;
    extern __shared__ __align__(16) double sp_sm[];
    double* sx = sp_sm;
    double* sg = sx + M;
    double* sxp = sg + M;
    double* sdp = sxp + M;
    double* sbs = sdp + M;
    double* sby = sbs + M;
    double* sy = sby + M;
    double* su = sy + M;   // sort scratch
    double* sgp = su + M;  // trial gradient
    double* smu = sgp + M;
    double* spart = smu + M;     // [2][MP]
    double* sW = spart + 2 * MP;  // [warps][MP]
    unsigned char* sact = reinterpret_cast<unsigned char*>(sW + kSpgCW * MP);
    const long long T = a.T;
    const long long r0 = T * crank / CS, r1 = T * (crank + 1) / CS;
    const int nloc = (int)(r1 - r0);
    const int lds = ld + 2;  // padded rows: the row groups of a warp on distinct bank groups
    double* sXp = sp_sm + (spg_cluster_smem_fixed() + 15) / 16 * 2;
    __shared__ SpgState sst;
    __shared__ double sbc[4];
    __shared__ uint64_t stage_bar;
    if (tid == 0) {
        mbar_init(&stage_bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&stage_bar, (uint32_t)((size_t)nloc * ld * sizeof(double)));
        sst = *a.st;
    }
    __syncthreads();
    {
        const uint64_t pol = policy_evict_last();
        for (int r = tid; r < nloc; r += blockDim.x)
            bulk_g2s(sXp + (size_t)r * lds, a.X + (r0 + r) * (long long)ld, (uint32_t)(ld * sizeof(double)),
                     &stage_bar, pol);
    }
    const int n = sst.n;
    for (int i = tid; i < M; i += blockDim.x) {
        const bool in = i < n;
        const double x = in ? __ldg(a.gb.x + i) : 0.0, g = in ? __ldg(a.gb.g + i) : 0.0;
        const double mu = in ? __ldg(a.mu + i) : 0.0;
        const unsigned char ac = in ? a.gb.act[i] : 0;
        sx[i] = x;
        sg[i] = g;
        smu[i] = mu;
        sact[i] = ac;
        sxp[i] = 0.0;  // zero past n: the FGRAD row's padding
    }
    mbar_wait(&stage_bar, 0u);
    __syncthreads();
    const SpgBufs sb{sx, sg, sxp, sdp, sbs, sby, sy, sact};

    constexpr int GPW = 32 / LPR;
    constexpr int NGC = kSpgCW * GPW;
    const int sub = lane % LPR;
    auto colp = [&](int j) { return 2 * ((j >> 1) * LPR + sub) + (j & 1); };
    int step = 0;
    const bool prof_on = a.prof && crank == 0 && tid == 0;
    unsigned long long pt[3] = {0, 0, 0}, tc = clock64();
    auto mark = [&](int i) {
        if (prof_on) {
            const unsigned long long now = clock64();
            pt[i] += now - tc;
            tc = now;
        }
    };
    while (!sst.done) {
        spg_prep_body<true>(&sst, sb, su, sbc);
        __syncthreads();
        mark(0);
        double fp = 0.0;
        if (sst.eval_flag) {
            // ---- FGRAD over this CTA's rows at xp (oracle.hpp:58-64, 82-83)
            double acc[CPL], xv[CPL];
#pragma unroll
            for (int j = 0; j < CPL; j += 2) {  // this lane's slice of xp, held for the pass
                const double2 v = *reinterpret_cast<const double2*>(sxp + colp(j));
                xv[j] = v.x;
                xv[j + 1] = v.y;
                acc[j] = acc[j + 1] = 0.0;
            }
            double s2 = 0.0, s3 = 0.0, s4 = 0.0;
            for (int lb = warp * GPW; lb < nloc; lb += NGC) {  // warp-uniform trip count
                const int tl = lb + lane / LPR;
                const bool rv = tl < nloc;
                const double* xr = sXp + (size_t)(rv ? tl : 0) * lds;
                double x[CPL];
#pragma unroll
                for (int j = 0; j < CPL; j += 2) {
                    double2 v = make_double2(0.0, 0.0);
                    if (rv && colp(j) < ld) v = *reinterpret_cast<const double2*>(xr + colp(j));
                    x[j] = v.x;
                    x[j + 1] = v.y;
                }
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int j = 0; j < CPL; j += 2) {
                    d0 = fma(x[j], xv[j], d0);
                    d1 = fma(x[j + 1], xv[j + 1], d1);
                }
                double zt = d0 + d1;
#pragma unroll
                for (int o = 1; o < LPR; o <<= 1) zt += __shfl_xor_sync(0xffffffffu, zt, o);
                const double z2 = zt * zt, z3 = z2 * zt;
                const double w = rv ? 2.0 * a.c2 * zt - 3.0 * a.c3 * z2 + 4.0 * a.c4 * z3 : 0.0;
#pragma unroll
                for (int j = 0; j < CPL; ++j) acc[j] = fma(x[j], w, acc[j]);
                if (rv && sub == 0) {
                    s2 += z2;
                    s3 += z3;
                    s4 += z2 * z2;
                }
            }
#pragma unroll
            for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
                for (int j = 0; j < CPL; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                s2 += __shfl_xor_sync(0xffffffffu, s2, o);
                s3 += __shfl_xor_sync(0xffffffffu, s3, o);
                s4 += __shfl_xor_sync(0xffffffffu, s4, o);
            }
            if (lane < LPR) {
#pragma unroll
                for (int j = 0; j < CPL; ++j)
                    if (colp(j) < M) sW[warp * MP + colp(j)] = acc[j];
            }
            if (lane == 0) {
                sW[warp * MP + M] = s2;
                sW[warp * MP + M + 1] = s3;
                sW[warp * MP + M + 2] = s4;
            }
            __syncthreads();
            double* buf = spart + (step & 1) * MP;
            for (int e = tid; e < MP; e += blockDim.x) {
                if (e >= ld && e < M) continue;
                double v = 0.0;
#pragma unroll
                for (int w2 = 0; w2 < kSpgCW; ++w2) v += sW[w2 * MP + e];
                buf[e] = v;
            }
            // ---- cluster combine: every CTA sums the CS partials in rank order
            cluster.sync();
            for (int e = tid; e < MP; e += blockDim.x) {
                if (e >= n && e < M) continue;
                if (e >= M + 3) continue;
                double pv[CS];
#pragma unroll
                for (int r = 0; r < CS; ++r) pv[r] = cluster.map_shared_rank(buf, r)[e];
                double v = 0.0;
#pragma unroll
                for (int r = 0; r < CS; ++r) v += pv[r];
                if (e < M)
                    sgp[e] = -a.c1 * smu[e] + v / a.Tg;  // oracle.hpp:82-84
                else
                    sbc[e - M + 1] = v;  // power sums (sbc[0] is the projection's broadcast)
            }
            __syncthreads();
            if (tid < 32) {  // mu'xp (fixed-order warp reduction), then f (oracle.hpp:62-64)
                const double mux = wdot(smu, sxp, n);
                if (tid == 0) sbc[0] = a.vo - a.c1 * mux + (a.c2 * sbc[1] - a.c3 * sbc[2] + a.c4 * sbc[3]) / a.Tg;
            }
            __syncthreads();
            fp = sbc[0];
            ++step;
        }
        mark(1);
        spg_accept_body<true>(&sst, sb, sgp, fp, su, sbc);
        __syncthreads();
        mark(2);
    }
    if (prof_on)
        for (int i = 0; i < 3; ++i) a.prof[i] += pt[i];
    if (crank == 0) {
        for (int i = tid; i < n; i += blockDim.x) a.gb.x[i] = sx[i];
        if (tid == 0) *a.st = sst;
    }
    cluster.sync();  // no CTA exits while a peer may still read its partials
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
    static const bool no_cluster = std::getenv("MVSK_NO_SPG_CLUSTER") != nullptr;
    const int n = (int)ctx->n;
    if (n < 2 || ctx->zoff_dev) return false;
    // narrow short panels: the whole preamble in one cluster launch (default)
    const long long nloc = (ctx->T_local + kSpgCS - 1) / kSpgCS;
    const size_t cl_smem = (spg_cluster_smem_fixed() + 15) / 16 * 16 + (size_t)nloc * (ctx->ld + 2) * sizeof(double);
    const void* cl_fn = ctx->ld <= 64 ? (const void*)&spg_cluster_kernel<4, 16> : (const void*)&spg_cluster_kernel<8, 16>;
    const bool cluster_ok = !no_cluster && ctx->nranks == 1 && ctx->ld <= kSpgCM &&  // no exchange at one rank
                            ctx->T_local >= kSpgCS && cl_smem <= ctx->max_smem &&
                            cluster_fits(cl_fn, kSpgCS, kSpgCW * 32, cl_smem);
    // wide panels (no cluster preamble): the conditional-while graph with the
    // block-parallel reductions by default (MVSK_NO_SPG_GRAPH: host loop);
    // MVSK_SPG_GRAPH keeps the bitwise-host-order variant for A/B
    static const bool no_graph = std::getenv("MVSK_NO_SPG_GRAPH") != nullptr;
    const bool par = !enabled;
    if (!cluster_ok && ((!enabled && (no_graph || ctx->ld <= kSpgCM)) || ctx->no_capture || n > kSpgMaxN)) return false;
    if (!ctx->spg) ctx->spg = new SpgWorkspace();
    SpgWorkspace& ws = *ctx->spg;
    if (ws.broken && !cluster_ok) return false;
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
    const void* prep_fn = par ? reinterpret_cast<const void*>(&spg_prep_kernel<true>)
                              : reinterpret_cast<const void*>(&spg_prep_kernel<false>);
    const void* acc_fn = par ? reinterpret_cast<const void*>(&spg_accept_kernel<true>)
                             : reinterpret_cast<const void*>(&spg_accept_kernel<false>);
    set_smem_attr(prep_fn, smem);
    set_smem_attr(acc_fn, smem);

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
    static const bool sort_proj = std::getenv("MVSK_SPG_SORT") != nullptr;
    static const bool prof_ph = std::getenv("MVSK_PROFILE") != nullptr;
    hs.sort = sort_proj ? 1 : 0;
    hs.prof = prof_ph ? 1 : 0;
    std::vector<unsigned char> act0((size_t)n);
    for (int i = 0; i < n; ++i) act0[(size_t)i] = x[(size_t)i] <= tau + 1e-12 ? 1 : 0;
    MVSK_CUDA(cudaMemcpyAsync(st, &hs, sizeof(SpgState), cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemcpyAsync(b.x, x.data(), n * sizeof(double), cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemcpyAsync(b.g, g0.data(), n * sizeof(double), cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemcpyAsync(b.act, act0.data(), (size_t)n, cudaMemcpyHostToDevice, sm));
    MVSK_CUDA(cudaMemsetAsync(b.xp, 0, ld * sizeof(double), sm));  // zero padding of the FGRAD row

    Slot& sl = ctx->slots[slot];
    if (cluster_ok) {
        SpgClusterArgs ca{};
        ca.st = st;
        ca.gb = b;
        ca.X = ctx->X;
        ca.mu = ctx->mu_dev;
        ca.T = ctx->T_local;
        ca.ld = (int)ld;
        ca.c1 = ctx->c.c1;
        ca.c2 = ctx->c.c2;
        ca.c3 = ctx->c.c3;
        ca.c4 = ctx->c.c4;
        ca.Tg = (double)ctx->T_global;
        ca.vo = ctx->value_offset;
        static unsigned long long* prof = nullptr;  // MVSK_SPG_PROF: cycle sums, printed at exit
        if (std::getenv("MVSK_SPG_PROF")) {
            if (!prof) {
                MVSK_CUDA(cudaMallocManaged(&prof, 4 * sizeof(unsigned long long)));
                std::memset(prof, 0, 4 * sizeof(unsigned long long));
                std::atexit([] {
                    cudaDeviceSynchronize();
                    std::fprintf(stderr, "[spg prof] prep %llu pass %llu accept %llu (cycles)\n", prof[0], prof[1],
                                 prof[2]);
                });
            }
            ca.prof = prof;
        }
        const void* fn = cl_fn;  // attributes set by cluster_fits
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kSpgCS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(kSpgCS);
        cfg.blockDim = dim3(kSpgCW * 32);
        cfg.dynamicSmemBytes = cl_smem;
        cfg.stream = sm;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        void* args[] = {&ca};
        ++ctx->launches;
        MVSK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
        MVSK_CUDA(cudaMemcpyAsync(&hs, st, sizeof(SpgState), cudaMemcpyDeviceToHost, sm));
        MVSK_CUDA(cudaMemcpyAsync(x.data(), b.x, n * sizeof(double), cudaMemcpyDeviceToHost, sm));
        MVSK_CUDA(cudaStreamSynchronize(sm));
        // a forward pass per evaluated trial, the memoised transpose per accepted one
        // (oracle.hpp:79-90), one physical pass per evaluation
        ctx->fwd += (uint64_t)hs.evals;
        ctx->tr += (uint64_t)hs.accepts;
        ctx->phys += (uint64_t)hs.evals;
        static const bool verbose = std::getenv("MVSK_PROFILE") != nullptr;
        if (verbose) std::fprintf(stderr, "[spg cluster] trials %d evals %d steps %d\n", hs.trials, hs.evals, hs.steps);
        sl.valid = false;
        sl.g_host_valid = false;
        sl.scalars_host_valid = false;
        steps_out = hs.steps;
        return true;
    }
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
                if (par)
                    spg_prep_kernel<true><<<1, kSpgThreads, smem, sm>>>(st, b);
                else
                    spg_prep_kernel<false><<<1, kSpgThreads, smem, sm>>>(st, b);
                run_pass(ctx, Op::FGRAD, 1, io);
                ++ctx->launches;
                if (par)
                    spg_accept_kernel<true><<<1, kSpgThreads, smem, sm>>>(st, b, sl.g, sl.sc, h, 1);
                else
                    spg_accept_kernel<false><<<1, kSpgThreads, smem, sm>>>(st, b, sl.g, sl.sc, h, 1);
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
    static const bool verbose_g = std::getenv("MVSK_PROFILE") != nullptr;
    if (verbose_g)
        std::fprintf(stderr,
                     "[spg graph] trials %d evals %d steps %d prep %.1f us accept %.1f us (sum, at 1.9 GHz) "
                     "sort %d rounds_max %d fallbacks %d phases us: L0 %.1f load %.1f theta %.1f out %.1f "
                     "reject %.1f update %.1f resid %.1f\n",
                     hs.trials, hs.evals, hs.steps, hs.cyc_prep / 1.9e3, hs.cyc_acc / 1.9e3, hs.sort, hs.rounds_max,
                     hs.sort_fallbacks, hs.cyc_ph[0] / 1.9e3, hs.cyc_ph[1] / 1.9e3, hs.cyc_ph[2] / 1.9e3,
                     hs.cyc_ph[3] / 1.9e3, hs.cyc_ph[4] / 1.9e3, hs.cyc_ph[5] / 1.9e3, hs.cyc_ph[6] / 1.9e3);
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
