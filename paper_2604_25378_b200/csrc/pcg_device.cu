// Device-resident PCG for the YAND direction (affine_normal.hpp:189-242).
//
// The reduced tangent operator H e = Q^T U^T grad2 f (U Q e) + lambda e is
// applied without leaving the device: the Householder reflectors (U:
// simplex.hpp:63-70, Q: affine_normal.hpp:28-33) lift every CG column into the
// HVP input rows (face -> full coordinates), one fused k-RHS HVP pass runs, and
// the step kernel gathers, applies Q^T U^T (:36-39, simplex.hpp:73-78),
// performs the capped-CG step of every column (cg_capped, :85-113: per-column
// alpha/beta, nonpositive curvature -> breakdown, ||r|| <= tol ||rhs|| or the
// cap -> stop) and lifts the next search direction. One CTA owns one column;
// every reduction has a fixed order.
//
// Scheduling: each Krylov loop is a conditional-while CUDA graph (the last
// column CTA sets the loop condition), and a whole Hutchinson / no-third
// direction - uploads, Jacobi diagonal, h, the probe block, the third-action
// pass, the rhs, the main CG and the readbacks - is captured once per shape
// (the loops spliced in as conditional nodes) and replayed with its
// parameters in device memory: one graph launch and one synchronisation per
// direction. The first direction of a shape runs eagerly (it sizes every
// workspace); exact-trace sweeps and > 16 probes stay eager.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#include <cooperative_groups.h>

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

// step parameters live in device memory so one instantiated graph serves every
// direction (the reflector scalars, face size, cap and tolerance change)
struct StepParams {
    Geo g;
    CGState s;
    double lambda;
};

__global__ void __launch_bounds__(kPT) cg_init_kernel(const StepParams* sp, const double* rhs, double* vin) {
    extern __shared__ double q[];
    __shared__ double sh[32];
    const Geo g = sp->g;
    const CGState s = sp->s;
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
// E rows have stride mm (apply_q) or m - 1 (U only), the face sizes of *gp
__global__ void __launch_bounds__(kPT) lift_kernel(const Geo* gp, const double* E, bool apply_q, const int* active,
                                                   double* vin) {
    extern __shared__ double q[];
    __shared__ double sh[32];
    const Geo g = *gp;
    const int ldE = apply_q ? g.m - 2 : g.m - 1;
    const int c = blockIdx.x;
    double* row = vin + (size_t)c * g.ld;
    if (active && !active[c]) {
        for (int i = threadIdx.x; i < g.ld; i += blockDim.x) row[i] = 0.0;
        return;
    }
    lift_col(g, E + (size_t)c * ldE, apply_q, row, q, sh);
}

// lift two source blocks of k columns each in one launch (the third-action
// pair u = U Q s_p, v = U Q r_p): blocks [0, k) lift E1 into vin1, [k, 2k) E2 into vin2
__global__ void __launch_bounds__(kPT) lift_pair_kernel(const Geo* gp, const double* E1, const double* E2, int k,
                                                        double* vin1, double* vin2) {
    extern __shared__ double q[];
    __shared__ double sh[32];
    const Geo g = *gp;
    const int ldE = g.m - 2;
    const bool second = (int)blockIdx.x >= k;
    const int c = second ? (int)blockIdx.x - k : (int)blockIdx.x;
    lift_col(g, (second ? E2 : E1) + (size_t)c * ldE, true, (second ? vin2 : vin1) + (size_t)c * g.ld, q, sh);
}

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
__global__ void __launch_bounds__(kPT) reduce_kernel(const Geo* gp, const double* H, bool apply_q, double* out) {
    extern __shared__ double t[];
    __shared__ double sh[32];
    const Geo g = *gp;
    const int ldo = g.m - 2;
    const int c = blockIdx.x;
    const double* r = reduce_col(g, H + (size_t)c * g.ld, apply_q, t, sh);
    const int len = apply_q ? g.m - 2 : g.m - 1;
    for (int i = threadIdx.x; i < len; i += blockDim.x) out[(size_t)c * ldo + i] = r[i];
}

// per-direction scalars of the elementwise kernels (device memory, graph-stable)
struct DirScalars {
    int mm;
    double lambda, fl, adiv, coef;
};

// Jacobi diagonal from the probe responses (:197-209): mean over probes of
// r o (Qt Ut H U Q r + lambda r), floored at max(1e-12, lambda); probe order fixed
__global__ void jacobi_diag_kernel(const DirScalars* ds, const double* probes, const double* rows, int k, double* jd) {
    const int mm = ds->mm;
    const double lambda = ds->lambda, fl = ds->fl;
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
__global__ void unit_probe_kernel(const DirScalars* ds, double* src, int k, int b0) {
    const int mm = ds->mm;
    const size_t tot = (size_t)k * mm;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        const int p = (int)(e / mm), i = (int)(e - (size_t)p * mm);
        src[e] = (i == b0 + p) ? 1.0 : 0.0;
    }
}

// a += sum of the block's third-action rows, in probe order (:225, :235)
__global__ void accum_rows_kernel(const DirScalars* ds, const double* rows, int k, double* a) {
    const int mm = ds->mm;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mm; i += gridDim.x * blockDim.x) {
        double v = a[i];
        for (int p = 0; p < k; ++p) v += rows[(size_t)p * mm + i];
        a[i] = v;
    }
}

// the last probe block's accumulation fused with the rhs (below): a += rows in
// probe order, then rhs = h - coef * a / adiv, elementwise as the two kernels
__global__ void accum_rhs_kernel(const DirScalars* ds, const double* rows, int k, double* a, const double* h,
                                 double* rhs) {
    const int mm = ds->mm;
    const double adiv = ds->adiv, coef = ds->coef;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mm; i += gridDim.x * blockDim.x) {
        double v = a[i];
        for (int p = 0; p < k; ++p) v += rows[(size_t)p * mm + i];
        a[i] = v;
        const double ai = adiv > 0 ? v / adiv : v;
        rhs[i] = h[i] - coef * ai;
    }
}

// rhs = h - (||gbar|| / n) a, a averaged over the Hutchinson probes (:236, :239)
__global__ void rhs_kernel(const DirScalars* ds, const double* h, const double* a, double* rhs) {
    const int mm = ds->mm;
    const double adiv = ds->adiv, coef = ds->coef;
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


// ---------------------------------------------------------------------------
// Cluster-resident Krylov loop for narrow panels (ld <= 128: compact faces,
// small problems). One thread-block cluster runs a whole capped-CG loop
// (cg_capped, affine_normal.hpp:85-113) for k <= 8 columns in lock-step:
// the CG state lives in shared memory, every HVP pass is streamed by all CTAs
// of the cluster (row groups of LPR lanes, the panel from L2/HBM), the CTA
// partials are combined through distributed shared memory in rank order (one
// cluster barrier per step, double-buffered), and the small per-column algebra
// (Householder lift / reduce, alpha, beta, the stop test) is computed
// redundantly by every CTA, one warp per column, on identical bits - so every
// CTA takes the same branches and no broadcast is needed. Replaces, per CG
// step, an HVP pass kernel and a cg_step kernel (~20 us on C4 faces) with
// in-cluster work and one barrier.
// ---------------------------------------------------------------------------
constexpr int kCcgMaxLd = 128;
constexpr int kCcgCS = 16;     // CTAs per cluster (non-portable size)
constexpr int kCcgWarps = 8;   // warps per CTA

struct CcgArgs {
    const StepParams* sp;  // geometry + CG state arrays (global) + lambda
    const double* rhs;     // k x mm
    const double* X;       // panel T x ld
    const double* z;       // cached z (T)
    long long T;
    int ld, k;
    double c2, c3, c4, invT;
    unsigned long long* prof;  // timing studies: per-phase clock64 sums of one CTA (or null)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// shared memory of cluster_cg_kernel: CG state and scratch, plus (PANEL) the
// CTA's rows of the panel (stride ld + 2) and their z
constexpr size_t ccg_smem_bytes() {
    constexpr int M = kCcgMaxLd;
    return (size_t)(4 * M + 2 * M + 2 * M + kCcgWarps * M + M + 3 * M + 2) * sizeof(double) +
           (size_t)(M + 8) * sizeof(int) + 16;
}

// Cluster-resident capped CG (cg_capped, affine_normal.hpp:85-113) for one
// column per cluster; k columns run as k clusters side by side. The column's
// state lives in shared memory; each HVP pass is streamed by the cluster's 16
// CTAs over contiguous row blocks (PANEL: the block is staged in shared memory
// once and re-read every step), the partials are combined through distributed
// shared memory in rank order (one cluster barrier per step, double-buffered)
// and the per-column algebra (Householder reduce / lift, alpha, beta, the stop
// test) is computed by warp 0 of every CTA on identical bits, so every CTA
// takes the same branches. LPR lanes per row, CPL columns per lane.
template <int LPR, int CPL, bool PANEL>
__global__ void __launch_bounds__(kCcgWarps * 32, 1) cluster_cg_kernel(const CcgArgs a) {
    namespace cgs = cooperative_groups;
    constexpr int M = kCcgMaxLd;
    constexpr int CS = kCcgCS;
    static_assert(LPR * CPL <= M && CPL % 2 == 0 && 32 % LPR == 0, "row layout");
    cgs::cluster_group cluster = cgs::this_cluster();
    const unsigned long long t_entry = clock64();
    const int crank = (int)cluster.block_rank();
    const int col = blockIdx.x / CS;  // the CG column of this cluster
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Geo g = a.sp->g;
    const CGState s = a.sp->s;
    const double lambda = a.sp->lambda;
    const int ld = a.ld, m = g.m, m1 = m - 1, mm = s.mm;

    extern __shared__ __align__(16) double ccg_sm[];
    double* sX = ccg_sm;
    double* sR = sX + M;
    double* sZ = sR + M;
    double* sP = sZ + M;
    double* sV = sP + M;          // lifted search direction (panel coordinates), zero past the face
    double* sH = sV + M;          // HVP row
    double* sPart = sH + M;       // [2][M] this CTA's pass partial (double-buffered)
    double* sW = sPart + 2 * M;   // [warps][M] warp partials
    double* sT = sW + kCcgWarps * M;  // reduce / lift scratch (warp 0)
    double* sU = sT + M;
    double* sQ = sU + M;
    double* sJ = sQ + M;
    double* sSc = sJ + M;         // [rz, target]
    int* sIdx = reinterpret_cast<int*>(sSc + 2);
    int* sFlag = sIdx + M;        // [active, iters, breakdown]
    const long long T = a.T;
    const long long r0 = T * crank / CS, r1 = T * (crank + 1) / CS;
    const int nloc = (int)(r1 - r0);
    // (offset from ccg_sm so the compiler keeps the shared address space)
    double* sXp = ccg_sm + ((size_t)(reinterpret_cast<char*>(sFlag + 8) - reinterpret_cast<char*>(ccg_sm)) + 15) / 16 * 2;
    // smem rows padded by one 16-byte pair (stride ld + 2): the row groups of a
    // warp fall on distinct bank groups
    const int lds = ld + 2;
    double* sZr = sXp + (size_t)nloc * lds;
    __shared__ uint64_t stage_bar;
    __shared__ double sCq;  // Q.U(+1) = sum_j Q_j U_{j+1}, fixed per direction
    if constexpr (PANEL) {
        // the CTA's row block -> shared memory by the bulk-copy engine (one
        // 16-byte-aligned copy per row, completion as tx-bytes on stage_bar)
        // The byte count is armed before the barrier below, so copies issued by
        // any warp afterwards cannot complete the phase early; every warp
        // issues a share of the rows (one issuing warp took ~10 us at C4)
        if (tid == 0) {
            mbar_init(&stage_bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(&stage_bar, (uint32_t)((size_t)nloc * ld * sizeof(double)));
        }
        __syncthreads();
        {
            const uint64_t pol = policy_evict_last();
            for (int r = tid; r < nloc; r += blockDim.x)
                bulk_g2s(sXp + (size_t)r * lds, a.X + (r0 + r) * (long long)ld, (uint32_t)(ld * sizeof(double)),
                         &stage_bar, pol);
        }
    }
    // every small operand in ONE batch of independent read-only loads (z rows,
    // U / Q reflectors, face map, Jacobi diagonal, the column's right-hand side
    // into sT): the separate loops were a chain of dependent global latencies
    // (~12 us of prologue per launch on C4 faces)
    const double* rhs_col = a.rhs + (size_t)col * mm;
    const int nmax = max(max(nloc, M), mm);
    for (int i = tid; i < nmax; i += blockDim.x) {
        const double zr = (PANEL && i < nloc) ? __ldg(a.z + r0 + i) : 0.0;
        const double u = i < m ? __ldg(g.vU + i) : 0.0;
        const long long ix = (i < m && g.idx) ? __ldg(g.idx + i) : (long long)i;
        const double q = i < m1 ? __ldg(g.vQ + i) : 0.0;
        const double j = (i < mm && s.jd) ? __ldg(s.jd + i) : 1.0;
        const double b = i < mm ? __ldg(rhs_col + i) : 0.0;
        if (PANEL && i < nloc) sZr[i] = zr;
        if (i < m) {
            sU[i] = u;
            sIdx[i] = (int)ix;
        }
        if (i < m1) sQ[i] = q;
        if (i < mm) {
            sJ[i] = j;
            sT[i] = b;
        }
        if (i < M) sV[i] = 0.0;
    }
    const unsigned long long t_loads = clock64();
    if constexpr (PANEL) mbar_wait(&stage_bar, 0u);
    __syncthreads();
    const unsigned long long t_staged = clock64();

    // lift: V = U Q (0, P) (lift_col), warp 0
    auto lift = [&]() {
        double* q = sT;
        double part = 0.0;
        for (int i = lane; i < m1; i += 32) {
            const double v = i == 0 ? 0.0 : sP[i - 1];
            q[i] = v;
            part += sQ[i] * v;
        }
        const double s1 = g.bQ * warp_sum(part);
        for (int i = lane; i < m1; i += 32) q[i] -= s1 * sQ[i];
        __syncwarp();
        double part2 = 0.0;
        for (int i = lane + 1; i < m; i += 32) part2 += sU[i] * q[i - 1];
        const double s2 = g.bU * warp_sum(part2);
        for (int i = lane; i < m; i += 32) sV[sIdx[i]] = (i == 0 ? 0.0 : q[i - 1]) - s2 * sU[i];
    };

    // ---- cg_init (cg_init_kernel) + the first lift, warp 0
    if (warp == 0) {
        double cq = 0.0;
        for (int i = lane; i < m1; i += 32) cq += sQ[i] * sU[i + 1];
        cq = warp_sum(cq);
        if (lane == 0) sCq = cq;
        double prz = 0.0, pbb = 0.0;
        for (int i = lane; i < mm; i += 32) {
            const double r = sT[i];  // the right-hand side, staged above
            const double zz = s.jd ? r / sJ[i] : r;
            sX[i] = 0.0;
            sR[i] = r;
            sZ[i] = zz;
            sP[i] = zz;
            prz += r * zz;
            pbb += r * r;
        }
        const double rz = warp_sum(prz), bb = warp_sum(pbb);
        const bool act = s.cap > 0 && sqrt(bb) > s.tol * sqrt(bb);  // :94 at it = 0
        if (lane == 0) {
            sSc[0] = rz;
            sSc[1] = s.tol * sqrt(bb);
            sFlag[0] = act ? 1 : 0;
            sFlag[1] = 0;
            sFlag[2] = 0;
        }
        __syncwarp();
        if (act) lift();
    }
    __syncthreads();

    constexpr int GPW = 32 / LPR;         // row groups per warp
    constexpr int NGC = kCcgWarps * GPW;  // row groups per CTA
    // column pairs interleaved over the LPR lanes of a row group: pair
    // j2 * LPR + sub holds columns 2p, 2p + 1, so a row group reads contiguous bytes
    const int sub = lane % LPR;
    auto colp = [&](int j) { return 2 * ((j >> 1) * LPR + sub) + (j & 1); };
    int step = 0;
    unsigned long long prof_t = clock64();
    int prof_last = -1;
    const bool prof_on = a.prof && crank == 0 && col == 0 && tid == 0;
    unsigned long long psum[5] = {prof_t - t_entry, 0, 0, 0, 0};  // [0]: staging + cg_init + first lift
    if (prof_on) {  // prologue parts: loads issued / staging landed / cg_init + lift
        atomicAdd(a.prof + 8, t_loads - t_entry);
        atomicAdd(a.prof + 9, t_staged - t_loads);
        atomicAdd(a.prof + 10, prof_t - t_staged);
    }
    auto prof_mark = [&](int i) {  // phase sums in registers, written once at exit
        if (prof_on) {
            const unsigned long long now = clock64();
#pragma unroll
            for (int q = 1; q < 5; ++q)
                if (prof_last == q) psum[q] += now - prof_t;
            prof_t = now;
            prof_last = i;
        }
    };
    while (sFlag[0]) {
        prof_mark(1);
        // ---- HVP pass over this CTA's rows: acc[j] += x_tj psi''(z_t) <x_t, V>
        double acc[CPL], vv[CPL];
#pragma unroll
        for (int j = 0; j < CPL; j += 2) {  // this lane's slice of V, held for the whole pass
            const double2 v = *reinterpret_cast<const double2*>(sV + colp(j));
            vv[j] = v.x;
            vv[j + 1] = v.y;
            acc[j] = acc[j + 1] = 0.0;
        }
        // every lane of a warp runs the same trip count (the shuffles need the
        // full warp); rows past the block contribute zeros
#pragma unroll 2
        for (int lb = warp * GPW; lb < nloc; lb += NGC) {
            const int tl = lb + lane / LPR;
            const bool rv = tl < nloc;
            double x[CPL];
            double zt = 0.0;
            const double* xr = PANEL ? sXp + (size_t)(rv ? tl : 0) * lds : a.X + (r0 + (rv ? tl : 0)) * (long long)ld;
#pragma unroll
            for (int j = 0; j < CPL; j += 2) {
                double2 v = make_double2(0.0, 0.0);
                if (rv && colp(j) < ld)
                    v = PANEL ? *reinterpret_cast<const double2*>(xr + colp(j))
                              : __ldg(reinterpret_cast<const double2*>(xr + colp(j)));
                x[j] = v.x;
                x[j + 1] = v.y;
            }
            if (rv) zt = PANEL ? sZr[tl] : __ldg(a.z + r0 + tl);
            const double psi2 = 2.0 * a.c2 - 6.0 * a.c3 * zt + 12.0 * a.c4 * (zt * zt);
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int j = 0; j < CPL; j += 2) {
                d0 = fma(x[j], vv[j], d0);
                d1 = fma(x[j + 1], vv[j + 1], d1);
            }
            double d = d0 + d1;
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            const double w = psi2 * d;
#pragma unroll
            for (int j = 0; j < CPL; ++j) acc[j] = fma(x[j], w, acc[j]);
        }
        prof_mark(2);
        // combine the warp's row groups (lanes with equal sub), then the warps in order
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
            for (int j = 0; j < CPL; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
        if (lane < LPR) {
#pragma unroll
            for (int j = 0; j < CPL; ++j) sW[warp * M + colp(j)] = acc[j];
        }
        __syncthreads();
        double* buf = sPart + (step & 1) * M;
        for (int e = tid; e < ld; e += blockDim.x) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < kCcgWarps; ++w) v += sW[w * M + e];
            buf[e] = v;
        }
        prof_mark(3);
        // ---- cluster combine: every CTA sums the CS partials in rank order
        cluster.sync();
        for (int e = tid; e < ld; e += blockDim.x) {
            double pv[CS];
#pragma unroll
            for (int r = 0; r < CS; ++r) pv[r] = cluster.map_shared_rank(buf, r)[e];
            double v = 0.0;
#pragma unroll
            for (int r = 0; r < CS; ++r) v += pv[r];
            sH[e] = v * a.invT;
        }
        __syncthreads();
        ++step;
        prof_mark(4);
        // ---- one capped-CG step (cg_step_col) and the next lift, warp 0. The
        // Householder reduce (two dependent sums), p'Hp, and the next lift (two
        // more) are regrouped by linearity into two rounds of independent sums:
        //   round 1: A1 = U.H, A2 = Q.H(+1), B1 = P.H(+2), B2 = P.U(+2),
        //            B3 = P.Q(+1), B4 = P.P  ->  s1, s2, p'Hp
        //   round 2: r'z, r'r, D1 = Q(+1).z, E1 = U(+2).z  ->  beta, lift s1', s2'
        // with C = Q.U(+1) fixed per direction (same products, regrouped sums)
        if (warp == 0) {
            const double rz_old = sSc[0];
            constexpr int U4 = M / 32;
            double a1 = 0.0, a2 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0, b4 = 0.0;
            double hh[U4];  // H'(j + 2) for j = lane + 32u
#pragma unroll
            for (int u = 0; u < U4; ++u) {
                const int i = lane + 32 * u;
                hh[u] = 0.0;
                if (i < m) {
                    const double h = sH[sIdx[i]];
                    a1 += sU[i] * h;
                    if (i >= 1) a2 += sQ[i - 1] * h;
                }
                if (i < mm) {
                    const double h2 = sH[sIdx[i + 2]];
                    const double p = sP[i];
                    hh[u] = h2;
                    b1 += p * h2;
                    b2 += p * sU[i + 2];
                    b3 += p * sQ[i + 1];
                    b4 += p * p;
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                a2 += __shfl_xor_sync(0xffffffffu, a2, o);
                b1 += __shfl_xor_sync(0xffffffffu, b1, o);
                b2 += __shfl_xor_sync(0xffffffffu, b2, o);
                b3 += __shfl_xor_sync(0xffffffffu, b3, o);
                b4 += __shfl_xor_sync(0xffffffffu, b4, o);
            }
            // (an xor butterfly leaves the same bits in every lane: each level adds
            // the same two operands, commuted)
            const double s1 = g.bU * a1;
            const double s2 = g.bQ * (a2 - s1 * sCq);
            const double pHp = b1 - s1 * b2 - s2 * b3 + lambda * b4;  // p'(red + lambda p) (:194)
            if (pHp <= 0.0) {  // :97-100
                if (lane == 0) {
                    sFlag[2] = 1;
                    sFlag[0] = 0;
                }
            } else {
                const double alpha = rz_old / pHp;
                double prz = 0.0, prr = 0.0, d1 = 0.0, e1 = 0.0;
                double zr[U4];
#pragma unroll
                for (int u = 0; u < U4; ++u) {
                    const int i = lane + 32 * u;
                    zr[u] = 0.0;
                    if (i < mm) {
                        const double hp = ((hh[u] - s1 * sU[i + 2]) - s2 * sQ[i + 1]) + lambda * sP[i];
                        sX[i] += alpha * sP[i];
                        const double r = sR[i] - alpha * hp;
                        sR[i] = r;
                        const double zz = s.jd ? r / sJ[i] : r;
                        sZ[i] = zz;
                        zr[u] = zz;
                        prz += r * zz;
                        prr += r * r;
                        d1 += sQ[i + 1] * zz;
                        e1 += sU[i + 2] * zz;
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    prz += __shfl_xor_sync(0xffffffffu, prz, o);
                    prr += __shfl_xor_sync(0xffffffffu, prr, o);
                    d1 += __shfl_xor_sync(0xffffffffu, d1, o);
                    e1 += __shfl_xor_sync(0xffffffffu, e1, o);
                }
                const double rz2 = prz, rr = prr;
                const double beta = rz2 / rz_old;
#pragma unroll
                for (int u = 0; u < U4; ++u) {
                    const int i = lane + 32 * u;
                    if (i < mm) sP[i] = zr[u] + beta * sP[i];
                }
                const int it = sFlag[1] + 1;
                const bool still = it < s.cap && sqrt(rr) > sSc[1];  // :94
                __syncwarp();
                if (lane == 0) {
                    sSc[0] = rz2;
                    sFlag[1] = it;
                    sFlag[0] = still ? 1 : 0;
                }
                if (still) {  // lift of the new p: V = U Q (0, p) (lift_col)
                    const double l1 = g.bQ * (d1 + beta * b3);
                    const double l2 = g.bU * ((e1 + beta * b2) - l1 * sCq);
                    for (int i = lane; i < m; i += 32) {
                        const double qv = i == 0 ? 0.0 : ((i >= 2 ? sP[i - 2] : 0.0) - l1 * sQ[i - 1]);
                        sV[sIdx[i]] = qv - l2 * sU[i];
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
    prof_mark(5);
    if (prof_on) {
#pragma unroll
        for (int q = 0; q < 5; ++q) a.prof[q] += psum[q];
        a.prof[6] += (unsigned long long)step;
        a.prof[7] += 1;
    }
    // ---- results to the global CG state (CTA 0 of the cluster)
    if (crank == 0) {
        for (int i = tid; i < mm; i += blockDim.x) {
            s.X[(size_t)col * mm + i] = sX[i];
            s.R[(size_t)col * mm + i] = sR[i];
            s.Z[(size_t)col * mm + i] = sZ[i];
            s.P[(size_t)col * mm + i] = sP[i];
        }
        if (tid == 0) {
            s.rz[col] = sSc[0];
            s.target[col] = sSc[1];
            s.active[col] = sFlag[0];
            s.iters[col] = sFlag[1];
            s.breakdown[col] = sFlag[2];
        }
    }
    cluster.sync();  // no CTA exits while a peer may still read its partials
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
    int* host_flags = nullptr;  // pinned [4 * kPcgMaxCols] (host-driven loop flags)
    int* host_counts = nullptr; // pinned [kMaxDeferred][2][K] iters / breakdown snapshots
    double* host_u = nullptr;   // pinned solution readback
    unsigned char* host_up = nullptr;  // pinned upload staging (parameters, geometry, probes)
    size_t host_up_bytes = 0;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t aux = nullptr;  // captures conditional-loop bodies while the direction is captured
    // device-resident Krylov loops of the eager path: a conditional-while graph per (k, slot)
    struct LoopGraph {
        int k, slot, role;
        uint64_t epoch;
        cudaGraphExec_t exec;
        uint64_t phys_per_step, launches_per_step;
    };
    std::vector<LoopGraph> graphs;
    std::vector<std::pair<int, int>> seen;  // (k, slot * 2 + role) keys that ran once at seen_epoch
    uint64_t seen_epoch = ~0ull;
    bool graphs_broken = false;
    // whole-direction graphs (Hutchinson / no-third directions), keyed by shape
    struct DirKey {
        int slot, mm, kp, kj, third;
        uint64_t epoch;
        bool operator==(const DirKey& o) const {
            return slot == o.slot && mm == o.mm && kp == o.kp && kj == o.kj && third == o.third && epoch == o.epoch;
        }
    };
    struct DirGraph {
        DirKey key;
        cudaGraphExec_t exec;
        uint64_t fwd, tr, phys, launches;  // counts of the non-loop part, per replay
        int nloops;
        int loop_k[2];
        uint64_t loop_pps[2], loop_lps[2];
    };
    std::vector<DirGraph> dgraphs;
    std::vector<DirKey> dseen;
    bool dir_broken = false;
};

void pcg_workspace_free(mvsk_gpu_ctx* ctx) {
    if (!ctx->pcg) return;
    PcgWorkspace& ws = *ctx->pcg;
    for (auto& lg : ws.graphs)
        if (lg.exec) cudaGraphExecDestroy(lg.exec);
    for (auto& dg : ws.dgraphs)
        if (dg.exec) cudaGraphExecDestroy(dg.exec);
    if (ws.host_counts) cudaFreeHost(ws.host_counts);
    if (ws.host_u) cudaFreeHost(ws.host_u);
    if (ws.host_up) cudaFreeHost(ws.host_up);
    if (ws.dev) cudaFree(ws.dev);
    if (ws.host_flags) cudaFreeHost(ws.host_flags);
    for (cudaEvent_t e : ws.ev)
        if (e) cudaEventDestroy(e);
    if (ws.aux) cudaStreamDestroy(ws.aux);
    delete ctx->pcg;
    ctx->pcg = nullptr;
}

namespace {
// parameters of one direction (device memory, uploaded from pinned staging)
struct DirDev {
    Geo g;
    StepParams sp[2];  // [0] probe block (cap = probe_cap), [1] main CG (cap = maxit)
    DirScalars ds;
};
}  // namespace

PcgOutput pcg_direction_device(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const PcgInput& in) {
    const int m = (int)in.m, m1 = m - 1, mm = m - 2;
    const int K = kPcgMaxCols;
    const size_t ld = (size_t)ctx->ld;
    const long long N = ctx->n;
    if (!ctx->pcg) ctx->pcg = new PcgWorkspace();
    PcgWorkspace& ws = *ctx->pcg;
    // ---- device workspace, carved for the full n so its pointers do not move
    // with the face size (they are baked into the instantiated graphs)
    unsigned char* base = nullptr;
    size_t off = 0;
    auto carve_d = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    const size_t o_dir = carve_d(sizeof(DirDev));
    const size_t o_vU = carve_d(N * 8), o_vQ = carve_d(N * 8), o_nu = carve_d(N * 8), o_idx = carve_d(N * 8);
    const size_t o_jsrc = carve_d((size_t)K * N * 8), o_psrc = carve_d((size_t)K * N * 8);
    const size_t up_bytes = off;  // the uploaded prefix: parameters, geometry, probes
    const size_t o_X = carve_d((size_t)K * N * 8), o_R = carve_d((size_t)K * N * 8), o_Z = carve_d((size_t)K * N * 8);
    const size_t o_P = carve_d((size_t)K * N * 8), o_src = carve_d((size_t)K * N * 8), o_rows = carve_d((size_t)K * N * 8);
    const size_t o_jd = carve_d(N * 8), o_h = carve_d(N * 8), o_a = carve_d(N * 8);
    const size_t o_rz = carve_d(K * 8), o_tg = carve_d(K * 8);
    const size_t o_act = carve_d(K * 4), o_it = carve_d(K * 4), o_bd = carve_d(K * 4), o_arr = carve_d(64);
    if (ws.bytes < off) {
        if (ws.dev) MVSK_CUDA(cudaFree(ws.dev));
        ws.dev = nullptr;
        MVSK_CUDA(cudaMalloc(&ws.dev, off));
        ws.bytes = off;
        ++ctx->epoch;
    }
    if (ws.host_up_bytes < up_bytes) {
        if (ws.host_up) MVSK_CUDA(cudaFreeHost(ws.host_up));
        ws.host_up = nullptr;
        ws.host_up_bytes = 0;
        MVSK_CUDA(cudaMallocHost(&ws.host_up, up_bytes));
        ws.host_up_bytes = up_bytes;
        ++ctx->epoch;
        if (ws.host_u) MVSK_CUDA(cudaFreeHost(ws.host_u));
        MVSK_CUDA(cudaMallocHost(&ws.host_u, (size_t)std::max<long long>(N, 1) * sizeof(double)));
    }
    if (!ws.host_flags) MVSK_CUDA(cudaMallocHost(&ws.host_flags, sizeof(int) * 4 * K));
    if (!ws.host_counts) MVSK_CUDA(cudaMallocHost(&ws.host_counts, sizeof(int) * kMaxDeferred * 2 * K));
    for (cudaEvent_t& e : ws.ev)
        if (!e) MVSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!ws.aux) MVSK_CUDA(cudaStreamCreateWithFlags(&ws.aux, cudaStreamNonBlocking));
    base = ws.dev;
    auto D = [&](size_t o) { return reinterpret_cast<double*>(base + o); };
    DirDev* dir = reinterpret_cast<DirDev*>(base + o_dir);
    double *vU = D(o_vU), *vQ = D(o_vQ), *nu = D(o_nu), *jsrc = D(o_jsrc), *psrc = D(o_psrc);
    long long* idx = reinterpret_cast<long long*>(base + o_idx);
    double *X = D(o_X), *Rm = D(o_R), *Z = D(o_Z), *P = D(o_P), *src = D(o_src), *rows = D(o_rows);
    double *jd = D(o_jd), *hvec = D(o_h), *avec = D(o_a), *rz = D(o_rz), *target = D(o_tg);
    int* active = reinterpret_cast<int*>(base + o_act);
    int* iters = reinterpret_cast<int*>(base + o_it);
    int* bdown = reinterpret_cast<int*>(base + o_bd);
    unsigned* arrive = reinterpret_cast<unsigned*>(base + o_arr);
    cudaStream_t st = ctx->stream;

    // ---- host staging of everything this direction uploads (same layout as the
    // device prefix [0, up_bytes)); one contiguous pinned buffer
    const bool jac = !in.jacobi_probes.empty();
    const int kj = jac ? (int)in.jacobi_probes.size() : 0;
    const int kp = in.has_third && !in.unit_probes ? (int)in.probes.size() : 0;
    unsigned char* hu = ws.host_up;
    auto HU = [&](size_t o) { return reinterpret_cast<double*>(hu + o); };
    {
        DirDev hd{};
        hd.g = Geo{vU, in.bU, vQ, in.bQ, fm.active ? idx : nullptr, m, (int)ld};
        const double* jdp = jac ? jd : nullptr;
        hd.sp[0] = StepParams{hd.g, CGState{X, Rm, Z, P, rz, target, active, iters, bdown, jdp, mm, in.probe_cap, in.tol},
                              in.lambda};
        hd.sp[1] = StepParams{hd.g, CGState{X, Rm, Z, P, rz, target, active, iters, bdown, jdp, mm, in.maxit, in.tol},
                              in.lambda};
        hd.ds = DirScalars{mm, in.lambda, std::max(1e-12, in.lambda),
                           (in.has_third && !in.unit_probes) ? (double)in.hutchinson_probes : 0.0, in.gn / (double)m};
        std::memcpy(hu + o_dir, &hd, sizeof(hd));
        std::copy(in.vU.begin(), in.vU.end(), HU(o_vU));
        std::copy(in.vQ.begin(), in.vQ.end(), HU(o_vQ));
        std::copy(in.nu.begin(), in.nu.end(), HU(o_nu));
        if (fm.active) std::memcpy(hu + o_idx, fm.idx.data(), (size_t)m * sizeof(long long));
        for (int p = 0; p < kj; ++p) std::copy(in.jacobi_probes[p].begin(), in.jacobi_probes[p].end(), HU(o_jsrc) + (size_t)p * mm);
        for (int p = 0; p < kp && p < K; ++p) std::copy(in.probes[p].begin(), in.probes[p].end(), HU(o_psrc) + (size_t)p * mm);
    }
    const size_t dsm_max = (size_t)2 * std::max<long long>(N, 1) * sizeof(double);
    // threads per column CTA from the context width (stable per context, so the
    // captured graphs stay valid): narrow faces run their block reductions on
    // two warps instead of sixteen
    const int pt = N <= 128 ? 64 : N <= 512 ? 128 : N <= 2048 ? 256 : kPT;
    for (const void* fn : {(const void*)lift_kernel, (const void*)lift_pair_kernel, (const void*)cg_step_kernel,
                           (const void*)reduce_kernel, (const void*)cg_init_kernel})
        set_smem_attr(fn, dsm_max);
    const int nb1 = (int)std::min<long long>(4LL * ctx->nsm, (N + 255) / 256 + 1);
    const Slot& sl = ctx->slots[slot];
    double* vin = ctx->vin;
    double* vin2 = ctx->vin + (size_t)MVSK_GPU_MAX_RHS * ld;
    double* H = ctx->outd;
    const Geo* gdev = &dir->g;
    const DirScalars* dsd = &dir->ds;

    PcgOutput out;
    // per-loop bookkeeping, settled after the direction's final sync
    struct Deferred {
        int k;
        int row;            // pinned row of [iters | breakdown] snapshots
        uint64_t pps, lps;  // passes / launches per step (graph loops); 0: counted live
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
            const int* hc = ws.host_counts + (size_t)d.row * 2 * K;
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

    // capture of a loop body on the aux stream (the direction itself may be
    // capturing on st); the passes inside go to the aux stream too
    auto capture_body = [&](cudaGraph_t body, int k, const StepParams* spd, cudaGraphConditionalHandle h) -> bool {
        if (cudaStreamBeginCaptureToGraph(ws.aux, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
            cudaSuccess)
            return false;
        bool threw = false;
        cudaStream_t saved = ctx->stream;
        ctx->stream = ws.aux;
        try {
            PassIO io;
            io.vin = vin;
            io.z = sl.z;
            io.out = H;
            io.ldo = (long long)ld;
            run_pass(ctx, Op::HVP, k, io);
            ++ctx->launches;
            cg_step_kernel<<<k, pt, dsm_max, ws.aux>>>(spd, H, vin, arrive, h, 1);
        } catch (...) {
            threw = true;
        }
        ctx->stream = saved;
        cudaGraph_t captured = nullptr;
        return cudaStreamEndCapture(ws.aux, &captured) == cudaSuccess && !threw;
    };
    // adds [decide] -> [while {pass, cg_step}] to graph gr after deps
    auto add_loop = [&](cudaGraph_t gr, const cudaGraphNode_t* deps, size_t ndeps, int k, const StepParams* spd,
                        cudaGraphNode_t* wn_out) -> bool {
        cudaGraphConditionalHandle h{};
        if (cudaGraphConditionalHandleCreate(&h, gr, 0, 0) != cudaSuccess) return false;
        int kk = k;
        int* act = active;
        void* args[] = {&act, &kk, &h};
        cudaKernelNodeParams kp{};
        kp.func = reinterpret_cast<void*>(&cg_decide_kernel);
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(32);
        kp.kernelParams = args;
        cudaGraphNode_t n0 = nullptr;
        if (cudaGraphAddKernelNode(&n0, gr, deps, ndeps, &kp) != cudaSuccess) return false;
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        if (cudaGraphAddNode(wn_out, gr, &n0, 1, &cp) != cudaSuccess) return false;
        return capture_body(cp.conditional.phGraph_out[0], k, spd, h);
    };

    // ---- the eager path's loop: a per-(k, slot) loop graph, or host-driven
    static const bool no_graph = std::getenv("MVSK_NO_CG_GRAPH") != nullptr;
    auto cg_graph = [&](int k, int role, const StepParams* spd) -> PcgWorkspace::LoopGraph* {
        if (no_graph || ctx->no_capture || ws.graphs_broken) return nullptr;
        if (ws.seen_epoch != ctx->epoch) {  // buffers may have been resized: size them eagerly again
            ws.seen.clear();
            ws.seen_epoch = ctx->epoch;
        }
        if (std::find(ws.seen.begin(), ws.seen.end(), std::make_pair(k, slot * 2 + role)) == ws.seen.end()) {
            ws.seen.emplace_back(k, slot * 2 + role);
            return nullptr;
        }
        for (auto& lg : ws.graphs)
            if (lg.k == k && lg.slot == slot && lg.role == role) {
                if (lg.epoch == ctx->epoch && lg.exec) return &lg;
                if (lg.exec) cudaGraphExecDestroy(lg.exec);
                lg.exec = nullptr;
            }
        cudaGraph_t gr = nullptr;
        cudaGraphExec_t exec = nullptr;
        const uint64_t p0 = ctx->phys, l0 = ctx->launches;
        cudaGraphNode_t wn = nullptr;
        bool ok = cudaGraphCreate(&gr, 0) == cudaSuccess && add_loop(gr, nullptr, 0, k, spd, &wn);
        if (ok) ok = cudaGraphInstantiate(&exec, gr, 0) == cudaSuccess;
        const uint64_t dp = ctx->phys - p0, dl = ctx->launches - l0;
        ctx->phys = p0;
        ctx->launches = l0;
        if (gr) cudaGraphDestroy(gr);
        cudaGetLastError();
        if (!ok) {
            if (exec) cudaGraphExecDestroy(exec);
            ws.graphs_broken = true;  // e.g. a launch kind a conditional body rejects: host loop
            return nullptr;
        }
        ws.graphs.push_back({k, slot, role, ctx->epoch, exec, dp, dl});
        return &ws.graphs.back();
    };

    // ---- the direction as a sequence of enqueues on st. `capture` != nullptr:
    // st is capturing the whole direction; each Krylov loop is spliced in as a
    // conditional-while node (its counts recorded in *capture)
    PcgWorkspace::DirGraph* capture = nullptr;
    // narrow panels: the whole Krylov loop in one thread-block cluster
    // (cluster_cg_kernel); MVSK_NO_CCG keeps the graph / host loops for A/B
    static const bool no_ccg = std::getenv("MVSK_NO_CCG") != nullptr;
    const bool ccg_ok = !no_ccg && ctx->nranks == 1 && ld <= (size_t)kCcgMaxLd && m <= (int)ld;
    auto ccg_launch = [&](int k, const StepParams* spd, const double* rhs) -> bool {
        if (!ccg_ok || k > 8) return false;
        // one 16-CTA cluster per column (k clusters side by side); each CTA keeps
        // its rows in shared memory
        const int CS = kCcgCS;
        const long long nloc = (ctx->T_local + CS - 1) / CS;
        const size_t panel = (size_t)nloc * (ld + 3) * sizeof(double);  // padded rows + z
        // only when each CTA's row block fits its shared memory: a taller narrow
        // panel streamed by 16 SMs per step would lose to the 148-CTA pass
        size_t smem = ccg_smem_bytes();
        if (smem + panel > ctx->max_smem) return false;
        smem += panel;
        const void* fn =
            ld <= 64 ? (const void*)&cluster_cg_kernel<4, 16, true> : (const void*)&cluster_cg_kernel<8, 16, true>;
        if (!cluster_fits(fn, CS, kCcgWarps * 32, smem)) return false;
        MVSK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CcgArgs ca{};
        ca.sp = spd;
        ca.rhs = rhs;
        ca.X = ctx->X;
        ca.z = sl.z;
        ca.T = ctx->T_local;
        ca.ld = (int)ld;
        ca.k = k;
        ca.c2 = ctx->c.c2;
        ca.c3 = ctx->c.c3;
        ca.c4 = ctx->c.c4;
        ca.invT = 1.0 / (double)ctx->T_global;
        static unsigned long long* prof = nullptr;  // MVSK_CCG_PROF: per-phase cycle sums, printed at exit
        if (std::getenv("MVSK_CCG_PROF")) {
            if (!prof) {
                MVSK_CUDA(cudaMallocManaged(&prof, 16 * sizeof(unsigned long long)));
                std::memset(prof, 0, 16 * sizeof(unsigned long long));
                std::atexit([] {
                    cudaDeviceSynchronize();
                    std::fprintf(stderr,
                                 "[ccg prof] launches %llu steps %llu | prologue %llu pass %llu combine %llu cluster %llu "
                                 "cg+lift %llu (cycles); prologue = loads %llu + staging wait %llu + init %llu\n",
                                 prof[7], prof[6], prof[0], prof[1], prof[2], prof[3], prof[4], prof[8], prof[9],
                                 prof[10]);
                });
            }
            ca.prof = prof;
        }
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(CS * k);
        cfg.blockDim = dim3(kCcgWarps * 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        void* args[] = {&ca};
        MVSK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
        return true;
    };
    auto cg = [&](int k, int role, const double* rhs) {
        const StepParams* spd = &dir->sp[role];
        if (ccg_launch(k, spd, rhs)) {
            // one launch and one physical pass per step, counted when the
            // iteration counts come back (settle_counts)
            if (capture) {
                const int li = capture->nloops++;
                capture->loop_k[li] = k;
                capture->loop_pps[li] = 1;
                capture->loop_lps[li] = 0;
            }
            defer_counts(k, true, 1, 0);
            return;
        }
        MVSK_CUDA(cudaMemsetAsync(arrive, 0, sizeof(unsigned), st));
        ++ctx->launches;
        cg_init_kernel<<<k, pt, dsm_max, st>>>(spd, rhs, vin);
        MVSK_CUDA(cudaGetLastError());
        if (capture) {
            cudaStreamCaptureStatus cs;
            cudaGraph_t gr = nullptr;
            const cudaGraphNode_t* deps = nullptr;
            size_t ndeps = 0;
            MVSK_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &gr, &deps, &ndeps));
            std::vector<cudaGraphNode_t> dv(deps, deps + ndeps);
            const uint64_t p0 = ctx->phys, l0 = ctx->launches;
            cudaGraphNode_t wn = nullptr;
            if (!add_loop(gr, dv.data(), dv.size(), k, spd, &wn))
                throw ApiError(MVSK_CUDA_ERROR, "pcg: conditional loop capture failed");
            MVSK_CUDA(cudaStreamUpdateCaptureDependencies(st, &wn, 1, cudaStreamSetCaptureDependencies));
            const int li = capture->nloops++;
            capture->loop_k[li] = k;
            capture->loop_pps[li] = ctx->phys - p0;
            capture->loop_lps[li] = ctx->launches - l0;
            ctx->phys = p0;
            ctx->launches = l0;
            defer_counts(k, true, capture->loop_pps[li], capture->loop_lps[li]);
            return;
        }
        if (PcgWorkspace::LoopGraph* lg = cg_graph(k, role, spd)) {
            MVSK_CUDA(cudaGraphLaunch(lg->exec, st));
            defer_counts(k, true, lg->phys_per_step, lg->launches_per_step);
            return;
        }
        int* hf = ws.host_flags;  // [2][K] flag snapshots
        MVSK_CUDA(cudaMemcpyAsync(hf, active, k * sizeof(int), cudaMemcpyDeviceToHost, st));
        MVSK_CUDA(cudaEventRecord(ws.ev[0], st));
        const int cap = role == 0 ? in.probe_cap : in.maxit;
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
            cg_step_kernel<<<k, pt, dsm_max, st>>>(spd, H, vin, arrive, cudaGraphConditionalHandle{}, 0);
            MVSK_CUDA(cudaGetLastError());
            const int nb = (step + 1) & 1;
            MVSK_CUDA(cudaMemcpyAsync(hf + nb * K, active, k * sizeof(int), cudaMemcpyDeviceToHost, st));
            MVSK_CUDA(cudaEventRecord(ws.ev[nb], st));
            MVSK_CUDA(cudaEventSynchronize(ws.ev[step & 1]));  // flags that gated this step
            int nact = 0;
            for (int c = 0; c < k; ++c) nact += hf[(step & 1) * K + c];
            if (!nact) {
                ctx->phys -= 1;  // the step ran as a no-op
                break;
            }
        }
        defer_counts(k, false, 0, 0);
    };
    auto hvp_rows = [&](int k) {
        PassIO io;
        io.vin = vin;
        io.z = sl.z;
        io.out = H;
        io.ldo = (long long)ld;
        run_pass(ctx, Op::HVP, k, io);
        ctx->fwd += k;  // reference contract: 2 passes per HVP
        ctx->tr += k;
    };
    auto enqueue = [&]() {
        // uploads: parameters, geometry, probes (exact sizes: the graph key has mm)
        if ((size_t)(N - m) * 3 * sizeof(double) <= 16384) {
            // parameters + U / Q reflectors + nu (+ face map) as ONE copy of the
            // staged prefix: the slack between the regions is small here
            const size_t end = fm.active ? o_idx + (size_t)m * sizeof(long long) : o_nu + (size_t)m1 * sizeof(double);
            MVSK_CUDA(cudaMemcpyAsync(base + o_dir, hu + o_dir, end - o_dir, cudaMemcpyHostToDevice, st));
        } else {
            MVSK_CUDA(cudaMemcpyAsync(base + o_dir, hu + o_dir, sizeof(DirDev), cudaMemcpyHostToDevice, st));
            MVSK_CUDA(cudaMemcpyAsync(vU, HU(o_vU), m * sizeof(double), cudaMemcpyHostToDevice, st));
            MVSK_CUDA(cudaMemcpyAsync(vQ, HU(o_vQ), m1 * sizeof(double), cudaMemcpyHostToDevice, st));
            MVSK_CUDA(cudaMemcpyAsync(nu, HU(o_nu), m1 * sizeof(double), cudaMemcpyHostToDevice, st));
            if (fm.active)
                MVSK_CUDA(cudaMemcpyAsync(idx, hu + o_idx, m * sizeof(long long), cudaMemcpyHostToDevice, st));
        }
        // ---- Jacobi diagonal (:197-209): 8 probes through Hop in one batch
        if (jac) {
            MVSK_CUDA(cudaMemcpyAsync(jsrc, HU(o_jsrc), (size_t)kj * mm * sizeof(double), cudaMemcpyHostToDevice, st));
            ++ctx->launches;
            lift_kernel<<<kj, pt, dsm_max, st>>>(gdev, jsrc, true, nullptr, vin);
            hvp_rows(kj);
            ++ctx->launches;
            reduce_kernel<<<kj, pt, dsm_max, st>>>(gdev, H, true, rows);
            ++ctx->launches;
            jacobi_diag_kernel<<<nb1, 256, 0, st>>>(dsd, jsrc, rows, kj, jd);
            MVSK_CUDA(cudaGetLastError());
        }
        // ---- h = Q^T U^T grad2 f (U nu)  (:212-213)
        ++ctx->launches;
        lift_kernel<<<1, pt, dsm_max, st>>>(gdev, nu, false, nullptr, vin);
        hvp_rows(1);
        ++ctx->launches;
        reduce_kernel<<<1, pt, dsm_max, st>>>(gdev, H, true, hvec);
        MVSK_CUDA(cudaGetLastError());
        // ---- a: Hutchinson probes or exact trace (:215-237), blocks of K
        // columns, accumulated on the device in probe order
        MVSK_CUDA(cudaMemsetAsync(avec, 0, mm * sizeof(double), st));
        bool rhs_done = false;
        if (in.has_third) {
            const int P_all = in.unit_probes ? mm : (int)in.probes.size();
            for (int b0 = 0; b0 < P_all; b0 += K) {
                const int k = std::min(K, P_all - b0);
                double* pb = src;
                if (in.unit_probes) {
                    ++ctx->launches;
                    unit_probe_kernel<<<nb1, 256, 0, st>>>(dsd, src, k, b0);
                } else if (b0 == 0) {
                    pb = psrc;
                    MVSK_CUDA(cudaMemcpyAsync(psrc, HU(o_psrc), (size_t)k * mm * sizeof(double), cudaMemcpyHostToDevice,
                                              st));
                } else {  // more than K Hutchinson probes: later blocks from pageable host memory
                    std::vector<double> buf((size_t)k * mm);
                    for (int p = 0; p < k; ++p)
                        std::copy(in.probes[b0 + p].begin(), in.probes[b0 + p].end(), buf.begin() + (size_t)p * mm);
                    MVSK_CUDA(cudaMemcpy(src, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice));
                }
                cg(k, 0, pb);
                // third_action(U Q s_p, U Q r_p) for the block, one fused pass
                ++ctx->launches;
                lift_pair_kernel<<<2 * k, pt, dsm_max, st>>>(gdev, X, pb, k, vin, vin2);
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
                reduce_kernel<<<k, pt, dsm_max, st>>>(gdev, H, true, rows);
                ++ctx->launches;
                if (b0 + K >= P_all) {  // last block: the rhs in the same kernel
                    accum_rhs_kernel<<<nb1, 256, 0, st>>>(dsd, rows, k, avec, hvec, src);
                    rhs_done = true;
                } else {
                    accum_rows_kernel<<<nb1, 256, 0, st>>>(dsd, rows, k, avec);
                }
                MVSK_CUDA(cudaGetLastError());
                if (!capture && in.unit_probes && deferred.size() + 2 >= (size_t)kMaxDeferred) {
                    // long exact-trace sweeps: settle the loop counts every few blocks
                    MVSK_CUDA(cudaStreamSynchronize(st));
                    settle_counts();
                }
            }
        }
        // rhs = h - (||gbar|| / n) a  (:239); a averaged over the Hutchinson probes (:236)
        if (!rhs_done) {
            ++ctx->launches;
            rhs_kernel<<<nb1, 256, 0, st>>>(dsd, hvec, avec, src);
            MVSK_CUDA(cudaGetLastError());
        }
        // main CG (:240-241)
        cg(1, 1, src);
        MVSK_CUDA(cudaMemcpyAsync(ws.host_u, X, mm * sizeof(double), cudaMemcpyDeviceToHost, st));
    };

    // ---- whole-direction graph: Hutchinson (<= K probes) or no-third directions.
    // The first direction of a shape runs eagerly (it sizes every workspace), the
    // second is captured, later ones replay it.
    static const bool no_dir_graph = std::getenv("MVSK_NO_DIR_GRAPH") != nullptr;
    const bool graphable = !no_dir_graph && !ctx->no_capture && !ws.dir_broken && !in.unit_probes && kp <= K && !no_graph &&
                           !ws.graphs_broken;
    const PcgWorkspace::DirKey key{slot, mm, kp, kj, in.has_third ? 1 : 0, ctx->epoch};
    PcgWorkspace::DirGraph* dg = nullptr;
    if (graphable) {
        for (auto& d : ws.dgraphs)
            if (d.key == key) dg = &d;
        if (!dg && std::find(ws.dseen.begin(), ws.dseen.end(), key) != ws.dseen.end()) {
            // capture it now
            PcgWorkspace::DirGraph ng{};
            ng.key = key;
            const uint64_t f0 = ctx->fwd, t0 = ctx->tr, p0 = ctx->phys, l0 = ctx->launches;
            cudaGraph_t gr = nullptr;
            bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                capture = &ng;
                try {
                    enqueue();
                } catch (...) {
                    ok = false;
                }
                capture = nullptr;
                ok = cudaStreamEndCapture(st, &gr) == cudaSuccess && ok;
            }
            cudaGraphExec_t exec = nullptr;
            if (ok) ok = cudaGraphInstantiate(&exec, gr, 0) == cudaSuccess;
            if (gr) cudaGraphDestroy(gr);
            cudaGetLastError();
            ng.fwd = ctx->fwd - f0;
            ng.tr = ctx->tr - t0;
            ng.phys = ctx->phys - p0;
            ng.launches = ctx->launches - l0;
            ctx->fwd = f0;
            ctx->tr = t0;
            ctx->phys = p0;
            ctx->launches = l0;
            deferred.clear();
            if (ok) {
                ng.exec = exec;
                if (ws.dgraphs.size() >= 8) {  // small cache of direction shapes
                    if (ws.dgraphs.front().exec) cudaGraphExecDestroy(ws.dgraphs.front().exec);
                    ws.dgraphs.erase(ws.dgraphs.begin());
                }
                ws.dgraphs.push_back(ng);
                dg = &ws.dgraphs.back();
            } else {
                if (exec) cudaGraphExecDestroy(exec);
                ws.dir_broken = true;
            }
        }
    }
    if (dg) {
        MVSK_CUDA(cudaGraphLaunch(dg->exec, st));
        ctx->fwd += dg->fwd;
        ctx->tr += dg->tr;
        ctx->phys += dg->phys;
        ctx->launches += 1 + dg->launches;
        int row = 0;
        for (int li = 0; li < dg->nloops; ++li)
            deferred.push_back({dg->loop_k[li], row++, dg->loop_pps[li], dg->loop_lps[li], true});
    } else {
        if (graphable && std::find(ws.dseen.begin(), ws.dseen.end(), key) == ws.dseen.end()) {
            if (ws.dseen.size() >= 32) ws.dseen.erase(ws.dseen.begin());
            ws.dseen.push_back(key);
        }
        enqueue();
    }
    MVSK_CUDA(cudaStreamSynchronize(st));
    settle_counts();
    out.u.assign(ws.host_u, ws.host_u + mm);
    return out;
}

}  // namespace mvsk_b200
