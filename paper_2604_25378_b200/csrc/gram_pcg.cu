// PCG direction through the reduced Hessian (affine_normal.hpp:189-242) for
// narrow faces.
//
// Every Krylov step of the PCG branch applies the tangent operator
//   Hop(e) = Q^T U^T grad2f (U Q e) + lambda e,   grad2f = A_f^T diag(psi'') A_f / T,
// which the reference evaluates matrix-free (oracle.hvp: two passes over the
// T x m face panel per step, ~56 steps per direction). For a face of m <= 112
// assets that operator is a small dense matrix: with the weighted Gram
// G = A_f^T diag(psi''(z)) A_f / T (one DMMA pass, gram_kernels.cu),
//   M = (U Q)^T G (U Q) = [H_Q [H_U G H_U]_11 H_Q]_11   ((m-2) x (m-2)),
// and every Hop is Me + lambda e — the same linear map, evaluated in a
// different summation order. A direction then costs one Gram pass, one CTA
// running every capped CG (cg_capped, :85-113: the Hutchinson probes in
// lock-step, one warp per column for the per-column algebra, the 8-column
// M P product by the whole CTA), the one 8-pair third-action pass the
// probes need (:233-235), and one CTA for a, the rhs and the main CG — four
// kernels in one graph, one readback. The matrix-free path remains for wider
// faces, exact traces and > 8 probes (pcg_device.cu).
//
// The logical pass counters follow the reference's contract (2 per Hop,
// 3 per third action; common.hpp:27-37), from the per-column HVP counts.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "host_ops.hpp"
#include "pcg_device.hpp"

namespace mvsk_b200 {

void run_graphed(mvsk_gpu_ctx* ctx, int op, int k, int slot, const std::function<void()>& enqueue);
void ensure_tvec2(mvsk_gpu_ctx* ctx);

namespace {

constexpr int kGpMaxM = 112;     // face width limit (two m x m fp64 buffers in shared memory)
constexpr int kGpMaxCols = 8;    // Hutchinson probes handled in one lock-step block
constexpr int kGpThreads = 512;
constexpr int kDirectDeviceMinLd = 64;  // narrower panels take the host LU / Cholesky direct branch
constexpr int kDirectDeviceMaxLd = 512;
constexpr int kGraphGramPcg = 102;
constexpr int kGraphGramDirect = 103;

// per-direction scalars; they live in the device parameter buffer (doubles
// [0, 16)) so one captured graph serves every direction of a face shape
struct GpParams {
    int m, mm, np, probe_cap, maxit, jacobi, has_third, face_active;
    double bU, bQ, gn, lambda, tol, n_d;
    __host__ __device__ void store(double* d) const {
        const double v[14] = {(double)m, (double)mm, (double)np, (double)probe_cap, (double)maxit, (double)jacobi,
                              (double)has_third, (double)face_active, bU, bQ, gn, lambda, tol, n_d};
        for (int i = 0; i < 14; ++i) d[i] = v[i];
    }
    __host__ __device__ static GpParams load(const double* d) {
        GpParams p;
        p.m = (int)d[0];
        p.mm = (int)d[1];
        p.np = (int)d[2];
        p.probe_cap = (int)d[3];
        p.maxit = (int)d[4];
        p.jacobi = (int)d[5];
        p.has_third = (int)d[6];
        p.face_active = (int)d[7];
        p.bU = d[8];
        p.bQ = d[9];
        p.gn = d[10];
        p.lambda = d[11];
        p.tol = d[12];
        p.n_d = d[13];
        return p;
    }
};
}  // namespace

// device workspace of the Gram-PCG path (lazy, per context; ctx->gpcg)
struct GramPcgWs {
    size_t cap_m = 0, cap_ld = 0;
    double* par = nullptr;       // device copy of the parameter doubles
    double* h_par = nullptr;     // pinned host staging of the same
    size_t par_elems = 0;
    double* Mg = nullptr;        // M, mm x (mm + 1)
    double* vec = nullptr;       // h (mm), jd (mm)
    double* vin1 = nullptr;      // lifted U Q s_p rows (np x ld)
    double* vin2 = nullptr;      // lifted U Q r_p rows (np x ld)
    double* t3 = nullptr;        // third-action rows (np x ld)
    double* res = nullptr;       // u (mm), counters (16)
    double* h_res = nullptr;     // pinned readback
    double* Gf = nullptr;        // group members: the m x m face Gram before / after the allreduce
};

namespace {

// parameter doubles: [scalars 16][vU m][vQ m-1][nu m-1][jprobes 8 x mm][probes np x mm][idx m]
struct GpLayout {
    size_t vU, vQ, nu, jp, pr, idx, total;
    __host__ __device__ GpLayout(int m, int mm, int np) {
        vU = 16;
        vQ = vU + (size_t)m;
        nu = vQ + (size_t)(m - 1);
        jp = nu + (size_t)(m - 1);
        pr = jp + (size_t)8 * mm;
        idx = pr + (size_t)np * mm;
        total = idx + (size_t)m;
    }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide sequential dot of two smem vectors by one warp (lane-strided
// partial sums, then a fixed butterfly): identical in every call
__device__ __forceinline__ double warp_dot(const double* a, const double* b, int n, int lane) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s = fma(a[i], b[i], s);
    return warp_sum(s);
}

// Householder helpers on shared vectors (one warp): y <- y - beta (v.y) v
__device__ void warp_reflect(double* y, const double* v, double beta, int n, int lane) {
    const double c = beta * warp_dot(v, y, n, lane);
    __syncwarp();
    for (int i = lane; i < n; i += 32) y[i] -= c * v[i];
    __syncwarp();
}

// row stride of M in shared / global memory: = 1 (mod 16), so the lanes of a
// warp reading rows i = lane + 32k hit distinct bank pairs
__host__ __device__ inline int m_stride(int mm) { return (mm + 15) / 16 * 16 + 1; }

// Capped CG (cg_capped, affine_normal.hpp:85-113) on M + lambda I, one warp per
// column, no block synchronisation: Hop(p) = M p + lambda p with each lane
// computing rows lane, lane + 32, ... (two FMA chains, index order), the dots
// as lane-strided sums + a fixed butterfly. Jacobi-preconditioned when jd !=
// null. b: rhs; x: solution; r, z, p, hp: scratch (mm each). Returns through
// it (iterations, the reference's `it`), nh (operator applications) and bd
// (nonpositive curvature).
__device__ void cg_warp(const double* M, int ldm, int mm, double lambda, const double* jd, double tol, int cap,
                        const double* b, double* x, double* r, double* z, double* p, double* hp, int& it, int& nh,
                        int& bd) {
    const int lane = threadIdx.x & 31;
    double srz = 0.0, sbb = 0.0;
    for (int i = lane; i < mm; i += 32) {
        const double bi = b[i];
        const double zi = jd ? bi / jd[i] : bi;
        x[i] = 0.0;
        r[i] = bi;
        z[i] = zi;
        p[i] = zi;
        srz = fma(bi, zi, srz);
        sbb = fma(bi, bi, sbb);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        srz += __shfl_xor_sync(0xffffffffu, srz, o);
        sbb += __shfl_xor_sync(0xffffffffu, sbb, o);
    }
    __syncwarp();
    double rz = srz;
    const double target = tol * sqrt(sbb);
    double rn = sqrt(sbb);  // r = b
    it = 0;
    nh = 0;
    bd = 0;
    while (it < cap && rn > target) {
        // M p: a lane's rows i, i + 32 run together, four accumulators each, so
        // eight independent FMA chains hide the fp64 latency (one row at a time
        // with two chains made the matvec ~80 % of a CG step)
        for (int i0 = lane; i0 < mm; i0 += 64) {
            const int i1 = i0 + 32;
            const bool two = i1 < mm;
            const double* m0 = M + (size_t)i0 * ldm;
            const double* m1 = M + (size_t)(two ? i1 : i0) * ldm;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
            int j = 0;
#pragma unroll 2
            for (; j + 3 < mm; j += 4) {
                const double p0 = p[j], p1 = p[j + 1], p2 = p[j + 2], p3 = p[j + 3];
                a0 = fma(m0[j], p0, a0);
                a1 = fma(m0[j + 1], p1, a1);
                a2 = fma(m0[j + 2], p2, a2);
                a3 = fma(m0[j + 3], p3, a3);
                b0 = fma(m1[j], p0, b0);
                b1 = fma(m1[j + 1], p1, b1);
                b2 = fma(m1[j + 2], p2, b2);
                b3 = fma(m1[j + 3], p3, b3);
            }
            for (; j < mm; ++j) {
                a0 = fma(m0[j], p[j], a0);
                b0 = fma(m1[j], p[j], b0);
            }
            hp[i0] = ((a0 + a1) + (a2 + a3)) + lambda * p[i0];
            if (two) hp[i1] = ((b0 + b1) + (b2 + b3)) + lambda * p[i1];
        }
        __syncwarp();
        const double pHp = warp_dot(p, hp, mm, lane);
        ++nh;
        if (pHp <= 0.0) {
            bd = 1;
            break;
        }
        const double alpha = rz / pHp;
        double a_rz = 0.0, a_rr = 0.0;
        for (int i = lane; i < mm; i += 32) {
            x[i] += alpha * p[i];
            const double ri = r[i] - alpha * hp[i];
            const double zi = jd ? ri / jd[i] : ri;
            r[i] = ri;
            z[i] = zi;
            a_rz = fma(ri, zi, a_rz);
            a_rr = fma(ri, ri, a_rr);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            a_rz += __shfl_xor_sync(0xffffffffu, a_rz, o);
            a_rr += __shfl_xor_sync(0xffffffffu, a_rr, o);
        }
        const double beta = a_rz / rz;
        for (int i = lane; i < mm; i += 32) p[i] = z[i] + beta * p[i];
        __syncwarp();
        rz = a_rz;
        rn = sqrt(a_rr);
        ++it;
    }
    __syncwarp();
}

// [H S H]_11 (reflect_sym, driver.cu): S k x k (stride lds) -> O (k-1) x (k-1)
// (stride ldo); a = S v by rows, c = beta^2 (v . a)
__device__ void reflect_sym_block(const double* S, int lds, int k, const double* v, double beta, double* O, int ldo,
                                  double* a, double* cbuf) {
    const int tid = threadIdx.x;
    for (int i = tid; i < k; i += blockDim.x) {
        double s = 0.0;
        const double* sr = S + (size_t)i * lds;
        for (int j = 0; j < k; ++j) s += sr[j] * v[j];
        a[i] = s;
    }
    __syncthreads();
    if (tid < 32) {
        const double s = warp_dot(v, a, k, tid);
        if (tid == 0) cbuf[0] = beta * beta * s;
    }
    __syncthreads();
    const double c = cbuf[0];
    const int r = k - 1;
    for (int e = tid; e < r * r; e += blockDim.x) {
        const int i = 1 + e / r, j = 1 + (e - (e / r) * r);
        if (j > i) continue;
        const double val = S[(size_t)i * lds + j] - (beta * v[i] * a[j] + beta * a[i] * v[j]) + c * v[i] * v[j];
        O[(size_t)(i - 1) * ldo + (j - 1)] = val;
        O[(size_t)(j - 1) * ldo + (i - 1)] = val;
    }
    __syncthreads();
}

struct SetupArgs {
    const double* par; // parameter doubles (GpParams first)
    int ld;            // panel row stride (lifted rows)
    double* Mg;        // out: M (mm x m_stride(mm))
    double* vec;       // out: h (mm), jd (mm)
    double* vin1;      // out: U Q s_p rows
    double* vin2;      // out: U Q r_p rows
    double* res;       // out: counters [16 + ...]
    double* pmat;      // direct: out: P in ld x ld (zero outside the face)
};

// the face Gram on one cluster: G_f = sum_t psi''(z_t) a_t a_t^T * scale over
// this rank's rows, a_t the face columns of row t (gathered through the
// face index), the CTAs splitting the rows
struct GramArgsC {
    const double* X;   // T_local x ld panel rows
    long long T;
    int ld;
    const double* z;   // slot z
    double c2, c3, c4, scale;
    double* Gout;      // !FUSED: the m x m face Gram (row-major)
    int stage_rows;    // rows staged in shared memory per chunk
};

// shared-memory plan (doubles): [region: S | W, also the row staging][ws stage_rows][tail 6m + 64]
__host__ __device__ inline size_t gp_s_doubles(int m) {
    const int mm = m - 2;
    return std::max((size_t)m * m, (size_t)mm * m_stride(mm));
}
__host__ __device__ inline size_t gp_w_doubles(int m) {
    const int mm = m - 2;
    return std::max(std::max((size_t)m * m, (size_t)mm * m_stride(mm)), (size_t)kGpMaxCols * mm * 6);
}
// staged row stride: the face width padded to whole 8-column DMMA tiles, then
// to 4 (mod 16) doubles, so the 16 lanes of a half-warp fragment load (4 rows
// x 4 columns) hit distinct banks
// Narrow panels (ld <= 128: the compact face contexts) stage whole rows by
// bulk copy, with a zero column at ld for the tile padding, and the face
// columns are picked in the fragment loads; wide panels gather the face
// columns into the staging rows
__host__ __device__ inline bool gp_bulk_rows(int ld) { return ld <= 128 && ld % 2 == 0; }
__host__ __device__ inline int gp_stage_stride(int m, int ld) {
    const int w = gp_bulk_rows(ld) ? (m > ld + 1 ? m : ld + 1) : m;
    const int mp8 = (w + 7) & ~7;
    return mp8 + (mp8 % 16 == 0 ? 4 : 12);
}
__host__ __device__ inline size_t gp_region_doubles(int m, int ld, int stage_rows) {
    return std::max(gp_s_doubles(m) + gp_w_doubles(m), (size_t)stage_rows * gp_stage_stride(m, ld));
}
__host__ __device__ inline size_t gp_setup_smem_doubles(int m, int ld, int stage_rows) {
    return gp_region_doubles(m, ld, stage_rows) + (size_t)stage_rows + 6 * (size_t)m + 64;
}

// Everything of the direction that precedes the third-action pass, on one CTA,
// with the face Gram already in S (m x m): h, M, the Jacobi diagonal, the
// probe CGs and the lifted third-action inputs.
__device__ void setup_phases(const SetupArgs& a, const GpParams& P, double* S, double* W, double* tail) {
    const int m = P.m, mm = P.mm, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const GpLayout L(m, mm, P.np);
    double* vU = tail;
    double* vQ = vU + m;
    double* av = vQ + m;   // scratch a (m)
    double* w = av + m;    // U nu, then G U nu (m)
    double* t = w + m;     // scratch (m)
    double* jd = t + m;    // jacobi diagonal (mm)
    double* misc = jd + m; // 64 doubles: scalars
    __shared__ int s_it[kGpMaxCols], s_nh[kGpMaxCols], s_bd[kGpMaxCols];
    const double* par = a.par;
    auto col = [&](int i) -> int { return P.face_active ? (int)par[L.idx + i] : i; };
    const long long tp0 = clock64();
    for (int i = tid; i < m; i += blockDim.x) {
        vU[i] = par[L.vU + i];
        if (i < m - 1) vQ[i] = par[L.vQ + i];
    }
    __syncthreads();
    // ---- h = Q^T U^T G (U nu)  (:212-213)
    if (warp == 0) {
        // U nu: pad (0, nu) then reflect with vU (simplex.hpp:66-70)
        for (int i = lane; i < m; i += 32) w[i] = i == 0 ? 0.0 : par[L.nu + i - 1];
        __syncwarp();
        warp_reflect(w, vU, P.bU, m, lane);
    }
    __syncthreads();
    for (int i = tid; i < m; i += blockDim.x) {
        double s = 0.0;
        const double* sr = S + (size_t)i * m;
        for (int j = 0; j < m; ++j) s += sr[j] * w[j];
        t[i] = s;
    }
    __syncthreads();
    if (warp == 0) {
        warp_reflect(t, vU, P.bU, m, lane);          // U^T: reflect, drop entry 0
        warp_reflect(t + 1, vQ, P.bQ, m - 1, lane);  // Q^T: reflect, drop entry 0
        for (int i = lane; i < mm; i += 32) a.vec[i] = t[2 + i];
    }
    __syncthreads();
    if (tid == 0) a.res[52] = (double)(clock64() - tp0);
    // ---- M = [H_Q [H_U G H_U]_11 H_Q]_11 (lambda enters Hop)
    reflect_sym_block(S, m, m, vU, P.bU, W, m - 1, av, misc);
    const int ldm = m_stride(mm);
    reflect_sym_block(W, m - 1, m - 1, vQ, P.bQ, S, ldm, av, misc);
    for (int e = tid; e < mm * ldm; e += blockDim.x) a.Mg[e] = S[e];
    if (tid == 0) a.res[53] = (double)(clock64() - tp0);
    // ---- Jacobi diagonal (:197-209): mean over 8 probes of r o Hop(r), floored
    double* B = W;
    double* X = B + (size_t)kGpMaxCols * mm;
    double* R = X + (size_t)kGpMaxCols * mm;
    double* Z = R + (size_t)kGpMaxCols * mm;
    double* PP = Z + (size_t)kGpMaxCols * mm;
    double* HP = PP + (size_t)kGpMaxCols * mm;
    const double* jdp = nullptr;
    if (P.jacobi) {
        for (int e = tid; e < 8 * mm; e += blockDim.x) B[e] = par[L.jp + e];
        __syncthreads();
        for (int e = tid; e < 8 * mm; e += blockDim.x) {
            const int c = e / mm, i = e - c * mm;
            const double* mr = S + (size_t)i * ldm;
            const double* r = B + c * mm;
            double s0 = 0.0, s1 = 0.0;
            int j = 0;
            for (; j + 1 < mm; j += 2) {
                s0 = fma(mr[j], r[j], s0);
                s1 = fma(mr[j + 1], r[j + 1], s1);
            }
            if (j < mm) s0 = fma(mr[j], r[j], s0);
            HP[e] = (s0 + s1) + P.lambda * r[i];
        }
        __syncthreads();
        const double fl = fmax(1e-12, P.lambda);
        for (int i = tid; i < mm; i += blockDim.x) {
            double s = 0.0;
            for (int c = 0; c < 8; ++c) s += B[c * mm + i] * HP[c * mm + i];
            jd[i] = fmax(s / 8.0, fl);
            a.vec[mm + i] = jd[i];
        }
        __syncthreads();
        jdp = jd;
    }
    if (tid == 0) a.res[54] = (double)(clock64() - tp0);
    // ---- Hutchinson probe CGs, one warp per probe (:227-233)
    if (P.has_third && P.np > 0) {
        for (int e = tid; e < P.np * mm; e += blockDim.x) B[e] = par[L.pr + e];
        for (int e = tid; e < P.np * a.ld; e += blockDim.x) {
            a.vin1[e] = 0.0;
            a.vin2[e] = 0.0;
        }
        __syncthreads();
        if (warp < P.np) {
            const int c = warp;
            int itc, nhc, bdc;
            cg_warp(S, ldm, mm, P.lambda, jdp, P.tol, P.probe_cap, B + c * mm, X + c * mm, R + c * mm, Z + c * mm,
                    PP + c * mm, HP + c * mm, itc, nhc, bdc);
            if (lane == 0) {
                s_it[c] = itc;
                s_nh[c] = nhc;
                s_bd[c] = bdc;
            }
        }
        __syncthreads();
        if (tid == 0) a.res[55] = (double)(clock64() - tp0);
        // lift U Q s_p (into vin1) and U Q r_p (into vin2), full-row coordinates
        if (warp < 2 * P.np) {
            const int c = warp % P.np;
            const double* src = (warp < P.np ? X : B) + c * mm;
            double* y = R + (size_t)warp * m;  // R..HP scratch: 2 np rows of m
            for (int i = lane; i < m; i += 32) y[i] = (i < 2) ? 0.0 : src[i - 2];
            __syncwarp();
            warp_reflect(y + 1, vQ, P.bQ, m - 1, lane);  // Q e (pad, reflect)
            warp_reflect(y, vU, P.bU, m, lane);          // U q
            double* dst = (warp < P.np ? a.vin1 : a.vin2) + (size_t)c * a.ld;
            for (int i = lane; i < m; i += 32) dst[col(i)] = y[i];
        }
        if (tid < P.np) {
            a.res[16 + tid] = s_it[tid];
            a.res[16 + kGpMaxCols + tid] = s_nh[tid];
            a.res[16 + 2 * kGpMaxCols + tid] = s_bd[tid];
        }
    }
}

// H [0 0; 0 D] H for D r x r (stride ldd) -> O (r+1) x (r+1) (stride ldo): the
// lift unreflect (driver.cu) that P = (UQ) M^-1 (UQ)^T applies twice:
// Dp - beta v (v^T Dp) - beta (Dp v) v^T + beta^2 (v^T Dp v) v v^T
__device__ void unreflect_block(const double* D, int ldd, int r, const double* v, double beta, double* O, int ldo,
                                double* dv, double* vd, double* cbuf) {
    const int k = r + 1, tid = threadIdx.x;
    for (int i = tid; i < k; i += blockDim.x) {
        double s = 0.0, t = 0.0;
        if (i > 0)
            for (int j = 1; j < k; ++j) s += D[(size_t)(i - 1) * ldd + (j - 1)] * v[j];
        if (i > 0)
            for (int j = 1; j < k; ++j) t += v[j] * D[(size_t)(j - 1) * ldd + (i - 1)];
        dv[i] = s;
        vd[i] = t;
    }
    __syncthreads();
    if (tid < 32) {
        const double s = warp_dot(v, dv, k, tid);
        if (tid == 0) cbuf[0] = beta * beta * s;
    }
    __syncthreads();
    const double c = cbuf[0];
    for (int e = tid; e < k * k; e += blockDim.x) {
        const int i = e / k, j = e - i * k;
        const double dij = (i > 0 && j > 0) ? D[(size_t)(i - 1) * ldd + (j - 1)] : 0.0;
        O[(size_t)i * ldo + j] = dij - (beta * v[i] * vd[j] + beta * dv[i] * v[j]) + c * v[i] * v[j];
    }
    __syncthreads();
}

// In-place Gauss-Jordan inverse of an SPD matrix without pivoting, the matrix
// held in registers: thread (ty, tx) of the 16 x 32 grid owns rows ty + 16 a
// (a < 7) and columns tx + 32 b (b < 4), i.e. up to 112 x 128 >= kGpMaxM - 2.
// Per pivot k the owners of row k publish the scaled pivot row (one warp: the
// pivot is broadcast by a shuffle), the owners of column k publish the column,
// one block barrier, then every thread applies its rank-1 update from
// registers; the buffers are double-buffered so the next pivot's owners may
// publish while slower threads still read. Sweep (classic in-place form):
//   row k /= d; a_ij -= a_ik a_kj (i, j != k); a_ik = -a_ik / d; a_kk = 1 / d
// (one reciprocal per pivot, then multiplications). The pivot loop is nested
// k = 16 KA + kty with KA a compile-time index, so the owners' register
// elements r[KA][.] / r[.][KA / 2] are static (a flat loop with runtime
// selects over the 28 elements issued ~680 instructions per pivot: 2.5k cycles).
// Returns false (W undefined, S untouched) when a pivot is not positive (or NaN);
// an infinite pivot surfaces in the caller's finite check of P.
constexpr int kGjRT = 7, kGjCT = 4;
static_assert(16 * kGjRT >= kGpMaxM - 2 && 32 * kGjCT >= kGpMaxM - 2 && kGpThreads == 512, "tile grid");

template <int KA>
__device__ __forceinline__ void gj_pivot_block(double (&r)[kGjRT][kGjCT], int mm, double (*gj_row)[32 * kGjCT],
                                               double (*gj_col)[16 * kGjRT], double* gj_piv, int* gj_bad, int tx, int ty) {
    constexpr int KB = KA / 2;  // column tile of k = 16 KA + kty
    // every thread updates its whole 7 x 4 tile (the padding is the identity):
    // guarding the inactive tiles of a narrow face costs more issue slots than
    // the 28 FMAs it would save
    for (int kty = 0; kty < 16; ++kty) {
        const int k = 16 * KA + kty;
        if (k >= mm) break;  // uniform
        const int buf = k & 1;
        const int ktx = k & 31;
        if (ty == kty) {  // one warp holds row k
            const double d = __shfl_sync(0xffffffffu, r[KA][KB], ktx);
            const double dinv = 1.0 / d;  // one division per pivot: fp64 division is a ~100-cycle routine
            const bool diag_lane = tx == ktx;
            if (diag_lane) {
                gj_piv[buf] = dinv;
                if (!(d > 0.0)) *gj_bad = 1;  // not positive (or NaN)
            }
#pragma unroll
            for (int b = 0; b < kGjCT; ++b) {
                const bool diag = (b == KB) && diag_lane;
                const double v = diag ? 0.0 : r[KA][b] * dinv;
                gj_row[buf][tx + 32 * b] = v;
                r[KA][b] = diag ? dinv : v;  // row k is final for this pivot
            }
        }
        if (tx == ktx) {  // 16 threads hold column k
#pragma unroll
            for (int a = 0; a < kGjRT; ++a) gj_col[buf][ty + 16 * a] = (a == KA && ty == kty) ? 0.0 : r[a][KB];
        }
        __syncthreads();
        double rw[kGjCT], cl[kGjRT];
#pragma unroll
        for (int b = 0; b < kGjCT; ++b) rw[b] = gj_row[buf][tx + 32 * b];
#pragma unroll
        for (int a = 0; a < kGjRT; ++a) cl[a] = gj_col[buf][ty + 16 * a];
        const double ndinv = -gj_piv[buf];
#pragma unroll
        for (int a = 0; a < kGjRT; ++a)
#pragma unroll
            for (int b = 0; b < kGjCT; ++b)
                r[a][b] = fma(-cl[a], rw[b], r[a][b]);  // row k (cl = 0), column k (rw = 0): unchanged
        if (tx == ktx) {  // column k: a_ik = -a_ik / d (the diagonal keeps 1 / d)
#pragma unroll
            for (int a = 0; a < kGjRT; ++a)
                if (!(a == KA && ty == kty)) r[a][KB] = cl[a] * ndinv;
        }
    }
}

__device__ bool spd_inverse_tiled(const double* S, double* W, int ldm, int mm) {
    constexpr int RT = kGjRT, CT = kGjCT;
    __shared__ double gj_row[2][32 * CT], gj_col[2][16 * RT], gj_piv[2];
    __shared__ int gj_bad;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    double r[RT][CT];
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < CT; ++b) {
            const int i = ty + 16 * a, j = tx + 32 * b;
            r[a][b] = (i < mm && j < mm) ? S[(size_t)i * ldm + j] : (i == j ? 1.0 : 0.0);
        }
    if (tid == 0) gj_bad = 0;
    __syncthreads();
    gj_pivot_block<0>(r, mm, gj_row, gj_col, gj_piv, &gj_bad, tx, ty);
    gj_pivot_block<1>(r, mm, gj_row, gj_col, gj_piv, &gj_bad, tx, ty);
    gj_pivot_block<2>(r, mm, gj_row, gj_col, gj_piv, &gj_bad, tx, ty);
    gj_pivot_block<3>(r, mm, gj_row, gj_col, gj_piv, &gj_bad, tx, ty);
    gj_pivot_block<4>(r, mm, gj_row, gj_col, gj_piv, &gj_bad, tx, ty);
    gj_pivot_block<5>(r, mm, gj_row, gj_col, gj_piv, &gj_bad, tx, ty);
    gj_pivot_block<6>(r, mm, gj_row, gj_col, gj_piv, &gj_bad, tx, ty);
    __syncthreads();
    if (gj_bad) return false;
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < CT; ++b) {
            const int i = ty + 16 * a, j = tx + 32 * b;
            if (i < mm && j < mm) W[(size_t)i * ldm + j] = r[a][b];
        }
    __syncthreads();
    return true;
}

// Direct branch (affine_normal.hpp:151-188) after the Gram, one CTA: h, M + lambda I,
// its inverse by Gauss-Jordan with partial pivoting (the pivots of the
// reference's PartialPivLU: the largest remaining magnitude, first index on
// ties; an all-zero pivot column flags the operator singular, which sends the
// caller to the lambda fallback like the reference's non-finite solve), then
// P = (UQ) M^-1 (UQ)^T scattered into the ld x ld trace matrix (zero outside the
// face). Outputs: h (vec), M^-1 (Mg, stride m_stride), P (pmat), flags (res[3]).
__device__ void direct_phases(const SetupArgs& a, const GpParams& P, double* S, double* W, double* tail, int ld) {
    const int m = P.m, mm = P.mm, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const GpLayout L(m, mm, P.np);
    double* vU = tail;
    double* vQ = vU + m;
    double* av = vQ + m;   // scratch (m)
    double* w = av + m;    // U nu, then G U nu (m)
    double* t = w + m;     // scratch (m)
    double* fc = t + m;    // pivot column (m)
    double* misc = fc + m; // scalars
    __shared__ int s_piv, s_sing;
    const double* par = a.par;
    auto col = [&](int i) -> int { return P.face_active ? (int)par[L.idx + i] : i; };
    for (int i = tid; i < m; i += blockDim.x) {
        vU[i] = par[L.vU + i];
        if (i < m - 1) vQ[i] = par[L.vQ + i];
    }
    __syncthreads();
    const long long td0 = clock64();
    // h = Q^T U^T G (U nu)  (:164-166)
    if (warp == 0) {
        for (int i = lane; i < m; i += 32) w[i] = i == 0 ? 0.0 : par[L.nu + i - 1];
        __syncwarp();
        warp_reflect(w, vU, P.bU, m, lane);
    }
    __syncthreads();
    for (int i = tid; i < m; i += blockDim.x) {
        double s = 0.0;
        const double* sr = S + (size_t)i * m;
        for (int j = 0; j < m; ++j) s += sr[j] * w[j];
        t[i] = s;
    }
    __syncthreads();
    if (warp == 0) {
        warp_reflect(t, vU, P.bU, m, lane);
        warp_reflect(t + 1, vQ, P.bQ, m - 1, lane);
        for (int i = lane; i < mm; i += 32) a.vec[i] = t[2 + i];
    }
    __syncthreads();
    if (tid == 0) a.res[52] = (double)(clock64() - td0);
    // M = (UQ)^T G (UQ) + lambda I  (:169-170)
    reflect_sym_block(S, m, m, vU, P.bU, W, m - 1, av, misc);
    const int ldm = m_stride(mm);
    reflect_sym_block(W, m - 1, m - 1, vQ, P.bQ, S, ldm, av, misc);
    for (int i = tid; i < mm; i += blockDim.x) S[(size_t)i * ldm + i] += P.lambda;
    for (int e = tid; e < mm * ldm; e += blockDim.x) {
        const int i = e / ldm, j = e - i * ldm;
        W[e] = (i == j) ? 1.0 : 0.0;
    }
    if (tid == 0) {
        s_sing = 0;
        a.res[3] = 0.0;
        a.res[4] = 0.0;
    }
    __syncthreads();
    if (tid == 0) a.res[53] = (double)(clock64() - td0);
    // SPD fast path: when every pivot of the unpivoted sweep is positive and
    // finite (M = W^T D W / T + lambda I with psi'' > 0, the normal case) the
    // inverse comes from the register-tiled in-place sweep, one block barrier
    // per pivot; otherwise the pivoted sweep below runs on the untouched S
    const bool spd_done = spd_inverse_tiled(S, W, ldm, mm);
    if (tid == 0) {
        a.res[56] = spd_done ? 1.0 : 0.0;
        a.res[57] = (double)(clock64() - td0);
    }
    // Gauss-Jordan on [M | I] with partial pivoting: W <- M^-1
    for (int k = 0; k < mm && !spd_done; ++k) {
        if (warp == 0) {
            double big = -1.0;
            int piv = k;
            for (int r = k + lane; r < mm; r += 32) {
                const double v = fabs(S[(size_t)r * ldm + k]);
                if (v > big) {
                    big = v;
                    piv = r;
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, big, o);
                const int op = __shfl_xor_sync(0xffffffffu, piv, o);
                if (ob > big || (ob == big && op < piv)) {
                    big = ob;
                    piv = op;
                }
            }
            if (lane == 0) {
                s_piv = piv;
                if (!(big > 0.0)) s_sing = 1;  // zero (or NaN) pivot column
            }
        }
        __syncthreads();
        if (s_sing) break;
        const int piv = s_piv;
        if (piv != k) {
            for (int j = tid; j < mm; j += blockDim.x) {
                double* a0 = S + (size_t)k * ldm + j;
                double* a1 = S + (size_t)piv * ldm + j;
                const double x0 = *a0;
                *a0 = *a1;
                *a1 = x0;
                double* b0 = W + (size_t)k * ldm + j;
                double* b1 = W + (size_t)piv * ldm + j;
                const double y0 = *b0;
                *b0 = *b1;
                *b1 = y0;
            }
            __syncthreads();
        }
        const double pv = S[(size_t)k * ldm + k];
        for (int r = tid; r < mm; r += blockDim.x) fc[r] = S[(size_t)r * ldm + k];
        __syncthreads();
        for (int j = tid; j < mm; j += blockDim.x) {
            S[(size_t)k * ldm + j] /= pv;
            W[(size_t)k * ldm + j] /= pv;
        }
        __syncthreads();
        for (int e = tid; e < mm * mm; e += blockDim.x) {
            const int r = e / mm, j = e - r * mm;
            if (r == k) continue;
            const double f = fc[r];
            if (f == 0.0) continue;
            if (j > k) S[(size_t)r * ldm + j] -= f * S[(size_t)k * ldm + j];
            W[(size_t)r * ldm + j] -= f * W[(size_t)k * ldm + j];
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.res[3] = s_sing ? 1.0 : 0.0;
        a.res[54] = (double)(clock64() - td0);
    }
    for (int e = tid; e < mm * ldm; e += blockDim.x) a.Mg[e] = W[e];
    __syncthreads();
    if (!a.pmat) return;
    // P = U [H_Q [0 0; 0 M^-1] H_Q] U^T: (m-1)^2 into S, then m^2 scattered
    unreflect_block(W, ldm, mm, vQ, P.bQ, S, m - 1, av, t, misc);
    double* Pm = W;  // M^-1 is saved in Mg; reuse W for P (m x m)
    unreflect_block(S, m - 1, m - 1, vU, P.bU, Pm, m, av, t, misc);
    for (int e = tid; e < ld * ld; e += blockDim.x) a.pmat[e] = 0.0;
    __syncthreads();
    int bad = 0;
    for (int e = tid; e < m * m; e += blockDim.x) {
        const int i = e / m, j = e - i * m;
        const double v = Pm[e];
        if (!isfinite(v)) bad = 1;
        a.pmat[(size_t)col(i) * ld + col(j)] = v;
    }
    if (bad) atomicOr(&s_sing, 2);
    __syncthreads();
    if (tid == 0) {
        a.res[4] = (s_sing & 2) ? 1.0 : 0.0;
        a.res[55] = (double)(clock64() - td0);
    }
}

__device__ __forceinline__ void gp_dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}

// One cluster of CS CTAs: the face Gram (rows split over the CTAs; each CTA
// stages its rows' face columns in shared memory with 8-byte async copies and
// accumulates 4 x 4 register blocks of the lower block triangle), the
// partials summed over the cluster through distributed shared memory in rank
// order (each CTA reduces a slice and stores it into CTA 0), then - FUSED -
// CTA 0 continues with the setup phases; otherwise it writes G_f for the
// group allreduce.
// MODE 0: write G_f (group members), 1: PCG setup, 2: direct setup
template <int MODE>
__global__ void __launch_bounds__(kGpThreads, 1) gram_pcg_cluster_kernel(const GramArgsC g, const SetupArgs a) {
    extern __shared__ __align__(16) double sm[];
    namespace cgx = cooperative_groups;
    cgx::cluster_group cluster = cgx::this_cluster();
    const GpParams P = GpParams::load(a.par);
    const int m = P.m, mp = (m + 3) & ~3, tid = threadIdx.x;
    const GpLayout L(m, P.mm, P.np);
    const int rank = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
    const long long tg0 = clock64();
    const int SR = g.stage_rows;
    double* S = sm;
    double* W = S + gp_s_doubles(m);
    double* xs = sm;  // the staging area overlays S | W
    double* ws = sm + gp_region_doubles(m, g.ld, SR);
    double* tail = ws + SR;
    const double* par = a.par;
    int* cols = reinterpret_cast<int*>(tail);
    for (int j = tid; j < mp; j += blockDim.x) cols[j] = j < m ? (P.face_active ? (int)par[L.idx + j] : j) : -1;
    // ---- face Gram on the tensor pipe: 8 x 8 lower-triangle tiles of
    // sum_t (psi''(z_t) x_t,I)(x_t,J) as mma.m8n8k4 f64 over 4-row k-steps; warp
    // w owns tiles w, w + nwarps, ... over all of this CTA's rows, so no
    // cross-warp reduction (fragment layout: A row-major lane -> (l/4, l%4),
    // B col-major lane -> (l%4, l/4), C lane -> (l/4, 2 (l%4) + {0, 1}))
    const int ms = gp_stage_stride(m, g.ld);
    const int nt = (m + 7) / 8, ntiles = nt * (nt + 1) / 2;
    const int lane = tid & 31, warp = tid >> 5, nwarps = (int)blockDim.x >> 5;
    const int tpw = (ntiles + nwarps - 1) / nwarps;  // tiles per warp (<= 8: kGpMaxM = 112, 16 warps)
    static_assert((kGpMaxM / 8) * (kGpMaxM / 8 + 1) / 2 <= 8 * (kGpThreads / 32), "tiles per warp");
    const bool bulk = gp_bulk_rows(g.ld);
    __shared__ uint64_t sbar;
    if (tid == 0) {
        mbar_init(&sbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const long long r0 = g.T * rank / CS, r1 = g.T * (rank + 1) / CS;
    long long tq = clock64(), tstage = 0, twait = 0, tmma = 0, tpre = tq - tg0;
    // the DMMA accumulate chain is long-latency (~440 cycles per dependent
    // step measured on C4), so every warp keeps ~8 independent chains: TW
    // tiles x U interleaved k-step accumulators, summed in a fixed order
    auto run = [&](auto tw_c, auto u_c) {
        constexpr int TW = decltype(tw_c)::value, U = decltype(u_c)::value;
        double acc[TW][U][2];
        int tI[TW], tJ[TW], cI[TW], cJ[TW];  // tiles; this lane's staged column of each
#pragma unroll
        for (int q = 0; q < TW; ++q) {
#pragma unroll
            for (int u = 0; u < U; ++u) acc[q][u][0] = acc[q][u][1] = 0.0;
            const int tl = warp + q * nwarps;
            int r = 0, e = tl;
            while (e > r) {  // lower tile triangle, row-major
                e -= r + 1;
                ++r;
            }
            // slots past the last tile redo tile 0 (discarded): branch-free k-loop
            tI[q] = tl < ntiles ? r : 0;
            tJ[q] = tl < ntiles ? e : 0;
            // bulk rows: the face column of fragment column l/4 (the zero column
            // ld past the face); gathered rows: the staged position itself
            const int fi = 8 * r + (lane >> 2), fj = 8 * e + (lane >> 2);
            cI[q] = !bulk ? fi : (fi < m ? cols[fi] : g.ld);
            cJ[q] = !bulk ? fj : (fj < m ? cols[fj] : g.ld);
        }
        uint32_t phase = 0;
        for (long long c0 = r0; c0 < r1; c0 += SR) {
            const int rows = (int)min((long long)SR, r1 - c0);
            const int rows4 = (rows + 3) & ~3;
            if (bulk) {
                if (tid == 0) mbar_arrive_expect_tx(&sbar, (uint32_t)((size_t)rows * g.ld * sizeof(double)));
                __syncthreads();
                for (int t = tid; t < rows; t += blockDim.x)
                    bulk_g2s(xs + (size_t)t * ms, g.X + (c0 + t) * g.ld, (uint32_t)(g.ld * sizeof(double)), &sbar,
                             policy_evict_last());
                for (int t = warp; t < rows4; t += nwarps)  // pad columns, pad rows
                    for (int j = (t < rows ? g.ld : 0) + lane; j < ms; j += 32) xs[(size_t)t * ms + j] = 0.0;
            } else {  // a warp per row, a lane per column: no index arithmetic per element
                for (int t = warp; t < rows4; t += nwarps) {
                    const double* src = g.X + (c0 + t) * g.ld;
                    for (int j = lane; j < ms; j += 32) {
                        if (t < rows && j < m)
                            cp_async8(xs + (size_t)t * ms + j, src + cols[j]);
                        else
                            xs[(size_t)t * ms + j] = 0.0;
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            for (int t = tid; t < rows4; t += blockDim.x) {
                const double zt = t < rows ? g.z[c0 + t] : 0.0;
                ws[t] = t < rows ? 2.0 * g.c2 - 6.0 * g.c3 * zt + 12.0 * g.c4 * (zt * zt) : 0.0;  // oracle.hpp:116-119
            }
            tstage += clock64() - tq;
            tq = clock64();
            if (bulk) {
                mbar_wait(&sbar, phase);
                phase ^= 1u;
            } else {
                asm volatile("cp.async.wait_all;" ::: "memory");
            }
            __syncthreads();
            twait += clock64() - tq;
            tq = clock64();
            const int kr = lane & 3;
            for (int t0 = 0; t0 < rows4; t0 += 4 * U) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int tk = t0 + 4 * u;
                    if (tk >= rows4) break;
                    const double* xr = xs + (size_t)(tk + kr) * ms;
                    const double wt = ws[tk + kr];
#pragma unroll
                    for (int q = 0; q < TW; ++q) {
                        const double b = xr[cJ[q]];
                        const double a = xr[cI[q]] * wt;
                        gp_dmma(acc[q][u], a, b);
                    }
                }
            }
            __syncthreads();
            tmma += clock64() - tq;
            tq = clock64();
        }
        // partial -> W (m x m, lower triangle of the face)
#pragma unroll
        for (int q = 0; q < TW; ++q) {
            if (warp + q * nwarps >= ntiles) continue;
            const int i = 8 * tI[q] + (lane >> 2);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double v = acc[q][0][h];
#pragma unroll
                for (int u = 1; u < U; ++u) v += acc[q][u][h];
                const int j = 8 * tJ[q] + 2 * (lane & 3) + h;
                if (i < m && j <= i) W[(size_t)i * m + j] = v;
            }
        }
    };
    if (tpw <= 1)
        run(std::integral_constant<int, 1>{}, std::integral_constant<int, 16>{});
    else if (tpw <= 2)
        run(std::integral_constant<int, 2>{}, std::integral_constant<int, 8>{});
    else if (tpw <= 4)
        run(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{});
    else
        run(std::integral_constant<int, 8>{}, std::integral_constant<int, 2>{});  // kGpMaxM = 112: <= 7 tiles
    const long long tg1 = clock64();
    cluster.sync();
    // ---- each CTA sums a slice of the entries over the cluster (rank order)
    // and stores it, mirrored and scaled, into CTA 0's S
    {
        double* S0 = cluster.map_shared_rank(S, 0);
        const int ntri = m * (m + 1) / 2;
        for (int e = rank * (int)blockDim.x + tid; e < ntri; e += CS * (int)blockDim.x) {
            int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
            while (i * (i + 1) / 2 > e) --i;
            while ((i + 1) * (i + 2) / 2 <= e) ++i;
            const int j = e - i * (i + 1) / 2;
            const size_t off = (size_t)i * m + j;
            double pv[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) pv[q] = q < CS ? cluster.map_shared_rank(W, q)[off] : 0.0;
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (q < CS) v += pv[q];
            v *= g.scale;
            S0[(size_t)i * m + j] = v;
            S0[(size_t)j * m + i] = v;
        }
    }
    cluster.sync();  // CTA 0 holds G_f; no CTA leaves while its partial may still be read
    if (rank != 0) return;
    if (tid == 0) {
        a.res[48] = (double)(tg1 - tg0);
        a.res[49] = (double)(clock64() - tg1);
        a.res[58] = (double)tpre;
        a.res[59] = (double)tstage;
        a.res[60] = (double)twait;
        a.res[61] = (double)tmma;
    }
    if constexpr (MODE == 0) {
        for (int e = tid; e < m * m; e += blockDim.x) g.Gout[e] = S[e];
    } else if constexpr (MODE == 1) {
        setup_phases(a, P, S, W, tail);
    } else {
        direct_phases(a, P, S, W, tail, g.ld);
    }
}

// group members: the allreduced face Gram from global memory, then the setup
__global__ void __launch_bounds__(kGpThreads, 1) gram_pcg_setup_kernel(const double* Gf, const SetupArgs a,
                                                                       int stage_rows) {
    extern __shared__ __align__(16) double sm[];
    const GpParams P = GpParams::load(a.par);
    const int m = P.m;
    double* S = sm;
    double* W = S + gp_s_doubles(m);
    double* tail = sm + gp_region_doubles(m, a.ld, stage_rows) + stage_rows;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) S[e] = Gf[e];
    __syncthreads();
    setup_phases(a, P, S, W, tail);
}

struct MainArgs {
    const double* par;
    int ld;
    const double* Mg;
    const double* vec;  // h, jd
    const double* t3;   // third-action rows (np x ld)
    double* res;        // u (mm) at [64...], counters at [0..16)
};

__global__ void __launch_bounds__(kGpThreads, 1) gram_pcg_main_kernel(const MainArgs a) {
    extern __shared__ __align__(16) double sm[];
    const GpParams P = GpParams::load(a.par);
    const int m = P.m, mm = P.mm, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const GpLayout L(m, mm, P.np);
    const int ldm = m_stride(mm);
    double* M = sm;
    double* rhs = M + (size_t)mm * ldm;
    double* X = rhs + mm;
    double* R = X + mm;
    double* Z = R + mm;
    double* PP = Z + mm;
    double* HP = PP + mm;
    double* jd = HP + mm;
    double* av = jd + mm;                // a (mm)
    double* rows = av + mm;              // np x m reduced third actions
    double* vU = rows + (size_t)kGpMaxCols * m;
    double* vQ = vU + m;
    const long long tm0 = clock64();
    const double* par = a.par;
    auto col = [&](int i) -> int { return P.face_active ? (int)par[L.idx + i] : i; };
    for (int e = tid; e < mm * ldm; e += blockDim.x) M[e] = a.Mg[e];
    for (int i = tid; i < m; i += blockDim.x) {
        vU[i] = par[L.vU + i];
        if (i < m - 1) vQ[i] = par[L.vQ + i];
    }
    for (int i = tid; i < mm; i += blockDim.x) {
        jd[i] = P.jacobi ? a.vec[mm + i] : 1.0;
        av[i] = 0.0;
    }
    __syncthreads();
    // a = (1/np) sum_p Q^T U^T T3_p in probe order (:233-236)
    if (P.has_third && P.np > 0) {
        if (warp < P.np) {
            double* y = rows + (size_t)warp * m;
            const double* src = a.t3 + (size_t)warp * a.ld;
            for (int i = lane; i < m; i += 32) y[i] = src[col(i)];
            __syncwarp();
            warp_reflect(y, vU, P.bU, m, lane);
            warp_reflect(y + 1, vQ, P.bQ, m - 1, lane);
        }
        __syncthreads();
        for (int i = tid; i < mm; i += blockDim.x) {
            double s = 0.0;
            for (int c = 0; c < P.np; ++c) s += rows[(size_t)c * m + 2 + i];
            av[i] = s / (double)P.np;
        }
        __syncthreads();
    }
    const long long tm1 = clock64();
    // rhs = h - (||gbar|| / n) a  (:239), then the main CG (:240-241) on warp 0
    const double coef = P.gn / P.n_d;
    for (int i = tid; i < mm; i += blockDim.x) rhs[i] = a.vec[i] - coef * av[i];
    __syncthreads();
    if (warp == 0) {
        int itc, nhc, bdc;
        cg_warp(M, ldm, mm, P.lambda, P.jacobi ? jd : nullptr, P.tol, P.maxit, rhs, X, R, Z, PP, HP, itc, nhc, bdc);
        for (int i = lane; i < mm; i += 32) a.res[64 + i] = X[i];
        if (lane == 0) {
            a.res[0] = itc;
            a.res[1] = nhc;
            a.res[2] = bdc;
            a.res[56] = (double)(tm1 - tm0);
            a.res[57] = (double)(clock64() - tm1);
        }
    }
}

// direct branch tail (:173-180): a = Q^T U^T (A_f^T tw) from the trace pass,
// rhs = h - (||gbar|| / n) a, u = M^-1 rhs; non-finite when the operator was
// singular or P non-finite (the caller retries with the fallback ridge)
__global__ void __launch_bounds__(kGpThreads, 1) gram_direct_main_kernel(const MainArgs a, const double* af) {
    extern __shared__ __align__(16) double sm[];
    const GpParams P = GpParams::load(a.par);
    const int m = P.m, mm = P.mm, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const GpLayout L(m, mm, P.np);
    const int ldm = m_stride(mm);
    double* y = sm;          // m
    double* rhs = y + m;     // mm
    double* vU = rhs + mm;   // m
    double* vQ = vU + m;     // m
    const double* par = a.par;
    auto col = [&](int i) -> int { return P.face_active ? (int)par[L.idx + i] : i; };
    for (int i = tid; i < m; i += blockDim.x) {
        vU[i] = par[L.vU + i];
        if (i < m - 1) vQ[i] = par[L.vQ + i];
        y[i] = (P.has_third && af) ? af[col(i)] : 0.0;
    }
    __syncthreads();
    if (warp == 0 && P.has_third && af) {
        warp_reflect(y, vU, P.bU, m, lane);
        warp_reflect(y + 1, vQ, P.bQ, m - 1, lane);
    }
    __syncthreads();
    const double coef = P.gn / P.n_d;
    for (int i = tid; i < mm; i += blockDim.x) rhs[i] = a.vec[i] - coef * ((P.has_third && af) ? y[2 + i] : 0.0);
    __syncthreads();
    const bool bad = a.res[3] != 0.0 || a.res[4] != 0.0;
    for (int i = tid; i < mm; i += blockDim.x) {
        const double* yr = a.Mg + (size_t)i * ldm;
        double s0 = 0.0, s1 = 0.0;
        int j = 0;
        for (; j + 1 < mm; j += 2) {
            s0 = fma(yr[j], rhs[j], s0);
            s1 = fma(yr[j + 1], rhs[j + 1], s1);
        }
        if (j < mm) s0 = fma(yr[j], rhs[j], s0);
        a.res[64 + i] = bad ? NAN : s0 + s1;
    }
}

size_t main_smem_bytes(int m) {
    const int mm = m - 2;
    return ((size_t)mm * m_stride(mm) + 9 * (size_t)mm + (size_t)kGpMaxCols * m + 2 * (size_t)m + 16) *
           sizeof(double);
}

}  // namespace

void gram_pcg_alloc(mvsk_gpu_ctx* ctx, GramPcgWs& ws, size_t ld) {
    for (double* p : {ws.par, ws.Mg, ws.vec, ws.vin1, ws.vin2, ws.t3, ws.res, ws.Gf})
        if (p) MVSK_CUDA(cudaFree(p));
    for (double* p : {ws.h_par, ws.h_res})
        if (p) MVSK_CUDA(cudaFreeHost(p));
    const GpLayout Lmax(kGpMaxM, kGpMaxM - 2, kGpMaxCols);
    ws.par_elems = Lmax.total;
    MVSK_CUDA(cudaMalloc(&ws.par, ws.par_elems * sizeof(double)));
    MVSK_CUDA(cudaMallocHost(&ws.h_par, ws.par_elems * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&ws.Mg, (size_t)kGpMaxM * (kGpMaxM + 1) * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&ws.Gf, (size_t)kGpMaxM * kGpMaxM * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&ws.vec, (size_t)2 * kGpMaxM * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&ws.vin1, (size_t)kGpMaxCols * ld * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&ws.vin2, (size_t)kGpMaxCols * ld * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&ws.t3, (size_t)kGpMaxCols * ld * sizeof(double)));
    MVSK_CUDA(cudaMalloc(&ws.res, (size_t)(64 + kGpMaxM) * sizeof(double)));
    MVSK_CUDA(cudaMallocHost(&ws.h_res, (size_t)(64 + kGpMaxM) * sizeof(double)));
    MVSK_CUDA(cudaMemset(ws.res, 0, (size_t)(64 + kGpMaxM) * sizeof(double)));
    ws.cap_m = kGpMaxM;
    ws.cap_ld = ld;
    ++ctx->epoch;
}

bool pcg_direction_gram(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const PcgInput& in, PcgOutput& out) {
    const int m = (int)in.m;
    const int np = in.has_third ? (int)in.probes.size() : 0;
    if (in.exact_trace || m < 4 || m > kGpMaxM || np > kGpMaxCols || (in.has_third && np == 0)) return false;
    if (in.jacobi_probes.size() != 0 && in.jacobi_probes.size() != 8) return false;
    const int mm = m - 2;
    // rows staged per chunk: as many as fit beside the setup's vectors, at most
    // one 8-CTA share of this rank's rows
    const int mp = gp_stage_stride(m, (int)ctx->ld);
    const long long avail = (long long)(ctx->max_smem / sizeof(double)) - (6LL * m + 64) - 64;
    long long SR = std::min<long long>(avail / (mp + 1), (ctx->T_local + 7) / 8);
    SR = std::max<long long>(SR & ~3LL, 4);  // whole 4-row DMMA k-steps
    const int stage_rows = (int)SR;
    const size_t setup_smem = gp_setup_smem_doubles(m, (int)ctx->ld, stage_rows) * sizeof(double);
    if (setup_smem > ctx->max_smem || main_smem_bytes(m) > ctx->max_smem) return false;
    if (!ctx->gpcg) ctx->gpcg = new GramPcgWs();
    GramPcgWs& ws = *ctx->gpcg;
    const GpLayout L(m, mm, np);
    const size_t ld = (size_t)ctx->ld;
    // workspace (sized for the largest face seen; growth invalidates graphs)
    if (ws.cap_m < (size_t)kGpMaxM || ws.cap_ld < ld) gram_pcg_alloc(ctx, ws, ld);
    // the Gram cluster: 16 CTAs where a non-portable cluster of this size is
    // resident, else 8 (portable)
    const bool sharded = is_sharded(ctx);
    const void* cfn = sharded ? reinterpret_cast<const void*>(&gram_pcg_cluster_kernel<0>)
                              : reinterpret_cast<const void*>(&gram_pcg_cluster_kernel<1>);
    int CS = 0;
    for (int cs : {16, 8})
        if (!CS && cluster_fits(cfn, cs, kGpThreads, setup_smem)) CS = cs;
    if (!CS) return false;
    // parameters -> pinned staging (read by the graph's H2D node at replay)
    double* hp = ws.h_par;
    std::copy(in.vU.begin(), in.vU.end(), hp + L.vU);
    std::copy(in.vQ.begin(), in.vQ.end(), hp + L.vQ);
    std::copy(in.nu.begin(), in.nu.end(), hp + L.nu);
    for (size_t p = 0; p < in.jacobi_probes.size(); ++p)
        std::copy(in.jacobi_probes[p].begin(), in.jacobi_probes[p].end(), hp + L.jp + p * mm);
    for (int p = 0; p < np; ++p) std::copy(in.probes[p].begin(), in.probes[p].end(), hp + L.pr + (size_t)p * mm);
    for (int i = 0; i < m; ++i) hp[L.idx + i] = (double)(fm.active ? fm.idx[(size_t)i] : i);
    GpParams P{};
    P.m = m;
    P.mm = mm;
    P.np = np;
    P.probe_cap = in.probe_cap;
    P.maxit = in.maxit;
    P.jacobi = in.jacobi_probes.empty() ? 0 : 1;
    P.has_third = in.has_third ? 1 : 0;
    P.face_active = fm.active ? 1 : 0;
    P.bU = in.bU;
    P.bQ = in.bQ;
    P.gn = in.gn;
    P.lambda = in.lambda;
    P.tol = in.tol;
    P.n_d = (double)m;
    P.store(hp);
    const Slot& sl = ctx->slots[slot];
    // graph key: the face width and probe count fix every launch shape
    const int key = m * 64 + np * 2 + P.jacobi;
    (void)mp;
    run_graphed(ctx, kGraphGramPcg, key, slot, [&] {
        MVSK_CUDA(cudaMemcpyAsync(ws.par, ws.h_par, L.total * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        SetupArgs sa{};
        sa.par = ws.par;
        sa.ld = (int)ld;
        sa.Mg = ws.Mg;
        sa.vec = ws.vec;
        sa.vin1 = ws.vin1;
        sa.vin2 = ws.vin2;
        sa.res = ws.res;
        GramArgsC ga{};
        ga.X = ctx->X;
        ga.T = ctx->T_local;
        ga.ld = (int)ld;
        ga.z = sl.z;
        ga.c2 = ctx->c.c2;
        ga.c3 = ctx->c.c3;
        ga.c4 = ctx->c.c4;
        ga.scale = 1.0 / (double)ctx->T_global;
        ga.Gout = ws.Gf;
        ga.stage_rows = stage_rows;
        set_smem_attr(cfn, setup_smem);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(CS);
        cfg.blockDim = dim3(kGpThreads);
        cfg.dynamicSmemBytes = setup_smem;
        cfg.stream = ctx->stream;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        void* cargs[] = {&ga, &sa};
        ++ctx->launches;
        MVSK_CUDA(cudaLaunchKernelExC(&cfg, cfn, cargs));
        ctx->phys += 1;  // the Gram streams the face panel once
        if (sharded) {
            allreduce_sum(ctx, ws.Gf, (size_t)m * m);
            set_smem_attr(reinterpret_cast<const void*>(&gram_pcg_setup_kernel), setup_smem);
            ++ctx->launches;
            gram_pcg_setup_kernel<<<1, kGpThreads, setup_smem, ctx->stream>>>(ws.Gf, sa, stage_rows);
            MVSK_CUDA(cudaGetLastError());
        }
        if (np > 0) {
            PassIO io;
            io.vin = ws.vin1;
            io.vin2 = ws.vin2;
            io.z = sl.z;
            io.out = ws.t3;
            io.ldo = (long long)ld;
            run_pass(ctx, Op::THIRD, np, io);
        }
        MainArgs ma{};
        ma.par = ws.par;
        ma.ld = (int)ld;
        ma.Mg = ws.Mg;
        ma.vec = ws.vec;
        ma.t3 = ws.t3;
        ma.res = ws.res;
        const size_t msm = main_smem_bytes(m);
        set_smem_attr(reinterpret_cast<const void*>(&gram_pcg_main_kernel), msm);
        ++ctx->launches;
        gram_pcg_main_kernel<<<1, kGpThreads, msm, ctx->stream>>>(ma);
        MVSK_CUDA(cudaGetLastError());
        MVSK_CUDA(cudaMemcpyAsync(ws.h_res, ws.res, (size_t)(64 + mm) * sizeof(double), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    });
    MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
    const double* r = ws.h_res;
    out.u.assign(r + 64, r + 64 + mm);
    long long hvps = 1 + (P.jacobi ? 8 : 0) + (long long)r[1];
    int iters = (int)r[0];
    bool bd = r[2] != 0.0;
    for (int p = 0; p < np; ++p) {
        iters += (int)r[16 + p];
        hvps += (long long)r[16 + kGpMaxCols + p];
        bd = bd || r[16 + 2 * kGpMaxCols + p] != 0.0;
    }
    out.iters = iters;
    out.breakdown = bd;
    static const bool prof = std::getenv("MVSK_GPCG_PROF") != nullptr;
    if (prof)
        std::fprintf(stderr,
                     "[gpcg] m=%d np=%d face_gather %d ld %lld T %lld cycles: gram %.0f reduce %.0f | setup h %.0f M %.0f "
                     "jacobi %.0f probes %.0f | main a %.0f cg %.0f | iters %d | gram: pre %.0f issue %.0f wait %.0f "
                     "mma %.0f\n",
                     m, np, fm.active ? 1 : 0, (long long)ctx->ld, (long long)ctx->T_local, r[48], r[49], r[52], r[53] - r[52], r[54] - r[53], r[55] - r[54], r[56], r[57], iters, r[58], r[59], r[60], r[61]);
    // reference contract (common.hpp:27-37): 2 passes per Hop, 3 per third action
    ctx->fwd += (uint64_t)(hvps + 2LL * np);
    ctx->tr += (uint64_t)(hvps + np);
    return true;
}

bool direct_direction_device(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const DirectInput& in,
                             std::vector<double>& u) {
    const int m = (int)in.m;
    if (m < 4 || m > kGpMaxM || is_sharded(ctx)) return false;
    // Device-resident by default on panels of >= kDirectDeviceMinLd columns: one
    // graph (Gram + h + M + register-tiled SPD inverse + P in one cluster
    // kernel, trace quadform, X^T pass, solve) and one round trip per
    // direction. Measured (profiles/r02_direct_device_ab.txt): C2-small solve
    // (n = 100, T = 1000) 5.04 ms on the host LU path (112 us per direction) vs
    // 4.31 ms here (94 us); C1 (n = 20, T = 500) 42 us per direction on the host
    // vs 60 us here - the kernel's fixed phase latencies (~26 us) and its three
    // trailing launches exceed two short round trips around an 18 x 18
    // factorisation, so narrow panels keep the host path.
    // MVSK_DEVICE_DIRECT=1 / MVSK_NO_DEVICE_DIRECT=1 force either side (A/B runs).
    static const bool force_on = std::getenv("MVSK_DEVICE_DIRECT") != nullptr;
    static const bool force_off = std::getenv("MVSK_NO_DEVICE_DIRECT") != nullptr;
    if (force_off || (!force_on && ctx->ld < kDirectDeviceMinLd)) return false;
    // P is scattered into a zero-filled ld x ld matrix by one CTA: index-map faces of wide panels (only
    // reachable with face compaction switched off) stay on the host path
    if (ctx->ld > kDirectDeviceMaxLd) return false;
    const int mm = m - 2;
    const int mp = gp_stage_stride(m, (int)ctx->ld);
    // 512 doubles less than the PCG setup: the static buffers of spd_inverse_tiled
    const long long avail = (long long)(ctx->max_smem / sizeof(double)) - (6LL * m + 64) - 64 - 512;
    long long SR = std::min<long long>(avail / (mp + 1), (ctx->T_local + 7) / 8);
    SR = std::max<long long>(SR & ~3LL, 4);  // whole 4-row DMMA k-steps
    const int stage_rows = (int)SR;
    const size_t setup_smem = gp_setup_smem_doubles(m, (int)ctx->ld, stage_rows) * sizeof(double);
    if (setup_smem > ctx->max_smem) return false;
    const void* cfn = reinterpret_cast<const void*>(&gram_pcg_cluster_kernel<2>);
    int CS = 0;
    for (int cs : {16, 8})
        if (!CS && cluster_fits(cfn, cs, kGpThreads, setup_smem)) CS = cs;
    if (!CS) return false;
    if (!ctx->gpcg) ctx->gpcg = new GramPcgWs();
    GramPcgWs& ws = *ctx->gpcg;
    const size_t ld = (size_t)ctx->ld;
    if (ws.cap_m < (size_t)kGpMaxM || ws.cap_ld < ld) gram_pcg_alloc(ctx, ws, ld);
    if (!ctx->pmat) {
        MVSK_CUDA(cudaMalloc(&ctx->pmat, ld * ld * sizeof(double)));
        ++ctx->epoch;
    }
    ensure_tvec2(ctx);
    const GpLayout L(m, mm, 0);
    double* hp = ws.h_par;
    std::copy(in.vU.begin(), in.vU.end(), hp + L.vU);
    std::copy(in.vQ.begin(), in.vQ.end(), hp + L.vQ);
    std::copy(in.nu.begin(), in.nu.end(), hp + L.nu);
    for (int i = 0; i < m; ++i) hp[L.idx + i] = (double)(fm.active ? fm.idx[(size_t)i] : i);
    GpParams P{};
    P.m = m;
    P.mm = mm;
    P.np = 0;
    P.has_third = in.has_third ? 1 : 0;
    P.face_active = fm.active ? 1 : 0;
    P.bU = in.bU;
    P.bQ = in.bQ;
    P.gn = in.gn;
    P.lambda = in.lambda;
    P.n_d = (double)m;
    P.store(hp);
    const Slot& sl = ctx->slots[slot];
    const int key = m * 64 + (in.has_third ? 1 : 0);
    run_graphed(ctx, kGraphGramDirect, key, slot, [&] {
        MVSK_CUDA(cudaMemcpyAsync(ws.par, ws.h_par, L.total * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        SetupArgs sa{};
        sa.par = ws.par;
        sa.ld = (int)ld;
        sa.Mg = ws.Mg;
        sa.vec = ws.vec;
        sa.res = ws.res;
        sa.pmat = in.has_third ? ctx->pmat : nullptr;
        GramArgsC ga{};
        ga.X = ctx->X;
        ga.T = ctx->T_local;
        ga.ld = (int)ld;
        ga.z = sl.z;
        ga.c2 = ctx->c.c2;
        ga.c3 = ctx->c.c3;
        ga.c4 = ctx->c.c4;
        ga.scale = 1.0 / (double)ctx->T_global;
        ga.Gout = nullptr;
        ga.stage_rows = stage_rows;
        set_smem_attr(cfn, setup_smem);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(CS);
        cfg.blockDim = dim3(kGpThreads);
        cfg.dynamicSmemBytes = setup_smem;
        cfg.stream = ctx->stream;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        void* cargs[] = {&ga, &sa};
        ++ctx->launches;
        MVSK_CUDA(cudaLaunchKernelExC(&cfg, cfn, cargs));
        ctx->phys += 1;
        const double* af = nullptr;
        if (in.has_third) {
            // q_t = a_t^T P a_t and tw_t = psi'''(z_t) q_t / T, then A^T tw (:174-177)
            run_quadform(ctx, ctx->pmat, ctx->tvec2, sl.z, ctx->tvec);
            PassIO io;
            io.tw = ctx->tvec;
            io.out = ctx->outd;
            io.ldo = (long long)ld;
            run_pass(ctx, Op::XTW, 1, io);
            af = ctx->outd;
        }
        MainArgs ma{};
        ma.par = ws.par;
        ma.ld = (int)ld;
        ma.Mg = ws.Mg;
        ma.vec = ws.vec;
        ma.res = ws.res;
        const size_t msm = (size_t)(3 * m + mm + 16) * sizeof(double);
        ++ctx->launches;
        gram_direct_main_kernel<<<1, kGpThreads, msm, ctx->stream>>>(ma, af);
        MVSK_CUDA(cudaGetLastError());
        MVSK_CUDA(cudaMemcpyAsync(ws.h_res, ws.res, (size_t)(64 + mm) * sizeof(double), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    });
    MVSK_CUDA(cudaStreamSynchronize(ctx->stream));
    u.assign(ws.h_res + 64, ws.h_res + 64 + mm);
    static const bool prof = std::getenv("MVSK_GPCG_PROF") != nullptr;
    if (prof) {
        const double* r = ws.h_res;
        std::fprintf(stderr,
                     "[gdirect] m=%d ld %lld T %lld spd %.0f (%.0f) cycles: gram %.0f reduce %.0f | h %.0f M %.0f inverse %.0f P %.0f | "
                     "gram: pre %.0f issue %.0f wait %.0f mma %.0f\n",
                     m, (long long)ctx->ld, (long long)ctx->T_local, r[56], r[57] - r[53], r[48], r[49], r[52], r[53] - r[52],
                     r[54] - r[53], r[55] - r[54], r[58], r[59], r[60], r[61]);
    }
    return true;
}

void gram_pcg_workspace_free(mvsk_gpu_ctx* ctx) {
    if (!ctx->gpcg) return;
    GramPcgWs& ws = *ctx->gpcg;
    for (double* p : {ws.par, ws.Mg, ws.vec, ws.vin1, ws.vin2, ws.t3, ws.res, ws.Gf})
        if (p) cudaFree(p);
    for (double* p : {ws.h_par, ws.h_res})
        if (p) cudaFreeHost(p);
    delete ctx->gpcg;
    ctx->gpcg = nullptr;
}

}  // namespace mvsk_b200
