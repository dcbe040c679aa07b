// Single-pass streaming kernels over the row-major sample panel X (T x ld fp64).
//
// One persistent CTA per SM (or several for small rows) owns a contiguous row
// block. Rows are staged global -> shared by the bulk-copy engine (TMA 1-D,
// mbarrier completion) into an S-deep ring; each staged row is read ONCE from
// shared memory into registers and serves both halves of the fused op:
//   phase 1  row dots  y_t = <x_t, v_k>         (warp shuffle + block combine)
//   phase 2  weights   w_t = phi^(j)(z_t) ...    (registers)
//   phase 3  X^T       acc_k += w_tk * x_t       (per-thread column registers)
// so f+grad, Hv, T3(u,v), the line-search power sums and X^T w all cost one
// HBM pass of X. Per-CTA partials are reduced by a second kernel in a fixed
// order (deterministic; no fp64 atomics).
//
// Thread layout: the CTA is G groups ("row teams") of P threads. Thread p of a
// team owns column pairs j = p + q*P, q < Q (double2 = 16 B smem reads,
// conflict-free); team g handles rows g, g+G, ... of each stage (RG rows).
//
// Reference: oracle.hpp:54-69 (make_cache), :79-90 (gradient), :92-101 (hvp),
// :103-113 (third_action), linesearch.hpp:22-44 (power_sums), oracle.hpp:137-140
// (transpose_apply).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include "ptx.cuh"

namespace mvsk_b200 {
namespace cg = cooperative_groups;

enum class Op : int { FGRAD = 0, HVP = 1, THIRD = 2, LINESUMS = 3, XTW = 4 };

constexpr int kMaxStages = 8;
constexpr int kNumScalars = 16;  // per-CTA scalar partial slots

}  // namespace mvsk_b200
#include "finish.cuh"
namespace mvsk_b200 {

struct StreamArgs {
    const double* X;   // T_local x ld, row-major, 16-B aligned rows (ld even)
    long long T;       // local rows
    int ld;            // padded row length (even)
    int npairs;        // ld / 2
    int P, G, RG, S;   // team size, teams per CTA, rows per team per stage, ring depth
    int evict_first;   // L2 policy for the streamed panel
    const double* vin;   // K input vectors, stride ld (FGRAD: x; HVP: V; THIRD: U; LINESUMS: d)
    const double* vin2;  // THIRD: V (stride ld)
    const double* z;     // cached z (HVP / THIRD / LINESUMS); FGRAD: z offset or null
    const double* tw;    // XTW: per-row weights
    double* zout;        // FGRAD: z out; LINESUMS: A d out (optional)
    double* part_acc;    // [gridDim][K][ld]
    double* part_sc;     // [gridDim][kNumScalars]
    double c2, c3, c4;
    double Tglob;        // global T (the reference divides by T = A.rows())
    const int* skip;     // optional: skip the pass when all nskip flags are 0
    int nskip;
    // cooperative launch only: after the partials, a grid-wide barrier and the
    // cross-CTA reduction + epilogue in the same kernel (no finish launch)
    int fused;
    int fin_ng, fin_nvb;
    FinishArgs fin;
};

// Device-side early exit for speculatively enqueued Krylov steps: the pass is a
// no-op when no CG column is still active (pcg_device.cu).
__device__ __forceinline__ bool pass_skipped(const int* skip, int nskip) {
    if (!skip) return false;
    int any = 0;
    for (int i = 0; i < nskip; ++i) any |= skip[i];
    return any == 0;
}

// number of dot products per row and accumulator sets per op
template <Op OP, int K>
struct OpShape {
    static constexpr int NDOT = (OP == Op::FGRAD || OP == Op::LINESUMS) ? 1
                                : (OP == Op::THIRD)                     ? 2 * K
                                : (OP == Op::XTW)                       ? 0
                                                                        : K;
    static constexpr int NACC = (OP == Op::LINESUMS) ? 0 : (OP == Op::HVP || OP == Op::THIRD) ? K : 1;
};

// fp64 values a thread keeps live across a stage: input vectors, accumulators
// and the staged row slice. Heavy variants are capped at 384 / 256 threads so
// they may use up to 168 / 255 registers; light ones allow 512 (128 registers).
// VS: the input vectors live in shared memory instead of registers (wide rows
// on short panels: the freed registers let two row teams share a CTA).
template <Op OP, int K, int Q, int RG, bool VS = false>
struct StreamRegs {
    static constexpr int NV = VS ? 0 : (OpShape<OP, K>::NDOT > 0 ? OpShape<OP, K>::NDOT : 1);
    static constexpr int NA = OpShape<OP, K>::NACC > 0 ? OpShape<OP, K>::NACC : 1;
    static constexpr int live = 2 * Q * (NV + NA + RG);
    static constexpr int max_threads = live <= 48 ? 512 : (live <= 64 ? 384 : 256);
};

template <Op OP, int K, int Q, int RG, bool VS = false>
__global__ void __launch_bounds__(StreamRegs<OP, K, Q, RG, VS>::max_threads, 1) stream_kernel(const StreamArgs a) {
    using Sh = OpShape<OP, K>;
    constexpr int NDOT = Sh::NDOT;
    constexpr int NACC = Sh::NACC;
    static_assert(!VS || NDOT > 0, "VS needs input vectors");
    constexpr int NV = (NDOT > 0 && !VS) ? NDOT : 1;
    constexpr int NA = NACC > 0 ? NACC : 1;
    constexpr int NDR = NDOT > 0 ? NDOT : 1;

    if (pass_skipped(a.skip, a.nskip)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int P = a.P, G = a.G, S = a.S;
    const int R = G * RG;  // rows per stage
    const int g = tid / P;
    const int p = tid - g * P;
    const int lane = tid & 31;
    const int nwp = P >= 32 ? P / 32 : 1;  // warps per team
    const int wg = P >= 32 ? p >> 5 : 0;   // warp index within team
    const long long ld = a.ld;

    // ---- shared memory carve: [mbar S][red 2 x R x NDR x nwp][VS: NDOT x ld][stages S x R x ld]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    double* red = reinterpret_cast<double*>(smem_raw + 128);
    const int red_elems = 2 * R * NDR * nwp;
    size_t off = 128 + (((size_t)red_elems * sizeof(double) + 127) & ~(size_t)127);
    double* vsm = reinterpret_cast<double*>(smem_raw + off);
    if constexpr (VS) off += ((size_t)NDOT * ld * sizeof(double) + 127) & ~(size_t)127;
    const size_t stage_bytes = ((size_t)R * ld * sizeof(double) + 127) & ~(size_t)127;
    unsigned char* stage_base = smem_raw + off;

    // ---- row range of this CTA
    const long long T = a.T;
    const long long r0 = T * blockIdx.x / gridDim.x;
    const long long r1 = T * (blockIdx.x + 1) / gridDim.x;
    const long long nrows = r1 - r0;
    const int nst = (int)((nrows + R - 1) / R);

    uint64_t policy = 0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    if constexpr (VS) {  // input vectors -> shared memory once (L2-resident, a few KB)
        for (int e = tid; e < NDOT * (int)a.npairs; e += (int)blockDim.x) {
            const int k = e / a.npairs, j = e - k * a.npairs;
            const double* src;
            if constexpr (OP == Op::THIRD)
                src = (k < K) ? a.vin + (long long)k * ld : a.vin2 + (long long)(k - K) * ld;
            else
                src = a.vin + (long long)k * ld;
            reinterpret_cast<double2*>(vsm + (long long)k * ld)[j] = reinterpret_cast<const double2*>(src)[j];
        }
    }
    __syncthreads();
    if (tid == 0) {
        policy = a.evict_first ? policy_evict_first() : policy_evict_last();
        const int pre = nst < S ? nst : S;
        for (int s = 0; s < pre; ++s) {
            const long long rows = (nrows - (long long)s * R) < R ? (nrows - (long long)s * R) : R;
            const uint32_t bytes = (uint32_t)(rows * ld * sizeof(double));
            mbar_arrive_expect_tx(&full[s], bytes);
            bulk_g2s(stage_base + s * stage_bytes, a.X + (r0 + (long long)s * R) * ld, bytes, &full[s], policy);
        }
    }

    // ---- per-thread input vectors (registers) and accumulators
    double2 vreg[NV][Q];
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int j = p + q * P;
            double2 v = make_double2(0.0, 0.0);
            if constexpr (NDOT > 0 && !VS) {
                if (j < a.npairs) {
                    const double* src;
                    if constexpr (OP == Op::THIRD)
                        src = (k < K) ? a.vin + (long long)k * ld : a.vin2 + (long long)(k - K) * ld;
                    else
                        src = a.vin + (long long)k * ld;
                    v = reinterpret_cast<const double2*>(src)[j];
                }
            }
            vreg[k][q] = v;
        }
    double2 acc[NA][Q];
#pragma unroll
    for (int k = 0; k < NA; ++k)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[k][q] = make_double2(0.0, 0.0);

    double sc[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) sc[i] = 0.0;

    const double c2 = a.c2, c3 = a.c3, c4 = a.c4;

    // per-row sample inputs (z, z offset or X^T weights) are prefetched one
    // stage ahead so their global-load latency never sits on the row's path
    constexpr bool NEEDS_ROWVAL = (OP != Op::FGRAD);
    const double* rowval = (OP == Op::XTW) ? a.tw : a.z;
    double znext[RG];
    auto load_rowvals = [&](int s_, double (&dst)[RG]) {
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) {
            const long long r = (long long)s_ * R + g + rr * G;
            dst[rr] = (rowval && s_ < nst && r < nrows) ? __ldg(rowval + r0 + r) : 0.0;
        }
    };
    if (NEEDS_ROWVAL || a.z) load_rowvals(0, znext);

    for (int s = 0; s < nst; ++s) {
        const int slot = s % S;
        const uint32_t parity = (uint32_t)((s / S) & 1);
        const long long srow0 = r0 + (long long)s * R;
        const long long left = r1 - srow0;
        const int rows_here = left < R ? (int)left : R;
        double zcur[RG];
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) zcur[rr] = znext[rr];
        if (NEEDS_ROWVAL || a.z) load_rowvals(s + 1, znext);
        mbar_wait(&full[slot], parity);
        const double* st = reinterpret_cast<const double*>(stage_base + slot * stage_bytes);

        // phase 0: this thread's slice of its team's rows -> registers
        double2 x[RG][Q];
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) {
            const int r = g + rr * G;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int j = p + q * P;
                double2 v = make_double2(0.0, 0.0);
                if (r < rows_here && j < a.npairs) v = reinterpret_cast<const double2*>(st + (long long)r * ld)[j];
                x[rr][q] = v;
            }
        }

        // phase 1: row dots
        double dot[RG][NDR];
#pragma unroll
        for (int rr = 0; rr < RG; ++rr)
#pragma unroll
            for (int k = 0; k < NDR; ++k) {
                double d0 = 0.0, d1 = 0.0;  // two independent FMA chains
                if constexpr (NDOT > 0) {
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        double2 vv;
                        if constexpr (VS) {
                            const int j = p + q * P;
                            vv = j < a.npairs ? reinterpret_cast<const double2*>(vsm + (long long)k * ld)[j]
                                              : make_double2(0.0, 0.0);
                        } else {
                            vv = vreg[k][q];
                        }
                        d0 = fma(x[rr][q].x, vv.x, d0);
                        d1 = fma(x[rr][q].y, vv.y, d1);
                    }
                }
                dot[rr][k] = d0 + d1;
            }
        if constexpr (NDOT > 0) {
            if (P >= 32) {
                // full-warp butterfly, unrolled so the RG x NDOT chains interleave
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
                    for (int rr = 0; rr < RG; ++rr)
#pragma unroll
                        for (int k = 0; k < NDOT; ++k) dot[rr][k] += __shfl_xor_sync(0xffffffffu, dot[rr][k], o);
            } else {
#pragma unroll
                for (int rr = 0; rr < RG; ++rr)
#pragma unroll
                    for (int k = 0; k < NDOT; ++k) {
                        double d = dot[rr][k];
                        for (int o = P >> 1; o >= 1; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o, P);
                        dot[rr][k] = d;
                    }
            }
            if (P > 32 && lane == 0) {
                double* rb = red + (size_t)(s & 1) * R * NDOT * nwp;
#pragma unroll
                for (int rr = 0; rr < RG; ++rr)
#pragma unroll
                    for (int k = 0; k < NDOT; ++k) rb[((g * RG + rr) * NDOT + k) * nwp + wg] = dot[rr][k];
            }
        }
        // every thread has pulled its stage slice into registers and published
        // its warp partials: the slot can be refilled and partials combined
        __syncthreads();
        if (tid == 0 && s + S < nst) {
            const long long s2 = s + S;
            const long long rows = (nrows - s2 * R) < R ? (nrows - s2 * R) : R;
            const uint32_t bytes = (uint32_t)(rows * ld * sizeof(double));
            mbar_arrive_expect_tx(&full[slot], bytes);
            bulk_g2s(stage_base + slot * stage_bytes, a.X + (r0 + s2 * R) * ld, bytes, &full[slot], policy);
        }
        if constexpr (NDOT > 0) {
            if (P > 32) {
                const double* rb = red + (size_t)(s & 1) * R * NDOT * nwp;
#pragma unroll
                for (int rr = 0; rr < RG; ++rr)
#pragma unroll
                    for (int k = 0; k < NDOT; ++k) {
                        // fixed-order pairwise combine of the team's warp partials
                        // (two independent chains instead of one serial one)
                        const double* src = rb + ((g * RG + rr) * NDOT + k) * nwp;
                        double d0 = 0.0, d1 = 0.0;
                        int w = 0;
                        for (; w + 1 < nwp; w += 2) {
                            d0 += src[w];
                            d1 += src[w + 1];
                        }
                        if (w < nwp) d0 += src[w];
                        dot[rr][k] = d0 + d1;
                    }
            }
        }

        // phase 2 + 3: per-row weights, then X^T accumulation from registers
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) {
            const int r = g + rr * G;
            const bool valid = r < rows_here;
            const long long t = srow0 + r;
            double w[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k) w[k] = 0.0;
            if (valid) {
                if constexpr (OP == Op::FGRAD) {
                    // oracle.hpp:58-64, 82-83
                    double zt = dot[rr][0];
                    if (a.z) zt += zcur[rr];
                    const double z2 = zt * zt;
                    const double z3 = z2 * zt;
                    w[0] = 2.0 * c2 * zt - 3.0 * c3 * z2 + 4.0 * c4 * z3;  // 1/T applied in the epilogue
                    if (p == 0) {
                        sc[0] += z2;
                        sc[1] += z3;
                        sc[2] += z2 * z2;
                        a.zout[t] = zt;
                    }
                } else if constexpr (OP == Op::HVP) {
                    // oracle.hpp:95-96
                    const double zt = zcur[rr];
                    const double psi2 = 2.0 * c2 - 6.0 * c3 * zt + 12.0 * c4 * (zt * zt);
#pragma unroll
                    for (int k = 0; k < K; ++k) w[k] = psi2 * dot[rr][k];
                } else if constexpr (OP == Op::THIRD) {
                    // oracle.hpp:107-108
                    const double zt = zcur[rr];
                    const double psi3 = -6.0 * c3 + 24.0 * c4 * zt;
#pragma unroll
                    for (int k = 0; k < K; ++k) w[k] = psi3 * dot[rr][k] * dot[rr][K + k];
                } else if constexpr (OP == Op::LINESUMS) {
                    // linesearch.hpp:26-38
                    if (p == 0) {
                        const double zt = zcur[rr], wt = dot[rr][0];
                        const double w2 = wt * wt, z2 = zt * zt;
                        sc[0] += zt * wt;
                        sc[1] += z2 * wt;
                        sc[2] += z2 * zt * wt;
                        sc[3] += w2;
                        sc[4] += zt * w2;
                        sc[5] += z2 * w2;
                        sc[6] += w2 * wt;
                        sc[7] += zt * w2 * wt;
                        sc[8] += w2 * w2;
                        if (a.zout) a.zout[t] = wt;
                    }
                } else {  // XTW
                    w[0] = zcur[rr];
                }
            }
            if constexpr (NACC > 0) {
#pragma unroll
                for (int k = 0; k < NACC; ++k)
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        acc[k][q].x = fma(w[k], x[rr][q].x, acc[k][q].x);
                        acc[k][q].y = fma(w[k], x[rr][q].y, acc[k][q].y);
                    }
            }
        }
    }

    // ---- CTA epilogue: combine teams (fixed order) and publish partials
    __syncthreads();  // all stages consumed; smem ring is free
    double* cmb = reinterpret_cast<double*>(stage_base);
    if constexpr (NACC > 0) {
        if (G == 1) {
#pragma unroll
            for (int k = 0; k < NACC; ++k)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const int j = p + q * P;
                    if (j < a.npairs)
                        reinterpret_cast<double2*>(a.part_acc + ((size_t)blockIdx.x * NACC + k) * ld)[j] = acc[k][q];
                }
        } else {
            // teams write [g][k][ld] into the free ring, then reduce over g
#pragma unroll
            for (int k = 0; k < NACC; ++k)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const int j = p + q * P;
                    if (j < a.npairs) reinterpret_cast<double2*>(cmb + ((size_t)g * NACC + k) * ld)[j] = acc[k][q];
                }
            __syncthreads();
            const int tot = NACC * a.ld;
            for (int i = tid; i < tot; i += blockDim.x) {
                double v = 0.0;
                for (int gg = 0; gg < G; ++gg) v += cmb[(size_t)gg * tot + i];
                a.part_acc[(size_t)blockIdx.x * tot + i] = v;
            }
        }
    }
    if constexpr (OP == Op::FGRAD || OP == Op::LINESUMS) {
        constexpr int NS = (OP == Op::FGRAD) ? 3 : 9;
        __syncthreads();
        double* scb = cmb + (size_t)G * NA * ld + 16;  // past the team buffer
        if (p == 0)
#pragma unroll
            for (int i = 0; i < NS; ++i) scb[g * NS + i] = sc[i];
        __syncthreads();
        for (int i = tid; i < NS; i += blockDim.x) {  // tiny CTAs may have < NS threads
            double v = 0.0;
            for (int gg = 0; gg < G; ++gg) v += scb[gg * NS + i];
            a.part_sc[(size_t)blockIdx.x * kNumScalars + i] = v;
        }
    }
    if (a.fused) {
        // every CTA's partials are in global memory before any CTA reduces them
        __threadfence();
        cg::this_grid().sync();
        double* part = reinterpret_cast<double*>(stage_base);  // the ring is free
        for (int vb = blockIdx.x; vb < a.fin_nvb; vb += gridDim.x)
            finish_block(a.fin, a.fin_ng, vb, tid, (int)blockDim.x, part);
    }
}

}  // namespace mvsk_b200
