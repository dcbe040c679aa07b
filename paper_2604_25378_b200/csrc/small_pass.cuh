// One-launch oracle passes for short, narrow panels (ld <= 128, a few thousand
// rows: the C1 / C2 panels and the compact faces of C3 / C4): ONE cluster of
// kSpCS CTAs holds the whole panel in shared memory for the duration of the
// pass, so the pass is a single launch with no grid barrier and no partials
// round trip through global memory:
//
//   load      each CTA stages its contiguous row block with one bulk copy per
//             row (mbarrier completion) and its per-row sample inputs (z, the
//             FGRAD z offset, the X^T weights) with plain loads, in parallel
//   rows      LPR lanes per row, CPL columns per lane (column pairs interleaved
//             across the LPR lanes: conflict-free 16-B shared reads); the row
//             dot(s), the op's per-row weight and the X^T accumulation in
//             registers, exactly the arithmetic of stream_kernel
//   combine   lanes -> warp (shuffles), warps -> CTA (fixed order in shared
//             memory), CTAs -> result over DSMEM in cluster-rank order; each
//             CTA finishes a slice of the columns and CTA 0 the scalars, with
//             the epilogues of finish_block (finish.cuh)
//
// The streaming kernel needs ~9 us for a C1 f+grad pass (32 CTAs stepping
// through 16 rows each, a grid barrier, then the partials reduction); here the
// critical path is one bulk load, ~nloc / 32 row steps and one cluster barrier.
// Reference: oracle.hpp:54-69 (make_cache), :79-90 (gradient), :92-101 (hvp),
// :103-113 (third_action), linesearch.hpp:22-44 (power_sums), oracle.hpp:137-140.
#pragma once
#include <cooperative_groups.h>

#include "finish.cuh"
#include "ptx.cuh"
#include "stream_kernels.cuh"

namespace mvsk_b200 {

constexpr int kSpCS = 16;           // CTAs per cluster (non-portable size)
constexpr int kSpW = 8;             // warps per CTA
constexpr int kSpM = 128;           // max ld
constexpr int kSpMP = kSpM + 12;    // a partial row: ld accumulator entries + 9 scalars (+ pad)

struct SmallPassArgs {
    const double* X;
    long long T;       // local rows
    int ld;
    const double* vin;   // FGRAD x, HVP v, THIRD u, LINESUMS d
    const double* vin2;  // THIRD v
    const double* rowv;  // FGRAD z offset (or null), HVP / THIRD / LINESUMS z, XTW weights
    double* zout;        // FGRAD z, LINESUMS A d (optional)
    FinishArgs fin;      // epilogue targets and constants (k = 1)
    unsigned long long* prof;  // MVSK_SMALL_PROF: CTA 0 phase cycle sums [load, rows, combine, epilogue, n]
};

__host__ __device__ constexpr size_t small_pass_smem(long long nloc, int ld) {
    return ((size_t)(kSpW + 1) * kSpMP + (size_t)nloc * (ld + 2) + (size_t)((nloc + 1) / 2 * 2)) * sizeof(double);
}

template <Op OP, int LPR, int CPL>
__global__ void __launch_bounds__(kSpW * 32, 1) small_pass_kernel(const SmallPassArgs a) {
    namespace cgs = cooperative_groups;
    static_assert(LPR * CPL <= kSpM && CPL % 2 == 0 && 32 % LPR == 0, "row layout");
    constexpr int NDOT = OP == Op::THIRD ? 2 : (OP == Op::XTW ? 0 : 1);
    constexpr int NS = OP == Op::FGRAD ? 3 : (OP == Op::LINESUMS ? 9 : 0);
    constexpr bool ACC = OP != Op::LINESUMS;
    constexpr int M = kSpM, MP = kSpMP, CS = kSpCS, GPW = 32 / LPR, NGC = kSpW * GPW;
    const FinishArgs& f = a.fin;
    if (pass_skipped(f.skip, f.nskip)) return;  // uniform over the cluster
    const bool prof = a.prof && threadIdx.x == 0 && blockIdx.x == 0;
    unsigned long long tp = prof ? clock64() : 0;
    auto mark = [&](int i) {
        if (prof) {
            const unsigned long long now = clock64();
            atomicAdd(a.prof + i, now - tp);
            tp = now;
        }
    };
    cgs::cluster_group cluster = cgs::this_cluster();
    const int crank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ld = a.ld, lds = ld + 2;
    extern __shared__ __align__(16) double sp[];
    double* sW = sp;                // [kSpW][MP] warp partials
    double* buf = sW + kSpW * MP;   // [MP] this CTA's partial, read by the cluster
    double* sX = buf + MP;          // [nloc][lds] staged rows
    const long long r0 = a.T * crank / CS, r1 = a.T * (crank + 1) / CS;
    const int nloc = (int)(r1 - r0);
    double* sZ = sX + (size_t)nloc * lds;  // [nloc] per-row inputs
    __shared__ uint64_t bar;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        if (nloc > 0) mbar_arrive_expect_tx(&bar, (uint32_t)((size_t)nloc * ld * sizeof(double)));
    }
    __syncthreads();
    {
        const uint64_t pol = policy_evict_last();
        for (int r = tid; r < nloc; r += blockDim.x)
            bulk_g2s(sX + (size_t)r * lds, a.X + (r0 + r) * (long long)ld, (uint32_t)(ld * sizeof(double)), &bar, pol);
    }
    constexpr bool ROWV = OP != Op::FGRAD;  // FGRAD: only the optional z offset
    if (ROWV || a.rowv)
        for (int r = tid; r < nloc; r += blockDim.x) sZ[r] = __ldg(a.rowv + r0 + r);

    const int sub = lane % LPR;
    auto colp = [&](int j) { return 2 * ((j >> 1) * LPR + sub) + (j & 1); };
    double v1[NDOT > 0 ? CPL : 1], v2[NDOT > 1 ? CPL : 1];
    if constexpr (NDOT > 0) {
#pragma unroll
        for (int j = 0; j < CPL; j += 2) {
            double2 v = make_double2(0.0, 0.0), w = make_double2(0.0, 0.0);
            if (colp(j) < ld) {
                v = *reinterpret_cast<const double2*>(a.vin + colp(j));
                if constexpr (NDOT > 1) w = *reinterpret_cast<const double2*>(a.vin2 + colp(j));
            }
            v1[j] = v.x;
            v1[j + 1] = v.y;
            if constexpr (NDOT > 1) {
                v2[j] = w.x;
                v2[j + 1] = w.y;
            }
        }
    }
    double acc[ACC ? CPL : 1];
#pragma unroll
    for (int j = 0; j < (ACC ? CPL : 1); ++j) acc[j] = 0.0;
    double s[NS > 0 ? NS : 1];
#pragma unroll
    for (int i = 0; i < (NS > 0 ? NS : 1); ++i) s[i] = 0.0;
    const double c2 = f.c2, c3 = f.c3, c4 = f.c4;
    if (nloc > 0) mbar_wait(&bar, 0u);
    __syncthreads();  // sZ
    mark(0);

    for (int lb = warp * GPW; lb < nloc; lb += NGC) {  // warp-uniform trip count
        const int tl = lb + lane / LPR;
        const bool rv = tl < nloc;
        const double* xr = sX + (size_t)(rv ? tl : 0) * lds;
        double x[CPL];
#pragma unroll
        for (int j = 0; j < CPL; j += 2) {
            double2 v = make_double2(0.0, 0.0);
            if (rv && colp(j) < ld) v = *reinterpret_cast<const double2*>(xr + colp(j));
            x[j] = v.x;
            x[j + 1] = v.y;
        }
        double d = 0.0, e = 0.0;
        if constexpr (NDOT > 0) {
            double d0 = 0.0, d1 = 0.0;  // two independent FMA chains, as stream_kernel
#pragma unroll
            for (int j = 0; j < CPL; j += 2) {
                d0 = fma(x[j], v1[j], d0);
                d1 = fma(x[j + 1], v1[j + 1], d1);
            }
            d = d0 + d1;
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        }
        if constexpr (NDOT > 1) {
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int j = 0; j < CPL; j += 2) {
                d0 = fma(x[j], v2[j], d0);
                d1 = fma(x[j + 1], v2[j + 1], d1);
            }
            e = d0 + d1;
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        }
        const double zr = rv && (ROWV || a.rowv) ? sZ[tl] : 0.0;
        const long long t = r0 + tl;
        double w = 0.0;
        if constexpr (OP == Op::FGRAD) {  // oracle.hpp:58-64, 82-83
            const double zt = a.rowv ? d + zr : d;
            const double z2 = zt * zt, z3 = z2 * zt;
            w = 2.0 * c2 * zt - 3.0 * c3 * z2 + 4.0 * c4 * z3;  // 1/T in the epilogue
            if (rv && sub == 0) {
                s[0] += z2;
                s[1] += z3;
                s[2] += z2 * z2;
                a.zout[t] = zt;
            }
        } else if constexpr (OP == Op::HVP) {  // oracle.hpp:95-96
            const double psi2 = 2.0 * c2 - 6.0 * c3 * zr + 12.0 * c4 * (zr * zr);
            w = psi2 * d;
        } else if constexpr (OP == Op::THIRD) {  // oracle.hpp:107-108
            const double psi3 = -6.0 * c3 + 24.0 * c4 * zr;
            w = psi3 * d * e;
        } else if constexpr (OP == Op::LINESUMS) {  // linesearch.hpp:26-38
            if (rv && sub == 0) {
                const double zt = zr, wt = d;
                const double w2 = wt * wt, z2 = zt * zt;
                s[0] += zt * wt;
                s[1] += z2 * wt;
                s[2] += z2 * zt * wt;
                s[3] += w2;
                s[4] += zt * w2;
                s[5] += z2 * w2;
                s[6] += w2 * wt;
                s[7] += zt * w2 * wt;
                s[8] += w2 * w2;
                if (a.zout) a.zout[t] = wt;
            }
        } else {  // XTW
            w = zr;
        }
        if constexpr (ACC) {
            if (!rv) w = 0.0;
#pragma unroll
            for (int j = 0; j < CPL; ++j) acc[j] = fma(x[j], w, acc[j]);
        }
    }
    // lanes of one column slice -> lane sub (fixed butterfly order)
    if constexpr (ACC) {
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
            for (int j = 0; j < CPL; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
        if (lane < LPR) {
#pragma unroll
            for (int j = 0; j < CPL; ++j)
                if (colp(j) < ld) sW[warp * MP + colp(j)] = acc[j];
        }
    }
    if constexpr (NS > 0) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
#pragma unroll
            for (int i = 0; i < NS; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
        if (lane == 0)
#pragma unroll
            for (int i = 0; i < NS; ++i) sW[warp * MP + M + i] = s[i];
    }
    __syncthreads();
    mark(1);
    for (int el = tid; el < MP; el += blockDim.x) {  // warps in a fixed order
        if ((el >= ld && el < M) || (el >= M + NS) || (!ACC && el < M)) continue;
        double v = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kSpW; ++w2) v += sW[w2 * MP + el];
        buf[el] = v;
    }
    cluster.sync();
    mark(2);
    // ---- columns: CTA c finishes the slice [c * chunk, (c + 1) * chunk)
    if constexpr (ACC) {
        const int chunk = (ld + CS - 1) / CS;
        const int el = crank * chunk + tid;
        if (tid < chunk && el < ld) {
            double pv[CS];
#pragma unroll
            for (int r = 0; r < CS; ++r) pv[r] = cluster.map_shared_rank(buf, r)[el];
            double v = 0.0;
#pragma unroll
            for (int r = 0; r < CS; ++r) v += pv[r];  // cluster-rank order
            if (!f.do_epi) {  // row-sharded: the raw sums go to the allreduce, then finish_kernel
                f.red[el] = v;
            } else if constexpr (OP == Op::FGRAD) {  // oracle.hpp:82-84
                const double gi = el < f.n ? (-f.c1 * f.mu[el] + v / f.T) : 0.0;
                f.g[el] = gi;
                if (f.hout) f.hout[8 + el] = gi;
            } else if (el < f.n) {
                const double o = OP == Op::XTW ? v : v / f.T;  // HVP / THIRD: the 1/T folded out of the weights
                f.out[el] = o;
                if (f.hout) f.hout[el] = o;
            }
        }
    }
    // ---- scalars on CTA 0
    if constexpr (NS > 0) {
        double mux = 0.0;
        if constexpr (OP == Op::FGRAD) {
            // mu'x in finish_block's order (one element per thread, warp
            // butterflies, warps in order), so the in-kernel epilogue and the
            // row-sharded finish_kernel epilogue agree bit for bit
            if (crank == 0 && f.do_epi) {
                double sacc = 0.0;
                for (int j = tid; j < f.n; j += blockDim.x) sacc += f.mu[j] * f.x[j];
#pragma unroll
                for (int o = 16; o; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
                if (lane == 0) sW[warp] = sacc;  // sW is free after the cluster barrier
                __syncthreads();
                for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) mux += sW[w2];
            }
        }
        if (crank == 0 && warp == 0) {
            double sv = 0.0;
            if (lane < NS) {
                double pv[CS];
#pragma unroll
                for (int r = 0; r < CS; ++r) pv[r] = cluster.map_shared_rank(buf, r)[M + lane];
#pragma unroll
                for (int r = 0; r < CS; ++r) sv += pv[r];
            }
            if (!f.do_epi) {
                if (lane < NS) f.red[(ACC ? ld : 0) + lane] = sv;
            } else if constexpr (OP == Op::FGRAD) {  // oracle.hpp:62-64
                const double s2 = __shfl_sync(0xffffffffu, sv, 0), s3 = __shfl_sync(0xffffffffu, sv, 1),
                             s4 = __shfl_sync(0xffffffffu, sv, 2);
                if (lane == 0) {
                    const double vo = f.value_offset_dev ? *f.value_offset_dev : f.value_offset;
                    double o5[5];
                    o5[0] = vo - f.c1 * mux + (f.c2 * s2 - f.c3 * s3 + f.c4 * s4) / f.T;
                    o5[1] = mux;
                    o5[2] = s2 / f.T;
                    o5[3] = s3 / f.T;
                    o5[4] = s4 / f.T;
                    for (int q = 0; q < 5; ++q) {
                        f.sc[q] = o5[q];
                        if (f.hout) f.hout[q] = o5[q];
                    }
                }
            } else if (lane < NS) {  // LINESUMS
                const double o = sv / f.T;
                f.out[lane] = o;
                if (f.hout) f.hout[lane] = o;
            }
        }
    }
    // (no system fence for hout: kernel completion orders the mapped writes
    // before the stream synchronisation the host waits on)
    mark(3);
    cluster.sync();  // no CTA leaves while its partial may still be read
    mark(4);
    if (prof) atomicAdd(a.prof + 5, 1ull);
}

}  // namespace mvsk_b200

namespace mvsk_b200 {

// ---- the direct branch's weighted Gram G = X^T diag(psi''(z)) X / T for the
// same short narrow panels (affine_normal.hpp:151-170 assemble it from n + 1
// passes; here one launch): the panel rows staged in the cluster's shared
// memory as above, 8 x 8 lower-triangle output tiles as mma.m8n8k4 f64 over
// 4-row k-steps (warp w owns tiles w, w + 8, ..., with enough interleaved
// accumulators per tile for ~8 independent chains: the accumulate chain is
// long-latency), the CTA partial tiles summed over DSMEM in cluster-rank
// order, G written mirrored to device memory and to the mapped host buffer.
constexpr int kSgW = 8;  // warps per CTA

__host__ __device__ constexpr int small_gram_stride(int ld) {  // 4 (mod 16) doubles: conflict-free fragments
    return ((ld + 7) & ~7) + ((((ld + 7) & ~7) % 16 == 0) ? 4 : 12);
}
__host__ __device__ constexpr size_t small_gram_smem(long long nloc, int ld) {
    const long long nt = (ld + 7) / 8;
    return ((size_t)((nloc + 3) & ~3LL) * (small_gram_stride(ld) + 1) + (size_t)(nt * (nt + 1) / 2) * 64) * sizeof(double);
}

struct SmallGramArgs {
    const double* X;
    long long T;
    int ld, n;
    const double* z;
    double c2, c3, c4, scale;
    double* G;   // n x n device
    double* Gh;  // n x n mapped host mirror (or null)
    double* packed;  // row-sharded: the lower triangle packed (n (n + 1) / 2) for the allreduce, instead of G
    unsigned long long* prof;  // MVSK_SMALL_PROF: CTA 0 phase cycle sums [load, tiles, reduce, exit, -, n]
};

__device__ __forceinline__ void sg_dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

template <int TW, int U>
__device__ __forceinline__ void small_gram_tiles(const double* xs, const double* ws, int ms, int rows4, int ntiles,
                                                 double* tb) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[TW][U][2];
    int tI[TW], tJ[TW];
#pragma unroll
    for (int q = 0; q < TW; ++q) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc[q][u][0] = acc[q][u][1] = 0.0;
        const int tl = warp + q * kSgW;
        int r = 0, e = tl;
        while (e > r) {
            e -= r + 1;
            ++r;
        }
        // slots past the last tile redo tile 0 (discarded): the k-loop stays
        // branch-free, so the warp issues its DMMAs back to back
        tI[q] = tl < ntiles ? r : 0;
        tJ[q] = tl < ntiles ? e : 0;
    }
    const int kr = lane & 3, kc = lane >> 2;
    for (int t0 = 0; t0 < rows4; t0 += 4 * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int tk = t0 + 4 * u;
            if (tk >= rows4) break;
            const double* xr = xs + (size_t)(tk + kr) * ms + kc;
            const double wt = ws[tk + kr];
#pragma unroll
            for (int q = 0; q < TW; ++q) {
                const double b = xr[8 * tJ[q]];
                const double a = xr[8 * tI[q]] * wt;
                sg_dmma(acc[q][u], a, b);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < TW; ++q) {
        const int tl = warp + q * kSgW;
        if (tl >= ntiles) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double v = acc[q][0][h];
#pragma unroll
            for (int u = 1; u < U; ++u) v += acc[q][u][h];
            tb[(size_t)tl * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + h] = v;
        }
    }
}

__global__ void __launch_bounds__(kSgW * 32, 1) small_gram_kernel(const SmallGramArgs a) {
    namespace cgs = cooperative_groups;
    cgs::cluster_group cluster = cgs::this_cluster();
    const int crank = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
    const int tid = threadIdx.x;
    const int ld = a.ld, ms = small_gram_stride(ld);
    const int nt = (a.n + 7) / 8, ntiles = nt * (nt + 1) / 2;
    const bool prof = a.prof && tid == 0 && blockIdx.x == 0;
    unsigned long long tp = prof ? clock64() : 0;
    auto mark = [&](int i) {
        if (prof) {
            const unsigned long long now = clock64();
            atomicAdd(a.prof + i, now - tp);
            tp = now;
        }
    };
    extern __shared__ __align__(16) double sg[];
    const long long r0 = a.T * crank / CS, r1 = a.T * (crank + 1) / CS;
    const int nloc = (int)(r1 - r0), rows4 = (nloc + 3) & ~3;
    // tb first: the cluster reads it by offset, which must not depend on this
    // CTA's row count
    double* tb = sg;                           // [ntiles][64] this CTA's tiles
    double* xs = tb + (size_t)ntiles * 64;     // [rows4][ms]
    double* ws = xs + (size_t)rows4 * ms;      // [rows4]
    __shared__ uint64_t bar;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        if (nloc > 0) mbar_arrive_expect_tx(&bar, (uint32_t)((size_t)nloc * ld * sizeof(double)));
    }
    __syncthreads();
    for (int r = tid; r < nloc; r += blockDim.x)
        bulk_g2s(xs + (size_t)r * ms, a.X + (r0 + r) * (long long)ld, (uint32_t)(ld * sizeof(double)), &bar,
                 policy_evict_last());
    for (int e = tid; e < rows4 * ms; e += blockDim.x) {  // pad columns and pad rows
        const int t = e / ms, j = e - t * ms;
        if (t >= nloc || j >= ld) xs[e] = 0.0;
    }
    for (int t = tid; t < rows4; t += blockDim.x) {  // oracle.hpp:116-119
        const double zt = t < nloc ? __ldg(a.z + r0 + t) : 0.0;
        ws[t] = t < nloc ? 2.0 * a.c2 - 6.0 * a.c3 * zt + 12.0 * a.c4 * (zt * zt) : 0.0;
    }
    if (nloc > 0) mbar_wait(&bar, 0u);
    __syncthreads();
    mark(0);
    const int tpw = (ntiles + kSgW - 1) / kSgW;
    // several independent accumulate chains per warp (the DMMA accumulate
    // latency is several hundred cycles); past ~12 chains the fragment loads
    // (2 LDS.64 per DMMA) and the register file bound it instead (C2: 12
    // tiles x 1 chain 13.4k cycles, 12 x 2 14.8k)
    if (tpw <= 1)
        small_gram_tiles<1, 16>(xs, ws, ms, rows4, ntiles, tb);
    else if (tpw <= 2)
        small_gram_tiles<2, 12>(xs, ws, ms, rows4, ntiles, tb);
    else if (tpw <= 4)
        small_gram_tiles<4, 6>(xs, ws, ms, rows4, ntiles, tb);
    else if (tpw <= 6)
        small_gram_tiles<6, 4>(xs, ws, ms, rows4, ntiles, tb);
    else if (tpw <= 8)
        small_gram_tiles<8, 2>(xs, ws, ms, rows4, ntiles, tb);
    else if (tpw <= 12)
        small_gram_tiles<12, 1>(xs, ws, ms, rows4, ntiles, tb);
    else
        small_gram_tiles<17, 1>(xs, ws, ms, rows4, ntiles, tb);  // n <= 128: 136 tiles
    __syncthreads();
    mark(1);
    cluster.sync();
    // tile entries split over the cluster; each summed over the CTAs in rank order
    const int tot = ntiles * 64;
    for (int e = crank * (int)blockDim.x + tid; e < tot; e += CS * (int)blockDim.x) {
        const int tl = e >> 6, w = e & 63;
        int ti = 0, tj = tl;
        while (tj > ti) {
            tj -= ti + 1;
            ++ti;
        }
        const int i = 8 * ti + (w >> 3), j = 8 * tj + (w & 7);
        if (i >= a.n || j > i) continue;
        double pv[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) pv[r] = r < CS ? cluster.map_shared_rank(tb, r)[e] : 0.0;
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < 16; ++r)
            if (r < CS) v += pv[r];
        v *= a.scale;
        if (a.packed) {
            a.packed[(size_t)i * (i + 1) / 2 + j] = v;
            continue;
        }
        a.G[(size_t)i * a.n + j] = v;
        a.G[(size_t)j * a.n + i] = v;
        if (a.Gh) {
            a.Gh[(size_t)i * a.n + j] = v;
            a.Gh[(size_t)j * a.n + i] = v;
        }
    }
    mark(2);
    cluster.sync();
    mark(3);
    if (prof) atomicAdd(a.prof + 5, 1ull);
}

}  // namespace mvsk_b200
