// Multi-RHS fused passes with a thread-block-cluster column split.
//
// For k right-hand sides the per-thread state (k inputs + k accumulators per
// owned column) does not fit one SM's registers at n ~ 4096. A cluster of C
// CTAs (on C SMs) therefore splits every row by columns: CTA r owns columns
// [r*cw, (r+1)*cw), stages only its segment of each row (1-D bulk copies, one
// per row), computes partial row dots for all k vectors, and exchanges the C
// partial dots of a stage through distributed shared memory. X is still read
// from HBM exactly once.
//
// Exchange protocol (no per-stage cluster barrier — v1's barrier.cluster +
// MEMBAR.GPU was 34 % of stall samples, profiles/r01_ncu_cluster_v1.txt):
//   * CTA r pushes its V partials of stage s into slot e = s % E of every peer
//     with st.async ... mbarrier::complete_tx (8 bytes each, landing on the
//     peer's xfull[e]);
//   * a consumer arms xfull[e] with expect_tx(C*V*8), waits, and sums the C
//     partials in rank order (identical bits in every CTA);
//   * slot reuse is ordered by the pipeline itself (E = 4 >= pipeline depth
//     + 2), so no release handshake / cluster-scope fence is needed (a remote
//     mbarrier.arrive.release cost 28 % of stall samples in the first try).
// The exchange of stage s is software-pipelined behind the row dots of stage
// s+1 (two register copies of the staged row slice).
//
//   HVP  (K rhs):    w_tk = psi''(z_t) <x_t, v_k>                   (oracle.hpp:92-101)
//   THIRD (K pairs): w_tk = psi'''(z_t) <x_t, u_k> <x_t, v_k>        (oracle.hpp:103-113)
// The warp-level reduction of the RG*NDOT partial dots is a butterfly
// reduce-scatter (31 shuffles for 32 values instead of 160).
#pragma once
#include <cooperative_groups.h>

#include "stream_kernels.cuh"

namespace mvsk_b200 {

namespace cg = cooperative_groups;

constexpr int kXSlots = 4;  // exchange ring depth E

struct ClusterArgs {
    const double* X;  // T_local x ld
    long long T;
    int ld;
    int cw;           // columns per CTA (even)
    int P;            // threads per CTA
    int S;            // TMA ring depth
    int evict_first;
    const double* vin;   // K vectors (stride ld)
    const double* vin2;  // THIRD: K vectors (stride ld)
    const double* z;     // cached z
    double* part_acc;    // [ncluster][K][ld]
    double c2, c3, c4;
    const int* skip;
    int nskip;
};

// Butterfly reduce-scatter of V <= 32 values over the 32 lanes of a warp.
// On return, lane l holds in v[0] the warp sum of value index vidx(l).
template <int V>
__device__ __forceinline__ int warp_reduce_scatter(double (&v)[V], int lane) {
    int idx_base = 0;
    int m = V;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (m > 1) {
            const int h = m / 2;
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < V / 2; ++i) {
                if (i < h) {
                    const double send = upper ? v[i] : v[i + h];
                    const double keep = upper ? v[i + h] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            if (upper) idx_base += h;
            m = h;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return idx_base;
}

template <Op OP, int K, int Q, int RG>
struct ClusterShape {
    static constexpr int NDOT = OP == Op::THIRD ? 2 * K : K;
    static constexpr int V = RG * NDOT;  // partial dots per stage
};

template <Op OP, int K, int Q, int RG>
__global__ void __launch_bounds__(256, 1) stream_cluster_kernel(const ClusterArgs a) {
    using Sh = ClusterShape<OP, K, Q, RG>;
    constexpr int NDOT = Sh::NDOT;
    constexpr int V = Sh::V;
    constexpr int E = kXSlots;
    static_assert(V <= 32, "partial dots per stage must fit one warp");
    if (pass_skipped(a.skip, a.nskip)) return;  // uniform over the whole grid
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks();
    const int crank = (int)cluster.block_rank();
    const int ncl = gridDim.x / C;
    const int ci = blockIdx.x / C;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = a.P, S = a.S, nw = P / 32;
    const int cw = a.cw, npairs = cw / 2;
    const long long ld = a.ld;
    const int col0 = crank * cw;

    // smem: [full S | xfull E] (mbarriers, 256 B)
    //       [red 2 x V x nw][xchg E x 16 x V][fdot 2 x V][ring S x RG x cw]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* xfull = full + 8;
    double* red = reinterpret_cast<double*>(smem_raw + 256);
    double* xchg = red + 2 * V * nw;
    double* fdot = xchg + E * 16 * V;
    size_t off = 256 + (size_t)(2 * V * nw + E * 16 * V + 2 * V) * sizeof(double);
    off = (off + 127) & ~(size_t)127;
    const size_t stage_bytes = ((size_t)RG * cw * sizeof(double) + 127) & ~(size_t)127;
    unsigned char* ring = smem_raw + off;

    const long long T = a.T;
    const long long r0 = T * ci / ncl, r1 = T * (ci + 1) / ncl;
    const long long nrows = r1 - r0;
    const int nst = (int)((nrows + RG - 1) / RG);

    uint64_t policy = 0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        for (int e = 0; e < E; ++e) mbar_init(&xfull[e], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int slot = s % S;
        const long long rows = (nrows - (long long)s * RG) < RG ? (nrows - (long long)s * RG) : RG;
        const uint32_t bytes = (uint32_t)(rows * cw * sizeof(double));
        mbar_arrive_expect_tx(&full[slot], bytes);
        for (int r = 0; r < rows; ++r)
            bulk_g2s(ring + slot * stage_bytes + (size_t)r * cw * sizeof(double),
                     a.X + (r0 + (long long)s * RG + r) * ld + col0, (uint32_t)(cw * sizeof(double)), &full[slot],
                     policy);
    };
    if (tid == 0) {
        policy = a.evict_first ? policy_evict_first() : policy_evict_last();
        const int pre = nst < S ? nst : S;
        for (int s = 0; s < pre; ++s) issue(s);
    }
    // peers' barriers are initialised before any remote push / arrive
    cluster.sync();

    double2 vreg[NDOT][Q];
#pragma unroll
    for (int k = 0; k < NDOT; ++k)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int j = tid + q * P;
            double2 v = make_double2(0.0, 0.0);
            if (j < npairs) {
                const double* src = (OP == Op::THIRD && k >= K) ? a.vin2 + (long long)(k - K) * ld
                                                                 : a.vin + (long long)k * ld;
                v = reinterpret_cast<const double2*>(src + col0)[j];
            }
            vreg[k][q] = v;
        }
    double2 acc[K][Q];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[k][q] = make_double2(0.0, 0.0);
    const double c2 = a.c2, c3 = a.c3, c4 = a.c4;

    // remote addresses (shared::cluster) of the exchange slots / barriers of every peer
    const int myv = tid < V ? tid : 0;

    // ---- produce(s): stage rows -> registers, partial dots, push partials to peers
    auto produce = [&](int s, double2 (&x)[RG][Q]) {
        const int slot = s % S;
        const long long srow0 = r0 + (long long)s * RG;
        const int rows_here = (r1 - srow0) < RG ? (int)(r1 - srow0) : RG;
        mbar_wait(&full[slot], (uint32_t)((s / S) & 1));
        const double* st = reinterpret_cast<const double*>(ring + slot * stage_bytes);
#pragma unroll
        for (int rr = 0; rr < RG; ++rr)
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int j = tid + q * P;
                x[rr][q] = (rr < rows_here && j < npairs) ? reinterpret_cast<const double2*>(st + (size_t)rr * cw)[j]
                                                           : make_double2(0.0, 0.0);
            }
        double dv[V];
#pragma unroll
        for (int rr = 0; rr < RG; ++rr)
#pragma unroll
            for (int k = 0; k < NDOT; ++k) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    d0 = fma(x[rr][q].x, vreg[k][q].x, d0);
                    d1 = fma(x[rr][q].y, vreg[k][q].y, d1);
                }
                dv[rr * NDOT + k] = d0 + d1;
            }
        const int vid = warp_reduce_scatter<V>(dv, lane);
        double* rb = red + (s & 1) * V * nw;
        if ((lane & ((32 / V) - 1)) == 0) rb[vid * nw + warp] = dv[0];
        __syncthreads();  // (A) stage slice in registers, warp partials published
        if (tid == 0 && s + S < nst) issue(s + S);
        if (tid < V) {
            double sum = 0.0;
            for (int w = 0; w < nw; ++w) sum += rb[myv * nw + w];
            const int e = s % E;
            // slot reuse needs no release handshake: this thread's push of
            // stage s follows its consume(s-2), which observed every peer's
            // stage s-2 push, which each peer issued after its own consume(s-4)
            // (same threads) finished reading slot (s-4) % E == e.
            double* slotp = xchg + ((size_t)e * 16 + crank) * V + myv;
            for (int r = 0; r < C; ++r) st_async_f64(mapa_u32(slotp, r), sum, mapa_u32(&xfull[e], r));
        }
    };

    // ---- consume(s): gather full dots, release the slot, weights + X^T accumulation
    auto consume = [&](int s, const double2 (&x)[RG][Q]) {
        const int e = s % E;
        const long long srow0 = r0 + (long long)s * RG;
        const int rows_here = (r1 - srow0) < RG ? (int)(r1 - srow0) : RG;
        double zc[RG];
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) zc[rr] = (rr < rows_here) ? __ldg(a.z + srow0 + rr) : 0.0;
        double* fb = fdot + (s & 1) * V;
        if (tid == 0) mbar_arrive_expect_tx(&xfull[e], (uint32_t)(C * V * sizeof(double)));
        if (tid < V) {
            mbar_wait_cluster(&xfull[e], (uint32_t)((s / E) & 1));
            const double* xb = xchg + (size_t)e * 16 * V;
            double sum = 0.0;
            for (int r = 0; r < C; ++r) sum += xb[r * V + myv];
            fb[myv] = sum;
        }
        __syncthreads();  // (B) full dots visible
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) {
            double w[K];
            const bool valid = rr < rows_here;
            if constexpr (OP == Op::HVP) {
                const double zt = zc[rr];
                const double psi2 = 2.0 * c2 - 6.0 * c3 * zt + 12.0 * c4 * (zt * zt);
#pragma unroll
                for (int k = 0; k < K; ++k) w[k] = valid ? psi2 * fb[rr * NDOT + k] : 0.0;
            } else {
                const double zt = zc[rr];
                const double psi3 = -6.0 * c3 + 24.0 * c4 * zt;
#pragma unroll
                for (int k = 0; k < K; ++k) w[k] = valid ? psi3 * fb[rr * NDOT + k] * fb[rr * NDOT + K + k] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    acc[k][q].x = fma(w[k], x[rr][q].x, acc[k][q].x);
                    acc[k][q].y = fma(w[k], x[rr][q].y, acc[k][q].y);
                }
        }
    };

    double2 xa[RG][Q], xb[RG][Q];
    if (nst > 0) produce(0, xa);
    int s = 0;
    for (; s + 1 < nst; s += 2) {
        produce(s + 1, xb);
        consume(s, xa);
        if (s + 2 < nst) produce(s + 2, xa);
        consume(s + 1, xb);
    }
    if (s < nst) consume(s, xa);

    // publish this CTA's column block of the cluster partial: part[ci][k][col0 + 2j]
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int j = tid + q * P;
            if (j < npairs)
                reinterpret_cast<double2*>(a.part_acc + ((size_t)ci * K + k) * ld + col0)[j] = acc[k][q];
        }
    // no CTA may exit while a peer can still push into its shared memory
    cluster.sync();
}

}  // namespace mvsk_b200
