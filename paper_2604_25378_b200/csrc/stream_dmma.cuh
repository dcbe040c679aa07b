// Multi-RHS fused passes on the fp64 tensor cores (DMMA.8x8x4) with a
// thread-block-cluster column split.
//
// A stage is 8 sample rows. For k right-hand sides both halves of the fused
// op are small dense products:
//   phase 1  Y (8 x k)  = X_s (8 x cw) . V (cw x k)        row dots
//   phase 2  G (cw x k) += X_s^T (cw x 8) . W (8 x k)      X^T accumulation
// with W = psi''(z) o Y (HVP) or psi'''(z) o Y_u o Y_v (THIRD). Both run as
// mma.sync.m8n8k4.f64 on the staged tile in shared memory: one warp
// instruction does 256 FMAs instead of 32, which is what lets 8 right-hand
// sides ride one HBM pass. The cw columns of a CTA are split over its 8 warps
// (WC each); the per-warp phase-1 partials are summed in a fixed order, the C
// CTA partials of the cluster are exchanged through DSMEM (st.async +
// mbarrier complete_tx, as in stream_cluster.cuh) and summed in rank order,
// so every CTA holds bit-identical Y. X is read from HBM once.
//
// Reference: oracle.hpp:92-101 (hvp), :103-113 (third_action).
#pragma once
#include <cooperative_groups.h>

#include "stream_cluster.cuh"

#ifndef MVSK_NCH1
#define MVSK_NCH1 4  // phase-1 accumulator chains (1 n-tile)
#endif
#ifndef MVSK_NCH2
#define MVSK_NCH2 2  // phase-1 accumulator chains (2 n-tiles)
#endif

namespace mvsk_b200 {

struct DmmaArgs {
    const double* X;  // T_local x ld
    long long T;
    int ld;
    int cw;   // columns owned by a CTA (even)
    int S;    // ring depth (>= 3)
    int evict_first;
    const double* vin;   // HVP: K vectors; THIRD: K u-vectors (stride ld)
    const double* vin2;  // THIRD: K v-vectors
    const double* z;
    double* part_acc;    // [ncluster][K][ld]
    double c2, c3, c4;
    const int* skip;
    int nskip;
    int early_refill;  // barrier at the top of produce() and refill there
};

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    // not volatile: a pure function of its operands, so ptxas may interleave
    // independent accumulator chains
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <Op OP, int K>
struct DmmaShape {
    static constexpr int NDOT = OP == Op::THIRD ? 2 * K : K;  // phase-1 columns
    static constexpr int NT1 = (NDOT + 7) / 8;                // phase-1 n-tiles
    static constexpr int V = 8 * NDOT;                        // partial dots per stage
};

// D = exchange pipelining depth: produce(s + D) is issued before consume(s),
// so D stages of DSMEM exchange are in flight (needs a TMA ring S >= D + 2 and
// E = 2D + 2 exchange slots, see the slot-reuse argument in stream_cluster.cuh).
template <Op OP, int K, int WC, int D>
__global__ void __launch_bounds__(256, 1) stream_dmma_kernel(const DmmaArgs a) {
    using Sh = DmmaShape<OP, K>;
    constexpr int NDOT = Sh::NDOT, NT1 = Sh::NT1, V = Sh::V;
    constexpr int KS1 = WC / 4;  // phase-1 k-steps per warp
    constexpr int MT = WC / 8;   // phase-2 m-tiles per warp
    constexpr int E = 2 * D + 2;
    constexpr int RS = 8 * WC + 4;  // smem row stride (doubles): conflict-free fragment loads
    static_assert(K <= 8, "phase 2 uses one n-tile");
    if (pass_skipped(a.skip, a.nskip)) return;  // uniform over the whole grid
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks();
    const int crank = (int)cluster.block_rank();
    const int ncl = gridDim.x / C;
    const int ci = blockIdx.x / C;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;  // fragment coordinates
    const int cw = a.cw, S = a.S;
    const long long ld = a.ld;
    const int col0 = crank * cw;
    const int wcol = warp * WC;  // warp's first column inside the CTA slice

    // smem: [full S | xfull E] mbarriers (256 B) [red 8 x V][xchg E x C x V][fdot 2 x V][ring S x 8 x RS]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* xfull = full + 8;
    double* red = reinterpret_cast<double*>(smem_raw + 256);
    double* xchg = red + 8 * V;
    double* fdot = xchg + E * C * V;
    size_t off = 256 + (size_t)(8 * V + E * C * V + 2 * V) * sizeof(double);
    off = (off + 127) & ~(size_t)127;
    constexpr size_t stage_elems = (size_t)8 * RS;
    double* ring = reinterpret_cast<double*>(smem_raw + off);

    const long long T = a.T;
    const long long r0 = T * ci / ncl, r1 = T * (ci + 1) / ncl;
    const long long nrows = r1 - r0;
    const int nst = (int)((nrows + 7) / 8);

    // zero the whole ring once: the pad columns [cw, RS) are never written by
    // the TMA, and the rows past the block end of a partial last stage keep
    // finite (stale or zero) values, so 0-weighted products stay 0
    for (size_t i = tid; i < (size_t)S * stage_elems; i += 256) ring[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes before the async-proxy fills
    uint64_t policy = 0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        for (int e = 0; e < E; ++e) mbar_init(&xfull[e], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        const int slot = s % S;
        const long long rows = (nrows - (long long)s * 8) < 8 ? (nrows - (long long)s * 8) : 8;
        mbar_arrive_expect_tx(&full[slot], (uint32_t)(rows * cw * sizeof(double)));
        for (int r = 0; r < rows; ++r)
            bulk_g2s(ring + slot * stage_elems + (size_t)r * RS, a.X + (r0 + (long long)s * 8 + r) * ld + col0,
                     (uint32_t)(cw * sizeof(double)), &full[slot], policy);
    };
    if (tid == 0) {
        policy = a.evict_first ? policy_evict_first() : policy_evict_last();
        const int pre = nst < S ? nst : S;
        for (int s = 0; s < pre; ++s) issue(s);
    }
    cluster.sync();  // peers' barriers initialised before any push

    // phase-1 B fragments: B[k = t4][n = g4] of every k-step = V[col][j]
    double vb[NT1][KS1];
#pragma unroll
    for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
        for (int ks = 0; ks < KS1; ++ks) {
            const int c = wcol + ks * 4 + t4;
            const int j = nt * 8 + g4;
            double v = 0.0;
            if (c < cw && j < NDOT) {
                const double* src = (OP == Op::THIRD && j >= K) ? a.vin2 + (long long)(j - K) * ld
                                                                 : a.vin + (long long)j * ld;
                v = src[col0 + c];
            }
            vb[nt][ks] = v;
        }
    double acc[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    const double c2 = a.c2, c3 = a.c3, c4 = a.c4;

    // ---- produce(s): wait for the tile, phase 1, warp partials, push the CTA partial
    auto produce = [&](int s, double (&zr)[2]) {
        const int slot = s % S;
        const long long srow0 = r0 + (long long)s * 8;
        zr[0] = (srow0 + t4 < r1) ? __ldg(a.z + srow0 + t4) : 0.0;
        zr[1] = (srow0 + 4 + t4 < r1) ? __ldg(a.z + srow0 + 4 + t4) : 0.0;
        if (a.early_refill) {
            // every warp is past its last read of the slot consumed one stage
            // earlier: refill it now rather than after this stage's phase 1
            __syncthreads();
            if (tid == 0 && s >= D + 1 && s - D - 1 + S < nst) issue(s - D - 1 + S);
        }
        mbar_wait(&full[slot], (uint32_t)((s / S) & 1));
        const double* X = ring + slot * stage_elems;  // rows past the block end: finite stale data,
                                                      // their dots are never used (zero weights)
        // NCH independent accumulator chains per n-tile hide the DMMA latency
        constexpr int NCH = NT1 >= 2 ? MVSK_NCH2 : MVSK_NCH1;
        double cfr[NCH][NT1][2];
#pragma unroll
        for (int h = 0; h < NCH; ++h)
#pragma unroll
            for (int nt = 0; nt < NT1; ++nt) cfr[h][nt][0] = cfr[h][nt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS1; ++ks) {
            const double av = X[g4 * RS + wcol + ks * 4 + t4];
#pragma unroll
            for (int nt = 0; nt < NT1; ++nt) dmma884(cfr[ks % NCH][nt], av, vb[nt][ks]);
        }
#pragma unroll
        for (int h = 1; h < NCH; ++h)
#pragma unroll
            for (int nt = 0; nt < NT1; ++nt) {
                cfr[0][nt][0] += cfr[h][nt][0];
                cfr[0][nt][1] += cfr[h][nt][1];
            }
        // Y partial: C[row = g4][j = nt*8 + 2*t4 + i]
        double* rb = red + warp * V;
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int j = nt * 8 + 2 * t4 + i;
                if (j < NDOT) rb[g4 * NDOT + j] = cfr[0][nt][i];
            }
        __syncthreads();  // (A) warp partials published; all consumes up to s-D-1 done
        if (!a.early_refill && tid == 0 && s >= D + 1 && s - D - 1 + S < nst) issue(s - D - 1 + S);
        if (tid < V) {
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) sum += red[w * V + tid];
            const int e = s % E;
            double* slotp = xchg + ((size_t)e * C + crank) * V + tid;
            for (int r = 0; r < C; ++r) st_async_f64(mapa_u32(slotp, r), sum, mapa_u32(&xfull[e], r));
        }
    };

    // ---- consume(s): full dots, weights, phase 2
    auto consume = [&](int s, const double (&zr)[2]) {
        const int slot = s % S;
        const int e = s % E;
        const long long srow0 = r0 + (long long)s * 8;
        double* fb = fdot + (s & 1) * V;
        if (tid == 0) mbar_arrive_expect_tx(&xfull[e], (uint32_t)(C * V * sizeof(double)));
        if (tid < V) {
            mbar_wait_cluster(&xfull[e], (uint32_t)((s / E) & 1));
            const double* xb = xchg + (size_t)e * C * V;
            double sum = 0.0;
            for (int r = 0; r < C; ++r) sum += xb[r * V + tid];
            fb[tid] = sum;
        }
        __syncthreads();  // (B) full dots visible
        // W fragments: B2[k = row = kh*4 + t4][n = g4]
        double wf[2];
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
            const int r = kh * 4 + t4;
            const bool valid = (srow0 + r < r1) && g4 < K;
            double w = 0.0;
            if (valid) {
                const double zt = zr[kh];
                if constexpr (OP == Op::HVP) {
                    const double psi2 = 2.0 * c2 - 6.0 * c3 * zt + 12.0 * c4 * (zt * zt);
                    w = psi2 * fb[r * NDOT + g4];
                } else {
                    const double psi3 = -6.0 * c3 + 24.0 * c4 * zt;
                    w = psi3 * fb[r * NDOT + g4] * fb[r * NDOT + K + g4];
                }
            }
            wf[kh] = w;
        }
        const double* X = ring + slot * stage_elems;
        // k-half outer: the MT accumulators form independent chains
#pragma unroll
        for (int kh = 0; kh < 2; ++kh)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const double av = X[(kh * 4 + t4) * RS + wcol + mt * 8 + g4];
                dmma884(acc[mt], av, wf[kh]);
            }
    };

    double zr[D + 1][2];
#pragma unroll
    for (int i = 0; i < D; ++i)
        if (i < nst) produce(i, zr[i]);
    for (int s0 = 0; s0 < nst; s0 += D + 1) {
#pragma unroll
        for (int j = 0; j <= D; ++j) {
            const int s = s0 + j;
            if (s < nst) {
                if (s + D < nst) produce(s + D, zr[(j + D) % (D + 1)]);
                consume(s, zr[j]);
            }
        }
    }

    // G fragment: D[m = col = g4][n = k = 2*t4 + i]
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int c = wcol + mt * 8 + g4;
            const int k = 2 * t4 + i;
            if (c < cw && k < K) a.part_acc[((size_t)ci * K + k) * ld + col0 + c] = acc[mt][i];
        }
    cluster.sync();  // no CTA exits while a peer may still push into it
}

// ---------------------------------------------------------------------------
// Warp-specialised variant: 8 math warps + one helper warpgroup.
//
// An intermediate generation (barrier-free stage loop, all 8 warps doing skeleton
// and DMMA in lock-step; profiles/r01_dmma_pipe.txt: 2.06 ms on the C5 8-RHS
// HVP) was bounded by its per-stage skeleton and has been removed. Here the
// skeleton moves to a helper warpgroup (registers rebalanced with
// setmaxnreg: 232 per math thread, 40 per helper thread):
//   warp 8   TMA producer: refills a ring slot once the 8 math warps released it
//   warp 9   reducer: sums the 8 warp partials of a stage, pushes the C-CTA
//            exchange (st.async + tx-count mbarrier on every peer)
//   warp 10  W builder: waits for the stage's cluster dots, forms
//            W = psi(z) o Y (rows past the block end -> 0) into a smem buffer
// and a math warp only runs  phase1(i) -> partial -> [W(i-1) ready] ->
// phase2(i-1) -> frag(i) -> release.
// Slot reuse: red[R] and the ring are guarded by empty barriers; the exchange
// ring E = 4 by the argument: a reducer pushes stage j+4 after its math warps
// finished phase1(j+4), hence passed W(j+2) ready, hence every CTA pushed j+2,
// hence every CTA's math warps finished phase1(j+2) and passed W(j) ready, so
// every W builder consumed stage j. The W buffer (2 deep) is rewritten for
// stage j+2 only after xfull(j+2), i.e. after this CTA's math warps finished
// phase1(j+2) and with it phase2(j).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void reg_alloc_232() { asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory"); }
__device__ __forceinline__ void reg_dealloc_40() { asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory"); }

// Ring layout of the warp-specialised kernel. A staged row r of a slot starts at
// r * RS + ws_row_swz(r) doubles with RS = 8 WC + 8, i.e. at 16-byte chunk
// (4 r + 2 ((r >> 1) & 1)) mod 8 of the 128-byte bank window: rows 2a and
// 2a + 1 sit 64 bytes apart (the phase-1 fragments: a quarter-warp reads 4
// chunks of each of two adjacent rows) and rows 0..3 / 4..7 start at chunks
// {0, 4, 2, 6} (the phase-2 fragments: 2 chunks of each of four rows), so both
// 16-byte fragment loads are bank-conflict-free. With the earlier uniform
// 8 WC + 4 stride the phase-1 loads were 2-way conflicted (ncu: 82 M conflict
// wavefronts of 227 M shared-load wavefronts on the C5 8-RHS HVP).
#ifndef MVSK_WS_SWZ
#define MVSK_WS_SWZ 1  // 0: the uniform 8 WC + 4 stride (A/B builds only)
#endif
__host__ __device__ constexpr int kWsRowStride(int wc) { return 8 * wc + (MVSK_WS_SWZ ? 8 : 4); }
__device__ __forceinline__ int ws_row_swz(int r) { return MVSK_WS_SWZ ? ((r >> 1) & 1) * 4 : 0; }

// F2REG = false (the 8 third-action pairs at 128-column slices, whose doubled
// V fragments leave no room for held phase-2 fragments): phase 2 reads the
// tile from the ring slot, which is then released after phase 2 instead of
// after phase 1 (one fill fewer in flight).
template <Op OP, int K, int WC, int C, bool F2REG = true>
__global__ void __launch_bounds__(384, 1) stream_dmma_ws_kernel(const DmmaArgs a) {
    using Sh = DmmaShape<OP, K>;
    constexpr int NDOT = Sh::NDOT, NT1 = Sh::NT1, V = Sh::V;
    constexpr int NW = 8;            // math warps
    constexpr int E = 4, R = 2;      // exchange / partial ring depths
    constexpr int KP = WC / 8;
    constexpr int MP = WC / 16;
    constexpr int MT = 2 * MP;
    constexpr int VPL = (V + 31) / 32;  // dots per reducer lane
    constexpr int RS = kWsRowStride(WC);
    constexpr int NCH = NT1 >= 2 ? MVSK_NCH2 : MVSK_NCH1;
    static_assert(K <= 8 && WC % 16 == 0 && C % 2 == 0, "shape");
    if (pass_skipped(a.skip, a.nskip)) return;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = (int)cluster.block_rank();
    const int ncl = gridDim.x / C;
    const int ci = blockIdx.x / C;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cw = a.cw, S = a.S;
    const long long ld = a.ld;
    const int col0 = crank * cw;

    // smem: mbarriers [full 8 | empty 8 | xfull 4 | pfull 2 | pempty 2 | wready 2] (256 B)
    //       [red R x NW x V][xchg E x V x C][wbuf 2 x 64][ring S x 8 x RS]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + 8;
    uint64_t* xfull = full + 16;
    uint64_t* pfull = full + 20;
    uint64_t* pempty = full + 22;
    uint64_t* wready = full + 24;
    double* red = reinterpret_cast<double*>(smem_raw + 256);
    double* xchg = red + R * NW * V;
    double* wbuf = xchg + E * V * C;
    size_t off = 256 + (size_t)(R * NW * V + E * V * C + 2 * 64) * sizeof(double);
    off = (off + 127) & ~(size_t)127;
    constexpr size_t stage_elems = (size_t)8 * RS;
    double* ring = reinterpret_cast<double*>(smem_raw + off);

    const long long T = a.T;
    const long long r0 = T * ci / ncl, r1 = T * (ci + 1) / ncl;
    const long long nrows = r1 - r0;
    const int nst = (int)((nrows + 7) / 8);
    constexpr uint32_t kXBytes = (uint32_t)(C * V * sizeof(double));

    for (size_t i = tid; i < (size_t)S * stage_elems; i += blockDim.x) ring[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        for (int e = 0; e < E; ++e) mbar_init(&xfull[e], 1);
        for (int r = 0; r < R; ++r) {
            mbar_init(&pfull[r], NW);
            mbar_init(&pempty[r], 1);
        }
        for (int r = 0; r < 2; ++r) mbar_init(&wready[r], 1);
        for (int e = 0; e < E && e < nst; ++e) mbar_arrive_expect_tx(&xfull[e], kXBytes);
        fence_mbar_init();
    }
    __syncthreads();
    cluster.sync();  // peers' barriers initialised (and armed) before any push

    if (warp >= NW) {
        // ======================= helper warpgroup =======================
        reg_dealloc_40();
        if (warp == NW) {
            // ---- TMA producer
            if (lane == 0) {
                const uint64_t policy = a.evict_first ? policy_evict_first() : policy_evict_last();
                int slot = 0;
                for (int s = 0; s < nst; ++s) {
                    // the slot's previous stage (s - S) released by all 8 math warps
                    if (s >= S) mbar_wait(&empty[slot], (uint32_t)(((s / S) - 1) & 1));
                    const long long rows = (nrows - (long long)s * 8) < 8 ? (nrows - (long long)s * 8) : 8;
                    mbar_arrive_expect_tx(&full[slot], (uint32_t)(rows * cw * sizeof(double)));
                    const double* src = a.X + (r0 + (long long)s * 8) * ld + col0;
                    double* dst = ring + slot * stage_elems;
                    for (int r = 0; r < rows; ++r)
                        bulk_g2s(dst + (size_t)r * RS + ws_row_swz(r), src + (long long)r * ld,
                                 (uint32_t)(cw * sizeof(double)), &full[slot], policy);
                    if (++slot == S) slot = 0;
                }
            }
        } else if (warp == NW + 1) {
            // ---- reducer
            const uint32_t xb_self = smem_u32(xchg);
            for (int j = 0; j < nst; ++j) {
                const int r = j % R;
                mbar_wait(&pfull[r], (uint32_t)((j / R) & 1));
                const double* rb = red + (size_t)r * NW * V;
                double sum[VPL];
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    const int v = lane + 32 * q;
                    double sacc = 0.0;
                    if (v < V) {
#pragma unroll
                        for (int w = 0; w < NW; ++w) sacc += rb[w * V + v];
                    }
                    sum[q] = sacc;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&pempty[r]);
                const int e = j % E;
                const uint32_t lb = smem_u32(&xfull[e]);
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    const int v = lane + 32 * q;
                    if (v < V) {
                        const uint32_t la = xb_self + (uint32_t)(((e * V + v) * C + crank) * sizeof(double));
#pragma unroll
                        for (int rr = 0; rr < C; ++rr) {
                            uint32_t ra, rbar;
                            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rr));
                            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(lb), "r"(rr));
                            st_async_f64(ra, sum[q], rbar);
                        }
                    }
                }
            }
        } else if (warp == NW + 2) {
            // ---- W builder: lane -> (row, g) pairs of the 8 x 8 W tile
            const double c2 = a.c2, c3 = a.c3, c4 = a.c4;
            for (int j = 0; j < nst; ++j) {
                const int e = j % E;
                const long long srow0 = r0 + (long long)j * 8;
                double zr[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int row = (lane + 32 * q) >> 3;
                    zr[q] = (srow0 + row < r1) ? __ldg(a.z + srow0 + row) : 0.0;
                }
                mbar_wait(&xfull[e], (uint32_t)((j / E) & 1));
                if (lane == 0 && j + E < nst) mbar_arrive_expect_tx(&xfull[e], kXBytes);
                const double* xb = xchg + (size_t)e * V * C;
                double* wb = wbuf + (j & 1) * 64;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int idx = lane + 32 * q;
                    const int row = idx >> 3, g = idx & 7;
                    double w = 0.0;
                    if (g < K && srow0 + row < r1) {
                        const double* yp = xb + (size_t)(row * NDOT + g) * C;
                        double y = 0.0;
#pragma unroll
                        for (int c = 0; c < C; c += 2) {
                            const double2 t = *reinterpret_cast<const double2*>(yp + c);
                            y += t.x;
                            y += t.y;
                        }
                        const double zt = zr[q];
                        if constexpr (OP == Op::HVP) {
                            w = (2.0 * c2 - 6.0 * c3 * zt + 12.0 * c4 * (zt * zt)) * y;
                        } else {
                            const double* yq = yp + (size_t)K * C;
                            double yv = 0.0;
#pragma unroll
                            for (int c = 0; c < C; c += 2) {
                                const double2 t = *reinterpret_cast<const double2*>(yq + c);
                                yv += t.x;
                                yv += t.y;
                            }
                            w = (-6.0 * c3 + 24.0 * c4 * zt) * y * yv;
                        }
                    }
                    wb[idx] = w;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&wready[j & 1]);
            }
        }
    } else {
        // ========================= math warps ==========================
        reg_alloc_232();
        const int g4 = lane >> 2, t4 = lane & 3;
        const int wcol = warp * WC;
        double vb[NT1][2 * KP];
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
            for (int ks = 0; ks < 2 * KP; ++ks) {
                const int c = wcol + 8 * (ks >> 1) + 2 * t4 + (ks & 1);
                const int j = nt * 8 + g4;
                double v = 0.0;
                if (c < cw && j < NDOT) {
                    const double* src = (OP == Op::THIRD && j >= K) ? a.vin2 + (long long)(j - K) * ld
                                                                     : a.vin + (long long)j * ld;
                    v = src[col0 + c];
                }
                vb[nt][ks] = v;
            }
        double acc[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
        double f2[F2REG ? 2 : 1][F2REG ? MT : 1];
        const int p1_off = g4 * RS + ws_row_swz(g4) + wcol + 2 * t4;
        const int p2_off = t4 * RS + ws_row_swz(t4) + wcol + 2 * g4;  // rows t4 and 4 + t4 share the offset
        int slot = 0, prev_slot = 0;
        uint32_t fpar = 0;
        for (int i = 0; i <= nst; ++i) {
            if (i < nst) {
                // phase 1
                mbar_wait(&full[slot], fpar);
                const double* X = ring + slot * stage_elems + p1_off;
                double cfr[NCH][NT1][2];
#pragma unroll
                for (int h = 0; h < NCH; ++h)
#pragma unroll
                    for (int nt = 0; nt < NT1; ++nt) cfr[h][nt][0] = cfr[h][nt][1] = 0.0;
#pragma unroll
                for (int m = 0; m < KP; ++m) {
                    const double2 av = *reinterpret_cast<const double2*>(X + 8 * m);
#pragma unroll
                    for (int nt = 0; nt < NT1; ++nt) {
                        dmma884(cfr[(2 * m) % NCH][nt], av.x, vb[nt][2 * m]);
                        dmma884(cfr[(2 * m + 1) % NCH][nt], av.y, vb[nt][2 * m + 1]);
                    }
                }
#pragma unroll
                for (int h = 1; h < NCH; ++h)
#pragma unroll
                    for (int nt = 0; nt < NT1; ++nt) {
                        cfr[0][nt][0] += cfr[h][nt][0];
                        cfr[0][nt][1] += cfr[h][nt][1];
                    }
                const int r = i % R;
                if (i >= R) mbar_wait(&pempty[r], (uint32_t)(((i / R) - 1) & 1));
                double* rb = red + (size_t)r * NW * V + warp * V + g4 * NDOT;
#pragma unroll
                for (int nt = 0; nt < NT1; ++nt)
                    if (nt * 8 + 2 * t4 < NDOT)
                        *reinterpret_cast<double2*>(rb + nt * 8 + 2 * t4) = make_double2(cfr[0][nt][0], cfr[0][nt][1]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull[r]);
            }
            if (i >= 1) {
                // phase 2 of stage i-1
                const int j = i - 1;
                mbar_wait(&wready[j & 1], (uint32_t)((j >> 1) & 1));
                const double* wb = wbuf + (j & 1) * 64;
                const double wf0 = wb[t4 * 8 + g4], wf1 = wb[(4 + t4) * 8 + g4];
                if constexpr (F2REG) {
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt], f2[0][mt], wf0);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt], f2[1][mt], wf1);
                } else {
                    const double* X = ring + prev_slot * stage_elems + p2_off;
#pragma unroll
                    for (int kh = 0; kh < 2; ++kh)
#pragma unroll
                        for (int p = 0; p < MP; ++p) {
                            const double2 v = *reinterpret_cast<const double2*>(X + kh * 4 * RS + 16 * p);
                            dmma884(acc[2 * p], v.x, kh ? wf1 : wf0);
                            dmma884(acc[2 * p + 1], v.y, kh ? wf1 : wf0);
                        }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[prev_slot]);
                }
            }
            if (i < nst) {
                // frag(i), release the slot
                if constexpr (F2REG) {
                    const double* X = ring + slot * stage_elems + p2_off;
#pragma unroll
                    for (int kh = 0; kh < 2; ++kh)
#pragma unroll
                        for (int p = 0; p < MP; ++p) {
                            const double2 v = *reinterpret_cast<const double2*>(X + kh * 4 * RS + 16 * p);
                            f2[kh][2 * p] = v.x;
                            f2[kh][2 * p + 1] = v.y;
                        }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[slot]);
                }
                prev_slot = slot;
                if (++slot == S) {
                    slot = 0;
                    fpar ^= 1;
                }
            }
        }
#pragma unroll
        for (int p = 0; p < MP; ++p)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int c = wcol + 16 * p + 2 * g4 + h;
                    const int k = 2 * t4 + q;
                    if (c < cw && k < K) a.part_acc[((size_t)ci * K + k) * ld + col0 + c] = acc[2 * p + h][q];
                }
    }
    cluster.sync();  // no CTA exits while a peer may still push into it
}

}  // namespace mvsk_b200
