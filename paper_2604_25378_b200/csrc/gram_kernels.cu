// Dense contractions of the direct branch (affine_normal.hpp:151-188):
//   * weighted Gram  G = X^T diag(w) X        — fp64 tensor cores (DMMA,
//     mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4), 128x128 output tiles, lower
//     triangle only, cp.async double-buffered row chunks, deterministic
//     split-K over samples;
//   * per-row quadratic forms q_t = x_t^T P x_t (the diag(W M^-1 W^T) of
//     affine_normal.hpp:175-176, with P = UQ M^-1 (UQ)^T).
// fp64 has no tcgen05 kind on sm_100a (CUDA 12.9 exposes f16/tf32/f8f6f4/i8/
// mxf4 only), so DMMA through mma.sync is the tensor-core path for fp64.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "oracle_ops.cuh"

namespace mvsk_b200 {

namespace {

constexpr int GBM = 128;            // output tile (square)
constexpr int GBK = 32;             // sample rows per chunk
constexpr int GST = 3;              // cp.async ring depth
constexpr int GPAD = 4;             // smem row pad (doubles): conflict-free fragment loads
constexpr int GLDS = GBM + GPAD;    // smem row stride

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct GramArgs {
    const double* X;  // T x ld
    const double* w;  // T sample weights (or null: psi''(z) from z below)
    const double* z;  // cached z when the weights are psi''(z) (oracle.hpp:116-119)
    double c2, c3, c4;
    long long T;
    int ld;
    int n;              // valid columns (fragments wholly past n are skipped)
    int ntile;          // tiles per dimension
    int nsplit;         // sample splits
    double* part;       // [nsplit][npairs][GBM*GBM]
};

// tile pair index -> (ti, tj), ti >= tj
__device__ __forceinline__ void pair_of(int p, int& ti, int& tj) {
    int i = (int)((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= p) ++i;
    while (i * (i + 1) / 2 > p) --i;
    ti = i;
    tj = p - i * (i + 1) / 2;
}

// WM x WN warps, warp tile (8 FM) x (8 FN); the sample weight scales the A
// fragments (WA) or the B fragments. GUARD (n not a multiple of the tile):
// fragments wholly past n are skipped (C1: 9 of the 512 per k-step are
// live); the guards cost registers and DMMA interleaving, so full-tile panels
// (C5: 179 vs 149 ms) use the unguarded instantiation
template <int WM, int WN, int FM, int FN, bool WA, bool GUARD = false>
__global__ void __launch_bounds__(WM * WN * 32, 1) syrk_dmma_kernel(const GramArgs a) {
    static_assert(WM * FM * 8 == GBM && WN * FN * 8 == GBM, "warp grid must cover the tile");
    constexpr int NT = WM * WN * 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* sA = reinterpret_cast<double*>(smem_raw);           // [GST][GBK][GLDS]
    double* sB = sA + GST * GBK * GLDS;                          // [GST][GBK][GLDS]
    double* sw = sB + GST * GBK * GLDS;                          // [GST][GBK]
    int ti, tj;
    pair_of(blockIdx.x, ti, tj);
    const int i0 = ti * GBM, j0 = tj * GBM;
    const int split = blockIdx.y;
    const long long t_lo = a.T * split / a.nsplit, t_hi = a.T * (split + 1) / a.nsplit;
    const int nchunk = (int)((t_hi - t_lo + GBK - 1) / GBK);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;  // warp tile origin (wm*8FM, wn*8FN)

    // columns of each operand that any computed fragment reads: the valid
    // extent rounded up to the 8-column fragment (zero-filled past ld)
    const int wa = min(GBM, (a.n - i0 + 7) & ~7), wb = min(GBM, (a.n - j0 + 7) & ~7);
    const int pieces = GUARD ? max(wa, wb) / 2 : GBM / 2;  // 16-byte pieces per row
    auto load_chunk = [&](int c, int buf) {
        const long long t0 = t_lo + (long long)c * GBK;
        // GBK rows x (<= 128) doubles per operand = 16-byte pieces spread over the CTA
        for (int e = tid; e < GBK * pieces; e += NT) {
            const int r = e / pieces, cp = e - r * pieces;
            const long long t = t0 + r;
            const bool rv = t < t_hi;
            const int ca = i0 + 2 * cp, cb = j0 + 2 * cp;
            const double* ga = a.X + (rv ? t : 0) * (long long)a.ld + (ca < a.ld ? ca : 0);
            const double* gb = a.X + (rv ? t : 0) * (long long)a.ld + (cb < a.ld ? cb : 0);
            cp_async16(sA + (buf * GBK + r) * GLDS + 2 * cp, ga, (rv && ca < a.ld) ? 16 : 0);
            cp_async16(sB + (buf * GBK + r) * GLDS + 2 * cp, gb, (rv && cb < a.ld) ? 16 : 0);
        }
        if (tid < GBK) {
            const long long t = t0 + tid;
            double wt = 0.0;
            if (t < t_hi) {
                if (GUARD && a.z) {  // edge-tile (small-n) instantiation: the psi2 weights fused
                    const double zt = a.z[t];  // into the load, one kernel fewer per round trip
                    wt = 2.0 * a.c2 - 6.0 * a.c3 * zt + 12.0 * a.c4 * (zt * zt);
                } else {
                    wt = a.w[t];
                }
            }
            sw[buf * GBK + tid] = wt;
        }
    };

    double acc[FM][FN][2];
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;

    // GST-deep cp.async ring: one commit group per chunk (possibly empty)
    for (int c = 0; c < GST - 1; ++c) {
        if (c < nchunk) load_chunk(c, c);
        cp_async_commit();
    }
    for (int c = 0; c < nchunk; ++c) {
        const int buf = c % GST;
        cp_async_wait<GST - 2>();  // chunk c landed
        __syncthreads();           // ... for every thread; chunk c-1's buffer is free
        if (c + GST - 1 < nchunk) load_chunk(c + GST - 1, (c + GST - 1) % GST);
        cp_async_commit();
        const double* A = sA + buf * GBK * GLDS;
        const double* B = sB + buf * GBK * GLDS;
        const double* W = sw + buf * GBK;
#pragma unroll
        for (int k0 = 0; k0 < GBK; k0 += 4) {
            const int kr = k0 + (lane & 3);
            const double wk = W[kr];
            double af[FM], bf[FN];
#pragma unroll
            for (int fm = 0; fm < FM; ++fm) af[fm] = A[kr * GLDS + wm * 8 * FM + fm * 8 + (lane >> 2)];
#pragma unroll
            for (int fn = 0; fn < FN; ++fn) bf[fn] = B[kr * GLDS + wn * 8 * FN + fn * 8 + (lane >> 2)];
            if constexpr (WA) {
#pragma unroll
                for (int fm = 0; fm < FM; ++fm) af[fm] *= wk;
            } else {
#pragma unroll
                for (int fn = 0; fn < FN; ++fn) bf[fn] *= wk;
            }
#pragma unroll
            for (int fm = 0; fm < FM; ++fm)
#pragma unroll
                for (int fn = 0; fn < FN; ++fn)
                    if (!GUARD || (wm * 8 * FM + fm * 8 < wa && wn * 8 * FN + fn * 8 < wb))
                        dmma_8x8x4(acc[fm][fn], af[fm], bf[fn]);
        }
    }
    // partial tile out (row-major 128 x 128)
    double* out = a.part + ((size_t)split * gridDim.x + blockIdx.x) * (GBM * GBM);
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
            const int r = wm * 8 * FM + fm * 8 + (lane >> 2);
            const int cc = wn * 8 * FN + fn * 8 + (lane & 3) * 2;
            if (!GUARD || (r < wa && cc < wb))  // the finish reads only the valid block
                *reinterpret_cast<double2*>(out + r * GBM + cc) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
        }
}

// sum splits in order, scale, mirror into the dense n x n result. One element
// per thread (blockIdx.y: 256-element slice of the tile) and the split loads
// issued 8 at a time before the in-order sum: a single-tile Gram (C1 / C2) is
// otherwise a chain of dependent L2 round trips (26 us at C2)
// With `packed` set (a sharded group), only the lower triangle is written, as
// packed rows (i, j <= i) at i (i + 1) / 2 + j: the allreduce then moves
// n (n + 1) / 2 values instead of n^2, and gram_unpack_kernel mirrors after it.
__global__ void gram_finish_kernel(const double* part, int npairs, int nsplit, int n, double scale, double* G,
                                   long long ldg, double* packed, double* Gh) {
    const int p = blockIdx.x;
    int ti, tj;
    pair_of(p, ti, tj);
    const int e = blockIdx.y * 256 + threadIdx.x;
    const int r = e / GBM, c = e - r * GBM;
    const int i = ti * GBM + r, j = tj * GBM + c;
    if (i >= n || j >= n) return;
    if (ti == tj && j > i) return;
    double v = 0.0;
    for (int s0 = 0; s0 < nsplit; s0 += 8) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = s0 + u < nsplit ? part[((size_t)(s0 + u) * npairs + p) * (GBM * GBM) + e] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (s0 + u < nsplit) v += t[u];
    }
    v *= scale;
    if (packed) {
        const int hi = i > j ? i : j, lo = i > j ? j : i;
        packed[(long long)hi * (hi + 1) / 2 + lo] = v;
        return;
    }
    G[(long long)i * ldg + j] = v;
    G[(long long)j * ldg + i] = v;
    if (Gh) {  // mapped host mirror (host-API readback without a copy node)
        Gh[(long long)i * ldg + j] = v;
        Gh[(long long)j * ldg + i] = v;
    }
}

// dense symmetric G from the allreduced packed lower triangle
__global__ void gram_unpack_kernel(const double* __restrict__ packed, int n, double* __restrict__ G, double* Gh) {
    const long long tot = (long long)n * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), j = (int)(e - (long long)i * n);
        const int hi = i > j ? i : j, lo = i > j ? j : i;
        const double v = packed[(long long)hi * (hi + 1) / 2 + lo];
        G[e] = v;
        if (Gh) Gh[e] = v;
    }
}

// q_t = x_t^T P x_t for RB rows per block; P is ld x ld (zero outside the
// face). PS: P staged in shared memory beside the row block. Both stagings
// are cp.async 16-byte pieces issued all at once (one memory latency per CTA
// instead of one per loop trip: these panels are latency-bound, C2 28 -> a
// few us). With tw set, the kernel writes tw_t = psi3(z_t) q_t / T
// (affine_normal.hpp:174-177) instead of q. Same summation order on both paths.
template <int RB, bool PS>
__global__ void quadform_kernel(const double* X, long long T, int ld, const double* P, double* q, const double* z,
                                double* tw, double c3, double c4, double Tg) {
    extern __shared__ __align__(16) double xs[];  // [RB][ld] (+ [ld][ld] when PS)
    const long long t0 = (long long)blockIdx.x * RB;
    const int rows = (int)min((long long)RB, T - t0);
    const int hp = ld / 2;  // ld is even: 16-byte pieces per row
    for (int e = threadIdx.x; e < RB * hp; e += blockDim.x) {
        const int r = e / hp, cp = e - r * hp;
        const bool rv = r < rows;
        cp_async16(xs + r * ld + 2 * cp, X + (t0 + (rv ? r : 0)) * ld + 2 * cp, rv ? 16 : 0);
    }
    const double* Pr = P;
    if constexpr (PS) {
        double* ps = xs + RB * ld;
        for (int e = threadIdx.x; e < ld * hp; e += blockDim.x) cp_async16(ps + 2 * e, P + 2 * e, 16);
        Pr = ps;
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    double part[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) part[r] = 0.0;
    for (int c = threadIdx.x; c < ld; c += blockDim.x) {
        double y[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) y[r] = 0.0;
#pragma unroll 8
        for (int i = 0; i < ld; ++i) {
            const double pic = PS ? Pr[(long long)i * ld + c] : __ldg(Pr + (long long)i * ld + c);
#pragma unroll
            for (int r = 0; r < RB; ++r) y[r] = fma(xs[r * ld + i], pic, y[r]);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r) part[r] = fma(y[r], xs[r * ld + c], part[r]);
    }
    __shared__ double red[RB][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        double v = part[r];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[r][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < RB && threadIdx.x < rows) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
        const long long t = t0 + threadIdx.x;
        if (tw) {
            const double psi3 = -6.0 * c3 + 24.0 * c4 * z[t];
            tw[t] = psi3 * v / Tg;
        } else {
            q[t] = v;
        }
    }
}

// tw_t = psi'''(z_t) q_t / T   (affine_normal.hpp:174-177)
__global__ void third_weights_kernel(const double* z, const double* q, double* tw, long long T, double c3, double c4,
                                     double Tg) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
        const double psi3 = -6.0 * c3 + 24.0 * c4 * z[t];
        tw[t] = psi3 * q[t] / Tg;
    }
}

}  // namespace

void run_weighted_gram(mvsk_gpu_ctx* ctx, const double* w_rows, double* G_dev, double scale, const double* z,
                       double* G_host) {
    if (!w_rows && z && !is_sharded(ctx) && run_small_gram(ctx, z, G_dev, scale, G_host)) return;
    if (!w_rows && z && is_sharded(ctx)) {  // the same one-cluster Gram, packed for the allreduce
        const size_t npk = (size_t)ctx->n * (ctx->n + 1) / 2;
        if (ctx->gram_part_elems < npk) {
            if (ctx->gram_part) MVSK_CUDA(cudaFree(ctx->gram_part));
            ctx->gram_part = nullptr;
            MVSK_CUDA(cudaMalloc(&ctx->gram_part, npk * sizeof(double)));
            ctx->gram_part_elems = npk;
            ++ctx->epoch;
        }
        if (run_small_gram(ctx, z, G_dev, scale, G_host, ctx->gram_part)) {
            allreduce_sum(ctx, ctx->gram_part, npk);
            ++ctx->launches;
            const int nb = (int)std::min<long long>(4LL * ctx->nsm, ((long long)ctx->n * ctx->n + 255) / 256);
            gram_unpack_kernel<<<nb, 256, 0, ctx->stream>>>(ctx->gram_part, (int)ctx->n, G_dev, G_host);
            MVSK_CUDA(cudaGetLastError());
            return;
        }
    }
    const int n = (int)ctx->n;
    const int ntile = (n + GBM - 1) / GBM;
    const int npairs = ntile * (ntile + 1) / 2;
    // split the sample range so that >= 1 wave of CTAs is busy, min one chunk
    // (32 rows) per split: a single-tile Gram (n <= 128, C1/C2) otherwise runs
    // on one or a few SMs, DMMA-bound per CTA (C2 at 64+ rows per split: 22 us)
    int nsplit = std::max(1, ctx->nsm / npairs);
    nsplit = (int)std::max<long long>(1, std::min<long long>(nsplit, (ctx->T_local + GBK - 1) / GBK));
    if (npairs >= ctx->nsm) {
        // one CTA per SM: pick the split whose (tiles x splits) work items fill
        // the last wave best (C5: 528 tiles = 3.57 waves -> 7 splits = 24.97
        // waves); the split partials cost one extra 128 KB write + read per item
        double best = 0.0;
        for (int s = 1; s <= 16; ++s) {
            if (ctx->T_local / s < 64LL * GBK) break;
            const double w = (double)npairs * s / ctx->nsm;
            const double eff = w / std::ceil(w);
            if (eff > best + 0.005) {
                best = eff;
                nsplit = s;
            }
        }
    }
    const size_t need = (size_t)nsplit * npairs * GBM * GBM;
    if (ctx->gram_part_elems < need) {
        if (ctx->gram_part) MVSK_CUDA(cudaFree(ctx->gram_part));
        ctx->gram_part = nullptr;
        MVSK_CUDA(cudaMalloc(&ctx->gram_part, need * sizeof(double)));
        ctx->gram_part_elems = need;
        ++ctx->epoch;
    }
    // warp layout: 1 = 8 warps of 32 x 64, weights on the 4 A fragments
    // (C5 148.7 ms), 0 = the same with the weights on the 8 B fragments
    // (151.6 ms), 2 = 16 warps of 32 x 32 (151.8 ms: more warps per scheduler
    // do not raise the DMMA pipe's 81 % active; scripts/gram_ab.py)
    static const int var = [] {
        const char* e = std::getenv("MVSK_GRAM_VAR");
        return e ? std::atoi(e) : 1;
    }();
    const bool guard = n % GBM != 0;
    if (z && !(var == 1 && guard)) {  // only the edge-tile kernel computes psi2 itself;
        run_psi2(ctx, z, ctx->tvec, ctx->T_local);  // the full-tile one keeps its 184 registers
        w_rows = ctx->tvec;
        z = nullptr;
    }
    GramArgs a{};
    a.X = ctx->X;
    a.w = w_rows;
    a.z = z;
    a.c2 = ctx->c.c2;
    a.c3 = ctx->c.c3;
    a.c4 = ctx->c.c4;
    a.T = ctx->T_local;
    a.ld = (int)ctx->ld;
    a.n = n;
    a.ntile = ntile;
    a.nsplit = nsplit;
    a.part = ctx->gram_part;
    const size_t smem = (size_t)(2 * GST * GBK * GLDS + GST * GBK) * sizeof(double);
    const void* fn = var == 2   ? reinterpret_cast<const void*>(&syrk_dmma_kernel<4, 4, 4, 4, true>)
                     : var == 0 ? reinterpret_cast<const void*>(&syrk_dmma_kernel<4, 2, 4, 8, false>)
                     : guard    ? reinterpret_cast<const void*>(&syrk_dmma_kernel<4, 2, 4, 8, true, true>)
                                : reinterpret_cast<const void*>(&syrk_dmma_kernel<4, 2, 4, 8, true>);
    const int nthr = var == 2 ? 512 : 256;
    // a sharded group exchanges the packed lower triangle (n (n + 1) / 2
    // values); the tail of the split-partial buffer holds it
    const size_t npk = (size_t)n * (n + 1) / 2;
    double* packed = nullptr;
    if (is_sharded(ctx)) {
        if (ctx->gram_part_elems < need + npk) {
            // grow keeping nothing: the partials are rewritten by the launch below
            MVSK_CUDA(cudaFree(ctx->gram_part));
            MVSK_CUDA(cudaMalloc(&ctx->gram_part, (need + npk) * sizeof(double)));
            ctx->gram_part_elems = need + npk;
            ++ctx->epoch;
            a.part = ctx->gram_part;
        }
        packed = ctx->gram_part + need;
    }
    set_smem_attr(fn, smem);
    ++ctx->launches;
    void* args[] = {&a};
    MVSK_CUDA(cudaLaunchKernel(fn, dim3(npairs, nsplit), dim3(nthr), args, smem, ctx->stream));
    ++ctx->launches;
    gram_finish_kernel<<<dim3(npairs, GBM * GBM / 256), 256, 0, ctx->stream>>>(ctx->gram_part, npairs, nsplit, n, scale,
                                                                                G_dev, n, packed,
                                                                                packed ? nullptr : G_host);
    MVSK_CUDA(cudaGetLastError());
    ctx->phys += 1;
    if (packed) {
        allreduce_sum(ctx, packed, npk);
        ++ctx->launches;
        const int nb = (int)std::min<long long>(4LL * ctx->nsm, ((long long)n * n + 255) / 256);
        gram_unpack_kernel<<<nb, 256, 0, ctx->stream>>>(packed, n, G_dev, G_host);
        MVSK_CUDA(cudaGetLastError());
    }
}

void run_quadform(mvsk_gpu_ctx* ctx, const double* P_dev, double* q_dev, const double* z, double* tw) {
    const long long T = ctx->T_local;
    if (T <= 0) return;
    const long long ld = ctx->ld;
    const double c3 = ctx->c.c3, c4 = ctx->c.c4, Tg = (double)ctx->T_global;
    const int thr = ld <= 128 ? 128 : 256;
    // 8-row blocks (C1 / C2: 63 / 125 CTAs); P beside them in shared memory
    // when it fits (n <= ~160, the direct-mode sizes)
    constexpr int RB = 8;
    const int nb = (int)((T + RB - 1) / RB);
    const size_t smem_ps = (size_t)(RB * ld + ld * ld) * sizeof(double);
    ++ctx->launches;
    if (smem_ps <= ctx->max_smem) {
        const void* fn = reinterpret_cast<const void*>(&quadform_kernel<RB, true>);
        if (smem_ps > 48 * 1024) set_smem_attr(fn, smem_ps);
        quadform_kernel<RB, true><<<nb, thr, smem_ps, ctx->stream>>>(ctx->X, T, (int)ld, P_dev, q_dev, z, tw, c3, c4, Tg);
    } else {
        const size_t smem = (size_t)RB * ld * sizeof(double);
        if (smem > 48 * 1024) set_smem_attr(reinterpret_cast<const void*>(&quadform_kernel<RB, false>), smem);
        quadform_kernel<RB, false><<<nb, thr, smem, ctx->stream>>>(ctx->X, T, (int)ld, P_dev, q_dev, z, tw, c3, c4, Tg);
    }
    MVSK_CUDA(cudaGetLastError());
}

void run_third_weights(mvsk_gpu_ctx* ctx, const double* z, const double* q, double* tw) {
    const long long T = ctx->T_local;
    if (T <= 0) return;
    const int nb = (int)std::min<long long>(4 * ctx->nsm, (T + 255) / 256);
    ++ctx->launches;
    third_weights_kernel<<<nb, 256, 0, ctx->stream>>>(z, q, tw, T, ctx->c.c3, ctx->c.c4, (double)ctx->T_global);
    MVSK_CUDA(cudaGetLastError());
}

}  // namespace mvsk_b200
