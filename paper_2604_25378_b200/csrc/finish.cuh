// Cross-CTA reduction + op epilogue of a streaming pass, shared by the
// stand-alone finish_kernel (oracle_ops.cu) and the grid-synchronised tail of
// the cooperative stream_kernel launch (stream_kernels.cuh).
//
// A virtual block owns `cols` consecutive entries of the k x ld accumulator
// (cols = nthr / ng); its ng thread groups sum disjoint ranges of the CTA
// partials (4 independent accumulators each) and the groups are combined in a
// fixed order, so the result is bitwise deterministic. Scalars (FGRAD 3,
// LINESUMS 9) are reduced by virtual block 0, one warp per scalar.
// Reference epilogues: oracle.hpp:58-64, 82-84 (f, gradient), :95-96 / :107-108
// (HVP / third action, the 1/T folded out of the per-row weights),
// linesearch.hpp:26-38 (power sums).
#pragma once

namespace mvsk_b200 {

struct FinishArgs {
    int op;
    int k;
    int ld, n;
    long long ldo;
    int nb;
    int do_reduce, do_epi;
    const double* part_acc;
    const double* part_sc;
    double* red;  // [k*ld + kNumScalars]
    // epilogue
    double* out;
    double* g;         // FGRAD gradient
    double* sc;        // FGRAD scalars
    const double* mu;  // ld
    const double* x;   // ld (FGRAD mu'x)
    double c1, c2, c3, c4, T, value_offset;
    const double* value_offset_dev;  // if set, read at run time (graph-stable across face rebuilds)
    const int* skip;
    int nskip;
    double* hout;  // optional mapped host mirror of the results (PassIO::hout)
};

// one virtual block `vb`; every thread of the CTA calls it (it synchronises)
__device__ __forceinline__ void finish_block(const FinishArgs& f, int ng, int vb, int tid, int nthr, double* part) {
    const int nacc = (f.op == 3 /* LINESUMS */) ? 0 : f.k;
    const int tot = nacc * f.ld;
    const int nsc = f.op == 0 /* FGRAD */ ? 3 : (f.op == 3 ? 9 : 0);
    const int cols = nthr / ng;
    const int cl = tid % cols, grp = tid / cols;
    const int i = vb * cols + cl;
    auto qsum = [&](const double* base, size_t stride, int lo, int hi) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int b = lo;
        for (; b + 3 < hi; b += 4) {
            a0 += base[(size_t)b * stride];
            a1 += base[(size_t)(b + 1) * stride];
            a2 += base[(size_t)(b + 2) * stride];
            a3 += base[(size_t)(b + 3) * stride];
        }
        for (; b < hi; ++b) a0 += base[(size_t)b * stride];
        return (a0 + a1) + (a2 + a3);
    };
    // 1) fixed-order reduction over CTA partials
    if (f.do_reduce) {
        if (i < tot && grp < ng) part[grp * cols + cl] = qsum(f.part_acc + i, (size_t)tot, f.nb * grp / ng, f.nb * (grp + 1) / ng);
        if (vb == 0) {  // each scalar by one warp: lanes split the CTAs, fixed-order combine
            const int lane = tid & 31, w = tid >> 5;
            for (int sidx = w; sidx < nsc; sidx += nthr / 32) {
                double v = 0.0;
                for (int b = lane; b < f.nb; b += 32) v += f.part_sc[(size_t)b * kNumScalars + sidx];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) f.red[tot + sidx] = v;
            }
        }
        __syncthreads();
        if (grp == 0 && i < tot) {
            double v = part[cl];
            for (int q = 1; q < ng; ++q) v += part[q * cols + cl];
            f.red[i] = v;
        }
        __syncthreads();
    }
    if (!f.do_epi) return;
    // 2) epilogue (each element by the thread that reduced it; scalars by block 0)
    if (f.op == 0) {
        if (grp == 0 && i < f.ld) {
            const double gi = i < f.n ? (-f.c1 * f.mu[i] + f.red[i] / f.T) : 0.0;  // oracle.hpp:82-84
            f.g[i] = gi;
            if (f.hout) f.hout[8 + i] = gi;
        }
        if (vb == 0) {
            double sacc = 0.0;
            for (int j = tid; j < f.n; j += nthr) sacc += f.mu[j] * f.x[j];
            for (int o = 16; o; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
            __syncthreads();  // part[] reuse
            if ((tid & 31) == 0) part[tid >> 5] = sacc;
            __syncthreads();
            if (tid == 0) {
                double mux = 0.0;
                for (int w = 0; w < nthr / 32; ++w) mux += part[w];
                const double s2 = f.red[tot], s3 = f.red[tot + 1], s4 = f.red[tot + 2];
                // oracle.hpp:62-64
                const double vo = f.value_offset_dev ? *f.value_offset_dev : f.value_offset;
                f.sc[0] = vo - f.c1 * mux + (f.c2 * s2 - f.c3 * s3 + f.c4 * s4) / f.T;
                f.sc[1] = mux;
                f.sc[2] = s2 / f.T;
                f.sc[3] = s3 / f.T;
                f.sc[4] = s4 / f.T;
                if (f.hout)
                    for (int q = 0; q < 5; ++q) f.hout[q] = f.sc[q];
            }
            __syncthreads();
        }
    } else if (f.op == 3) {
        if (vb == 0 && tid < 9) {
            const double v = f.red[tot + tid] / f.T;
            f.out[tid] = v;
            if (f.hout) f.hout[tid] = v;
        }
    } else if (grp == 0 && i < tot) {
        const int k = i / f.ld, c = i - k * f.ld;
        // HVP / THIRD: A^T(w)/T with the 1/T folded out of the per-row weights
        if (c < f.n) {
            const double v = f.op == 4 /* XTW */ ? f.red[i] : f.red[i] / f.T;
            f.out[(size_t)k * f.ldo + c] = v;
            if (f.hout) f.hout[(size_t)k * f.ldo + c] = v;
        }
    }
}

}  // namespace mvsk_b200
