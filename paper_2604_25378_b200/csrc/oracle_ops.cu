// Launch planning, dispatch and epilogues for the streaming oracle kernels.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "oracle_ops.cuh"
#include "stream_cluster.cuh"
#include "stream_dmma.cuh"
#include "small_pass.cuh"

namespace mvsk_b200 {

namespace {


struct Plan {
    int Q = 1, P = 32, G = 1, RG = 1, S = 2;
    bool VS = false;  // input vectors in shared memory (stream_kernel<..., VS>)
    size_t smem = 0;
    int nb = 1;
    const void* fn = nullptr;
};

template <Op OP, int K, int Q, int RG, bool VS = false>
const void* kfn() {
    return reinterpret_cast<const void*>(&stream_kernel<OP, K, Q, RG, VS>);
}

// wide rows on short panels (C4: 34 rows of 40 KB per SM): the input vector in
// shared memory frees the registers for two 160-thread row teams per CTA
const void* select_kernel_vs(Op op, int K, int Q, int RG) {
    if (K != 1) return nullptr;
    if (RG == 2) {
        if (Q == 8 && op == Op::FGRAD) return kfn<Op::FGRAD, 1, 8, 2, true>();
        if (Q == 8 && op == Op::HVP) return kfn<Op::HVP, 1, 8, 2, true>();
        return nullptr;
    }
    if (RG != 1) return nullptr;
    switch (op) {
    case Op::FGRAD:
        if (Q == 8) return kfn<Op::FGRAD, 1, 8, 1, true>();
        if (Q == 16) return kfn<Op::FGRAD, 1, 16, 1, true>();
        break;
    case Op::LINESUMS:
        if (Q == 8) return kfn<Op::LINESUMS, 1, 8, 1, true>();
        if (Q == 16) return kfn<Op::LINESUMS, 1, 16, 1, true>();
        break;
    case Op::HVP:
        if (Q == 8) return kfn<Op::HVP, 1, 8, 1, true>();
        if (Q == 16) return kfn<Op::HVP, 1, 16, 1, true>();
        break;
    default: break;
    }
    return nullptr;
}

// (Q, RG) pairs instantiated for every op: RG * Q <= 8 keeps the staged row
// slice within 16 fp64 registers per thread.
#define MVSK_QRG(OP, K)                                                         \
    if (Q == 1 && RG == 1) return kfn<OP, K, 1, 1>();                           \
    if (Q == 1 && RG == 2) return kfn<OP, K, 1, 2>();                           \
    if (Q == 1 && RG == 4) return kfn<OP, K, 1, 4>();                           \
    if (Q == 2 && RG == 1) return kfn<OP, K, 2, 1>();                           \
    if (Q == 2 && RG == 2) return kfn<OP, K, 2, 2>();                           \
    if (Q == 2 && RG == 4) return kfn<OP, K, 2, 4>();                           \
    if (Q == 4 && RG == 1) return kfn<OP, K, 4, 1>();                           \
    if (Q == 4 && RG == 2) return kfn<OP, K, 4, 2>();

const void* select_kernel(Op op, int K, int Q, int RG) {
    switch (op) {
    case Op::FGRAD:
        MVSK_QRG(Op::FGRAD, 1)
        if (Q == 8 && RG == 1) return kfn<Op::FGRAD, 1, 8, 1>();
        if (Q == 8 && RG == 2) return kfn<Op::FGRAD, 1, 8, 2>();
        break;
    case Op::LINESUMS:
        MVSK_QRG(Op::LINESUMS, 1)
        if (Q == 8 && RG == 1) return kfn<Op::LINESUMS, 1, 8, 1>();
        if (Q == 8 && RG == 2) return kfn<Op::LINESUMS, 1, 8, 2>();
        break;
    case Op::XTW:
        MVSK_QRG(Op::XTW, 1)
        if (Q == 8 && RG == 1) return kfn<Op::XTW, 1, 8, 1>();
        break;
    case Op::HVP:
        if (K == 1) {
            MVSK_QRG(Op::HVP, 1)
            if (Q == 8 && RG == 1) return kfn<Op::HVP, 1, 8, 1>();
            if (Q == 8 && RG == 2) return kfn<Op::HVP, 1, 8, 2>();
        } else if (K == 2) {
            MVSK_QRG(Op::HVP, 2)
            if (Q == 8 && RG == 1) return kfn<Op::HVP, 2, 8, 1>();
            if (Q == 8 && RG == 2) return kfn<Op::HVP, 2, 8, 2>();
        } else if (K == 4) {
            if (Q == 1 && RG == 1) return kfn<Op::HVP, 4, 1, 1>();
            if (Q == 1 && RG == 2) return kfn<Op::HVP, 4, 1, 2>();
            if (Q == 2 && RG == 1) return kfn<Op::HVP, 4, 2, 1>();
        } else if (K == 8) {  // narrow panels (compact faces): one column pair per thread
            if (Q == 1 && RG == 1) return kfn<Op::HVP, 8, 1, 1>();
        }
        break;
    case Op::THIRD:
        if (K == 8 || K == 4) {  // narrow panels
            if (Q == 1 && RG == 1) return K == 8 ? kfn<Op::THIRD, 8, 1, 1>() : kfn<Op::THIRD, 4, 1, 1>();
            break;
        }
        if (K == 1) {
            MVSK_QRG(Op::THIRD, 1)
            if (Q == 8 && RG == 1) return kfn<Op::THIRD, 1, 8, 1>();
            if (Q == 8 && RG == 2) return kfn<Op::THIRD, 1, 8, 2>();
        }
        break;
    }
    return nullptr;
}
#undef MVSK_QRG

// largest Q allowed per (op, K) given register budgets (<= ~110 live fp64)
int max_q(Op op, int K) {
    if (op == Op::HVP) return K == 1 ? 8 : K == 2 ? 8 : K == 4 ? 2 : 1;
    if (op == Op::THIRD) return K == 1 ? 8 : 1;
    return 8;
}

int op_ndot(Op op, int K) {
    return (op == Op::FGRAD || op == Op::LINESUMS) ? 1 : (op == Op::THIRD ? 2 * K : (op == Op::XTW ? 0 : K));
}
int op_nacc(Op op, int K) { return (op == Op::HVP || op == Op::THIRD) ? K : (op == Op::LINESUMS ? 0 : 1); }

// mirror of StreamRegs<>::max_threads (stream_kernels.cuh)
int max_threads(Op op, int K, int Q, int RG, bool vs = false) {
    const int nv = vs ? 0 : std::max(op_ndot(op, K), 1), na = std::max(op_nacc(op, K), 1);
    const int live = 2 * Q * (nv + na + RG);
    return live <= 48 ? 512 : (live <= 64 ? 384 : 256);
}

int round_team(int need) {
    if (need <= 32) {
        int p = 1;
        while (p < need) p <<= 1;
        return std::max(p, 2);
    }
    return (need + 31) / 32 * 32;
}

// MVSK_TUNE="Q,G,RG,S,OCC" (0 = heuristic) overrides the plan; used by the
// tuning sweep only (scripts/tune_stream.py)
struct TuneOverride {
    int Q = 0, G = 0, RG = 0, S = 0, OCC = 0, VS = -1;
};
TuneOverride tune_override() {
    TuneOverride t;
    if (const char* e = std::getenv("MVSK_TUNE"))
        std::sscanf(e, "%d,%d,%d,%d,%d,%d", &t.Q, &t.G, &t.RG, &t.S, &t.OCC, &t.VS);
    return t;
}

// wide-row plan for short panels: the input vector in shared memory, Q = 16
// column pairs per thread, two row teams per CTA (MVSK_TUNE 6th field: 1/0
// forces it on / off for the ops that have it)
// An A/B variant (MVSK_TUNE 6th field = 1): it beat the one-row plan for
// f+grad at C4 (50.6 -> 46.6 us) but two rows per team in registers beat both
// (42.6 us; profiles/r02_tune_c4_vs.txt), so it is not a default
bool make_plan_vs(const mvsk_gpu_ctx* ctx, Op op, int K, const TuneOverride& tov, Plan& pl) {
    const long long npairs = ctx->ld / 2;
    const bool want = tov.VS == 1;
    // the same width range as every other op of this build (n <= 8192)
    if (!want || npairs > 4096) return false;
    const int Q = tov.Q > 0 ? tov.Q : 16;
    const int RG = tov.RG > 0 ? tov.RG : 1;
    if (!select_kernel_vs(op, K, Q, RG)) return false;
    const int P = round_team((int)((npairs + Q - 1) / Q));
    const int mt = max_threads(op, K, Q, RG, true);
    int G = tov.G > 0 ? tov.G : std::max(1, std::min(4, mt / P));
    if (G * P > mt) return false;
    const size_t row_bytes = (size_t)ctx->ld * sizeof(double);
    const size_t stage_bytes = ((size_t)G * RG * row_bytes + 127) & ~(size_t)127;
    const int ndot = op_ndot(op, K), nacc = op_nacc(op, K);
    const int nwp = P >= 32 ? P / 32 : 1;
    const size_t red_bytes = (((size_t)2 * G * RG * std::max(ndot, 1) * nwp * sizeof(double)) + 127) & ~(size_t)127;
    const size_t vs_bytes = ((size_t)ndot * ctx->ld * sizeof(double) + 127) & ~(size_t)127;
    const size_t combine = ((size_t)G * std::max(nacc, 1) * ctx->ld + 16 + (size_t)G * 16) * sizeof(double);
    const size_t combine_all = std::max(combine, (size_t)(G * P) * sizeof(double));
    const int nst_total = (int)std::max<long long>(1, (ctx->T_local + G * RG - 1) / (G * RG));
    int S = tov.S >= 2 ? tov.S : 3;
    S = std::min(S, std::max(2, nst_total));
    auto smem_of = [&](int s) { return 128 + red_bytes + vs_bytes + std::max((size_t)s * stage_bytes, combine_all); };
    while (S > 2 && smem_of(S) > ctx->max_smem) --S;
    if (smem_of(S) > ctx->max_smem) return false;
    pl.Q = Q;
    pl.P = P;
    pl.G = G;
    pl.RG = RG;
    pl.S = S;
    pl.VS = true;
    pl.smem = smem_of(S);
    pl.fn = select_kernel_vs(op, K, Q, RG);
    pl.nb = (int)std::min<long long>(ctx->nsm, std::max<long long>(1, (ctx->T_local + G * RG - 1) / (G * RG)));
    return true;
}

// Launch plan. Measured on B200 at C5 (profiles/r01_tune_c5.txt): teams of
// <= 256 threads (8 column pairs each at n=4096), two teams per CTA on
// different rows, a 2-deep ring of 64 KB stages -> 7.1-7.4 TB/s streamed.
bool make_plan(const mvsk_gpu_ctx* ctx, Op op, int K, Plan& pl) {
    const TuneOverride tov = tune_override();
    if (make_plan_vs(ctx, op, K, tov, pl)) return true;
    const long long npairs = ctx->ld / 2;
    const int qmax = max_q(op, K);
    // small panels (< 64 rows per SM) are latency-bound: favour short teams and
    // several teams per CTA so more rows are in flight (C3: 63 -> 34 us / HVP)
    const bool small = ctx->T_local < 64LL * ctx->nsm;
    int Q = -1;
    if (small) {
        // short teams, many of them: the most column pairs per thread that
        // fits, so up to 16 teams share a CTA and a CTA's few rows are in
        // flight in one or two stages (profiles/r01_tune_small_panels.txt:
        // T=5000 n=64 12.3 -> 8.3 us, n=256 15.4 -> 10.3 us per HVP)
        for (int q = qmax; q >= 1 && Q < 0; q >>= 1)
            if (round_team((int)((npairs + q - 1) / q)) <= max_threads(op, K, q, 1) && select_kernel(op, K, q, 1))
                Q = q;
    }
    for (int q = 1; Q < 0 && q <= qmax; q <<= 1)
        if ((npairs + q - 1) / q <= 256) {
            Q = q;
            break;
        }
    if (Q < 0)
        for (int q = 1; q <= qmax; q <<= 1)
            if ((npairs + q - 1) / q <= max_threads(op, K, q, 1)) {
                Q = q;
                break;
            }
    if (tov.Q > 0 && tov.Q <= qmax && (npairs + tov.Q - 1) / tov.Q <= max_threads(op, K, tov.Q, 1)) Q = tov.Q;
    if (Q < 0) return false;
    const int P = round_team((int)((npairs + Q - 1) / Q));
    if (P > max_threads(op, K, Q, 1)) return false;
    const size_t row_bytes = (size_t)ctx->ld * sizeof(double);
    const size_t stage_target = 64 * 1024;
    // teams per CTA (each team streams its own rows)
    int G = small ? std::max(1, std::min(16, max_threads(op, K, Q, 1) / P))
                  : std::max(1, max_threads(op, K, Q, 1) / P);
    const long long want_rows = std::max<long long>(1, (long long)(stage_target / row_bytes));
    while (G > 1 && G > want_rows) G >>= 1;
    int RG = 1;
    while (!small && RG < 4 && RG * 2 * Q <= 8 && (long long)G * RG * 2 <= want_rows &&
           G * P <= max_threads(op, K, Q, RG * 2))
        RG <<= 1;
    if (small) {  // enough rows per stage to cover a CTA's share in one stage
        const long long rows_cta = (ctx->T_local + ctx->nsm - 1) / ctx->nsm;
        while (RG < 4 && (long long)G * RG < rows_cta && RG * 2 * Q <= 8 && G * P <= max_threads(op, K, Q, RG * 2) &&
               select_kernel(op, K, Q, RG * 2) && (long long)G * RG * 2 <= want_rows)
            RG <<= 1;
    }
    // a heavy op whose team fills the CTA (THIRD, 2-RHS HVP at n=4096) would
    // otherwise keep one row in flight per CTA and expose the per-row reduction
    // latency (C5 third: 8 warps/SM, 'wait' + short-scoreboard stalls); two rows
    // per team interleave two independent chains
    if (!small && G == 1 && RG == 1 && Q == 8 && P <= max_threads(op, K, Q, 2) &&
        select_kernel(op, K, Q, 2) != nullptr && want_rows >= 2)
        RG = 2;
    // short panels of wide rows (C4: 34 rows of 40 KB per SM, one 320-thread team):
    // two rows per team per stage interleave two reduction chains (f+grad
    // 48.3 -> 42.6 us, HVP 44.5 -> 40.5, line sums 40.4 -> 38.9;
    // profiles/r02_tune_c4_vs.txt)
    if (small && G == 1 && RG == 1 && Q == 8 && P >= 256 && select_kernel(op, K, 8, 2) &&
        G * P <= max_threads(op, K, 8, 2) && want_rows >= 1)
        RG = 2;
    if (tov.G > 0 && tov.G * P <= max_threads(op, K, Q, RG)) G = tov.G;
    if (tov.RG > 0 && (tov.RG * Q <= 8 || select_kernel(op, K, Q, tov.RG)) && G * P <= max_threads(op, K, Q, tov.RG))
        RG = tov.RG;
    if (op == Op::HVP && K == 4 && Q == 2) RG = 1;
    if (G * P > max_threads(op, K, Q, RG)) return false;
    const long long R = (long long)G * RG;
    const size_t stage_bytes = ((size_t)R * row_bytes + 127) & ~(size_t)127;
    const int nst_total = (int)std::max<long long>(1, (ctx->T_local + R - 1) / R);
    // one team: a deeper ring hides the per-row latency (C5: third 2.28 -> 1.80 ms,
    // 2-RHS HVP 2.44 -> 1.85 ms); two teams already overlap two rows per stage
    int S = (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, (G == 1 ? 128 * 1024 : 64 * 1024) / stage_bytes));
    if (tov.S >= 2 && tov.S <= kMaxStages) S = tov.S;
    S = std::min(S, std::max(2, nst_total));
    // team-combine and scalar scratch live in the ring after the last stage
    const int nacc = op_nacc(op, K);
    const int ndot = op_ndot(op, K);
    const int nwp = P >= 32 ? P / 32 : 1;
    const size_t red_bytes = (((size_t)2 * R * std::max(ndot, 1) * nwp * sizeof(double)) + 127) & ~(size_t)127;
    const size_t combine = ((size_t)G * std::max(nacc, 1) * ctx->ld + 16 + (size_t)G * 16) * sizeof(double);
    // the fused finish reuses the ring as a [threads] fp64 scratch
    const size_t combine_all = std::max(combine, (size_t)(G * P) * sizeof(double));
    size_t ring = std::max((size_t)S * stage_bytes, combine_all);
    pl.smem = 128 + red_bytes + ring;
    while (pl.smem > ctx->max_smem && S > 2) {
        --S;
        ring = std::max((size_t)S * stage_bytes, combine_all);
        pl.smem = 128 + red_bytes + ring;
    }
    if (pl.smem > ctx->max_smem) return false;
    pl.Q = Q;
    pl.P = P;
    pl.G = G;
    pl.RG = RG;
    pl.S = S;
    pl.fn = select_kernel(op, K, Q, RG);
    if (!pl.fn) return false;
    const int threads = G * P;
    int occ = (int)std::min<size_t>(4, (ctx->max_smem + 1024) / (pl.smem + 1024));
    occ = std::max(1, std::min(occ, 2048 / threads));
    if (small) occ = 1;  // fewer CTA partials: the cross-CTA reduction dominates small panels
    if (tov.OCC > 0) occ = std::min(occ, tov.OCC);
    const long long want_blocks = std::max<long long>(1, (ctx->T_local + R - 1) / R);
    pl.nb = (int)std::min<long long>((long long)ctx->nsm * occ, want_blocks);
    return true;
}

// ---- cluster column-split plans (multi-RHS HVP / THIRD) ------------------------
struct CPlan {
    int C = 4, Q = 1, RG = 1, P = 256, S = 2;
    size_t smem = 0;
    int ncl = 1;
    const void* fn = nullptr;
};

template <Op OP, int K, int Q, int RG>
const void* cfn() {
    return reinterpret_cast<const void*>(&stream_cluster_kernel<OP, K, Q, RG>);
}

// instantiated (K, Q, RG): the pipelined kernel keeps two copies of the staged
// row slice, so the register budget (<= 255) bounds Q * RG per K
const void* select_cluster(Op op, int K, int Q, int RG) {
    if (op == Op::HVP && K == 8) {
        if (Q == 1 && RG == 4) return cfn<Op::HVP, 8, 1, 4>();
        if (Q == 1 && RG == 2) return cfn<Op::HVP, 8, 1, 2>();
        if (Q == 2 && RG == 2) return cfn<Op::HVP, 8, 2, 2>();
        if (Q == 2 && RG == 1) return cfn<Op::HVP, 8, 2, 1>();
    } else if (op == Op::HVP && K == 4) {
        if (Q == 1 && RG == 4) return cfn<Op::HVP, 4, 1, 4>();
        if (Q == 2 && RG == 4) return cfn<Op::HVP, 4, 2, 4>();
        if (Q == 2 && RG == 2) return cfn<Op::HVP, 4, 2, 2>();
        if (Q == 4 && RG == 2) return cfn<Op::HVP, 4, 4, 2>();
        if (Q == 4 && RG == 1) return cfn<Op::HVP, 4, 4, 1>();
    } else if (op == Op::THIRD && K == 8) {
        if (Q == 1 && RG == 2) return cfn<Op::THIRD, 8, 1, 2>();
        if (Q == 1 && RG == 1) return cfn<Op::THIRD, 8, 1, 1>();
    } else if (op == Op::THIRD && K == 4) {
        if (Q == 1 && RG == 4) return cfn<Op::THIRD, 4, 1, 4>();
        if (Q == 2 && RG == 2) return cfn<Op::THIRD, 4, 2, 2>();
        if (Q == 2 && RG == 1) return cfn<Op::THIRD, 4, 2, 1>();
    }
    return nullptr;
}

bool make_cluster_plan(const mvsk_gpu_ctx* ctx, Op op, int K, CPlan& pl) {
    int forceC = 0, forceRG = 0;
    if (const char* e = std::getenv("MVSK_TUNE_CLUSTER")) std::sscanf(e, "%d,%d", &forceC, &forceRG);
    const int ndot = op == Op::THIRD ? 2 * K : K;
    const int Cs[3] = {4, 8, 2};
    for (int ci = 0; ci < 3; ++ci) {
        const int C = forceC ? forceC : Cs[ci];
        if (ctx->ld % (2 * C)) {
            if (forceC) return false;
            continue;
        }
        const int cw = (int)(ctx->ld / C);
        const int npc = cw / 2;
        int Q = 1;
        while (Q < 4 && (npc + Q - 1) / Q > 256) Q <<= 1;
        if ((npc + Q - 1) / Q > 256) {
            if (forceC) return false;
            continue;
        }
        int RG = 4;
        while (RG > 1 && (RG * ndot > 32 || !select_cluster(op, K, Q, RG))) RG >>= 1;
        if (forceRG && select_cluster(op, K, Q, forceRG) && forceRG * ndot <= 32) RG = forceRG;
        const void* fn = select_cluster(op, K, Q, RG);
        if (!fn) {
            if (forceC) return false;
            continue;
        }
        const int V = RG * ndot;
        const size_t stage = ((size_t)RG * cw * sizeof(double) + 127) & ~(size_t)127;
        int S = (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, (128 * 1024) / stage));
        size_t head = 256 + (size_t)(2 * V * 8 + kXSlots * 16 * V + 2 * V) * sizeof(double);
        head = (head + 127) & ~(size_t)127;
        while (S > 2 && head + S * stage > ctx->max_smem) --S;
        if (head + S * stage > ctx->max_smem) {
            if (forceC) return false;
            continue;
        }
        pl.C = C;
        pl.Q = Q;
        pl.RG = RG;
        pl.P = 256;
        pl.S = S;
        pl.smem = head + S * stage;
        pl.fn = fn;
        pl.ncl = std::max(1, ctx->nsm / C);
        return true;
    }
    return false;
}

// ---- DMMA cluster plans (multi-RHS HVP / THIRD on the fp64 tensor cores) -------
struct DPlan {
    int C = 4, WC = 128, S = 3, threads = 256;
    size_t smem = 0;
    int ncl = 1;
    const void* fn = nullptr;
};

template <Op OP, int K, int WC, int D>
const void* dfn() {
    return reinterpret_cast<const void*>(&stream_dmma_kernel<OP, K, WC, D>);
}

const void* select_dmma(Op op, int K, int WC, int D) {
#define MVSK_DWC(OP, K, D)                                 \
    if (WC == 32) return dfn<OP, K, 32, D>();               \
    if (WC == 64) return dfn<OP, K, 64, D>();               \
    if (WC == 80) return dfn<OP, K, 80, D>();               \
    if (WC == 128) return dfn<OP, K, 128, D>();
    if (D == 0) {
        if (op == Op::HVP && K == 8) {
            MVSK_DWC(Op::HVP, 8, 0)
            if (WC == 160) return dfn<Op::HVP, 8, 160, 0>();
        }
        if (op == Op::HVP && K == 4) { MVSK_DWC(Op::HVP, 4, 0) }
        if (op == Op::THIRD && K == 4) { MVSK_DWC(Op::THIRD, 4, 0) }
        if (op == Op::THIRD && K == 8) {
            if (WC == 64) return dfn<Op::THIRD, 8, 64, 0>();
            if (WC == 80) return dfn<Op::THIRD, 8, 80, 0>();
            if (WC == 128) return dfn<Op::THIRD, 8, 128, 0>();
        }
    }
    if (D == 1) {
        if (op == Op::HVP && K == 8) { MVSK_DWC(Op::HVP, 8, 1) }
        if (op == Op::HVP && K == 4) { MVSK_DWC(Op::HVP, 4, 1) }
        if (op == Op::THIRD && K == 4) { MVSK_DWC(Op::THIRD, 4, 1) }
        if (op == Op::THIRD && K == 8) {
            if (WC == 32) return dfn<Op::THIRD, 8, 32, 1>();
            if (WC == 64) return dfn<Op::THIRD, 8, 64, 1>();
            if (WC == 80) return dfn<Op::THIRD, 8, 80, 1>();
        }
    }
#undef MVSK_DWC
    return nullptr;
}

template <Op OP, int K, int WC, int C, bool F2REG = true>
const void* wfn() {
    return reinterpret_cast<const void*>(&stream_dmma_ws_kernel<OP, K, WC, C, F2REG>);
}

// warp-specialised variant (stream_dmma_ws_kernel): 8 math warps + a helper
// warpgroup. 4-CTA clusters with 64/128-column warp slices; 8-CTA clusters
// (64/80-column slices) where a 4-CTA split would not fit the registers: the
// 8 third-action pairs at n = 4096, and n = 5000 (C4)
const void* select_dmma_ws(Op op, int K, int WC, int C) {
    if (C == 4) {
        if (op == Op::HVP && K == 8) {
            if (WC == 64) return wfn<Op::HVP, 8, 64, 4>();
            if (WC == 128) return wfn<Op::HVP, 8, 128, 4>();
        }
        if (op == Op::HVP && K == 4) {
            if (WC == 64) return wfn<Op::HVP, 4, 64, 4>();
            if (WC == 128) return wfn<Op::HVP, 4, 128, 4>();
        }
        if (op == Op::THIRD && K == 4) {
            if (WC == 64) return wfn<Op::THIRD, 4, 64, 4>();
            if (WC == 128) return wfn<Op::THIRD, 4, 128, 4>();
        }
        if (op == Op::THIRD && K == 8) {  // 128-column slices: phase 2 from the ring (registers)
            if (WC == 64) return wfn<Op::THIRD, 8, 64, 4>();
            if (WC == 128) return wfn<Op::THIRD, 8, 128, 4, false>();
        }
    }
    if (C == 8) {
        if (op == Op::HVP && K == 8 && WC == 80) return wfn<Op::HVP, 8, 80, 8>();
        if (op == Op::HVP && K == 4 && WC == 80) return wfn<Op::HVP, 4, 80, 8>();
        if (op == Op::THIRD && K == 4 && WC == 80) return wfn<Op::THIRD, 4, 80, 8>();
        if (op == Op::THIRD && K == 8) {
            if (WC == 64) return wfn<Op::THIRD, 8, 64, 8>();
            if (WC == 80) return wfn<Op::THIRD, 8, 80, 8>();
        }
    }
    return nullptr;
}

bool make_dmma_ws_plan(const mvsk_gpu_ctx* ctx, Op op, int K, DPlan& pl) {
    const int ndot = op == Op::THIRD ? 2 * K : K;
    const int V = 8 * ndot;
    int forceC = 0;
    if (const char* e = std::getenv("MVSK_DMMA_WS_C")) forceC = std::atoi(e);
    // 8-CTA clusters only for small panels (< 64 rows per SM, latency-bound):
    // at C5 the 8 third-action pairs run 3.77 ms there vs 2.68 ms on v1, at C4
    // (T = 5000) the 4-RHS ops gain 25-30 % and the 8 pairs 4 %; the 8-RHS HVP
    // at C4 is 6 % faster on v1 (profiles/r01_dmma_pipe.txt)
    const bool small = ctx->T_local < 64LL * ctx->nsm;
    for (int C : {4, 8}) {
        if (forceC && C != forceC) continue;
        if (!forceC && C == 8 && (!small || (op == Op::HVP && K == 8))) continue;
        if (ctx->ld % (2 * C)) continue;
        const int cw = (int)(ctx->ld / C);
        int WC = 0;
        for (int w : {64, 80, 128})
            if (!WC && 8 * w >= cw && select_dmma_ws(op, K, w, C)) WC = w;
        if (!WC) continue;
        const size_t stage = (size_t)8 * kWsRowStride(WC) * sizeof(double);
        size_t head = 256 + (size_t)(2 * 8 * V + 4 * C * V + 128) * sizeof(double);
        head = (head + 127) & ~(size_t)127;
        const int S = (int)std::min<size_t>(8, (ctx->max_smem - head) / stage);
        if (S < 2) continue;
        pl.C = C;
        pl.WC = WC;
        pl.S = S;
        pl.threads = 384;
        pl.smem = head + (size_t)S * stage;
        pl.fn = select_dmma_ws(op, K, WC, C);
        pl.ncl = std::max(1, ctx->nsm / C);
        return true;
    }
    return false;
}

bool make_dmma_plan(const mvsk_gpu_ctx* ctx, Op op, int K, DPlan& pl) {
    if (std::getenv("MVSK_NO_DMMA")) return false;
    // warp-specialised kernel first (C5 8-RHS HVP 1.41 ms vs 2.23 v1,
    // profiles/r01_dmma_pipe.txt, r02_dmma_row_swizzle_ab.txt); v1 serves the
    // shapes the warp-specialised kernel has no instantiation for (160-column
    // slices at n = 5000) and MVSK_DMMA_V1 forces it for A/B runs
    const bool v1 = std::getenv("MVSK_DMMA_V1") || std::getenv("MVSK_TUNE_DMMA");
    if (!v1 && make_dmma_ws_plan(ctx, op, K, pl)) return true;
    int forceC = 0, forceD = 0;
    if (const char* e = std::getenv("MVSK_TUNE_DMMA")) std::sscanf(e, "%d,%d", &forceC, &forceD);
    const int ndot = op == Op::THIRD ? 2 * K : K;
    const int V = 8 * ndot;
    const int Cs[4] = {4, 8, 2, 1};
    for (int i = 0; i < 4; ++i) {
        const int C = forceC ? forceC : Cs[i];
        if (ctx->ld % (2 * C)) {
            if (forceC) return false;
            continue;
        }
        const int cw = (int)(ctx->ld / C);
        int WC = 0;
        for (int w : {32, 64, 80, 128, 160})
            if (!WC && 8 * w >= cw && select_dmma(op, K, w, forceD < 0 ? 0 : (forceD > 0 ? forceD : 0))) WC = w;
        if (!WC)
            for (int w : {32, 64, 80, 128, 160})
                if (!WC && 8 * w >= cw && select_dmma(op, K, w, 1)) WC = w;
        if (!WC) {
            if (forceC) return false;
            continue;
        }
        const size_t stage = (size_t)8 * (8 * WC + 4) * sizeof(double);
        // exchange depth D: produce(s + D) runs before consume(s). D = 0 frees a
        // ring slot one phase earlier (two fills in flight with S = 3 at cw = 1024)
        // and measured 1-4 % faster than D = 1 (C5 hvp8 2.30 vs 2.39 ms, C4 third8
        // 0.120 vs 0.124 ms, profiles/r01_tune_dmma_depth.txt); D = 2 was no faster
        int D = 0;
        const void* fn = nullptr;
        int S = 0;
        size_t head = 0;
        for (int d : {0, 1}) {
            if (fn || (forceD > 0 && d != forceD) || (forceD < 0 && d != 0)) continue;  // -1 forces D = 0
            const void* f = select_dmma(op, K, WC, d);
            if (!f) continue;
            size_t h = 256 + (size_t)(8 * V + (2 * d + 2) * C * V + 2 * V) * sizeof(double);
            h = (h + 127) & ~(size_t)127;
            const int s = (int)std::min<size_t>(6, (ctx->max_smem - h) / stage);
            if (s < d + 2) continue;
            fn = f;
            D = d;
            S = s;
            head = h;
        }
        if (!fn) {
            if (forceC) return false;
            continue;
        }
        (void)D;
        pl.C = C;
        pl.WC = WC;
        pl.S = S;
        pl.smem = head + (size_t)S * stage;
        pl.fn = fn;
        pl.ncl = std::max(1, ctx->nsm / C);
        return true;
    }
    return false;
}



constexpr int kFinThreads = 256;
__global__ void __launch_bounds__(kFinThreads) finish_kernel(const FinishArgs f, int ng) {
    if (pass_skipped(f.skip, f.nskip)) return;
    __shared__ double part[kFinThreads];
    finish_block(f, ng, blockIdx.x, threadIdx.x, kFinThreads, part);
}

__global__ void psi2_kernel(const double* z, double* out, long long T, double c2, double c3, double c4) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
        const double zt = z[t];
        out[t] = 2.0 * c2 - 6.0 * c3 * zt + 12.0 * c4 * (zt * zt);  // oracle.hpp:116-119
    }
}

void ensure_part(mvsk_gpu_ctx* ctx, size_t elems) {
    if (ctx->part_acc_elems >= elems) return;
    if (ctx->part_acc) MVSK_CUDA(cudaFree(ctx->part_acc));
    ctx->part_acc = nullptr;
    MVSK_CUDA(cudaMalloc(&ctx->part_acc, elems * sizeof(double)));
    ctx->part_acc_elems = elems;
    ++ctx->epoch;
}

}  // namespace

namespace {
std::mutex g_attr_mu;
}

// cudaFuncSetAttribute once per (device, kernel, size): a driver call, not free,
// and per-device (one process may drive several GPUs)
static bool cluster_fits_query(const void* fn, int cs, int threads, size_t smem);

// whether at least one cluster of `cs` CTAs x `threads` with `smem` bytes of
// dynamic shared memory can be resident (non-portable sizes need the opt-in
// attribute; MIG / MPS partitions may not fit one): the cluster-resident
// kernels fall back to their launch-per-step paths when it cannot
bool cluster_fits(const void* fn, int cs, int threads, size_t smem) {
    struct Entry {
        int dev;
        const void* fn;
        int cs, threads;
        size_t smem;
        bool ok;
    };
    static std::vector<Entry> seen;  // answers cached per device / kernel / shape
    static std::mutex mu;
    int dev = 0;
    MVSK_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Entry& e : seen)
            if (e.dev == dev && e.fn == fn && e.cs == cs && e.threads == threads && e.smem == smem) return e.ok;
    }
    const bool ok = cluster_fits_query(fn, cs, threads, smem);
    std::lock_guard<std::mutex> lk(mu);
    seen.push_back({dev, fn, cs, threads, smem, ok});
    return ok;
}

static bool cluster_fits_query(const void* fn, int cs, int threads, size_t smem) {
    if (cs > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    set_smem_attr(fn, smem);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int maxcl = 0;
    if (cudaOccupancyMaxActiveClusters(&maxcl, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return maxcl > 0;
}

void set_smem_attr(const void* fn, size_t smem) {
    struct Entry {
        int dev;
        const void* fn;
        size_t smem;
    };
    static std::vector<Entry> done;
    int dev = 0;
    MVSK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (auto& d : done)
        if (d.dev == dev && d.fn == fn) {
            if (d.smem >= smem) return;
            MVSK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            d.smem = smem;
            return;
        }
    MVSK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done.push_back({dev, fn, smem});
}

void ensure_host_staging(mvsk_gpu_ctx* ctx, size_t elems) {
    if (ctx->h_elems >= elems) return;
    if (ctx->h_in) cudaFreeHost(ctx->h_in);
    if (ctx->h_out) cudaFreeHost(ctx->h_out);
    ctx->h_in = ctx->h_out = ctx->h_out_dev = nullptr;
    MVSK_CUDA(cudaMallocHost(&ctx->h_in, elems * sizeof(double)));
    // results come back through the mapped alias (PassIO::hout): the epilogue
    // writes them over the bus, no device-to-host copy node per op
    MVSK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_out), elems * sizeof(double), cudaHostAllocMapped));
    MVSK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->h_out_dev), ctx->h_out, 0));
    ctx->h_elems = elems;
    ++ctx->epoch;
}

static void run_single(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io);
static bool run_cluster(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io);
static bool run_dmma(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io);

void run_pass(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io) {
    if ((op == Op::HVP || op == Op::THIRD) && k > 1) {
        // widest supported RHS block per pass: cluster column-split for 8 / 4,
        // single-CTA rows for 2 / 1; chunked over k
        int done = 0;
        while (done < k) {
            const int left = k - done;
            PassIO sub = io;
            sub.vin = io.vin + (size_t)done * ctx->ld;
            if (io.vin2) sub.vin2 = io.vin2 + (size_t)done * ctx->ld;
            sub.out = io.out + (size_t)done * io.ldo;
            if (io.hout) sub.hout = io.hout + (size_t)done * io.ldo;
            int kk = 0;
            // narrow panels (compact faces, ld <= 256): the k-RHS pass as one
            // cooperative streaming kernel (fused reduction) beats the cluster
            // tensor-core kernel, whose per-stage exchange dominates tiny rows
            if (ctx->ld <= 256)
                for (int w : {8, 4}) {
                    Plan tmp;
                    if (!kk && left >= w && make_plan(ctx, op, w, tmp)) {
                        run_single(ctx, op, w, sub);
                        kk = w;
                    }
                }
            for (int w : {8, 4})
                if (!kk && left >= w && run_dmma(ctx, op, w, sub)) kk = w;
            for (int w : {8, 4})
                if (!kk && left >= w && run_cluster(ctx, op, w, sub)) kk = w;
            if (!kk) {
                kk = (op == Op::HVP && left >= 2) ? 2 : 1;
                Plan tmp;
                while (kk > 1 && !make_plan(ctx, op, kk, tmp)) kk >>= 1;
                run_single(ctx, op, kk, sub);
            }
            done += kk;
        }
        return;
    }
    run_single(ctx, op, k, io);
}

// cross-CTA (or cross-cluster) fixed-order reduction, allreduce over the
// row-shard group, and the op epilogue
static FinishArgs finish_args(mvsk_gpu_ctx* ctx, Op op, int nacc, int nb, const PassIO& io, Slot* slot) {
    FinishArgs f{};
    f.op = (int)op;
    f.k = op == Op::LINESUMS ? 0 : std::max(nacc, 1);
    f.ld = (int)ctx->ld;
    f.n = (int)ctx->n;
    f.ldo = io.ldo;
    f.nb = ctx->T_local > 0 ? nb : 0;
    f.part_acc = ctx->part_acc;
    f.part_sc = ctx->part_sc;
    f.red = ctx->red;
    f.out = io.out;
    f.mu = ctx->mu_dev;
    f.x = io.x_for_mux;
    f.c1 = ctx->c.c1;
    f.c2 = ctx->c.c2;
    f.c3 = ctx->c.c3;
    f.c4 = ctx->c.c4;
    f.T = (double)ctx->T_global;
    f.value_offset = ctx->value_offset;
    f.value_offset_dev = ctx->value_offset_dev;
    f.skip = io.skip;
    f.nskip = io.nskip;
    f.hout = io.hout;
    if (slot) {
        f.g = slot->g;
        f.sc = slot->sc;
    }
    return f;
}

static int finish_groups(int nb) { return nb >= 512 ? 32 : nb >= 128 ? 8 : 4; }

// reduced: the CTA partials were already reduced into ctx->red inside the pass
// (cooperative launch with do_epi = 0); only the allreduce and epilogue remain
static void finish_pass(mvsk_gpu_ctx* ctx, Op op, int nacc, int nb, const PassIO& io, Slot* slot,
                        bool reduced = false) {
    FinishArgs f = finish_args(ctx, op, nacc, nb, io, slot);
    const int tot = std::max(f.k, 1) * f.ld;
    const int ng = finish_groups(nb);
    const int fb = std::max(1, (tot + kFinThreads / ng - 1) / (kFinThreads / ng));
    if (!is_sharded(ctx)) {
        f.do_reduce = 1;
        f.do_epi = 1;
        // scalars are reduced by block 0 and consumed by block 0 only
        ++ctx->launches;
        finish_kernel<<<fb, kFinThreads, 0, ctx->stream>>>(f, ng);
        MVSK_CUDA(cudaGetLastError());
    } else {
        if (!reduced) {
            f.do_reduce = 1;
            f.do_epi = 0;
            ++ctx->launches;
            finish_kernel<<<fb, kFinThreads, 0, ctx->stream>>>(f, ng);
            MVSK_CUDA(cudaGetLastError());
        }
        const int nsc = op == Op::FGRAD ? 3 : (op == Op::LINESUMS ? 9 : 0);
        const size_t cnt = (size_t)(op == Op::LINESUMS ? 0 : tot) + nsc;
        allreduce_sum(ctx, ctx->red, cnt);
        f.do_reduce = 0;
        f.do_epi = 1;
        ++ctx->launches;
        finish_kernel<<<fb, kFinThreads, 0, ctx->stream>>>(f, ng);
        MVSK_CUDA(cudaGetLastError());
    }
}

static bool run_cluster(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io) {
    CPlan pl;
    if (!make_cluster_plan(ctx, op, k, pl)) return false;
    set_smem_attr(pl.fn, pl.smem);
    // clusters that can be co-resident, at most one wave
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = pl.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(pl.P);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(pl.ncl * pl.C);
    int maxcl = 0;
    if (cudaOccupancyMaxActiveClusters(&maxcl, pl.fn, &cfg) == cudaSuccess && maxcl > 0)
        pl.ncl = std::min(pl.ncl, maxcl);
    else
        cudaGetLastError();
    pl.ncl = (int)std::max<long long>(1, std::min<long long>(pl.ncl, (ctx->T_local + pl.RG - 1) / pl.RG));
    cfg.gridDim = dim3(pl.ncl * pl.C);
    ensure_part(ctx, (size_t)pl.ncl * k * ctx->ld);
    ClusterArgs a{};
    a.X = ctx->X;
    a.T = ctx->T_local;
    a.ld = (int)ctx->ld;
    a.cw = (int)(ctx->ld / pl.C);
    a.P = pl.P;
    a.S = pl.S;
    a.evict_first = (size_t)ctx->T_local * ctx->ld * sizeof(double) > (size_t)96 * 1024 * 1024;
    a.vin = io.vin;
    a.vin2 = io.vin2;
    a.z = io.z;
    a.part_acc = ctx->part_acc;
    a.skip = io.skip;
    a.nskip = io.nskip;
    a.c2 = ctx->c.c2;
    a.c3 = ctx->c.c3;
    a.c4 = ctx->c.c4;
    if (ctx->T_local > 0) {
        void* args[] = {&a};
        ++ctx->launches;
        MVSK_CUDA(cudaLaunchKernelExC(&cfg, pl.fn, args));
    }
    ctx->phys += 1;
    finish_pass(ctx, op, k, pl.ncl, io, nullptr);
    return true;
}

static bool run_dmma(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io) {
    DPlan pl;
    if (!make_dmma_plan(ctx, op, k, pl)) return false;
    set_smem_attr(pl.fn, pl.smem);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = pl.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(pl.threads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(pl.ncl * pl.C);
    int maxcl = 0;
    if (cudaOccupancyMaxActiveClusters(&maxcl, pl.fn, &cfg) == cudaSuccess && maxcl > 0)
        pl.ncl = std::min(pl.ncl, maxcl);
    else
        cudaGetLastError();
    pl.ncl = (int)std::max<long long>(1, std::min<long long>(pl.ncl, (ctx->T_local + 7) / 8));
    cfg.gridDim = dim3(pl.ncl * pl.C);
    ensure_part(ctx, (size_t)pl.ncl * k * ctx->ld);
    DmmaArgs a{};
    a.X = ctx->X;
    a.T = ctx->T_local;
    a.ld = (int)ctx->ld;
    a.cw = (int)(ctx->ld / pl.C);
    a.S = pl.S;
    a.evict_first = (size_t)ctx->T_local * ctx->ld * sizeof(double) > (size_t)96 * 1024 * 1024;
    a.vin = io.vin;
    a.vin2 = io.vin2;
    a.z = io.z;
    a.part_acc = ctx->part_acc;
    a.skip = io.skip;
    a.nskip = io.nskip;
    a.c2 = ctx->c.c2;
    a.c3 = ctx->c.c3;
    a.c4 = ctx->c.c4;
    a.early_refill = 1;
    if (const char* e = std::getenv("MVSK_DMMA_EARLY")) a.early_refill = std::atoi(e);
    if (ctx->T_local > 0) {
        void* args[] = {&a};
        ++ctx->launches;
        MVSK_CUDA(cudaLaunchKernelExC(&cfg, pl.fn, args));
    }
    ctx->phys += 1;
    finish_pass(ctx, op, k, pl.ncl, io, nullptr);
    return true;
}

// MVSK_SMALL_PROF: per-phase cycle sums of CTA 0 of the one-cluster kernels
// (0: small_pass_kernel, 1: small_gram_kernel), printed at exit
static unsigned long long* small_prof(int which) {
    static const bool on = std::getenv("MVSK_SMALL_PROF") != nullptr;
    static unsigned long long* buf = nullptr;
    if (!on) return nullptr;
    if (!buf) {
        MVSK_CUDA(cudaMallocManaged(&buf, 16 * sizeof(unsigned long long)));
        std::memset(buf, 0, 16 * sizeof(unsigned long long));
        std::atexit([] {
            cudaDeviceSynchronize();
            for (int w = 0; w < 2; ++w) {
                const unsigned long long* p = buf + 8 * w;
                const double nn = p[5] ? (double)p[5] : 1.0;
                std::fprintf(stderr, "[%s] %llu launches, cycles/launch on CTA 0: %.0f | %.0f | %.0f | %.0f | %.0f\n",
                             w ? "small gram: load | tiles | reduce | exit" : "small pass: load | rows | combine | epilogue | exit",
                             p[5], p[0] / nn, p[1] / nn, p[2] / nn, p[3] / nn, p[4] / nn);
            }
        });
    }
    return buf + 8 * which;
}

template <Op OP>
static const void* small_pass_fn(int ld) {
    if (ld <= 32) return reinterpret_cast<const void*>(&small_pass_kernel<OP, 2, 16>);
    if (ld <= 64) return reinterpret_cast<const void*>(&small_pass_kernel<OP, 4, 16>);
    return reinterpret_cast<const void*>(&small_pass_kernel<OP, 8, 16>);
}

// the one-cluster pass (small_pass.cuh) when the whole local panel fits the
// cluster's shared memory: single rank, one right-hand side, ld <= 128
static bool run_small_pass(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io, Slot* slot) {
    static const bool off = std::getenv("MVSK_NO_SMALL_PASS") != nullptr;
    if (off || k != 1 || ctx->ld > kSpM || ctx->T_local < kSpCS) return false;
    const long long nloc = (ctx->T_local + kSpCS - 1) / kSpCS;
    const size_t smem = small_pass_smem(nloc, (int)ctx->ld);
    if (smem > ctx->max_smem) return false;
    const void* fn = nullptr;
    switch (op) {
    case Op::FGRAD: fn = small_pass_fn<Op::FGRAD>((int)ctx->ld); break;
    case Op::HVP: fn = small_pass_fn<Op::HVP>((int)ctx->ld); break;
    case Op::THIRD: fn = small_pass_fn<Op::THIRD>((int)ctx->ld); break;
    case Op::LINESUMS: fn = small_pass_fn<Op::LINESUMS>((int)ctx->ld); break;
    case Op::XTW: fn = small_pass_fn<Op::XTW>((int)ctx->ld); break;
    }
    if (!fn || !cluster_fits(fn, kSpCS, kSpW * 32, smem)) return false;
    set_smem_attr(fn, smem);
    SmallPassArgs a{};
    a.X = ctx->X;
    a.T = ctx->T_local;
    a.ld = (int)ctx->ld;
    a.vin = io.vin;
    a.vin2 = io.vin2;
    a.rowv = op == Op::FGRAD ? ctx->zoff_dev : (op == Op::XTW ? io.tw : io.z);
    a.zout = op == Op::FGRAD ? slot->z : io.zout;
    a.fin = finish_args(ctx, op, op == Op::LINESUMS ? 0 : 1, 1, io, slot);
    a.prof = small_prof(0);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kSpCS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kSpCS);
    cfg.blockDim = dim3(kSpW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&a};
    const bool sharded = is_sharded(ctx);
    a.fin.do_reduce = 0;
    a.fin.do_epi = sharded ? 0 : 1;
    MVSK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    ++ctx->launches;
    ctx->phys += 1;
    if (sharded) finish_pass(ctx, op, op == Op::LINESUMS ? 0 : 1, 1, io, slot, true);
    return true;
}

bool run_small_gram(mvsk_gpu_ctx* ctx, const double* z, double* G_dev, double scale, double* G_host, double* packed) {
    static const bool off = std::getenv("MVSK_NO_SMALL_PASS") != nullptr;
    if (off || !z || (is_sharded(ctx) && !packed) || ctx->ld > kSpM || ctx->T_local < kSpCS) return false;
    const long long nloc = (ctx->T_local + kSpCS - 1) / kSpCS;
    const size_t smem = small_gram_smem(nloc, (int)ctx->ld);
    const void* fn = reinterpret_cast<const void*>(&small_gram_kernel);
    if (smem > ctx->max_smem || !cluster_fits(fn, kSpCS, kSgW * 32, smem)) return false;
    set_smem_attr(fn, smem);
    SmallGramArgs a{};
    a.X = ctx->X;
    a.T = ctx->T_local;
    a.ld = (int)ctx->ld;
    a.n = (int)ctx->n;
    a.z = z;
    a.c2 = ctx->c.c2;
    a.c3 = ctx->c.c3;
    a.c4 = ctx->c.c4;
    a.scale = scale;
    a.G = G_dev;
    a.Gh = G_host;
    a.packed = packed;
    a.prof = small_prof(1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kSpCS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kSpCS);
    cfg.blockDim = dim3(kSgW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&a};
    MVSK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    ++ctx->launches;
    ctx->phys += 1;
    return true;
}

static void run_single(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io) {
    if (run_small_pass(ctx, op, k, io, op == Op::FGRAD ? &ctx->slots[io.slot] : nullptr)) return;
    Plan pl;
    if (!make_plan(ctx, op, k, pl))
        throw ApiError(MVSK_DIMENSION_ERROR, "no streaming-kernel plan for n=" + std::to_string(ctx->n) +
                                                 " (this build supports n <= 8192)");
    const int nacc = (op == Op::HVP || op == Op::THIRD) ? k : (op == Op::LINESUMS ? 0 : 1);
    ensure_part(ctx, (size_t)pl.nb * std::max(nacc, 1) * ctx->ld);
    set_smem_attr(pl.fn, pl.smem);

    StreamArgs a{};
    a.X = ctx->X;
    a.T = ctx->T_local;
    a.ld = (int)ctx->ld;
    a.npairs = (int)(ctx->ld / 2);
    a.P = pl.P;
    a.G = pl.G;
    a.RG = pl.RG;
    a.S = pl.S;
    a.evict_first = (size_t)ctx->T_local * ctx->ld * sizeof(double) > (size_t)96 * 1024 * 1024;
    a.vin = io.vin;
    a.vin2 = io.vin2;
    a.z = (op == Op::FGRAD) ? ctx->zoff_dev : io.z;
    a.tw = io.tw;
    a.part_acc = ctx->part_acc;
    a.part_sc = ctx->part_sc;
    a.skip = io.skip;
    a.nskip = io.nskip;
    a.c2 = ctx->c.c2;
    a.c3 = ctx->c.c3;
    a.c4 = ctx->c.c4;
    a.Tglob = (double)ctx->T_global;
    Slot* slot = nullptr;
    if (op == Op::FGRAD) {
        slot = &ctx->slots[io.slot];
        a.zout = slot->z;
    } else {
        a.zout = io.zout;
    }
    ctx->phys += 1;
    if (ctx->T_local <= 0) {
        finish_pass(ctx, op, nacc, pl.nb, io, slot);
        return;
    }
    // the cross-CTA reduction runs inside the stream kernel: a cooperative
    // launch (all CTAs co-resident by construction of the plan) lets the CTAs
    // reduce each other's partials after one grid barrier, which saves the
    // finish launch and its dependency gap (latency-bound small panels and
    // Krylov steps). Single rank: the epilogue runs there too; row-sharded
    // groups: the reduced buffer goes to the allreduce, then the epilogue kernel.
    const int threads = pl.G * pl.P;
    static const bool no_fuse = std::getenv("MVSK_NO_FUSED_FINISH") != nullptr;
    if (!no_fuse && threads % 32 == 0) {
        a.fused = 1;
        a.fin = finish_args(ctx, op, nacc, pl.nb, io, slot);
        a.fin.do_reduce = 1;
        a.fin.do_epi = is_sharded(ctx) ? 0 : 1;
        int ng = finish_groups(pl.nb);
        while (ng > 1 && threads / ng < 8) ng >>= 1;
        a.fin_ng = ng;
        const int cols = threads / ng;
        const int tot = std::max(a.fin.k, 1) * a.fin.ld;
        a.fin_nvb = std::max(1, (tot + cols - 1) / cols);
        void* args[] = {&a};
        const cudaError_t e =
            cudaLaunchCooperativeKernel(pl.fn, dim3(pl.nb), dim3(threads), args, pl.smem, ctx->stream);
        if (e == cudaSuccess) {
            ++ctx->launches;
            if (is_sharded(ctx)) finish_pass(ctx, op, nacc, pl.nb, io, slot, true);
            return;
        }
        if (e != cudaErrorCooperativeLaunchTooLarge) MVSK_CUDA(e);
        cudaGetLastError();  // not co-resident with this plan: separate finish
        a.fused = 0;
    }
    {
        void* args[] = {&a};
        ++ctx->launches;
        MVSK_CUDA(cudaLaunchKernel(pl.fn, dim3(pl.nb), dim3(threads), args, pl.smem, ctx->stream));
    }
    finish_pass(ctx, op, nacc, pl.nb, io, slot);
}

void run_psi2(mvsk_gpu_ctx* ctx, const double* z, double* out, long long T) {
    if (T <= 0) return;
    const int nb = (int)std::min<long long>(4 * ctx->nsm, (T + 255) / 256);
    ++ctx->launches;
    psi2_kernel<<<nb, 256, 0, ctx->stream>>>(z, out, T, ctx->c.c2, ctx->c.c3, ctx->c.c4);
    MVSK_CUDA(cudaGetLastError());
}

}  // namespace mvsk_b200
