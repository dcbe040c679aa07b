// C++ host driver over the device oracle: the YAND direction
// (affine_normal.hpp:127-245) and the Algorithm-1 solve driver
// (solver.hpp:116-655), restated B200-first:
//   * faces are index maps over the resident panel (no T x nf column gather,
//     solver.hpp:343-363): the face cache at x_f IS the full cache at the
//     merged point, so pins/releases cost nothing on the device;
//   * the Hutchinson probe CGs (affine_normal.hpp:227-237) and the Jacobi
//     probes (:197-209) run in lockstep, so every CG step issues ONE k-RHS
//     fused HVP pass instead of k sequential 2-pass HVPs; per-column CG
//     arithmetic is exactly cg_capped's (:85-113);
//   * the direct branch (:151-188) assembles G = A_F^T diag(psi'') A_F / T
//     on the fp64 tensor cores and reduces M = (UQ)^T G (UQ) with the
//     Householder structure on the host (O(n^2) + the mm^3 LU); h = (UQ)^T G U nu needs
//     no extra pass; a = (UQ)^T A^T(psi''' o q) / T with q_t = a_t^T P a_t.
// Host geometry (O(n) Householder applies, projections) stays on the host.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>

#include "host_ops.hpp"
#include "pcg_device.hpp"
#include "spg_device.hpp"

namespace mvsk_b200 {
namespace {

// ---- optional host-side profile of a solve (MVSK_PROFILE=1 -> stderr) --------
struct Prof {
    bool on = false;
    double proj = 0, dir = 0, cache = 0, grad = 0, line = 0, total = 0, face = 0, resid = 0, spg = 0;
    double dgram = 0, dquad = 0, dlu = 0;  // direct branch: Gram / trace round trips, host LU + inverse + P
    long nproj = 0, ndir = 0, ncache = 0, nline = 0, nface = 0, nresid = 0;
};
Prof g_prof;
struct Tick {
    double& acc;
    std::chrono::steady_clock::time_point t0;
    explicit Tick(double& a) : acc(a), t0(std::chrono::steady_clock::now()) {}
    ~Tick() {
        if (g_prof.on) acc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
};

// ---- small dense helpers -----------------------------------------------------
double dot(const Vec& a, const Vec& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
double norm(const Vec& a) { return std::sqrt(dot(a, a)); }
double vsum(const Vec& a) {
    double s = 0.0;
    for (double v : a) s += v;
    return s;
}
double vmean(const Vec& a) { return vsum(a) / (double)a.size(); }
bool all_finite(const Vec& a) {
    for (double v : a)
        if (!std::isfinite(v)) return false;
    return true;
}
void axpy(Vec& y, double a, const Vec& x) {
    for (size_t i = 0; i < y.size(); ++i) y[i] += a * x[i];
}

// ---- SplitMix64 (rng.hpp:12-43): the Hutchinson / Jacobi probe streams ------
struct SplitMix64 {
    uint64_t s;
    explicit SplitMix64(uint64_t seed) : s(seed) {}
    uint64_t next_u64() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double next_sign() { return (next_u64() >> 63) ? 1.0 : -1.0; }
};

// ---- tangent basis U (simplex.hpp:22-78) and reduced frame Q (affine_normal.hpp:19-56)
struct Basis {
    long long n;
    Vec v;
    double beta;
    explicit Basis(long long nn) : n(nn), v((size_t)nn, -1.0 / std::sqrt((double)nn)) {
        if (nn < 2) throw ApiError(MVSK_DIMENSION_ERROR, "tangent basis needs n >= 2");
        v[0] += 1.0;
        beta = 2.0 / dot(v, v);
    }
    Vec apply(const Vec& y) const {  // U y
        Vec p((size_t)n);
        p[0] = 0.0;
        for (long long i = 1; i < n; ++i) p[(size_t)i] = y[(size_t)i - 1];
        const double s = beta * dot(v, p);
        for (size_t i = 0; i < p.size(); ++i) p[i] -= s * v[i];
        return p;
    }
    Vec apply_t(const Vec& x) const {  // U^T x
        const double s = beta * dot(v, x);
        Vec o((size_t)n - 1);
        for (long long i = 1; i < n; ++i) o[(size_t)i - 1] = x[(size_t)i] - s * v[(size_t)i];
        return o;
    }
};

struct Frame {
    Vec nu, v;
    double gn = 0, beta = 0;
    Vec apply_Q(const Vec& eta) const {
        Vec p(nu.size());
        p[0] = 0.0;
        for (size_t i = 1; i < p.size(); ++i) p[i] = eta[i - 1];
        const double s = beta * dot(v, p);
        for (size_t i = 0; i < p.size(); ++i) p[i] -= s * v[i];
        return p;
    }
    Vec apply_Qt(const Vec& w) const {
        const double s = beta * dot(v, w);
        Vec o(nu.size() - 1);
        for (size_t i = 1; i < nu.size(); ++i) o[i - 1] = w[i] - s * v[i];
        return o;
    }
};

Frame householder_frame(const Vec& g) {
    const double gn = norm(g);
    if (!(gn > 0)) throw ApiError(MVSK_DOMAIN_ERROR, "householder_frame: zero reduced gradient (stationary)");
    if (g.size() < 2) throw ApiError(MVSK_DIMENSION_ERROR, "householder_frame: need m >= 2");
    Frame f;
    f.gn = gn;
    f.nu = g;
    for (double& x : f.nu) x /= gn;
    const double s = f.nu[0] >= 0.0 ? 1.0 : -1.0;
    f.v = f.nu;
    f.v[0] += s;
    f.beta = 2.0 / dot(f.v, f.v);
    return f;
}

// ---- dense partial-pivot LU (the role of Eigen::PartialPivLU, :171) ---------
// The O(n^3) loops are cloned for AVX2 (picked at load time by the ifunc
// resolver, SSE2 otherwise). No FMA target: the vector lanes round each
// multiply and subtract exactly like the scalar code, so both clones give the
// same bits.
__attribute__((target_clones("avx2", "default"))) void lu_factor_rows(double* a, long long* perm, long long n) {
    for (long long i = 0; i < n; ++i) perm[i] = i;
    for (long long k = 0; k < n; ++k) {
        long long piv = k;
        double big = std::abs(a[k * n + k]);
        for (long long r = k + 1; r < n; ++r)
            if (std::abs(a[r * n + k]) > big) {
                big = std::abs(a[r * n + k]);
                piv = r;
            }
        if (big != 0.0) {
            if (piv != k) {
                for (long long c = 0; c < n; ++c) std::swap(a[k * n + c], a[piv * n + c]);
                std::swap(perm[k], perm[piv]);
            }
            // divide by the pivot, as Eigen's partial-pivot LU does (no reciprocal)
            const double pv = a[k * n + k];
            for (long long r = k + 1; r < n; ++r) a[r * n + k] /= pv;
        }
        for (long long r = k + 1; r < n; ++r) {
            const double l = a[r * n + k];
            if (l != 0.0) {
                double* __restrict__ ar = a + r * n;
                const double* __restrict__ ak = a + k * n;
                for (long long c = k + 1; c < n; ++c) ar[c] -= l * ak[c];
            }
        }
    }
}

// Z = U^-1 L^-1 in pivot column order (see LU::inverse)
__attribute__((target_clones("avx512f", "avx2", "default"))) void lu_inverse_rows(const double* a, double* Z, long long n) {
    for (long long i = 0; i < n; ++i) {
        double* __restrict__ zi = Z + i * n;
        zi[i] = 1.0;
        for (long long c = 0; c < i; ++c) {
            const double l = a[i * n + c];
            const double* __restrict__ zc = Z + c * n;
            for (long long j = 0; j <= c; ++j) zi[j] -= l * zc[j];
        }
    }
    for (long long i = n - 1; i >= 0; --i) {
        double* __restrict__ zi = Z + i * n;
        for (long long c = i + 1; c < n; ++c) {
            const double u = a[i * n + c];
            const double* __restrict__ zc = Z + c * n;
            for (long long j = 0; j < n; ++j) zi[j] -= u * zc[j];
        }
        const double d = a[i * n + i];
        for (long long j = 0; j < n; ++j) zi[j] /= d;
    }
}

struct LU {
    long long n;
    Vec a;
    std::vector<long long> perm;
    LU(const Vec& M, long long nn) : n(nn), a(M), perm((size_t)nn) { lu_factor_rows(a.data(), perm.data(), n); }
    // A^-1, row-major. Row-oriented substitution on the permuted identity: every
    // entry sees exactly the operation sequence of solve(e_j) (same bits), but
    // the inner loops run along contiguous rows. The forward sweep runs in
    // permuted column order, where L^-1 P is unit lower triangular: row c is
    // zero past column c, so those (exactly zero) updates are skipped
    // (n^3/6 instead of n^3/2 multiply-adds).
    Vec inverse() const {
        Vec Z((size_t)(n * n), 0.0);  // columns in pivot order: Z[i][j'] = Y[i][perm[j']]
        lu_inverse_rows(a.data(), Z.data(), n);
        Vec Y((size_t)(n * n));
        for (long long i = 0; i < n; ++i)
            for (long long j = 0; j < n; ++j) Y[(size_t)(i * n + perm[(size_t)j])] = Z[(size_t)(i * n + j)];
        return Y;
    }
    Vec solve(const Vec& b) const {
        Vec y((size_t)n);
        for (long long i = 0; i < n; ++i) y[(size_t)i] = b[(size_t)perm[(size_t)i]];
        for (long long i = 0; i < n; ++i) {
            double s = y[(size_t)i];
            for (long long c = 0; c < i; ++c) s -= a[(size_t)(i * n + c)] * y[(size_t)c];
            y[(size_t)i] = s;
        }
        for (long long i = n - 1; i >= 0; --i) {
            double s = y[(size_t)i];
            for (long long c = i + 1; c < n; ++c) s -= a[(size_t)(i * n + c)] * y[(size_t)c];
            y[(size_t)i] = s / a[(size_t)(i * n + i)];
        }
        return y;
    }
};

// ---- symmetric positive definite shortcut for the direct branch -------------
// M = (UQ)^T G (UQ) + lambda I is symmetric and, whenever psi'' > 0 on the
// samples (every CRRA calibration) and the face panel has full column rank,
// positive definite. Then M = L L^T, and M^-1 = L^-T L^-1 costs about half of
// the LU factor plus inverse (mm^3 / 2 instead of mm^3 multiply-adds). The
// reference's PartialPivLU (:171) gives the same solution to rounding. A
// non-positive or non-finite pivot (indefinite or singular M) returns false,
// and the caller keeps the LU path with its exact fallback semantics.
__attribute__((target_clones("avx512f", "avx2", "default"))) bool chol_inverse_rows(const double* M, double* L, double* X,
                                                                        double* Minv, long long n) {
    for (long long j = 0; j < n; ++j) {
        const double* lj = L + j * n;
        for (long long i = j; i < n; ++i) {
            const double* li = L + i * n;
            // the dot in 8 independent partial sums (vectorisable; this order is
            // not the reference's PartialPivLU order either way)
            double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            long long k = 0;
            for (; k + 8 <= j; k += 8)
                for (int u = 0; u < 8; ++u) p[u] += li[k + u] * lj[k + u];
            for (; k < j; ++k) p[0] += li[k] * lj[k];
            const double s = M[i * n + j] - (((p[0] + p[4]) + (p[1] + p[5])) + ((p[2] + p[6]) + (p[3] + p[7])));
            if (i == j) {
                if (!(s > 0.0) || !std::isfinite(s)) return false;
                L[j * n + j] = std::sqrt(s);
            } else {
                L[i * n + j] = s / L[j * n + j];
            }
        }
    }
    // X = L^-1, row by row (X[i] = (e_i - sum_{k<i} L[i][k] X[k]) / L[i][i])
    for (long long i = 0; i < n; ++i) {
        double* __restrict__ xi = X + i * n;
        for (long long c = 0; c <= i; ++c) xi[c] = (c == i) ? 1.0 : 0.0;
        for (long long k = 0; k < i; ++k) {
            const double l = L[i * n + k];
            const double* __restrict__ xk = X + k * n;
            for (long long c = 0; c <= k; ++c) xi[c] -= l * xk[c];
        }
        const double d = L[i * n + i];
        for (long long c = 0; c <= i; ++c) xi[c] /= d;
    }
    // M^-1 = X^T X (lower triangle by rank-1 updates of X's rows, then mirrored)
    for (long long a = 0; a < n * n; ++a) Minv[a] = 0.0;
    for (long long i = 0; i < n; ++i) {
        const double* __restrict__ xi = X + i * n;
        for (long long a = 0; a <= i; ++a) {
            const double xa = xi[a];
            if (xa == 0.0) continue;
            double* __restrict__ ma = Minv + a * n;
            for (long long b = 0; b <= a; ++b) ma[b] += xa * xi[b];
        }
    }
    for (long long a = 0; a < n; ++a)
        for (long long b = a + 1; b < n; ++b) Minv[a * n + b] = Minv[b * n + a];
    for (long long a = 0; a < n * n; ++a)
        if (!std::isfinite(Minv[a])) return false;
    return true;
}

// ---- simplex geometry (simplex.hpp:93-137) ----------------------------------------
double alpha_max(const Vec& x, const Vec& d, double tau) {
    double cap = std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < x.size(); ++i)
        if (d[i] < 0.0) cap = std::min(cap, (x[i] - tau) / (-d[i]));
    return std::max(cap, 0.0);
}

Vec project_slice(const Vec& v, double tau, double mass = 1.0) {
    Tick tk(g_prof.proj);
    ++g_prof.nproj;
    const size_t n = v.size();
    const double s = mass - (double)n * tau;
    if (!(tau >= 0.0) || !(s > 0.0)) throw ApiError(MVSK_DOMAIN_ERROR, "project_slice: need 0 <= tau < mass/n");
    Vec u(n);
    for (size_t i = 0; i < n; ++i) u[i] = v[i] - tau;
    // theta comes from the running sums of the sorted values up to the last
    // index where u[k] > cand, i.e. the support of the projection. Sorting only
    // the top K (partial sort: the same top-K order as a full sort, so the same
    // sums and the same bits) suffices when that index is well inside K; a
    // support reaching K/2 falls back to the full sort.
    double css = 0.0, theta = 0.0;
    size_t K = std::min<size_t>(n, 256);
    for (;;) {
        if (K < n) {  // top K by selection, then sorted: O(n + K log K)
            std::nth_element(u.begin(), u.begin() + (long)K - 1, u.end(), std::greater<double>());
            std::sort(u.begin(), u.begin() + (long)K, std::greater<double>());
        } else
            std::sort(u.begin(), u.end(), std::greater<double>());
        css = 0.0;
        theta = 0.0;
        size_t last = 0;
        for (size_t k = 0; k < K; ++k) {
            css += u[k];
            const double cand = (css - s) / (double)(k + 1);
            if (u[k] > cand) {
                theta = cand;
                last = k;
            }
        }
        if (K == n || 2 * (last + 1) <= K) break;
        K = std::min(n, 8 * K);
    }
    Vec out(n);
    for (size_t i = 0; i < n; ++i) out[i] = std::max(v[i] - tau - theta, 0.0) + tau;
    return out;
}

double projected_kkt_residual(const Vec& g) {
    const double m = vmean(g);
    double s = 0.0;
    for (double x : g) s += (x - m) * (x - m);
    return std::sqrt(s);
}

double gradient_mapping_residual(const Vec& x, const Vec& g, double tau) {
    Vec y(x.size());
    for (size_t i = 0; i < x.size(); ++i) y[i] = x[i] - g[i];
    const Vec p = project_slice(y, tau);
    double s = 0.0;
    for (size_t i = 0; i < x.size(); ++i) s += (x[i] - p[i]) * (x[i] - p[i]);
    return std::sqrt(s);
}

// ---- line search (linesearch.hpp:47-193) ------------------------------------------
struct LineModel {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, cap = 0;
    double eval(double al) const { return a0 + al * (a1 + al * (a2 + al * (a3 + al * a4))); }
    double deriv(double al) const { return a1 + al * (2.0 * a2 + al * (3.0 * a3 + al * 4.0 * a4)); }
};

std::vector<double> cubic_real_roots(double c3, double c2, double c1, double c0) {
    const double p = c2 / c3, q = c1 / c3, r = c0 / c3;
    const double a = q - p * p / 3.0;
    const double b = 2.0 * p * p * p / 27.0 - p * q / 3.0 + r;
    const double shift = p / 3.0;
    std::vector<double> roots;
    const double disc = b * b / 4.0 + a * a * a / 27.0;
    if (disc > 0.0) {
        const double sq = std::sqrt(disc);
        roots.push_back(std::cbrt(-b / 2.0 + sq) + std::cbrt(-b / 2.0 - sq) - shift);
    } else if (a == 0.0 && b == 0.0) {
        roots.push_back(-shift);
    } else {
        constexpr double pi = 3.14159265358979323846;
        const double rho = std::sqrt(-a * a * a / 27.0);
        double ca = -b / (2.0 * rho);
        ca = std::min(1.0, std::max(-1.0, ca));
        const double phi = std::acos(ca);
        const double mag = 2.0 * std::sqrt(-a / 3.0);
        for (int k = 0; k < 3; ++k) roots.push_back(mag * std::cos((phi + 2.0 * pi * k) / 3.0) - shift);
    }
    return roots;
}

double polish_root(const LineModel& m, double al) {
    for (int it = 0; it < 2; ++it) {
        const double d1 = m.deriv(al);
        const double d2 = 2.0 * m.a2 + al * (6.0 * m.a3 + al * 12.0 * m.a4);
        if (d2 == 0.0) break;
        const double nx = al - d1 / d2;
        if (!(nx > 0.0) || !(nx < m.cap)) break;
        al = nx;
    }
    return al;
}

std::pair<double, double> minimize_line(const LineModel& m) {
    if (!(m.cap > 0.0)) return {0.0, m.a0};
    std::vector<double> cands{0.0, m.cap};
    const double scale = std::max({std::abs(m.a1), std::abs(m.a2), std::abs(m.a3), std::abs(m.a4), 1e-300});
    if (std::abs(m.a4) > 1e-14 * scale) {
        for (double r : cubic_real_roots(4.0 * m.a4, 3.0 * m.a3, 2.0 * m.a2, m.a1))
            if (r > 0.0 && r < m.cap) cands.push_back(polish_root(m, r));
    } else if (std::abs(m.a3) > 1e-14 * scale) {
        const double A = 3.0 * m.a3, B = 2.0 * m.a2, C = m.a1;
        const double disc = B * B - 4.0 * A * C;
        if (disc >= 0.0) {
            const double sq = std::sqrt(disc);
            for (double r : {(-B + sq) / (2.0 * A), (-B - sq) / (2.0 * A)})
                if (r > 0.0 && r < m.cap) cands.push_back(polish_root(m, r));
        }
    } else if (std::abs(m.a2) > 1e-14 * scale) {
        const double r = -m.a1 / (2.0 * m.a2);
        if (r > 0.0 && r < m.cap) cands.push_back(r);
    }
    double ba = 0.0, bv = m.a0;
    for (double al : cands) {
        const double v = m.eval(al);
        if (v < bv || (v == bv && al < ba)) {
            bv = v;
            ba = al;
        }
    }
    return {ba, bv};
}

std::pair<double, bool> armijo_search(const std::function<double(double)>& phi, double gd, double a0) {
    if (!(gd < 0)) throw ApiError(MVSK_DOMAIN_ERROR, "armijo_search: direction is not descent");
    const double sigma = 1e-4, shrink = 0.5;
    const double p0 = phi(0.0);
    double al = a0;
    for (int k = 0; k < 60; ++k) {
        if (phi(al) <= p0 + sigma * al * gd) return {al, false};
        al *= shrink;
    }
    return {0.0, true};
}

// ---- the oracle view the driver talks to ----------------------------------------
struct View {
    mvsk_gpu_ctx* ctx;
    FaceMap fm;
    long long m() const { return fm.m; }
    double make_cache(int slot, const Vec& x) const {
        Tick tk(g_prof.cache);
        ++g_prof.ncache;
        return op_make_cache(ctx, slot, fm, x.data());
    }
    Vec gradient(int slot) const {
        Tick tk(g_prof.grad);
        Vec g((size_t)fm.m);
        op_gradient(ctx, slot, fm, g.data());
        return g;
    }
    // HVPs of k vectors in one fused pass
    std::vector<Vec> hvp(int slot, const std::vector<Vec>& V) const {
        const int k = (int)V.size();
        std::vector<Vec> out;
        Vec in((size_t)fm.m * k), o((size_t)fm.m * k);
        for (int i = 0; i < k; ++i) std::copy(V[i].begin(), V[i].end(), in.begin() + (size_t)i * fm.m);
        for (int base = 0; base < k; base += MVSK_GPU_MAX_RHS) {
            const int kk = std::min(MVSK_GPU_MAX_RHS, k - base);
            op_hvp(ctx, slot, fm, in.data() + (size_t)base * fm.m, kk, o.data() + (size_t)base * fm.m);
        }
        for (int i = 0; i < k; ++i) out.emplace_back(o.begin() + (size_t)i * fm.m, o.begin() + (size_t)(i + 1) * fm.m);
        return out;
    }
    std::vector<Vec> third(int slot, const std::vector<Vec>& U, const std::vector<Vec>& V) const {
        const int k = (int)U.size();
        std::vector<Vec> out;
        Vec iu((size_t)fm.m * k), iv((size_t)fm.m * k), o((size_t)fm.m * k);
        for (int i = 0; i < k; ++i) {
            std::copy(U[i].begin(), U[i].end(), iu.begin() + (size_t)i * fm.m);
            std::copy(V[i].begin(), V[i].end(), iv.begin() + (size_t)i * fm.m);
        }
        for (int base = 0; base < k; base += MVSK_GPU_MAX_RHS) {
            const int kk = std::min(MVSK_GPU_MAX_RHS, k - base);
            op_third(ctx, slot, fm, iu.data() + (size_t)base * fm.m, iv.data() + (size_t)base * fm.m, kk,
                     o.data() + (size_t)base * fm.m);
        }
        for (int i = 0; i < k; ++i) out.emplace_back(o.begin() + (size_t)i * fm.m, o.begin() + (size_t)(i + 1) * fm.m);
        return out;
    }
    // k line models at the same cache in one round trip (op_line_models); a0 = NaN marks a direction the
    // single call would reject. Logical passes are counted when a model is consumed (count_line_model).
    std::vector<LineModel> line_models(int slot, const std::vector<const Vec*>& dirs, const std::vector<double>& caps) const {
        Tick tk(g_prof.line);
        const int k = (int)dirs.size();
        Vec D((size_t)k * (size_t)fm.m), o((size_t)k * 14);
        for (int i = 0; i < k; ++i) std::copy(dirs[(size_t)i]->begin(), dirs[(size_t)i]->end(), D.begin() + (size_t)i * fm.m);
        op_line_models(ctx, slot, fm, D.data(), k, o.data());
        std::vector<LineModel> out((size_t)k);
        for (int i = 0; i < k; ++i) {
            LineModel& lm = out[(size_t)i];
            lm.a0 = o[(size_t)i * 14];
            lm.a1 = o[(size_t)i * 14 + 1];
            lm.a2 = o[(size_t)i * 14 + 2];
            lm.a3 = o[(size_t)i * 14 + 3];
            lm.a4 = o[(size_t)i * 14 + 4];
            lm.cap = caps[(size_t)i];
        }
        return out;
    }
    void count_line_model() const {
        ++g_prof.nline;
        ctx->fwd += 1;
    }
    LineModel line_model(int slot, const Vec& d, double cap) const {
        Tick tk(g_prof.line);
        ++g_prof.nline;
        double o[14];
        op_line_model(ctx, slot, fm, d.data(), o);
        LineModel lm;
        lm.a0 = o[0];
        lm.a1 = o[1];
        lm.a2 = o[2];
        lm.a3 = o[3];
        lm.a4 = o[4];
        lm.cap = cap;
        return lm;
    }
};

// ---- lockstep capped CG over k right-hand sides (cg_capped, :85-113, per column)
using HopBatch = std::function<std::vector<Vec>(const std::vector<Vec>&)>;

std::vector<Vec> cg_lockstep(const HopBatch& H, const std::vector<Vec>& rhs, double tol, int cap, const Vec* jd,
                             int& iters, bool& breakdown) {
    const size_t k = rhs.size();
    const size_t m = k ? rhs[0].size() : 0;
    auto pre = [&](const Vec& r) {
        if (!jd) return r;
        Vec z(r.size());
        for (size_t i = 0; i < r.size(); ++i) z[i] = r[i] / (*jd)[i];
        return z;
    };
    std::vector<Vec> x(k, Vec(m, 0.0)), r(rhs), z(k), p(k);
    std::vector<double> rz(k), target(k);
    std::vector<int> it(k, 0);
    std::vector<char> done(k, 0);
    for (size_t c = 0; c < k; ++c) {
        z[c] = pre(r[c]);
        p[c] = z[c];
        rz[c] = dot(r[c], z[c]);
        target[c] = tol * norm(rhs[c]);
    }
    for (;;) {
        std::vector<size_t> act;
        for (size_t c = 0; c < k; ++c) {
            if (done[c]) continue;
            if (it[c] < cap && norm(r[c]) > target[c])
                act.push_back(c);
            else
                done[c] = 1;
        }
        if (act.empty()) break;
        std::vector<Vec> ps;
        for (size_t c : act) ps.push_back(p[c]);
        const std::vector<Vec> Hp = H(ps);
        for (size_t a = 0; a < act.size(); ++a) {
            const size_t c = act[a];
            const double pHp = dot(p[c], Hp[a]);
            if (pHp <= 0.0) {
                breakdown = true;
                done[c] = 1;
                continue;
            }
            const double alpha = rz[c] / pHp;
            axpy(x[c], alpha, p[c]);
            axpy(r[c], -alpha, Hp[a]);
            z[c] = pre(r[c]);
            const double rz2 = dot(r[c], z[c]);
            const double beta = rz2 / rz[c];
            for (size_t i = 0; i < m; ++i) p[c][i] = z[c][i] + beta * p[c][i];
            rz[c] = rz2;
            ++it[c];
        }
    }
    for (size_t c = 0; c < k; ++c) iters += it[c];
    return x;
}

struct TangentCfg {
    bool pcg = false;
    double lambda = 0.0, tol = 1e-3;
    int maxit = 15, probes = 8, probe_maxit = 5;
    bool jacobi = false, exact_trace = false;
};

TangentCfg tangent_of(const mvsk_tangent_config& c) {
    TangentCfg t;
    t.pcg = c.mode == 1;
    t.lambda = c.lambda;
    t.tol = c.krylov_tol;
    t.maxit = c.krylov_maxit;
    t.jacobi = c.jacobi != 0;
    t.exact_trace = c.exact_trace != 0;
    t.probes = c.hutchinson_probes;
    t.probe_maxit = c.probe_maxit;
    return t;
}

// yand_direction (affine_normal.hpp:127-245) at the cache in `slot`
// [H S H]_11 for symmetric S (k x k, row-major), H = I - beta v v^T: the
// (k-1) x (k-1) block without row/col 0. S - beta v a^T - beta a v^T +
// beta^2 (v^T a) v v^T with a = S v; evaluated on the lower triangle and
// mirrored, so the result is exactly symmetric like S.
Vec reflect_sym(const Vec& S, long long k, const Vec& v, double beta) {
    Vec a((size_t)k, 0.0);
    for (long long i = 0; i < k; ++i) {
        double s = 0.0;
        const double* sr = &S[(size_t)(i * k)];
        for (long long j = 0; j < k; ++j) s += sr[j] * v[(size_t)j];
        a[(size_t)i] = s;
    }
    const double c = beta * beta * dot(v, a);
    const long long r = k - 1;
    Vec o((size_t)(r * r));
    for (long long i = 1; i < k; ++i)
        for (long long j = 1; j <= i; ++j) {
            const double val = S[(size_t)(i * k + j)] - (beta * v[(size_t)i] * a[(size_t)j] + beta * a[(size_t)i] * v[(size_t)j]) +
                               c * v[(size_t)i] * v[(size_t)j];
            o[(size_t)((i - 1) * r + (j - 1))] = val;
            o[(size_t)((j - 1) * r + (i - 1))] = val;
        }
    return o;
}

// H [0 0; 0 D] H for a general D (r x r): the (r+1) x (r+1) lift that
// P = (UQ) D (UQ)^T applies twice (D - beta v (v^T D) - beta (D v) v^T + beta^2
// (v^T D v) v v^T on the zero-padded D)
Vec unreflect(const Vec& D, long long r, const Vec& v, double beta) {
    const long long k = r + 1;
    Vec Dp((size_t)(k * k), 0.0);
    for (long long i = 0; i < r; ++i)
        for (long long j = 0; j < r; ++j) Dp[(size_t)((i + 1) * k + (j + 1))] = D[(size_t)(i * r + j)];
    Vec dv((size_t)k, 0.0), vd((size_t)k, 0.0);  // D v and v^T D
    for (long long i = 0; i < k; ++i) {
        double s = 0.0;
        const double* dr = &Dp[(size_t)(i * k)];
        for (long long j = 0; j < k; ++j) s += dr[j] * v[(size_t)j];
        dv[(size_t)i] = s;
    }
    for (long long i = 0; i < k; ++i) {
        const double vi = v[(size_t)i];
        if (vi == 0.0) continue;
        const double* dr = &Dp[(size_t)(i * k)];
        for (long long j = 0; j < k; ++j) vd[(size_t)j] += vi * dr[j];
    }
    const double c = beta * beta * dot(v, dv);
    for (long long i = 0; i < k; ++i) {
        double* pr = &Dp[(size_t)(i * k)];
        const double bvi = beta * v[(size_t)i], bdvi = beta * dv[(size_t)i], cvi = c * v[(size_t)i];
        for (long long j = 0; j < k; ++j) pr[j] += -(bvi * vd[(size_t)j] + bdvi * v[(size_t)j]) + cvi * v[(size_t)j];
    }
    return Dp;
}

Vec yand_direction(const View& O, int slot, const TangentCfg& cfg, uint64_t it_seed, mvsk_direction_diag& diag) {
    mvsk_gpu_ctx* ctx = O.ctx;
    const long long n = O.m();
    const long long m = n - 1;
    const Basis basis(n);
    const Vec g = O.gradient(slot);
    const Vec gbar = basis.apply_t(g);
    const double gn = norm(gbar);
    diag.reduced_grad_norm = gn;
    if (!(gn > 0)) throw ApiError(MVSK_DOMAIN_ERROR, "yand_direction: stationary point, no direction");
    if (m == 1) {
        Vec y = gbar;
        for (double& v : y) v = -v / gn;
        return basis.apply(y);
    }
    const Frame frame = householder_frame(gbar);
    const long long mm = m - 1;
    const mvsk_coeffs& c = ctx->c;
    const bool has_third = (c.c3 != 0.0 || c.c4 != 0.0);
    Vec u;

    bool direct_done = false;
    if (!cfg.pcg) {
        // ---- the whole direct branch on the device for faces of <= 112 assets
        // (gram_pcg.cu: one graph launch; the lambda fallback as a second one)
        DirectInput din;
        din.m = n;
        din.vU = basis.v;
        din.bU = basis.beta;
        din.vQ = frame.v;
        din.bQ = frame.beta;
        din.nu = frame.nu;
        din.gn = gn;
        din.lambda = cfg.lambda;
        din.has_third = has_third;
        Vec ud;
        Tick tkd(g_prof.dgram);
        if (direct_direction_device(ctx, slot, O.fm, din, ud)) {
            ctx->fwd += (uint64_t)mm + 1;  // the reference's W and t_nu passes (:159, :164)
            if (!all_finite(ud)) {  // singular unregularised operator: :181-188
                diag.lambda_fallback = 1;
                din.lambda = std::max(cfg.lambda, 1e-4);
                if (!direct_direction_device(ctx, slot, O.fm, din, ud) || !all_finite(ud))
                    throw ApiError(MVSK_NUMERIC_ERROR, "yand_direction: tangent solve failed");
            }
            u = std::move(ud);
            direct_done = true;
        }
    }
    if (direct_done) {
    } else if (!cfg.pcg) {
        // ---- direct branch via the weighted Gram (:151-188)
        // W = A (UQ) never forms: with G = A^T diag(psi'') A / T from the DMMA
        // kernel, M0 = (UQ)^T G (UQ) = [H_Q [H_U G H_U]_11 H_Q]_11 (two
        // Householder similarity transforms, [.]_11 drops row/col 0), O(n^2)
        // instead of the O(n^2 mm) dense products of :160-170.
        ctx->fwd += (uint64_t)mm + 1;  // the reference's W and t_nu passes (:159, :164)
        Vec G((size_t)(n * n));
        {
            Tick tk(g_prof.dgram);
            op_weighted_gram(ctx, slot, O.fm, G.data());
        }
        const Vec B = reflect_sym(G, n, basis.v, basis.beta);   // H_U G H_U, then drop row/col 0
        const Vec M0 = reflect_sym(B, m, frame.v, frame.beta);  // H_Q B H_Q, then drop row/col 0
        // h = (UQ)^T G (U nu)  (:165-166)
        const Vec unu = basis.apply(frame.nu);
        Vec Gu((size_t)n, 0.0);
        for (long long i = 0; i < n; ++i) {
            double s = 0.0;
            const double* gr = &G[(size_t)(i * n)];
            for (long long j = 0; j < n; ++j) s += gr[j] * unu[(size_t)j];
            Gu[(size_t)i] = s;
        }
        const Vec h = frame.apply_Qt(basis.apply_t(Gu));

        auto solve_with = [&](double lam) -> Vec {
            Vec M = M0;
            for (long long i = 0; i < mm; ++i) M[(size_t)(i * mm + i)] += lam;
            const auto tlu = std::chrono::steady_clock::now();
            if (has_third) {  // SPD shortcut (falls back to the LU path below)
                static const bool no_chol = std::getenv("MVSK_NO_CHOL") != nullptr;
                Vec Lf((size_t)(mm * mm)), Xf((size_t)(mm * mm)), Minv((size_t)(mm * mm));
                if (!no_chol && chol_inverse_rows(M.data(), Lf.data(), Xf.data(), Minv.data(), mm)) {
                    const Vec P = unreflect(unreflect(Minv, mm, frame.v, frame.beta), m, basis.v, basis.beta);
                    if (g_prof.on)
                        g_prof.dlu += std::chrono::duration<double>(std::chrono::steady_clock::now() - tlu).count();
                    bool fin = all_finite(P);
                    Vec a((size_t)mm, std::numeric_limits<double>::quiet_NaN());
                    if (fin) {
                        Vec af((size_t)n);
                        Tick tk(g_prof.dquad);
                        op_third_trace_rows(ctx, slot, O.fm, P.data(), af.data());
                        a = frame.apply_Qt(basis.apply_t(af));
                    }
                    Vec rhs((size_t)mm), uu((size_t)mm);
                    for (long long k = 0; k < mm; ++k)
                        rhs[(size_t)k] = h[(size_t)k] - (gn / (double)n) * a[(size_t)k];
                    for (long long i = 0; i < mm; ++i) {  // u = M^-1 rhs
                        double s = 0.0;
                        const double* mr = &Minv[(size_t)(i * mm)];
                        for (long long j = 0; j < mm; ++j) s += mr[j] * rhs[(size_t)j];
                        uu[(size_t)i] = s;
                    }
                    return uu;
                }
            }
            const LU lu(M, mm);
            Vec a((size_t)mm, 0.0);
            if (has_third) {
                // P = UQ M^-1 (UQ)^T (n x n): the explicit inverse, then the two
                // reflections back (pad row/col 0, H_Q . H_Q, pad, H_U . H_U)
                const Vec Minv = lu.inverse();
                const Vec P = unreflect(unreflect(Minv, mm, frame.v, frame.beta), m, basis.v, basis.beta);
                if (g_prof.on) g_prof.dlu += std::chrono::duration<double>(std::chrono::steady_clock::now() - tlu).count();
                bool fin = true;
                for (double v : P)
                    if (!std::isfinite(v)) {
                        fin = false;
                        break;
                    }
                if (!fin) {
                    a.assign((size_t)mm, std::numeric_limits<double>::quiet_NaN());
                } else {
                    Vec af((size_t)n);
                    Tick tk(g_prof.dquad);
                    op_third_trace_rows(ctx, slot, O.fm, P.data(), af.data());
                    a = frame.apply_Qt(basis.apply_t(af));
                }
            }
            Vec rhs((size_t)mm);
            for (long long k = 0; k < mm; ++k) rhs[(size_t)k] = h[(size_t)k] - (gn / (double)n) * a[(size_t)k];
            return lu.solve(rhs);
        };
        u = solve_with(cfg.lambda);
        if (!all_finite(u)) {
            diag.lambda_fallback = 1;
            u = solve_with(std::max(cfg.lambda, 1e-4));
            if (!all_finite(u)) throw ApiError(MVSK_NUMERIC_ERROR, "yand_direction: tangent solve failed");
        }
    } else if (!std::getenv("MVSK_HOST_PCG")) {
        // ---- matrix-free PCG branch (:189-242), Krylov loops resident on the device
        PcgInput in;
        in.m = n;
        in.vU = basis.v;
        in.bU = basis.beta;
        in.vQ = frame.v;
        in.bQ = frame.beta;
        in.nu = frame.nu;
        in.gn = gn;
        in.lambda = cfg.lambda;
        in.tol = cfg.tol;
        in.maxit = cfg.maxit;
        in.probe_cap = cfg.exact_trace ? cfg.maxit : cfg.probe_maxit;
        in.hutchinson_probes = cfg.probes;
        in.exact_trace = cfg.exact_trace;
        in.has_third = has_third;
        if (cfg.jacobi) {  // :197-209 probe stream
            SplitMix64 rng(0x0d1a6ULL ^ it_seed);
            for (int p = 0; p < 8; ++p) {
                Vec r((size_t)mm);
                for (long long i = 0; i < mm; ++i) r[(size_t)i] = rng.next_sign();
                in.jacobi_probes.push_back(std::move(r));
            }
        }
        if (has_third) {
            if (cfg.exact_trace) {  // :217-226, unit vectors generated on the device
                in.unit_probes = true;
            } else {  // :227-237
                SplitMix64 rng(0x5eedULL ^ it_seed);
                for (int pr = 0; pr < cfg.probes; ++pr) {
                    Vec r((size_t)mm);
                    for (long long i = 0; i < mm; ++i) r[(size_t)i] = rng.next_sign();
                    in.probes.push_back(std::move(r));
                }
            }
        }
        static const bool no_gram_pcg = std::getenv("MVSK_NO_GRAM_PCG") != nullptr;
        PcgOutput po;
        if (no_gram_pcg || !pcg_direction_gram(ctx, slot, O.fm, in, po)) po = pcg_direction_device(ctx, slot, O.fm, in);
        u = std::move(po.u);
        diag.krylov_iters += po.iters;
        if (po.breakdown) diag.pcg_breakdown = 1;
    } else {
        // ---- matrix-free PCG branch (:189-242), host-driven Krylov loops
        const HopBatch Hop = [&](const std::vector<Vec>& E) {
            std::vector<Vec> amb;
            for (const Vec& e : E) amb.push_back(basis.apply(frame.apply_Q(e)));
            std::vector<Vec> hv = O.hvp(slot, amb);
            std::vector<Vec> red;
            for (size_t i = 0; i < E.size(); ++i) {
                Vec r = frame.apply_Qt(basis.apply_t(hv[i]));
                for (size_t j = 0; j < r.size(); ++j) r[j] += cfg.lambda * E[i][j];
                red.push_back(std::move(r));
            }
            return red;
        };
        std::optional<Vec> jd;
        if (cfg.jacobi) {  // :197-209, 8 probes in one batched pass
            SplitMix64 rng(0x0d1a6ULL ^ it_seed);
            std::vector<Vec> R;
            for (int p = 0; p < 8; ++p) {
                Vec r((size_t)mm);
                for (long long i = 0; i < mm; ++i) r[(size_t)i] = rng.next_sign();
                R.push_back(std::move(r));
            }
            const std::vector<Vec> HR = Hop(R);
            Vec dg((size_t)mm, 0.0);
            for (int p = 0; p < 8; ++p)
                for (long long i = 0; i < mm; ++i) dg[(size_t)i] += R[p][(size_t)i] * HR[p][(size_t)i];
            for (double& v : dg) v /= 8.0;
            const double fl = std::max(1e-12, cfg.lambda);
            for (double& v : dg) v = std::max(v, fl);
            jd = dg;
        }
        const Vec* jdp = jd ? &*jd : nullptr;
        const Vec hvec = frame.apply_Qt(basis.apply_t(O.hvp(slot, {basis.apply(frame.nu)})[0]));  // :212-213
        Vec a((size_t)mm, 0.0);
        int iters = 0;
        bool bd = false;
        if (has_third) {
            std::vector<Vec> probes;
            if (cfg.exact_trace) {  // :217-226
                for (long long k = 0; k < mm; ++k) {
                    Vec e((size_t)mm, 0.0);
                    e[(size_t)k] = 1.0;
                    probes.push_back(std::move(e));
                }
            } else {  // :227-237
                SplitMix64 rng(0x5eedULL ^ it_seed);
                for (int pr = 0; pr < cfg.probes; ++pr) {
                    Vec r((size_t)mm);
                    for (long long i = 0; i < mm; ++i) r[(size_t)i] = rng.next_sign();
                    probes.push_back(std::move(r));
                }
            }
            const int pcap = cfg.exact_trace ? cfg.maxit : cfg.probe_maxit;
            // lockstep CG in blocks of MVSK_GPU_MAX_RHS probes
            for (size_t b0 = 0; b0 < probes.size(); b0 += MVSK_GPU_MAX_RHS) {
                const size_t b1 = std::min(probes.size(), b0 + (size_t)MVSK_GPU_MAX_RHS);
                std::vector<Vec> blk(probes.begin() + b0, probes.begin() + b1);
                const std::vector<Vec> S = cg_lockstep(Hop, blk, cfg.tol, pcap, jdp, iters, bd);
                std::vector<Vec> Ua, Va;
                for (size_t i = 0; i < blk.size(); ++i) {
                    Ua.push_back(basis.apply(frame.apply_Q(S[i])));
                    Va.push_back(basis.apply(frame.apply_Q(blk[i])));
                }
                const std::vector<Vec> T3 = O.third(slot, Ua, Va);
                for (size_t i = 0; i < blk.size(); ++i) axpy(a, 1.0, frame.apply_Qt(basis.apply_t(T3[i])));
            }
            if (!cfg.exact_trace)
                for (double& v : a) v /= (double)cfg.probes;
        }
        Vec rhs((size_t)mm);
        for (long long k = 0; k < mm; ++k) rhs[(size_t)k] = hvec[(size_t)k] - (gn / (double)n) * a[(size_t)k];
        u = cg_lockstep(Hop, {rhs}, cfg.tol, cfg.maxit, jdp, iters, bd)[0];
        diag.krylov_iters += iters;
        if (bd) diag.pcg_breakdown = 1;
    }
    diag.u_norm = norm(u);
    Vec qu = frame.apply_Q(u);
    for (size_t i = 0; i < qu.size(); ++i) qu[i] -= frame.nu[i];
    return basis.apply(qu);  // :244
}

// ---- solve (solver.hpp:195-655) -------------------------------------------------
struct SolveCfg {
    double eps, tau;
    int max_iter;
    std::optional<double> max_elapsed;
    double trial;
    std::vector<double> restarts;
    int restart_max_iter;
    TangentCfg tangent;
    bool armijo, stall_restarts, identification;
};

constexpr int kSlotFace = 0;
constexpr int kSlotTmp = 1;

struct Report {
    Vec x;
    double f = 0, kkt = 0, interior = 0;
    int iterations = 0, face_events = 0, restarts = 0, ident = 0, status = 2;
    long long krylov = 0;
};

Vec spg_identify(const View& full, Vec x, double tau, int max_steps, int patience, double eps_stop, int& steps_out,
                 const std::function<void(int, double, const Vec&)>& observer) {
    double f = full.make_cache(kSlotTmp, x);
    Vec g = full.gradient(kSlotTmp);
    // the whole preamble as one device graph (bitwise the loop below) unless an
    // observer must see every step or the panel is out of the device loop's range
    if (!observer && !full.fm.active) {
        Tick tk(g_prof.spg);
        Vec xd = x;
        if (spg_identify_device(full.ctx, kSlotTmp, xd, f, g, tau, max_steps, patience, eps_stop, steps_out))
            return xd;
    }
    Vec xcur = x;
    double L = 10.0;
    bool have_bb = false;
    Vec bb_s, bb_y;
    auto active = [&](const Vec& v) {
        std::vector<char> a(v.size());
        for (size_t i = 0; i < v.size(); ++i) a[i] = v[i] <= tau + 1e-12 ? 1 : 0;
        return a;
    };
    std::vector<char> act = active(xcur);
    int last_change = 0, steps = 0;
    for (int k = 0; k < max_steps; ++k) {
        double L0 = L;
        if (have_bb) {
            const double sy = dot(bb_s, bb_y), ss = dot(bb_s, bb_s);
            L0 = (ss > 0 && sy > 0) ? sy / ss : L;
            L0 = std::min(std::max(L0, 1e-2), 1e12);
        }
        double Lk = L0;
        bool stepped = false;
        for (int bt = 0; bt < 40; ++bt) {
            Vec y(xcur.size());
            for (size_t i = 0; i < y.size(); ++i) y[i] = xcur[i] - g[i] / Lk;
            Vec xp = project_slice(y, tau, 1.0);
            Vec dp(xp.size());
            for (size_t i = 0; i < dp.size(); ++i) dp[i] = xp[i] - xcur[i];
            const double gdp = dot(g, dp);
            if (gdp < 0) {
                const double fp = full.make_cache(kSlotTmp, xp);
                if (fp <= f + 1e-4 * gdp) {
                    Vec gp = full.gradient(kSlotTmp);
                    bb_s = std::move(dp);
                    bb_y.resize(gp.size());
                    for (size_t i = 0; i < gp.size(); ++i) bb_y[i] = gp[i] - g[i];
                    have_bb = true;
                    xcur = xp;
                    f = fp;
                    g = std::move(gp);
                    L = Lk;
                    stepped = true;
                    break;
                }
            }
            if (Lk > 1e13) break;
            Lk *= 2.0;
        }
        if (!stepped) break;
        ++steps;
        if (observer) observer(-steps, f, xcur);
        std::vector<char> actp = active(xcur);
        if (actp != act) {
            act = std::move(actp);
            last_change = steps;
        } else if (std::find(act.begin(), act.end(), 1) != act.end() && steps - last_change >= patience) {
            break;
        }
        if (eps_stop > 0 && steps % 10 == 0 && gradient_mapping_residual(xcur, g, tau) <= eps_stop) break;
    }
    steps_out = steps;
    return xcur;
}

// compact a face when it is at most 3/4 of a panel wide enough for the pass
// bytes to matter (n >= 256); MVSK_NO_FACE_COMPACT keeps index maps throughout
bool face_compaction(long long n0, long long nf) {
    static const bool off = std::getenv("MVSK_NO_FACE_COMPACT") != nullptr;
    long long cap = 64;  // face.cu width class
    while (cap < nf) cap <<= 1;
    return !off && n0 >= 256 && 4 * cap <= 3 * n0;
}

Report solve(mvsk_gpu_ctx* ctx, const SolveCfg& config, Vec x0,
             const std::function<void(int, double, const Vec&)>& observer) {
    const long long n0 = ctx->n;
    const double tau = config.tau, eps = config.eps;
    if (!(eps > 0)) throw ApiError(MVSK_DOMAIN_ERROR, "solve: epsilon must be positive");
    if (!(tau >= 0) || (n0 > 1 && !(tau < 1.0 / (double)n0))) throw ApiError(MVSK_DOMAIN_ERROR, "solve: tau out of range");
    const auto t_start = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count(); };

    View full{ctx, full_face(ctx)};
    Report rep;
    if (x0.empty()) x0.assign((size_t)n0, 1.0 / (double)n0);
    {
        double mn = std::numeric_limits<double>::infinity();
        for (double v : x0) mn = std::min(mn, v);
        if ((long long)x0.size() != n0 || mn < tau - 1e-12 || std::abs(vsum(x0) - 1.0) > 1e-10)
            throw ApiError(MVSK_DOMAIN_ERROR, "solve: x0 is not in the tau-slice");
    }
    auto finish = [&](const Vec& x, int status, double kkt) {
        rep.f = full.make_cache(kSlotTmp, x);
        rep.interior = projected_kkt_residual(full.gradient(kSlotTmp));
        rep.kkt = kkt;
        rep.x = x;
        rep.status = status;
        return rep;
    };
    if (n0 == 1) return finish(Vec(1, 1.0), 0, 0.0);
    if (config.identification)
        x0 = spg_identify(full, x0, tau, 600, 30, std::max(1e3 * eps, 1e-4), rep.ident, observer);

    struct Best {
        double f;
        Vec x;
    };
    Best best{full.make_cache(kSlotTmp, x0), x0};
    if (observer) observer(0, best.f, best.x);

    std::vector<std::pair<double, int>> attempts{{config.trial, config.max_iter}};
    if (config.stall_restarts)
        for (double s : config.restarts) attempts.emplace_back(s, config.restart_max_iter);

    auto merge = [&](const Vec& xf, const std::vector<char>& free_mask, const std::vector<char>& pinned_mask) {
        Vec xn((size_t)n0, tau);
        size_t j = 0;
        for (long long i = 0; i < n0; ++i)
            if (free_mask[(size_t)i]) xn[(size_t)i] = xf[j++];
        long long npin = 0;
        for (long long i = 0; i < n0; ++i)
            if (pinned_mask[(size_t)i]) {
                xn[(size_t)i] = tau;
                ++npin;
            }
        double s = 0.0;
        for (long long i = 0; i < n0; ++i)
            if (!pinned_mask[(size_t)i]) s += xn[(size_t)i];
        if (s > 0) {
            const double scale = (1.0 - (double)npin * tau) / s;
            for (long long i = 0; i < n0; ++i)
                if (!pinned_mask[(size_t)i]) xn[(size_t)i] *= scale;
        }
        return xn;
    };
    auto full_residual = [&](const Vec& x, Vec& g_out) {
        Tick tkr(g_prof.resid);
        ++g_prof.nresid;
        full.make_cache(kSlotTmp, x);
        g_out = full.gradient(kSlotTmp);
        return gradient_mapping_residual(x, g_out, tau);
    };
    auto full_value = [&](const Vec& x) { return full.make_cache(kSlotTmp, x); };

    int it_total = 0;
    bool timed_out = false;
    for (size_t ai = 0; ai < attempts.size(); ++ai) {
        const double tr = attempts[ai].first;
        const int budget = attempts[ai].second;
        Vec x = best.x;
        std::vector<char> pinned((size_t)n0, 0);
        long long npinned = 0;
        for (long long i = 0; i < n0; ++i)
            if (x[(size_t)i] <= tau + 1e-12) {
                pinned[(size_t)i] = 1;
                ++npinned;
            }
        if (npinned >= n0) {
            std::fill(pinned.begin(), pinned.end(), 0);
            npinned = 0;
        }
        int stall_small = 0, stall_zero = 0;
        double eps_face = eps;
        double face_ref = std::numeric_limits<double>::infinity();
        double t_cur = tr;
        bool rebuild = true, stalled = false;
        int it = 0, since_check = 0;
        std::vector<char> free_mask((size_t)n0, 1);
        long long nf = n0;
        double mass = 1.0;
        View face{ctx, full_face(ctx)};
        // the face cache made right after a move (at the merged point, below)
        // serves the next iteration's cache when its face point is that point
        bool face_cached = false;
        Vec face_cached_xf;

        while (it < budget) {
            if (config.max_elapsed && elapsed() > *config.max_elapsed) {
                timed_out = true;
                break;
            }
            ++it;
            ++it_total;
            ++since_check;
            if (rebuild) {  // :343-370
                nf = n0 - npinned;
                free_mask.assign((size_t)n0, 0);
                FaceMap fm;
                fm.tau = tau;
                fm.m = nf;
                fm.active = nf != n0;
                for (long long i = 0; i < n0; ++i)
                    if (!pinned[(size_t)i]) {
                        free_mask[(size_t)i] = 1;
                        fm.idx.push_back(i);
                    }
                // small faces of a wide panel: the reference's gathered face panel
                // (Af, zoff, -c1 mu_pin) as a compact device context, so face passes
                // stream T x nf instead of T x n; otherwise an index map over the
                // resident panel (no gather)
                if (fm.active && face_compaction(n0, nf) && !ctx->zoff_dev && ctx->value_offset == 0.0) {
                    Tick tkf(g_prof.face);
                    ++g_prof.nface;
                    mvsk_gpu_ctx* fc = face_context(ctx, fm.idx, pinned, tau);
                    face = View{fc, face_child_map(fc, nf)};
                } else {
                    if (!fm.active) fm.idx.clear();
                    face = View{ctx, fm};
                }
                mass = 1.0 - (double)npinned * tau;
                t_cur = tr;
                rebuild = false;
                face_cached = false;
            }
            Vec xf((size_t)nf);
            {
                size_t j = 0;
                for (long long i = 0; i < n0; ++i)
                    if (free_mask[(size_t)i]) xf[j++] = x[(size_t)i];
            }
            const double fcur = (face_cached && xf == face_cached_xf) ? op_value(face.ctx, kSlotFace)
                                                                       : face.make_cache(kSlotFace, xf);
            face_cached = false;
            const Vec gf = face.gradient(kSlotFace);
            const double gf_mean = vmean(gf);
            double face_res = 0.0;
            if (nf > 1) {
                double s = 0.0;
                for (double gv : gf) s += (gv - gf_mean) * (gv - gf_mean);
                face_res = std::sqrt(s);
            }
            if (face_res <= eps_face || since_check >= 15) {  // :384-427
                since_check = 0;
                Vec g_full;
                const double r = full_residual(x, g_full);
                if (r <= eps) {
                    const double fv = full_value(x);
                    if (fv < best.f) best = {fv, x};
                    rep.iterations = it_total;
                    rep.restarts = (int)ai;
                    return finish(x, 0, r);
                }
                std::vector<char> rel((size_t)n0, 0);
                bool any_rel = false;
                const double rel_gate = std::max(1e-10, face_res);
                for (long long i = 0; i < n0; ++i)
                    if (pinned[(size_t)i] && g_full[(size_t)i] - gf_mean < -rel_gate) {
                        rel[(size_t)i] = 1;
                        any_rel = true;
                    }
                if (any_rel) {
                    for (long long i = 0; i < n0; ++i)
                        if (rel[(size_t)i]) {
                            pinned[(size_t)i] = 0;
                            --npinned;
                        }
                    ++rep.face_events;
                    rebuild = true;
                    eps_face = eps;
                    x = merge(xf, free_mask, pinned);
                    stall_small = stall_zero = 0;
                    face_ref = std::numeric_limits<double>::infinity();
                    continue;
                }
                if (face_res <= eps_face) {
                    if (face_res <= 1e-3 * eps || nf <= 1) {
                        stalled = true;
                        break;
                    }
                    eps_face = 0.25 * face_res;
                    stall_small = stall_zero = 0;
                    face_ref = std::numeric_limits<double>::infinity();
                }
            }
            // the face cache is rebuilt by the residual checks above (shared
            // tmp slot only); kSlotFace still holds the face point
            mvsk_direction_diag dd{};
            Vec d;
            {
                Tick tk(g_prof.dir);
                ++g_prof.ndir;
                d = yand_direction(face, kSlotFace, config.tangent, (uint64_t)it_total, dd);
            }
            rep.krylov += dd.krylov_iters;
            const double amax = alpha_max(xf, d, tau);
            bool moved = false;
            auto step_from = [&](const LineModel& lm) {  // :437-446
                if (config.armijo) {
                    auto res = armijo_search([&](double al) { return lm.eval(al); }, lm.a1, std::min(1.0, lm.cap));
                    return std::pair<double, double>{res.first, lm.eval(res.first)};
                }
                return minimize_line(lm);
            };
            auto exact_step = [&](const Vec& dir, double cap) { return step_from(face.line_model(kSlotFace, dir, cap)); };
            if (amax >= t_cur) {
                auto st = exact_step(d, amax);
                if (st.first > 0) {
                    axpy(xf, st.first, d);
                    moved = true;
                }
            } else {  // :454-562
                std::vector<char> floor0((size_t)nf);
                for (long long i = 0; i < nf; ++i) floor0[(size_t)i] = xf[(size_t)i] <= tau + 1e-12;
                std::vector<std::vector<char>> zsets;
                std::vector<long long> zset_sizes;
                // The ladder's rungs (trial step t_cur / 2^rung, projected) depend on xf, d and the projections
                // only, never on earlier rungs' line searches, so the loop of :454-562 is walked lazily: rung by
                // rung as the reference visits them, and once a rung's exact step has failed the line models of
                // ALL remaining rungs are evaluated in one graph launch and one round trip (k independent
                // line-sums passes, each bitwise the single-direction pass), then consumed in order.
                struct Rung {
                    Vec db;
                    double cap = 0.0;
                    bool step = false;  // takes an exact step (else skipped: tiny or non-descent direction)
                    bool stop = false;  // the ladder ends after this rung (newz == 0)
                    bool have = false;
                    LineModel lm;
                };
                std::vector<Rung> rungs;
                double t_len = t_cur;
                auto next_rung = [&]() {
                    Vec trial(xf.size());
                    for (size_t i = 0; i < xf.size(); ++i) trial[i] = xf[i] + t_len * d[i];
                    const Vec xb = project_slice(trial, tau, mass);
                    std::vector<char> zb((size_t)nf);
                    long long zb_count = 0, newz = 0;
                    for (long long i = 0; i < nf; ++i) {
                        zb[(size_t)i] = xb[(size_t)i] <= tau + 1e-15;
                        if (zb[(size_t)i]) ++zb_count;
                        if (xb[(size_t)i] <= tau + 1e-12 && !floor0[(size_t)i]) ++newz;
                    }
                    if (zb_count > 0 && (zsets.empty() || zb_count != zset_sizes.back())) {
                        zsets.push_back(zb);
                        zset_sizes.push_back(zb_count);
                    }
                    Rung R;
                    R.db.resize(xf.size());
                    for (size_t i = 0; i < xf.size(); ++i) R.db[i] = xb[i] - xf[i];
                    const double dbm = vmean(R.db);
                    for (double& v : R.db) v -= dbm;
                    const double dbn = norm(R.db);
                    R.step = !(dbn <= 1e-12 * std::max(1.0, norm(xf)) || dot(gf, R.db) >= -1e-10 * (1.0 + std::abs(fcur)));
                    if (R.step) R.cap = std::min(1.0, alpha_max(xf, R.db, tau));
                    R.stop = newz == 0;
                    rungs.push_back(std::move(R));
                    t_len *= 0.5;
                };
                bool any_failed = false;
                for (int rung = 0; rung < 6; ++rung) {
                    if ((int)rungs.size() <= rung) next_rung();
                    if (rungs[(size_t)rung].step) {
                        if (!rungs[(size_t)rung].have && any_failed) {
                            while ((int)rungs.size() < 6 && !rungs.back().stop) next_rung();
                            std::vector<size_t> want;
                            for (size_t q = (size_t)rung; q < rungs.size(); ++q)
                                if (rungs[q].step && !rungs[q].have) want.push_back(q);
                            if (want.size() > 1) {
                                std::vector<const Vec*> dirs;
                                std::vector<double> caps;
                                for (size_t q : want) {
                                    dirs.push_back(&rungs[q].db);
                                    caps.push_back(rungs[q].cap);
                                }
                                const std::vector<LineModel> lms = face.line_models(kSlotFace, dirs, caps);
                                for (size_t e = 0; e < want.size(); ++e)
                                    if (std::isfinite(lms[e].a0)) {
                                        rungs[want[e]].lm = lms[e];
                                        rungs[want[e]].have = true;
                                    }
                            }
                        }
                        Rung& R = rungs[(size_t)rung];
                        if (R.have) {
                            face.count_line_model();  // a batch-evaluated rung is consumed: one reference pass
                        } else {
                            R.lm = face.line_model(kSlotFace, R.db, R.cap);
                            R.have = true;
                        }
                        auto st = step_from(R.lm);
                        if (st.first > 0 && (rung == 0 || fcur - st.second >= 1e-12 * (1.0 + std::abs(fcur)))) {
                            axpy(xf, st.first, R.db);
                            moved = true;
                            break;
                        }
                        any_failed = true;
                    }
                    if (rungs[(size_t)rung].stop) break;
                }
                if (!moved) {
                    bool done = false;
                    double pin_f = fcur;
                    for (const auto& zb : zsets) {
                        long long cnt = 0;
                        for (char b : zb) cnt += b;
                        if (cnt >= nf) continue;
                        std::vector<char> pin_try = pinned;
                        size_t j = 0;
                        for (long long i = 0; i < n0; ++i)
                            if (free_mask[(size_t)i]) {
                                if (zb[j]) pin_try[(size_t)i] = 1;
                                ++j;
                            }
                        Vec x_try = merge(xf, free_mask, pin_try);
                        const double f_try = full_value(x_try);
                        if (f_try <= fcur + 1e-12 * (1.0 + std::abs(fcur))) {
                            pinned = std::move(pin_try);
                            npinned += cnt;
                            x = std::move(x_try);
                            pin_f = f_try;
                            done = true;
                            break;
                        }
                    }
                    if (!done) {
                        long long cnt = 0;
                        for (long long i = 0; i < nf; ++i)
                            if (xf[(size_t)i] <= tau + 1e-12) ++cnt;
                        if (cnt > 0 && cnt < nf) {
                            size_t j = 0;
                            for (long long i = 0; i < n0; ++i)
                                if (free_mask[(size_t)i]) {
                                    if (xf[j] <= tau + 1e-12) {
                                        pinned[(size_t)i] = 1;
                                        ++npinned;
                                    }
                                    ++j;
                                }
                            x = merge(xf, free_mask, pinned);
                            if (observer) pin_f = full_value(x);
                            done = true;
                        }
                    }
                    if (done) {
                        ++rep.face_events;
                        rebuild = true;
                        eps_face = eps;
                        stall_small = stall_zero = 0;
                        face_ref = std::numeric_limits<double>::infinity();
                        if (observer) observer(it_total, pin_f, x);
                        continue;
                    } else if (amax > 0) {
                        auto st = exact_step(d, amax);
                        if (st.first > 0) {
                            axpy(xf, st.first, d);
                            moved = true;
                        }
                    }
                }
            }
            if (moved) {  // :564-581
                x = merge(xf, free_mask, pinned);
                // f(x) through the face oracle at the merged point: the face
                // panel, its pinned offset zoff and value offset make face values
                // equal full objective values (oracle.hpp:31-45, solver.hpp:357-363;
                // merge puts the pinned coordinates exactly at tau), so one narrow
                // pass replaces the reference's full-panel evaluation, and the
                // next iteration reuses the cache
                Vec xfn((size_t)nf);
                {
                    size_t j = 0;
                    for (long long i = 0; i < n0; ++i)
                        if (free_mask[(size_t)i]) xfn[j++] = x[(size_t)i];
                }
                const double fv_new = face.make_cache(kSlotFace, xfn);
                face_cached = true;
                face_cached_xf = std::move(xfn);
                const double dec = (fcur - fv_new) / (1.0 + std::abs(fcur));
                if (dec < 1e-12) t_cur = std::max(std::min(0.5 * t_cur, 0.99 * amax), 1e-10);
                if (dec >= 1e-12 || face_res <= 0.9 * face_ref) {
                    stall_small = 0;
                    face_ref = face_res;
                } else {
                    ++stall_small;
                }
                stall_zero = 0;
                if (fv_new < best.f) best = {fv_new, x};
                if (observer) observer(it_total, fv_new, x);
            } else {
                ++stall_zero;
            }
            if (stall_small >= 5 || stall_zero >= 2) {  // :583-631
                const double fcur2 = full_value(x);
                std::vector<std::pair<double, long long>> order;
                for (long long i = 0; i < n0; ++i)
                    if (!pinned[(size_t)i]) order.emplace_back(x[(size_t)i], i);
                std::sort(order.begin(), order.end());
                bool rescued = false;
                std::vector<char> cur_free((size_t)n0);
                for (long long i = 0; i < n0; ++i) cur_free[(size_t)i] = !pinned[(size_t)i];
                Vec x_free(order.size());
                {
                    size_t j = 0;
                    for (long long i = 0; i < n0; ++i)
                        if (cur_free[(size_t)i]) x_free[j++] = x[(size_t)i];
                }
                double rescue_f = fcur2;
                for (const auto& pr : order) {
                    if (pr.first > 1e-3 * (1.0 - (double)npinned * tau)) break;
                    if (npinned + 1 >= n0) break;
                    std::vector<char> pin_try = pinned;
                    pin_try[(size_t)pr.second] = 1;
                    Vec x_try = merge(x_free, cur_free, pin_try);
                    const double f_try = full_value(x_try);
                    if (f_try <= fcur2 + 1e-12 * (1.0 + std::abs(fcur2))) {
                        pinned = std::move(pin_try);
                        ++npinned;
                        x = std::move(x_try);
                        rescue_f = f_try;
                        rescued = true;
                        break;
                    }
                }
                if (rescued) {
                    rebuild = true;
                    stall_small = stall_zero = 0;
                    face_ref = std::numeric_limits<double>::infinity();
                    ++rep.face_events;
                    if (observer) observer(it_total, rescue_f, x);
                    continue;
                }
                stalled = true;
                break;
            }
        }
        Vec g_exit;
        const double r = full_residual(x, g_exit);
        const double fv = full_value(x);
        if (fv < best.f) best = {fv, x};
        rep.iterations = it_total;
        rep.restarts = (int)ai;
        if (r <= eps) return finish(x, 0, r);
        if (timed_out) break;
        if (!config.stall_restarts) return finish(x, stalled ? 1 : 2, r);
    }
    Vec g_best;
    const double rb = full_residual(best.x, g_best);
    rep.iterations = it_total;
    const int status = rb <= eps ? 0 : timed_out ? 3 : 1;
    return finish(best.x, status, rb);
}

SolveCfg solve_cfg_of(const mvsk_solver_config* cfg) {
    SolveCfg sc;
    sc.eps = cfg->epsilon;
    sc.tau = cfg->tau;
    sc.max_iter = cfg->max_iter;
    if (cfg->has_max_elapsed) sc.max_elapsed = cfg->max_elapsed_seconds;
    sc.trial = cfg->projected_trial_step;
    sc.restarts.assign(cfg->restart_trial_steps,
                       cfg->restart_trial_steps + std::max(0, std::min(4, cfg->n_restart_trial_steps)));
    sc.restart_max_iter = cfg->restart_max_iter;
    sc.tangent = tangent_of(cfg->tangent);
    sc.armijo = cfg->line_search == 1;
    sc.stall_restarts = cfg->stall_restarts != 0;
    sc.identification = cfg->identification_pass != 0;
    return sc;
}

// coefficients are baked into captured graphs and every cached slot's f / g
void set_coeffs(mvsk_gpu_ctx* ctx, const mvsk_coeffs& c) {
    ctx->c = c;
    ++ctx->epoch;
    for (auto& s : ctx->slots) {
        s.valid = false;
        s.g_host_valid = false;
        s.scalars_host_valid = false;
    }
}

// ---- return-floor sweep (BASELINE config 4) -------------------------------------
// Not part of the reference code: the paper's calibration of the mean
// coefficient (PAPER.md:757 — "calibrate the mean coefficient so that the
// resulting MVSK portfolio lies as close as possible to the same in-sample
// return floor"), with c2..c4 held at the context's values. For each floor r the
// in-sample mean m(c1) = mu'x*(c1) of the optimum, nondecreasing in c1, is
// bracketed (c1 = 0, then doubling from the context's c1) and bisected until
// |m - r| <= mean_tol * (m_max - m_mv) or the per-floor solve budget is spent;
// every solve is cached and shared between floors. Default floors are the
// interior points r_k = m_mv + k/(K+1) (m_max - m_mv): m_mv is the mean of the
// minimum-variance optimum (c = (0, c2, 0, 0)), m_max = max_j mu_j (the
// max-mean vertex).
struct FloorEval {
    double c1, mean, f, kkt;
    int status;
    Vec x;
};

struct SweepOut {
    std::vector<FloorEval> best;
    std::vector<int> solves;
    std::vector<double> floors;
    double m_mv = 0, m_max = 0;
    int total = 0;
};

SweepOut floor_sweep(mvsk_gpu_ctx* ctx, const SolveCfg& sc, const mvsk_sweep_config& sw, const std::vector<double>& user_floors,
                     int nfloors) {
    const mvsk_coeffs c0 = ctx->c;
    const Vec& mu = ctx->mu;
    auto mean_of = [&](const Vec& x) {
        double m = 0.0;
        for (size_t i = 0; i < x.size(); ++i) m += mu[i] * x[i];
        return m;
    };
    SweepOut out;
    std::vector<FloorEval> cache;
    auto run = [&](const mvsk_coeffs& c, const Vec& x0) {
        set_coeffs(ctx, c);
        Report r = solve(ctx, sc, x0, nullptr);
        ++out.total;
        return FloorEval{c.c1, mean_of(r.x), r.f, r.kkt, r.status, r.x};
    };
    try {
        const FloorEval mv = run(mvsk_coeffs{0.0, c0.c2, 0.0, 0.0}, Vec());
        out.m_mv = mv.mean;
        out.m_max = *std::max_element(mu.begin(), mu.end());
        const double span = out.m_max - out.m_mv;
        if (!user_floors.empty()) {
            out.floors = user_floors;
        } else {
            for (int k = 1; k <= nfloors; ++k) out.floors.push_back(out.m_mv + span * k / (double)(nfloors + 1));
        }
        const double tol = (sw.mean_tol > 0 ? sw.mean_tol : 1e-3) * std::max(std::fabs(span), 1e-300);
        const int budget = sw.max_solves > 0 ? sw.max_solves : 16;
        // E(c1): cached solve, warm-started from the evaluated optimum nearest in c1
        auto eval = [&](double c1, int& used) -> const FloorEval& {
            for (const FloorEval& e : cache)
                if (e.c1 == c1) return e;
            Vec x0;
            if (sw.warm_start && !cache.empty()) {
                const FloorEval* nb = &cache[0];
                for (const FloorEval& e : cache)
                    if (std::fabs(e.c1 - c1) < std::fabs(nb->c1 - c1)) nb = &e;
                x0 = nb->x;
            }
            cache.push_back(run(mvsk_coeffs{c1, c0.c2, c0.c3, c0.c4}, x0));
            ++used;
            return cache.back();
        };
        const double c1_start = c0.c1 > 0 ? c0.c1 : 1.0;
        for (const double r : out.floors) {
            int used = 0;
            eval(0.0, used);
            auto closest = [&]() {
                const FloorEval* b = nullptr;
                for (const FloorEval& e : cache)
                    if (!b || std::fabs(e.mean - r) < std::fabs(b->mean - r) ||
                        (std::fabs(e.mean - r) == std::fabs(b->mean - r) && e.c1 < b->c1))
                        b = &e;
                return *b;
            };
            auto bracket = [&](double& lo, double& hi, bool& have_hi) {
                lo = 0.0;
                have_hi = false;
                hi = 0.0;
                for (const FloorEval& e : cache) {
                    if (e.mean < r && e.c1 > lo) lo = e.c1;
                    if (e.mean >= r && (!have_hi || e.c1 < hi)) {
                        hi = e.c1;
                        have_hi = true;
                    }
                }
            };
            double lo, hi;
            bool have_hi;
            bracket(lo, hi, have_hi);
            // grow the upper end until the optimum's mean reaches the floor
            double probe = c1_start;
            for (const FloorEval& e : cache) probe = std::max(probe, e.c1);
            while (!have_hi && used < budget && probe < 1e15) {
                const FloorEval& e = eval(probe, used);
                if (e.mean >= r) break;
                probe *= 2.0;
                bracket(lo, hi, have_hi);
            }
            bracket(lo, hi, have_hi);
            while (have_hi && used < budget && std::fabs(closest().mean - r) > tol && hi - lo > 1e-12 * hi) {
                eval(0.5 * (lo + hi), used);
                bracket(lo, hi, have_hi);
            }
            out.best.push_back(closest());
            out.solves.push_back(used);
        }
    } catch (...) {
        set_coeffs(ctx, c0);
        throw;
    }
    set_coeffs(ctx, c0);
    return out;
}

thread_local std::string g_err2;

template <class F>
int32_t guard(mvsk_gpu_ctx* ctx, F&& f) {
    try {
        f();
        return MVSK_OK;
    } catch (const ApiError& e) {
        if (ctx) ctx->err = e.what();
        g_err2 = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        g_err2 = e.what();
        return MVSK_INTERNAL_ERROR;
    }
}

}  // namespace
}  // namespace mvsk_b200

using namespace mvsk_b200;

extern "C" {

int32_t mvsk_gpu_preset(const char* name, mvsk_solver_config* out) {
    return guard(nullptr, [&] {
        const std::string s(name ? name : "");
        if (s != "small" && s != "large") throw ApiError(MVSK_DOMAIN_ERROR, "preset: unknown mode " + s);
        std::memset(out, 0, sizeof(*out));
        // SolverConfig defaults (solver.hpp:44-62) + TangentSolveConfig (affine_normal.hpp:59-69)
        out->epsilon = 1e-6;
        out->tau = 1e-8;
        out->projected_trial_step = 0.05;
        out->restart_trial_steps[0] = 0.045;
        out->restart_trial_steps[1] = 0.02;
        out->n_restart_trial_steps = 2;
        out->restart_max_iter = 120;
        out->tangent.krylov_tol = 1e-3;
        out->tangent.krylov_maxit = 15;
        out->tangent.hutchinson_probes = 8;
        out->tangent.probe_maxit = 5;
        if (s == "small") {  // :64-71
            out->max_iter = 300;
            out->tangent.mode = 0;
            out->tangent.lambda = 0.0;
        } else {  // :73-85
            out->max_iter = 40;
            out->has_max_elapsed = 1;
            out->max_elapsed_seconds = 60.0;
            out->tangent.mode = 1;
            out->tangent.lambda = 1e-4;
            out->stall_restarts = 1;
            out->identification_pass = 1;
        }
        std::strncpy(out->label, s.c_str(), sizeof(out->label) - 1);
    });
}

int32_t mvsk_gpu_yand_direction(mvsk_gpu_ctx* ctx, int32_t slot, const mvsk_tangent_config* cfg, uint64_t it_seed,
                                double* d_out, mvsk_direction_diag* diag) {
    return guard(ctx, [&] {
        MVSK_CUDA(cudaSetDevice(ctx->device));
        check_slot(ctx, slot);
        if (ctx->pub_face.m < 2) throw ApiError(MVSK_DIMENSION_ERROR, "tangent basis needs n >= 2");
        View v{ctx, ctx->pub_face};
        mvsk_direction_diag dd{};
        const Vec d = yand_direction(v, slot, tangent_of(*cfg), it_seed, dd);
        std::copy(d.begin(), d.end(), d_out);
        if (diag) *diag = dd;
    });
}

int32_t mvsk_gpu_solve(mvsk_gpu_ctx* ctx, const mvsk_solver_config* cfg, const double* x0, double* x_star,
                       mvsk_solve_report* report, mvsk_observer_fn observer, void* observer_user) {
    return guard(ctx, [&] {
        MVSK_CUDA(cudaSetDevice(ctx->device));
        const auto t0 = std::chrono::steady_clock::now();
        const SolveCfg sc = solve_cfg_of(cfg);
        const uint64_t f0 = ctx->fwd, t0p = ctx->tr, p0 = ctx->phys;
        std::function<void(int, double, const Vec&)> obs;
        if (observer)
            obs = [&](int it, double f, const Vec& x) { observer(observer_user, it, f, x.data(), (int64_t)x.size()); };
        const Vec xs = x0 ? Vec(x0, x0 + ctx->n) : Vec();
        const FaceMap saved = ctx->pub_face;
        g_prof = Prof();
        g_prof.on = std::getenv("MVSK_PROFILE") != nullptr;
        Report r = solve(ctx, sc, xs, obs);
        fold_face_counters(ctx);
        ctx->pub_face = saved;
        if (g_prof.on)
            std::fprintf(stderr,
                         "[mvsk profile] total %.3f ms | make_cache %.3f ms (%ld) | gradient %.3f ms | direction %.3f "
                         "ms (%ld) | line_model %.3f ms (%ld) | project_slice %.3f ms (%ld) | face rebuild %.3f ms (%ld) "
                         "| full residual %.3f ms (%ld) | spg %.3f ms | direct: gram %.3f ms, trace %.3f ms, lu+inv %.3f ms\n",
                         1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                         1e3 * g_prof.cache, g_prof.ncache, 1e3 * g_prof.grad, 1e3 * g_prof.dir, g_prof.ndir,
                         1e3 * g_prof.line, g_prof.nline, 1e3 * g_prof.proj, g_prof.nproj, 1e3 * g_prof.face,
                         g_prof.nface, 1e3 * g_prof.resid, g_prof.nresid, 1e3 * g_prof.spg, 1e3 * g_prof.dgram,
                         1e3 * g_prof.dquad, 1e3 * g_prof.dlu);
        std::copy(r.x.begin(), r.x.end(), x_star);
        std::memset(report, 0, sizeof(*report));
        report->f_star = r.f;
        report->kkt_residual = r.kkt;
        report->interior_residual = r.interior;
        report->iterations = r.iterations;
        report->face_events = r.face_events;
        report->restarts = r.restarts;
        report->identification_steps = r.ident;
        report->krylov_iters_total = r.krylov;
        report->oracle_passes = (ctx->fwd - f0) + (ctx->tr - t0p);
        report->physical_passes = ctx->phys - p0;
        report->status = r.status;
        report->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::strncpy(report->config_label, cfg->label, sizeof(report->config_label) - 1);
    });
}

int32_t mvsk_gpu_set_coeffs(mvsk_gpu_ctx* ctx, const mvsk_coeffs* c) {
    return guard(ctx, [&] {
        if (!c) throw ApiError(MVSK_DOMAIN_ERROR, "set_coeffs: null coefficients");
        if (!std::isfinite(c->c1) || !std::isfinite(c->c2) || !std::isfinite(c->c3) || !std::isfinite(c->c4))
            throw ApiError(MVSK_DOMAIN_ERROR, "set_coeffs: non-finite coefficient");
        set_coeffs(ctx, *c);
    });
}

int32_t mvsk_gpu_floor_sweep(mvsk_gpu_ctx* ctx, const mvsk_solver_config* cfg, const mvsk_sweep_config* sw,
                             int32_t nfloors, const double* floors, double* x_out, mvsk_floor_point* points,
                             double* m_mv, double* m_max, int32_t* total_solves) {
    return guard(ctx, [&] {
        MVSK_CUDA(cudaSetDevice(ctx->device));
        if (!cfg || nfloors < 1) throw ApiError(MVSK_DOMAIN_ERROR, "floor_sweep: need a solver config and nfloors >= 1");
        mvsk_sweep_config d{};
        d.mean_tol = 1e-3;
        d.max_solves = 16;
        d.warm_start = 1;
        const mvsk_sweep_config& s = sw ? *sw : d;
        std::vector<double> fl;
        if (floors) {
            fl.assign(floors, floors + nfloors);
            for (double v : fl)
                if (!std::isfinite(v)) throw ApiError(MVSK_DOMAIN_ERROR, "floor_sweep: non-finite floor");
        }
        const FaceMap saved = ctx->pub_face;
        const SweepOut o = floor_sweep(ctx, solve_cfg_of(cfg), s, fl, nfloors);
        fold_face_counters(ctx);
        ctx->pub_face = saved;
        for (int k = 0; k < nfloors; ++k) {
            const FloorEval& e = o.best[(size_t)k];
            if (x_out) std::copy(e.x.begin(), e.x.end(), x_out + (size_t)k * ctx->n);
            if (points) {
                mvsk_floor_point& p = points[k];
                p.floor = o.floors[(size_t)k];
                p.c1 = e.c1;
                p.mean = e.mean;
                p.f_star = e.f;
                p.kkt_residual = e.kkt;
                p.status = e.status;
                p.solves = o.solves[(size_t)k];
            }
        }
        if (m_mv) *m_mv = o.m_mv;
        if (m_max) *m_max = o.m_max;
        if (total_solves) *total_solves = o.total;
    });
}

}  // extern "C"
