// TEST INFRASTRUCTURE ONLY — see mvsk_oracle.hpp. CPU restatement of the
// reference (/root/reference/proj/include/mvsk/*.hpp), file:line cited per function.
#include "mvsk_oracle.hpp"

#include <thread>

namespace mo {

int& pass_threads() {
    static int t = 1;
    return t;
}

// Runs body(lo, hi) over [0, T) split into pass_threads() contiguous blocks.
template <class F>
static void parallel_rows(index_t T, F&& body) {
    const int nt = pass_threads();
    if (nt <= 1 || T < 2 * nt) {
        body(index_t(0), T, 0);
        return;
    }
    std::vector<std::thread> th;
    for (int id = 0; id < nt; ++id)
        th.emplace_back([&, id] { body(T * id / nt, T * (id + 1) / nt, id); });
    for (auto& t : th) t.join();
}

// Eigen row-major GEMV at oracle.hpp:128,135 — one streaming pass over rows.
void gemv(const Mat& A, const Vec& x, Vec& z) {
    const index_t T = A.rows, n = A.cols;
    z.assign(static_cast<size_t>(T), 0.0);
    const double* xp = x.data();
    parallel_rows(T, [&](index_t lo, index_t hi, int) {
        for (index_t t = lo; t < hi; ++t) {
            const double* r = A.row(t);
            double s = 0.0;
            for (index_t j = 0; j < n; ++j) s += r[j] * xp[j];
            z[static_cast<size_t>(t)] = s;
        }
    });
}

// A^T w at oracle.hpp:139 — one streaming pass; with >1 threads each thread
// owns a contiguous row block and the partials are summed in thread order.
void gemv_t(const Mat& A, const Vec& w, Vec& g) {
    const index_t T = A.rows, n = A.cols;
    g.assign(static_cast<size_t>(n), 0.0);
    const int nt = pass_threads();
    if (nt <= 1 || T < 2 * nt) {
        double* gp = g.data();
        for (index_t t = 0; t < T; ++t) {
            const double* r = A.row(t);
            const double wt = w[static_cast<size_t>(t)];
            for (index_t j = 0; j < n; ++j) gp[j] += r[j] * wt;
        }
        return;
    }
    std::vector<Vec> part(static_cast<size_t>(nt), Vec(static_cast<size_t>(n), 0.0));
    parallel_rows(T, [&](index_t lo, index_t hi, int id) {
        double* gp = part[static_cast<size_t>(id)].data();
        for (index_t t = lo; t < hi; ++t) {
            const double* r = A.row(t);
            const double wt = w[static_cast<size_t>(t)];
            for (index_t j = 0; j < n; ++j) gp[j] += r[j] * wt;
        }
    });
    for (int id = 0; id < nt; ++id)
        for (index_t j = 0; j < n; ++j) g[static_cast<size_t>(j)] += part[static_cast<size_t>(id)][static_cast<size_t>(j)];
}

// ---- panel.hpp ---------------------------------------------------------------
// center_panel, panel.hpp:32-44
ReturnPanel center_panel(Mat R) {
    if (R.rows < 2) throw dimension_error("center_panel: need at least two time periods");
    if (R.cols < 1) throw dimension_error("center_panel: need at least one asset");
    for (double v : R.a)
        if (!std::isfinite(v)) throw data_error("center_panel: non-finite return entry");
    ReturnPanel p;
    const index_t T = R.rows, n = R.cols;
    p.mu.assign(static_cast<size_t>(n), 0.0);
    for (index_t t = 0; t < T; ++t)
        for (index_t j = 0; j < n; ++j) p.mu[static_cast<size_t>(j)] += R(t, j);
    for (double& m : p.mu) m /= static_cast<double>(T);
    p.A = Mat(T, n);
    for (index_t t = 0; t < T; ++t)
        for (index_t j = 0; j < n; ++j) p.A(t, j) = R(t, j) - p.mu[static_cast<size_t>(j)];
    p.R = std::move(R);
    return p;
}

// make_coefficients, panel.hpp:64-72
PreferenceCoefficients make_coefficients(double c1, double c2, double c3, double c4) {
    if (c1 < 0 || c2 < 0 || c3 < 0 || c4 < 0) throw domain_error("coefficients must be nonnegative");
    if (c1 == 0 && c2 == 0 && c3 == 0 && c4 == 0) throw domain_error("coefficients must not all be zero");
    return PreferenceCoefficients{c1, c2, c3, c4};
}

// crra_coefficients, panel.hpp:76-87
PreferenceCoefficients crra_coefficients(double gamma) {
    if (!(gamma > 0)) throw domain_error("crra_coefficients: gamma must be positive");
    PreferenceCoefficients c;
    c.c1 = 1.0;
    c.c2 = gamma / 2.0;
    c.c3 = gamma * (gamma + 1.0) / 6.0;
    c.c4 = gamma * (gamma + 1.0) * (gamma + 2.0) / 24.0;
    return c;
}

// ---- oracle.hpp ----------------------------------------------------------------
// ctor, oracle.hpp:31-41
Oracle::Oracle(const Mat& A, Vec mu, PreferenceCoefficients coeffs,
               std::shared_ptr<PassCounter> counter, Vec zoff, double value_offset)
    : A_(&A), mu_(std::move(mu)), zoff_(std::move(zoff)), c_(coeffs), f_offset_(value_offset),
      passes_(counter ? std::move(counter) : std::make_shared<PassCounter>()) {
    if (sz(mu_) != A_->cols) throw dimension_error("oracle: mu length does not match panel columns");
    if (!zoff_.empty() && sz(zoff_) != A_->rows)
        throw dimension_error("oracle: offset length does not match panel rows");
}

// make_cache, oracle.hpp:54-69
OracleCache Oracle::make_cache(Vec x) const {
    if (sz(x) != A_->cols) throw dimension_error("oracle: iterate length does not match panel");
    OracleCache cache;
    cache.z = forward(x);
    const size_t T = cache.z.size();
    cache.z2.resize(T);
    cache.z3.resize(T);
    double s2 = 0, s3 = 0, s4 = 0;
    for (size_t t = 0; t < T; ++t) {
        cache.z2[t] = cache.z[t] * cache.z[t];
        cache.z3[t] = cache.z2[t] * cache.z[t];
        s2 += cache.z2[t];
        s3 += cache.z3[t];
        s4 += cache.z2[t] * cache.z2[t];
    }
    const double Td = static_cast<double>(A_->rows);
    cache.f_value = f_offset_ - c_.c1 * dot(mu_, x) + (c_.c2 * s2 - c_.c3 * s3 + c_.c4 * s4) / Td;
    cache.x = std::move(x);
    if (!std::isfinite(cache.f_value)) throw numeric_error("oracle: non-finite objective value");
    return cache;
}

// moments, oracle.hpp:73-77
std::tuple<double, double, double, double> Oracle::moments(const OracleCache& c) const {
    const double Td = static_cast<double>(A_->rows);
    double s2 = 0, s3 = 0, s4 = 0;
    for (size_t t = 0; t < c.z.size(); ++t) {
        s2 += c.z2[t];
        s3 += c.z3[t];
        s4 += c.z2[t] * c.z2[t];
    }
    return {dot(mu_, c.x), s2 / Td, s3 / Td, s4 / Td};
}

// gradient, oracle.hpp:79-90
const Vec& Oracle::gradient(const OracleCache& cache) const {
    if (!cache.has_grad) {
        const double Td = static_cast<double>(A_->rows);
        Vec w(cache.z.size());
        for (size_t t = 0; t < w.size(); ++t)
            w[t] = (2.0 * c_.c2 * cache.z[t] - 3.0 * c_.c3 * cache.z2[t] + 4.0 * c_.c4 * cache.z3[t]) / Td;
        Vec atw = transpose_apply(w);
        cache.grad.resize(atw.size());
        for (size_t j = 0; j < atw.size(); ++j) cache.grad[j] = -c_.c1 * mu_[j] + atw[j];
        if (!all_finite(cache.grad)) throw numeric_error("oracle: non-finite gradient");
        cache.has_grad = true;
    }
    return cache.grad;
}

// hvp, oracle.hpp:92-101
Vec Oracle::hvp(const OracleCache& cache, const Vec& v) const {
    const double Td = static_cast<double>(A_->rows);
    Vec Av = forward_tangent(v);
    Vec w(Av.size());
    for (size_t t = 0; t < w.size(); ++t)
        w[t] = (2.0 * c_.c2 - 6.0 * c_.c3 * cache.z[t] + 12.0 * c_.c4 * cache.z2[t]) * Av[t] / Td;
    Vec out = transpose_apply(w);
    if (!all_finite(out)) throw numeric_error("oracle: non-finite Hessian product");
    return out;
}

// third_action, oracle.hpp:103-113
Vec Oracle::third_action(const OracleCache& cache, const Vec& u, const Vec& v) const {
    const double Td = static_cast<double>(A_->rows);
    Vec Au = forward_tangent(u);
    Vec Av = forward_tangent(v);
    Vec w(Au.size());
    for (size_t t = 0; t < w.size(); ++t)
        w[t] = (-6.0 * c_.c3 + 24.0 * c_.c4 * cache.z[t]) * Au[t] * Av[t] / Td;
    Vec out = transpose_apply(w);
    if (!all_finite(out)) throw numeric_error("oracle: non-finite third-order action");
    return out;
}

// hessian_diag_weights, oracle.hpp:116-119
Vec Oracle::hessian_diag_weights(const OracleCache& cache) const {
    Vec w(cache.z.size());
    for (size_t t = 0; t < w.size(); ++t)
        w[t] = 2.0 * c_.c2 - 6.0 * c_.c3 * cache.z[t] + 12.0 * c_.c4 * cache.z2[t];
    return w;
}

// forward / forward_tangent / transpose_apply, oracle.hpp:126-140
Vec Oracle::forward(const Vec& x) const {
    ++passes_->forward;
    Vec z;
    gemv(*A_, x, z);
    if (!zoff_.empty())
        for (size_t t = 0; t < z.size(); ++t) z[t] += zoff_[t];
    return z;
}
Vec Oracle::forward_tangent(const Vec& v) const {
    ++passes_->forward;
    Vec z;
    gemv(*A_, v, z);
    return z;
}
Vec Oracle::transpose_apply(const Vec& w) const {
    ++passes_->transpose;
    Vec g;
    gemv_t(*A_, w, g);
    return g;
}

// ---- linesearch.hpp --------------------------------------------------------------
// power_sums, linesearch.hpp:22-44
PowerSums power_sums(const Vec& z, const Vec& w) {
    if (z.size() != w.size()) throw dimension_error("power_sums: length mismatch");
    PowerSums s;
    for (size_t t = 0; t < z.size(); ++t) {
        const double zt = z[t], wt = w[t];
        const double w2 = wt * wt, z2 = zt * zt;
        s.s11 += zt * wt;
        s.s21 += z2 * wt;
        s.s31 += z2 * zt * wt;
        s.s02 += w2;
        s.s12 += zt * w2;
        s.s22 += z2 * w2;
        s.s03 += w2 * wt;
        s.s13 += zt * w2 * wt;
        s.s04 += w2 * w2;
    }
    const double T = static_cast<double>(z.size());
    s.s11 /= T; s.s21 /= T; s.s31 /= T;
    s.s02 /= T; s.s12 /= T; s.s22 /= T;
    s.s03 /= T; s.s13 /= T; s.s04 /= T;
    return s;
}

// line_model, linesearch.hpp:62-81
LineModel line_model(const Oracle& oracle, const OracleCache& cache, const Vec& d, double cap) {
    const double dn = norm(d);
    if (!(dn > 0)) throw domain_error("line_model: zero direction");
    if (std::abs(vsum(d)) > 1e-10 * dn) throw domain_error("line_model: direction is not tangent to the simplex");
    LineModel m;
    Vec w = oracle.sample_direction(d);
    m.sums = power_sums(cache.z, w);
    const auto& c = oracle.coeffs();
    m.a0 = cache.f_value;
    m.a1 = -c.c1 * dot(oracle.mu(), d) + 2.0 * c.c2 * m.sums.s11 - 3.0 * c.c3 * m.sums.s21 +
           4.0 * c.c4 * m.sums.s31;
    m.a2 = c.c2 * m.sums.s02 - 3.0 * c.c3 * m.sums.s12 + 6.0 * c.c4 * m.sums.s22;
    m.a3 = -c.c3 * m.sums.s03 + 4.0 * c.c4 * m.sums.s13;
    m.a4 = c.c4 * m.sums.s04;
    m.alpha_cap = cap;
    return m;
}

// cubic_real_roots, linesearch.hpp:87-114
std::vector<double> cubic_real_roots(double c3, double c2, double c1, double c0) {
    const double p = c2 / c3, q = c1 / c3, r = c0 / c3;
    const double a = q - p * p / 3.0;
    const double b = 2.0 * p * p * p / 27.0 - p * q / 3.0 + r;
    const double shift = p / 3.0;
    std::vector<double> roots;
    const double disc = b * b / 4.0 + a * a * a / 27.0;
    if (disc > 0.0) {
        const double sq = std::sqrt(disc);
        const double u = std::cbrt(-b / 2.0 + sq);
        const double v = std::cbrt(-b / 2.0 - sq);
        roots.push_back(u + v - shift);
    } else if (a == 0.0 && b == 0.0) {
        roots.push_back(-shift);
    } else {
        constexpr double pi = 3.14159265358979323846;
        const double rho = std::sqrt(-a * a * a / 27.0);
        double cosarg = -b / (2.0 * rho);
        cosarg = std::min(1.0, std::max(-1.0, cosarg));
        const double phi = std::acos(cosarg);
        const double mag = 2.0 * std::sqrt(-a / 3.0);
        for (int k = 0; k < 3; ++k) roots.push_back(mag * std::cos((phi + 2.0 * pi * k) / 3.0) - shift);
    }
    return roots;
}

// polish_root, linesearch.hpp:118-128
double polish_root(const LineModel& m, double alpha) {
    for (int it = 0; it < 2; ++it) {
        const double d1 = m.deriv(alpha);
        const double d2 = 2.0 * m.a2 + alpha * (6.0 * m.a3 + alpha * 12.0 * m.a4);
        if (d2 == 0.0) break;
        double next = alpha - d1 / d2;
        if (!(next > 0.0) || !(next < m.alpha_cap)) break;
        alpha = next;
    }
    return alpha;
}

// minimize_line, linesearch.hpp:135-168
std::pair<double, double> minimize_line(const LineModel& m) {
    if (!(m.alpha_cap > 0.0)) return {0.0, m.a0};
    std::vector<double> cands{0.0, m.alpha_cap};
    const double scale = std::max({std::abs(m.a1), std::abs(m.a2), std::abs(m.a3), std::abs(m.a4), 1e-300});
    if (std::abs(m.a4) > 1e-14 * scale) {
        for (double r : cubic_real_roots(4.0 * m.a4, 3.0 * m.a3, 2.0 * m.a2, m.a1))
            if (r > 0.0 && r < m.alpha_cap) cands.push_back(polish_root(m, r));
    } else if (std::abs(m.a3) > 1e-14 * scale) {
        const double A = 3.0 * m.a3, B = 2.0 * m.a2, C = m.a1;
        const double disc = B * B - 4.0 * A * C;
        if (disc >= 0.0) {
            const double sq = std::sqrt(disc);
            for (double r : {(-B + sq) / (2.0 * A), (-B - sq) / (2.0 * A)})
                if (r > 0.0 && r < m.alpha_cap) cands.push_back(polish_root(m, r));
        }
    } else if (std::abs(m.a2) > 1e-14 * scale) {
        const double r = -m.a1 / (2.0 * m.a2);
        if (r > 0.0 && r < m.alpha_cap) cands.push_back(r);
    }
    double best_alpha = 0.0, best_val = m.a0;
    for (double alpha : cands) {
        const double v = m.eval(alpha);
        if (v < best_val || (v == best_val && alpha < best_alpha)) {
            best_val = v;
            best_alpha = alpha;
        }
    }
    return {best_alpha, best_val};
}

// armijo_search, linesearch.hpp:178-193
ArmijoResult armijo_search(const std::function<double(double)>& phi, double g_dot_d,
                           double alpha_init, double sigma, double shrink) {
    if (!(g_dot_d < 0)) throw domain_error("armijo_search: direction is not descent");
    if (!(sigma > 0 && sigma < 1) || !(shrink > 0 && shrink < 1)) throw domain_error("armijo_search: bad constants");
    const double phi0 = phi(0.0);
    double alpha = alpha_init;
    for (int k = 0; k < 60; ++k) {
        if (phi(alpha) <= phi0 + sigma * alpha * g_dot_d) return {alpha, false};
        alpha *= shrink;
    }
    return {0.0, true};
}

// ---- simplex.hpp -----------------------------------------------------------------
// TangentBasis ctor, simplex.hpp:22-45 (dense cache omitted: the matrix-free
// apply is what yand_direction and the solver use)
TangentBasis::TangentBasis(index_t n) : n_(n) {
    if (n < 2) throw dimension_error("tangent basis needs n >= 2");
    v_.assign(static_cast<size_t>(n), -1.0 / std::sqrt(static_cast<double>(n)));
    v_[0] += 1.0;
    beta_ = 2.0 / sqnorm(v_);
}

// apply, simplex.hpp:63-70
Vec TangentBasis::apply(const Vec& y) const {
    if (sz(y) != n_ - 1) throw dimension_error("tangent basis: bad reduced vector length");
    Vec p(static_cast<size_t>(n_));
    p[0] = 0.0;
    for (index_t i = 1; i < n_; ++i) p[static_cast<size_t>(i)] = y[static_cast<size_t>(i - 1)];
    const double s = beta_ * dot(v_, p);
    for (size_t i = 0; i < p.size(); ++i) p[i] -= s * v_[i];
    return p;
}

// apply_transpose, simplex.hpp:73-78
Vec TangentBasis::apply_transpose(const Vec& x) const {
    if (sz(x) != n_) throw dimension_error("tangent basis: bad ambient vector length");
    const double s = beta_ * dot(v_, x);
    Vec out(static_cast<size_t>(n_ - 1));
    for (index_t i = 1; i < n_; ++i) out[static_cast<size_t>(i - 1)] = x[static_cast<size_t>(i)] - s * v_[static_cast<size_t>(i)];
    return out;
}

// alpha_max, simplex.hpp:93-99
double alpha_max(const Vec& x, const Vec& d, double tau) {
    double cap = std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < x.size(); ++i)
        if (d[i] < 0.0) cap = std::min(cap, (x[i] - tau) / (-d[i]));
    return std::max(cap, 0.0);
}

// project_slice, simplex.hpp:104-122
Vec project_slice(const Vec& v, double tau, double mass) {
    const index_t n = sz(v);
    const double s = mass - static_cast<double>(n) * tau;
    if (!(tau >= 0.0) || !(s > 0.0)) throw domain_error("project_slice: need 0 <= tau < mass/n");
    std::vector<double> u(static_cast<size_t>(n));
    for (index_t i = 0; i < n; ++i) u[static_cast<size_t>(i)] = v[static_cast<size_t>(i)] - tau;
    std::sort(u.begin(), u.end(), std::greater<double>());
    double css = 0.0, theta = 0.0;
    for (index_t k = 0; k < n; ++k) {
        css += u[static_cast<size_t>(k)];
        const double cand = (css - s) / static_cast<double>(k + 1);
        if (u[static_cast<size_t>(k)] > cand) theta = cand;
    }
    Vec out(static_cast<size_t>(n));
    for (index_t i = 0; i < n; ++i) out[static_cast<size_t>(i)] = std::max(v[static_cast<size_t>(i)] - tau - theta, 0.0) + tau;
    return out;
}

// projected_kkt_residual, simplex.hpp:126-129
double projected_kkt_residual(const Vec& g) {
    const double mean = vmean(g);
    double s = 0.0;
    for (double x : g) s += (x - mean) * (x - mean);
    return std::sqrt(s);
}

// gradient_mapping_residual, simplex.hpp:135-137
double gradient_mapping_residual(const Vec& x, const Vec& g, double tau) {
    Vec y(x.size());
    for (size_t i = 0; i < x.size(); ++i) y[i] = x[i] - g[i];
    Vec p = project_slice(y, tau);
    double s = 0.0;
    for (size_t i = 0; i < x.size(); ++i) s += (x[i] - p[i]) * (x[i] - p[i]);
    return std::sqrt(s);
}

// restrict_to_face, simplex.hpp:161-192
FaceProblem restrict_to_face(const Mat& A, const Vec& mu, const Vec& x, double tau) {
    const index_t n = A.cols, T = A.rows;
    FaceProblem fp;
    for (index_t i = 0; i < n; ++i)
        if (x[static_cast<size_t>(i)] > tau + 1e-12) fp.free_indices.push_back(i);
    const index_t nf = static_cast<index_t>(fp.free_indices.size());
    if (nf == 0) throw domain_error("restrict_to_face: degenerate face, all coordinates pinned");
    fp.A = Mat(T, nf);
    fp.mu.resize(static_cast<size_t>(nf));
    for (index_t j = 0; j < nf; ++j) {
        const index_t src = fp.free_indices[static_cast<size_t>(j)];
        for (index_t t = 0; t < T; ++t) fp.A(t, j) = A(t, src);
        fp.mu[static_cast<size_t>(j)] = mu[static_cast<size_t>(src)];
    }
    fp.zoff.assign(static_cast<size_t>(T), 0.0);
    double mu_pin = 0.0;
    size_t next_free = 0;
    for (index_t i = 0; i < n; ++i) {
        if (next_free < fp.free_indices.size() && fp.free_indices[next_free] == i) {
            ++next_free;
        } else {
            for (index_t t = 0; t < T; ++t) fp.zoff[static_cast<size_t>(t)] += tau * A(t, i);
            mu_pin += tau * mu[static_cast<size_t>(i)];
        }
    }
    fp.mu_pinned_term = mu_pin;
    fp.free_mass = 1.0 - static_cast<double>(n - nf) * tau;
    return fp;
}

// ---- affine_normal.hpp -------------------------------------------------------------
// ReducedFrame::apply_Q, affine_normal.hpp:28-33
Vec ReducedFrame::apply_Q(const Vec& eta) const {
    Vec p(nu.size());
    p[0] = 0.0;
    for (size_t i = 1; i < p.size(); ++i) p[i] = eta[i - 1];
    const double s = beta * dot(v, p);
    for (size_t i = 0; i < p.size(); ++i) p[i] -= s * v[i];
    return p;
}
// ReducedFrame::apply_Qt, affine_normal.hpp:36-39
Vec ReducedFrame::apply_Qt(const Vec& w) const {
    const double s = beta * dot(v, w);
    Vec out(nu.size() - 1);
    for (size_t i = 1; i < nu.size(); ++i) out[i - 1] = w[i] - s * v[i];
    return out;
}

// householder_frame, affine_normal.hpp:42-56
ReducedFrame householder_frame(const Vec& reduced_grad) {
    const double gn = norm(reduced_grad);
    if (!(gn > 0)) throw domain_error("householder_frame: zero reduced gradient (stationary)");
    if (reduced_grad.size() < 2) throw dimension_error("householder_frame: need m >= 2");
    ReducedFrame f;
    f.nu = reduced_grad;  // reduced_grad / gn: Eigen's scalar quotient divides each coefficient
    for (double& x : f.nu) x /= gn;
    f.grad_norm = gn;
    const double s = f.nu[0] >= 0.0 ? 1.0 : -1.0;
    f.v = f.nu;
    f.v[0] += s;
    f.beta = 2.0 / sqnorm(f.v);
    return f;
}

// cg_capped, affine_normal.hpp:85-113
Vec cg_capped(const std::function<Vec(const Vec&)>& H, const Vec& rhs, double tol, int cap,
              const Vec* jacobi_diag, int& iters, bool& breakdown) {
    const size_t m = rhs.size();
    Vec x(m, 0.0);
    Vec r = rhs;
    auto precond = [&](const Vec& rr) {
        if (!jacobi_diag) return rr;
        Vec z(rr.size());
        for (size_t i = 0; i < rr.size(); ++i) z[i] = rr[i] / (*jacobi_diag)[i];
        return z;
    };
    Vec z = precond(r);
    Vec p = z;
    double rz = dot(r, z);
    const double target = tol * norm(rhs);
    int it = 0;
    while (it < cap && norm(r) > target) {
        Vec Hp = H(p);
        const double pHp = dot(p, Hp);
        if (pHp <= 0.0) {
            breakdown = true;
            break;
        }
        const double alpha = rz / pHp;
        axpy_inplace(x, alpha, p);
        axpy_inplace(r, -alpha, Hp);
        z = precond(r);
        const double rz2 = dot(r, z);
        const double beta = rz2 / rz;
        for (size_t i = 0; i < m; ++i) p[i] = z[i] + beta * p[i];
        rz = rz2;
        ++it;
    }
    iters += it;
    return x;
}

// PartialPivLU: Doolittle with row partial pivoting on the largest |entry|
// (Eigen::PartialPivLU semantics: a zero pivot column is skipped, the solve
// then divides by the zero diagonal and yields non-finite values).
PartialPivLU::PartialPivLU(const Mat& M) : n(M.rows), lu(M.a), perm(static_cast<size_t>(M.rows)) {
    for (index_t i = 0; i < n; ++i) perm[static_cast<size_t>(i)] = i;
    auto at = [&](index_t r, index_t c) -> double& { return lu[static_cast<size_t>(r * n + c)]; };
    for (index_t k = 0; k < n; ++k) {
        index_t piv = k;
        double big = std::abs(at(k, k));
        for (index_t r = k + 1; r < n; ++r)
            if (std::abs(at(r, k)) > big) {
                big = std::abs(at(r, k));
                piv = r;
            }
        if (big != 0.0) {
            if (piv != k) {
                for (index_t c = 0; c < n; ++c) std::swap(at(k, c), at(piv, c));
                std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(piv)]);
            }
            // Eigen's unblocked LU divides the column by the pivot (no reciprocal)
            const double piv_v = at(k, k);
            for (index_t r = k + 1; r < n; ++r) at(r, k) /= piv_v;
        }
        for (index_t r = k + 1; r < n; ++r) {
            const double l = at(r, k);
            if (l != 0.0)
                for (index_t c = k + 1; c < n; ++c) at(r, c) -= l * at(k, c);
        }
    }
}
Vec PartialPivLU::solve(const Vec& b) const {
    Vec y(static_cast<size_t>(n));
    for (index_t i = 0; i < n; ++i) y[static_cast<size_t>(i)] = b[static_cast<size_t>(perm[static_cast<size_t>(i)])];
    for (index_t i = 0; i < n; ++i) {
        double s = y[static_cast<size_t>(i)];
        for (index_t c = 0; c < i; ++c) s -= lu[static_cast<size_t>(i * n + c)] * y[static_cast<size_t>(c)];
        y[static_cast<size_t>(i)] = s;
    }
    for (index_t i = n - 1; i >= 0; --i) {
        double s = y[static_cast<size_t>(i)];
        for (index_t c = i + 1; c < n; ++c) s -= lu[static_cast<size_t>(i * n + c)] * y[static_cast<size_t>(c)];
        y[static_cast<size_t>(i)] = s / lu[static_cast<size_t>(i * n + i)];
    }
    return y;
}

// yand_direction, affine_normal.hpp:127-245
Vec yand_direction(const Oracle& oracle, const TangentBasis& basis, const OracleCache& cache,
                   const TangentSolveConfig& cfg, std::uint64_t it_seed, DirectionDiagnostics* diag_out) {
    const index_t n = oracle.assets();
    const index_t m = n - 1;
    DirectionDiagnostics local;
    DirectionDiagnostics& diag = diag_out ? *diag_out : local;

    const Vec& g = oracle.gradient(cache);
    Vec gbar = basis.apply_transpose(g);
    const double gn = norm(gbar);
    diag.reduced_grad_norm = gn;
    if (!(gn > 0)) throw domain_error("yand_direction: stationary point, no direction");
    if (m == 1) {
        Vec y = gbar;  // (-gbar) / gn, coefficient-wise
        for (double& v : y) v = -v / gn;
        return basis.apply(y);
    }

    const ReducedFrame frame = householder_frame(gbar);
    const index_t mm = m - 1;
    const auto& c = oracle.coeffs();
    const bool has_third = (c.c3 != 0.0 || c.c4 != 0.0);
    const index_t T = oracle.periods();
    const double Td = static_cast<double>(T);

    Vec u;
    if (cfg.mode == TangentSolveConfig::Mode::direct) {
        // :153-160 W = A U Q (T x mm)
        Mat UQ(n, mm);
        for (index_t k = 0; k < mm; ++k) {
            Vec e(static_cast<size_t>(mm), 0.0);
            e[static_cast<size_t>(k)] = 1.0;
            Vec col = basis.apply(frame.apply_Q(e));
            for (index_t i = 0; i < n; ++i) UQ(i, k) = col[static_cast<size_t>(i)];
        }
        oracle.counter()->forward += static_cast<std::uint64_t>(mm);
        const Mat& A = oracle.A();
        Mat W(T, mm);
        for (index_t t = 0; t < T; ++t) {
            const double* ar = A.row(t);
            double* wr = W.row(t);
            for (index_t i = 0; i < n; ++i) {
                const double a = ar[i];
                const double* uq = UQ.row(i);
                for (index_t k = 0; k < mm; ++k) wr[k] += a * uq[k];
            }
        }
        const Vec psi2 = oracle.hessian_diag_weights(cache);
        // :163-166
        oracle.counter()->forward += 1;
        Vec unu = basis.apply(frame.nu);
        Vec t_nu;
        gemv(A, unu, t_nu);
        Vec h(static_cast<size_t>(mm), 0.0);
        for (index_t t = 0; t < T; ++t) {
            const double s = psi2[static_cast<size_t>(t)] * t_nu[static_cast<size_t>(t)];
            const double* wr = W.row(t);
            for (index_t k = 0; k < mm; ++k) h[static_cast<size_t>(k)] += wr[k] * s;
        }
        for (double& hv : h) hv /= Td;

        auto solve_with = [&](double lam) -> Vec {
            // :169-170 M = W^T diag(psi'') W / T + lam I
            Mat M(mm, mm);
            for (index_t t = 0; t < T; ++t) {
                const double* wr = W.row(t);
                const double p2 = psi2[static_cast<size_t>(t)];
                for (index_t i = 0; i < mm; ++i) {
                    const double wi = wr[i] * p2;
                    double* mr = M.row(i);
                    for (index_t j = 0; j < mm; ++j) mr[j] += wi * wr[j];
                }
            }
            for (double& v : M.a) v /= Td;
            for (index_t i = 0; i < mm; ++i) M(i, i) += lam;
            PartialPivLU lu(M);
            Vec a(static_cast<size_t>(mm), 0.0);
            if (has_third) {
                // :173-178 S = M^-1 W^T, q_t = w_t^T S_t, a = W^T(psi''' o q)/T
                Vec q(static_cast<size_t>(T));
                Vec wt(static_cast<size_t>(mm));
                for (index_t t = 0; t < T; ++t) {
                    for (index_t k = 0; k < mm; ++k) wt[static_cast<size_t>(k)] = W(t, k);
                    Vec st = lu.solve(wt);
                    double s = 0.0;
                    for (index_t k = 0; k < mm; ++k) s += wt[static_cast<size_t>(k)] * st[static_cast<size_t>(k)];
                    q[static_cast<size_t>(t)] = s;
                }
                for (index_t t = 0; t < T; ++t) {
                    const double psi3 = -6.0 * c.c3 + 24.0 * c.c4 * cache.z[static_cast<size_t>(t)];
                    const double s = psi3 * q[static_cast<size_t>(t)];
                    const double* wr = W.row(t);
                    for (index_t k = 0; k < mm; ++k) a[static_cast<size_t>(k)] += wr[k] * s;
                }
                for (double& av : a) av /= Td;
            }
            Vec rhs(static_cast<size_t>(mm));
            for (index_t k = 0; k < mm; ++k)
                rhs[static_cast<size_t>(k)] = h[static_cast<size_t>(k)] - (gn / static_cast<double>(n)) * a[static_cast<size_t>(k)];
            return lu.solve(rhs);
        };
        u = solve_with(cfg.lambda);
        if (!all_finite(u)) {
            diag.lambda_fallback = true;
            u = solve_with(std::max(cfg.lambda, 1e-4));
            if (!all_finite(u)) throw numeric_error("yand_direction: tangent solve failed");
        }
    } else {
        // :190-195
        auto Hop = [&](const Vec& e) -> Vec {
            Vec amb = basis.apply(frame.apply_Q(e));
            Vec hv = oracle.hvp(cache, amb);
            Vec red = frame.apply_Qt(basis.apply_transpose(hv));
            for (size_t i = 0; i < red.size(); ++i) red[i] += cfg.lambda * e[i];
            return red;
        };
        std::optional<Vec> jd;
        if (cfg.jacobi) {
            // :197-209
            SplitMix64 rng(0x0d1a6ULL ^ it_seed);
            Vec dg(static_cast<size_t>(mm), 0.0);
            for (int p = 0; p < 8; ++p) {
                Vec r(static_cast<size_t>(mm));
                for (index_t i = 0; i < mm; ++i) r[static_cast<size_t>(i)] = rng.next_sign();
                Vec hr = Hop(r);
                for (index_t i = 0; i < mm; ++i) dg[static_cast<size_t>(i)] += r[static_cast<size_t>(i)] * hr[static_cast<size_t>(i)];
            }
            for (double& v : dg) v /= 8.0;
            const double floor_val = std::max(1e-12, cfg.lambda);
            for (double& v : dg) v = std::max(v, floor_val);
            jd = dg;
        }
        const Vec* jdp = jd ? &*jd : nullptr;
        // :212-213
        Vec hvec = frame.apply_Qt(basis.apply_transpose(oracle.hvp(cache, basis.apply(frame.nu))));

        Vec a(static_cast<size_t>(mm), 0.0);
        if (has_third) {
            if (cfg.exact_trace) {
                // :217-226
                for (index_t k = 0; k < mm; ++k) {
                    Vec e(static_cast<size_t>(mm), 0.0);
                    e[static_cast<size_t>(k)] = 1.0;
                    Vec p = cg_capped(Hop, e, cfg.krylov_tol, cfg.krylov_maxit, jdp, diag.krylov_iters, diag.pcg_breakdown);
                    Vec t3 = frame.apply_Qt(basis.apply_transpose(oracle.third_action(
                        cache, basis.apply(frame.apply_Q(p)), basis.apply(frame.apply_Q(e)))));
                    axpy_inplace(a, 1.0, t3);
                }
            } else {
                // :227-237
                SplitMix64 rng(0x5eedULL ^ it_seed);
                for (int pr = 0; pr < cfg.hutchinson_probes; ++pr) {
                    Vec r(static_cast<size_t>(mm));
                    for (index_t i = 0; i < mm; ++i) r[static_cast<size_t>(i)] = rng.next_sign();
                    Vec s = cg_capped(Hop, r, cfg.krylov_tol, cfg.probe_maxit, jdp, diag.krylov_iters, diag.pcg_breakdown);
                    Vec t3 = frame.apply_Qt(basis.apply_transpose(oracle.third_action(
                        cache, basis.apply(frame.apply_Q(s)), basis.apply(frame.apply_Q(r)))));
                    axpy_inplace(a, 1.0, t3);
                }
                for (double& v : a) v /= static_cast<double>(cfg.hutchinson_probes);
            }
        }
        // :239-241
        Vec rhs(static_cast<size_t>(mm));
        for (index_t k = 0; k < mm; ++k)
            rhs[static_cast<size_t>(k)] = hvec[static_cast<size_t>(k)] - (gn / static_cast<double>(n)) * a[static_cast<size_t>(k)];
        u = cg_capped(Hop, rhs, cfg.krylov_tol, cfg.krylov_maxit, jdp, diag.krylov_iters, diag.pcg_breakdown);
    }
    diag.u_norm = norm(u);
    // :244
    Vec qu = frame.apply_Q(u);
    for (size_t i = 0; i < qu.size(); ++i) qu[i] -= frame.nu[i];
    return basis.apply(qu);
}

// ---- solver.hpp ----------------------------------------------------------------------
SolverConfig small_preset() {  // :64-71
    SolverConfig c;
    c.label = "small";
    c.max_iter = 300;
    c.tangent.mode = TangentSolveConfig::Mode::direct;
    c.tangent.lambda = 0.0;
    return c;
}
SolverConfig large_preset() {  // :73-85
    SolverConfig c;
    c.label = "large";
    c.max_iter = 40;
    c.max_elapsed_seconds = 60.0;
    c.tangent.mode = TangentSolveConfig::Mode::pcg;
    c.tangent.lambda = 1e-4;
    c.tangent.krylov_tol = 1e-3;
    c.tangent.krylov_maxit = 15;
    c.stall_restarts = true;
    c.identification_pass = true;
    return c;
}

// spg_identify, solver.hpp:116-185
Vec spg_identify(const Oracle& oracle, Vec x, double tau, int max_steps, int patience,
                 double eps_stop, int& steps_out, const IterateObserver& observer) {
    OracleCache cache = oracle.make_cache(std::move(x));
    double f = oracle.value(cache);
    Vec g = oracle.gradient(cache);
    Vec xcur = cache.x;
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
            const double sy = dot(bb_s, bb_y), ss = sqnorm(bb_s);
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
                OracleCache cp = oracle.make_cache(std::move(xp));
                const double fp = oracle.value(cp);
                if (fp <= f + 1e-4 * gdp) {
                    Vec gp = oracle.gradient(cp);
                    bb_s = std::move(dp);
                    bb_y.resize(gp.size());
                    for (size_t i = 0; i < gp.size(); ++i) bb_y[i] = gp[i] - g[i];
                    have_bb = true;
                    xcur = cp.x;
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
        if (observer) observer({-steps, f, xcur});
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

// solve, solver.hpp:195-655
SolveReport solve(const ReturnPanel& panel, const PreferenceCoefficients& coeffs,
                  const SolverConfig& config, Vec x0) {
    const index_t n0 = panel.assets();
    const index_t T = panel.periods();
    const double tau = config.tau;
    const double eps = config.epsilon;
    if (!(eps > 0)) throw domain_error("solve: epsilon must be positive");
    if (!(tau >= 0) || (n0 > 1 && !(tau < 1.0 / static_cast<double>(n0)))) throw domain_error("solve: tau out of range");

    const auto t_start = std::chrono::steady_clock::now();
    auto elapsed = [&] {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    };
    auto counter = std::make_shared<PassCounter>();
    Oracle oracle(panel.A, panel.mu, coeffs, counter);
    SolveReport rep;
    rep.config_label = config.label;

    if (x0.empty()) x0.assign(static_cast<size_t>(n0), 1.0 / static_cast<double>(n0));
    {
        double mn = std::numeric_limits<double>::infinity();
        for (double v : x0) mn = std::min(mn, v);
        if (sz(x0) != n0 || mn < tau - 1e-12 || std::abs(vsum(x0) - 1.0) > 1e-10)
            throw domain_error("solve: x0 is not in the tau-slice");
    }

    auto finish = [&](Vec x, SolveStatus status, double kkt) {
        OracleCache cache = oracle.make_cache(std::move(x));
        rep.f_star = oracle.value(cache);
        rep.interior_residual = projected_kkt_residual(oracle.gradient(cache));
        rep.kkt_residual = kkt;
        rep.x_star = cache.x;
        rep.status = status;
        rep.oracle_passes = counter->total();
        rep.wall_seconds = elapsed();
        return rep;
    };

    if (n0 == 1) {
        rep.status = SolveStatus::converged;
        return finish(Vec(1, 1.0), SolveStatus::converged, 0.0);
    }
    if (config.identification_pass) {
        x0 = spg_identify(oracle, std::move(x0), tau, 600, 30, std::max(1e3 * eps, 1e-4),
                          rep.identification_steps, config.observer);
    }
    struct Best { double f; Vec x; };
    OracleCache c0 = oracle.make_cache(std::move(x0));
    Best best{oracle.value(c0), c0.x};
    if (config.observer) config.observer({0, best.f, best.x});

    std::vector<std::pair<double, int>> attempts{{config.projected_trial_step, config.max_iter}};
    if (config.stall_restarts)
        for (double s : config.restart_trial_steps) attempts.emplace_back(s, config.restart_max_iter);

    // :265-286
    auto merge = [&](const Vec& xf, const std::vector<char>& free_mask, const std::vector<char>& pinned_mask) {
        Vec xn(static_cast<size_t>(n0), tau);
        index_t j = 0;
        for (index_t i = 0; i < n0; ++i)
            if (free_mask[static_cast<size_t>(i)]) xn[static_cast<size_t>(i)] = xf[static_cast<size_t>(j++)];
        index_t npin = 0;
        for (index_t i = 0; i < n0; ++i)
            if (pinned_mask[static_cast<size_t>(i)]) {
                xn[static_cast<size_t>(i)] = tau;
                ++npin;
            }
        double s = 0.0;
        for (index_t i = 0; i < n0; ++i)
            if (!pinned_mask[static_cast<size_t>(i)]) s += xn[static_cast<size_t>(i)];
        if (s > 0) {
            const double scale = (1.0 - static_cast<double>(npin) * tau) / s;
            for (index_t i = 0; i < n0; ++i)
                if (!pinned_mask[static_cast<size_t>(i)]) xn[static_cast<size_t>(i)] *= scale;
        }
        return xn;
    };
    auto full_residual = [&](const Vec& x, Vec& g_out) {
        OracleCache cache = oracle.make_cache(x);
        g_out = oracle.gradient(cache);
        return gradient_mapping_residual(x, g_out, tau);
    };
    auto full_value = [&](const Vec& x) { return oracle.value(oracle.make_cache(x)); };

    int it_total = 0;
    bool timed_out = false;

    for (size_t ai = 0; ai < attempts.size(); ++ai) {
        const double tr = attempts[ai].first;
        const int budget = attempts[ai].second;
        Vec x = best.x;
        std::vector<char> pinned(static_cast<size_t>(n0), 0);
        index_t npinned = 0;
        for (index_t i = 0; i < n0; ++i)
            if (x[static_cast<size_t>(i)] <= tau + 1e-12) {
                pinned[static_cast<size_t>(i)] = 1;
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
        std::vector<char> free_mask(static_cast<size_t>(n0), 1);
        index_t nf = n0;
        Mat Af;
        Vec muf, zoff;
        double mass = 1.0, mu_pin = 0.0;
        std::optional<Oracle> face;
        std::optional<TangentBasis> U;

        while (it < budget) {
            if (config.max_elapsed_seconds && elapsed() > *config.max_elapsed_seconds) {
                timed_out = true;
                break;
            }
            ++it;
            ++it_total;
            ++since_check;
            if (rebuild) {  // :343-370
                nf = n0 - npinned;
                free_mask.assign(static_cast<size_t>(n0), 0);
                Af = Mat(T, nf);
                muf.assign(static_cast<size_t>(nf), 0.0);
                zoff.assign(static_cast<size_t>(T), 0.0);
                mu_pin = 0.0;
                index_t j = 0;
                for (index_t i = 0; i < n0; ++i) {
                    if (!pinned[static_cast<size_t>(i)]) {
                        free_mask[static_cast<size_t>(i)] = 1;
                        for (index_t t = 0; t < T; ++t) Af(t, j) = panel.A(t, i);
                        muf[static_cast<size_t>(j)] = panel.mu[static_cast<size_t>(i)];
                        ++j;
                    } else {
                        for (index_t t = 0; t < T; ++t) zoff[static_cast<size_t>(t)] += tau * panel.A(t, i);
                        mu_pin += tau * panel.mu[static_cast<size_t>(i)];
                    }
                }
                mass = 1.0 - static_cast<double>(npinned) * tau;
                face.emplace(Af, muf, coeffs, counter, zoff, -coeffs.c1 * mu_pin);
                if (nf > 1) U.emplace(nf);
                else U.reset();
                t_cur = tr;
                rebuild = false;
            }
            Vec xf(static_cast<size_t>(nf));
            {
                index_t j = 0;
                for (index_t i = 0; i < n0; ++i)
                    if (free_mask[static_cast<size_t>(i)]) xf[static_cast<size_t>(j++)] = x[static_cast<size_t>(i)];
            }
            OracleCache fc = face->make_cache(xf);
            const Vec& gf = face->gradient(fc);
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
                    rep.restarts = static_cast<int>(ai);
                    return finish(x, SolveStatus::converged, r);
                }
                std::vector<char> rel(static_cast<size_t>(n0), 0);
                bool any_rel = false;
                const double rel_gate = std::max(1e-10, face_res);
                for (index_t i = 0; i < n0; ++i)
                    if (pinned[static_cast<size_t>(i)] && g_full[static_cast<size_t>(i)] - gf_mean < -rel_gate) {
                        rel[static_cast<size_t>(i)] = 1;
                        any_rel = true;
                    }
                if (any_rel) {
                    for (index_t i = 0; i < n0; ++i)
                        if (rel[static_cast<size_t>(i)]) {
                            pinned[static_cast<size_t>(i)] = 0;
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

            const double fcur = face->value(fc);
            DirectionDiagnostics dd;
            Vec d = yand_direction(*face, *U, fc, config.tangent, static_cast<std::uint64_t>(it_total), &dd);
            rep.krylov_iters_total += dd.krylov_iters;
            const double amax = alpha_max(xf, d, tau);
            bool moved = false;

            auto exact_step = [&](const Vec& dir, double cap) {  // :437-446
                LineModel lm = line_model(*face, fc, dir, cap);
                if (config.line_search == SolverConfig::LineSearch::armijo) {
                    auto res = armijo_search([&](double al) { return lm.eval(al); }, lm.a1, std::min(1.0, cap));
                    return std::pair<double, double>{res.alpha, lm.eval(res.alpha)};
                }
                return minimize_line(lm);
            };

            if (amax >= t_cur) {  // :448-453
                auto [al, fv] = exact_step(d, amax);
                (void)fv;
                if (al > 0) {
                    axpy_inplace(xf, al, d);
                    moved = true;
                }
            } else {  // :454-562
                std::vector<char> floor0(static_cast<size_t>(nf));
                for (index_t i = 0; i < nf; ++i) floor0[static_cast<size_t>(i)] = xf[static_cast<size_t>(i)] <= tau + 1e-12;
                std::vector<std::vector<char>> zsets;
                std::vector<index_t> zset_sizes;
                double t_len = t_cur;
                for (int rung = 0; rung < 6; ++rung) {
                    Vec trial(xf.size());
                    for (size_t i = 0; i < xf.size(); ++i) trial[i] = xf[i] + t_len * d[i];
                    Vec xb = project_slice(trial, tau, mass);
                    std::vector<char> zb(static_cast<size_t>(nf));
                    index_t zb_count = 0, newz = 0;
                    for (index_t i = 0; i < nf; ++i) {
                        zb[static_cast<size_t>(i)] = xb[static_cast<size_t>(i)] <= tau + 1e-15;
                        if (zb[static_cast<size_t>(i)]) ++zb_count;
                        if (xb[static_cast<size_t>(i)] <= tau + 1e-12 && !floor0[static_cast<size_t>(i)]) ++newz;
                    }
                    if (zb_count > 0 && (zsets.empty() || zb_count != zset_sizes.back())) {
                        zsets.push_back(zb);
                        zset_sizes.push_back(zb_count);
                    }
                    Vec db(xf.size());
                    for (size_t i = 0; i < xf.size(); ++i) db[i] = xb[i] - xf[i];
                    const double dbm = vmean(db);
                    for (double& v : db) v -= dbm;
                    const double dbn = norm(db);
                    if (dbn <= 1e-12 * std::max(1.0, norm(xf)) || dot(gf, db) >= -1e-10 * (1.0 + std::abs(fcur))) {
                        if (newz == 0) break;
                        t_len *= 0.5;
                        continue;
                    }
                    const double cap = std::min(1.0, alpha_max(xf, db, tau));
                    auto [al, fv] = exact_step(db, cap);
                    if (al > 0 && (rung == 0 || fcur - fv >= 1e-12 * (1.0 + std::abs(fcur)))) {
                        axpy_inplace(xf, al, db);
                        moved = true;
                        break;
                    }
                    if (newz == 0) break;
                    t_len *= 0.5;
                }
                if (!moved) {
                    bool done = false;
                    double pin_f = fcur;
                    for (const auto& zb : zsets) {
                        index_t cnt = 0;
                        for (char b : zb) cnt += b;
                        if (cnt >= nf) continue;
                        std::vector<char> pin_try = pinned;
                        index_t j = 0;
                        for (index_t i = 0; i < n0; ++i)
                            if (free_mask[static_cast<size_t>(i)]) {
                                if (zb[static_cast<size_t>(j)]) pin_try[static_cast<size_t>(i)] = 1;
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
                        index_t cnt = 0;
                        for (index_t i = 0; i < nf; ++i)
                            if (xf[static_cast<size_t>(i)] <= tau + 1e-12) ++cnt;
                        if (cnt > 0 && cnt < nf) {
                            index_t j = 0;
                            for (index_t i = 0; i < n0; ++i)
                                if (free_mask[static_cast<size_t>(i)]) {
                                    if (xf[static_cast<size_t>(j)] <= tau + 1e-12) {
                                        pinned[static_cast<size_t>(i)] = 1;
                                        ++npinned;
                                    }
                                    ++j;
                                }
                            x = merge(xf, free_mask, pinned);
                            if (config.observer) pin_f = full_value(x);
                            done = true;
                        }
                    }
                    if (done) {
                        ++rep.face_events;
                        rebuild = true;
                        eps_face = eps;
                        stall_small = stall_zero = 0;
                        face_ref = std::numeric_limits<double>::infinity();
                        if (config.observer) config.observer({it_total, pin_f, x});
                        continue;
                    } else if (amax > 0) {
                        auto [al, fv] = exact_step(d, amax);
                        (void)fv;
                        if (al > 0) {
                            axpy_inplace(xf, al, d);
                            moved = true;
                        }
                    }
                }
            }

            if (moved) {  // :564-581
                x = merge(xf, free_mask, pinned);
                const double fv_new = full_value(x);
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
                if (config.observer) config.observer({it_total, fv_new, x});
            } else {
                ++stall_zero;
            }

            if (stall_small >= 5 || stall_zero >= 2) {  // :583-631
                const double fcur2 = full_value(x);
                std::vector<std::pair<double, index_t>> order;
                for (index_t i = 0; i < n0; ++i)
                    if (!pinned[static_cast<size_t>(i)]) order.emplace_back(x[static_cast<size_t>(i)], i);
                std::sort(order.begin(), order.end());
                bool rescued = false;
                std::vector<char> cur_free(static_cast<size_t>(n0));
                for (index_t i = 0; i < n0; ++i) cur_free[static_cast<size_t>(i)] = !pinned[static_cast<size_t>(i)];
                Vec x_free(order.size());
                {
                    index_t j = 0;
                    for (index_t i = 0; i < n0; ++i)
                        if (cur_free[static_cast<size_t>(i)]) x_free[static_cast<size_t>(j++)] = x[static_cast<size_t>(i)];
                }
                double rescue_f = fcur2;
                for (const auto& [mass_i, idx] : order) {
                    if (mass_i > 1e-3 * (1.0 - static_cast<double>(npinned) * tau)) break;
                    if (npinned + 1 >= n0) break;
                    std::vector<char> pin_try = pinned;
                    pin_try[static_cast<size_t>(idx)] = 1;
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
                    if (config.observer) config.observer({it_total, rescue_f, x});
                    continue;
                }
                stalled = true;
                break;
            }
        }

        // :634-645
        Vec g_exit;
        const double r = full_residual(x, g_exit);
        const double fv = full_value(x);
        if (fv < best.f) best = {fv, x};
        rep.iterations = it_total;
        rep.restarts = static_cast<int>(ai);
        if (r <= eps) return finish(x, SolveStatus::converged, r);
        if (timed_out) break;
        if (!config.stall_restarts)
            return finish(x, stalled ? SolveStatus::stalled : SolveStatus::max_iter, r);
    }
    // :648-654
    Vec g_best;
    const double rb = full_residual(best.x, g_best);
    rep.iterations = it_total;
    const SolveStatus status = rb <= eps ? SolveStatus::converged
                               : timed_out ? SolveStatus::max_elapsed
                                           : SolveStatus::stalled;
    return finish(best.x, status, rb);
}

}  // namespace mo
