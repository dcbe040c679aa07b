// TEST INFRASTRUCTURE ONLY — the CPU parity oracle.
//
// A plain C++17 restatement (no Eigen) of the reference YAND-MVSK CPU code
// under /root/reference/proj/include/mvsk/. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it, and only as
// the checker or the timed CPU baseline. The product (paper_2604_25378_b200/)
// never links, imports or calls anything here.
//
// Parity status: the reference cannot be compiled in this image (it needs
// Eigen >= 3.3, CMakeLists.txt:12, absent), and it stores no golden output
// vectors. This restatement is therefore pinned against every known-answer
// constant and relational test the reference suite holds for this path
// (tests/test_rng.cpp, test_linesearch.cpp, test_oracle.cpp, test_simplex.cpp,
// test_panel.cpp, test_affine_normal.cpp, test_solver.cpp), re-expressed in
// tests/test_oracle_pins.py. Eigen's summation order is not reproduced; the
// reference's own tolerances (1e-13 against plain loops) cover that.
//
// Every function cites the reference file:line it restates.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

namespace mo {

using index_t = std::int64_t;

// ---- common.hpp:14-37 ------------------------------------------------------
struct dimension_error : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct domain_error : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct data_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct numeric_error : std::runtime_error { using std::runtime_error::runtime_error; };

struct PassCounter {
    std::uint64_t forward = 0;
    std::uint64_t transpose = 0;
    std::uint64_t total() const { return forward + transpose; }
    void reset() { forward = transpose = 0; }
};

// ---- minimal dense vector / row-major matrix (stand-ins for Eigen) --------
using Vec = std::vector<double>;

struct Mat {  // row-major, panel.hpp:16
    index_t rows = 0, cols = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(index_t r, index_t c, double v = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r * c), v) {}
    double& operator()(index_t r, index_t c) { return a[static_cast<size_t>(r * cols + c)]; }
    double operator()(index_t r, index_t c) const { return a[static_cast<size_t>(r * cols + c)]; }
    const double* row(index_t r) const { return a.data() + r * cols; }
    double* row(index_t r) { return a.data() + r * cols; }
};

inline index_t sz(const Vec& v) { return static_cast<index_t>(v.size()); }
inline double dot(const Vec& a, const Vec& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
inline double sqnorm(const Vec& a) { return dot(a, a); }
inline double norm(const Vec& a) { return std::sqrt(sqnorm(a)); }
inline double vsum(const Vec& a) {
    double s = 0.0;
    for (double x : a) s += x;
    return s;
}
inline double vmean(const Vec& a) { return vsum(a) / static_cast<double>(a.size()); }
inline bool all_finite(const Vec& a) {
    for (double x : a)
        if (!std::isfinite(x)) return false;
    return true;
}
inline Vec axpby(double alpha, const Vec& x, double beta, const Vec& y) {  // alpha x + beta y
    Vec r(x.size());
    for (size_t i = 0; i < x.size(); ++i) r[i] = alpha * x[i] + beta * y[i];
    return r;
}
inline Vec scaled(const Vec& x, double s) {
    Vec r(x);
    for (double& v : r) v *= s;
    return r;
}
inline void axpy_inplace(Vec& y, double alpha, const Vec& x) {
    for (size_t i = 0; i < y.size(); ++i) y[i] += alpha * x[i];
}

// Host thread count for the passes (1 = reference-faithful, the reference has
// no threading: CMakeLists.txt:1-47). >1 is only used for the timed CPU arm.
int& pass_threads();

// z = A x (row-major GEMV), out-of-place
void gemv(const Mat& A, const Vec& x, Vec& z);
// g = A^T w
void gemv_t(const Mat& A, const Vec& w, Vec& g);

// ---- rng.hpp:12-43 ---------------------------------------------------------
class SplitMix64 {
public:
    explicit SplitMix64(std::uint64_t seed) : state_(seed) {}
    std::uint64_t next_u64() {
        std::uint64_t z = (state_ += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_uniform(double lo, double hi) { return lo + (hi - lo) * next_unit(); }
    double next_normal() {
        double u1 = next_unit(), u2 = next_unit();
        while (u1 <= 0.0) u1 = next_unit();
        constexpr double two_pi = 6.283185307179586476925286766559;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
    }
    double next_sign() { return (next_u64() >> 63) ? 1.0 : -1.0; }
    std::uint64_t state() const { return state_; }

private:
    std::uint64_t state_;
};

// ---- panel.hpp:22-87 -------------------------------------------------------
struct ReturnPanel {
    Mat R;
    Vec mu;
    Mat A;
    index_t periods() const { return A.rows; }
    index_t assets() const { return A.cols; }
};
ReturnPanel center_panel(Mat R);  // panel.hpp:32-44

struct PreferenceCoefficients { double c1 = 0, c2 = 0, c3 = 0, c4 = 0; };
PreferenceCoefficients make_coefficients(double c1, double c2, double c3, double c4);  // :64-72
PreferenceCoefficients crra_coefficients(double gamma);                                // :76-87

// ---- oracle.hpp:14-149 -----------------------------------------------------
struct OracleCache {
    Vec x;
    Vec z, z2, z3;
    double f_value = 0;
    mutable bool has_grad = false;
    mutable Vec grad;
};

class Oracle {
public:
    Oracle(const Mat& A, Vec mu, PreferenceCoefficients coeffs,
           std::shared_ptr<PassCounter> counter = nullptr, Vec zoff = Vec(),
           double value_offset = 0.0);
    index_t periods() const { return A_->rows; }
    index_t assets() const { return A_->cols; }
    const Mat& A() const { return *A_; }
    const Vec& mu() const { return mu_; }
    const PreferenceCoefficients& coeffs() const { return c_; }
    const std::shared_ptr<PassCounter>& counter() const { return passes_; }

    OracleCache make_cache(Vec x) const;
    double value(const OracleCache& c) const { return c.f_value; }
    std::tuple<double, double, double, double> moments(const OracleCache& c) const;
    const Vec& gradient(const OracleCache& c) const;
    Vec hvp(const OracleCache& c, const Vec& v) const;
    Vec third_action(const OracleCache& c, const Vec& u, const Vec& v) const;
    Vec hessian_diag_weights(const OracleCache& c) const;
    Vec sample_direction(const Vec& d) const { return forward_tangent(d); }

private:
    Vec forward(const Vec& x) const;
    Vec forward_tangent(const Vec& v) const;
    Vec transpose_apply(const Vec& w) const;

    const Mat* A_;
    Vec mu_;
    Vec zoff_;
    PreferenceCoefficients c_;
    double f_offset_ = 0.0;
    std::shared_ptr<PassCounter> passes_;
};

// ---- linesearch.hpp:16-193 -------------------------------------------------
struct PowerSums {
    double s11 = 0, s21 = 0, s31 = 0;
    double s02 = 0, s12 = 0, s22 = 0;
    double s03 = 0, s13 = 0, s04 = 0;
};
PowerSums power_sums(const Vec& z, const Vec& w);

struct LineModel {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
    double alpha_cap = 0;
    PowerSums sums;
    double eval(double alpha) const {
        return a0 + alpha * (a1 + alpha * (a2 + alpha * (a3 + alpha * a4)));
    }
    double deriv(double alpha) const {
        return a1 + alpha * (2.0 * a2 + alpha * (3.0 * a3 + alpha * 4.0 * a4));
    }
};
LineModel line_model(const Oracle& oracle, const OracleCache& cache, const Vec& d, double cap);
std::vector<double> cubic_real_roots(double c3, double c2, double c1, double c0);
double polish_root(const LineModel& m, double alpha);
std::pair<double, double> minimize_line(const LineModel& m);
struct ArmijoResult { double alpha = 0; bool stalled = false; };
ArmijoResult armijo_search(const std::function<double(double)>& phi, double g_dot_d,
                           double alpha_init, double sigma = 1e-4, double shrink = 0.5);

// ---- simplex.hpp:17-192 ----------------------------------------------------
class TangentBasis {
public:
    explicit TangentBasis(index_t n);
    index_t ambient_dim() const { return n_; }
    Vec apply(const Vec& y) const;            // :63-70
    Vec apply_transpose(const Vec& x) const;  // :73-78
    const Vec& reflector() const { return v_; }
    double beta() const { return beta_; }

private:
    index_t n_;
    Vec v_;
    double beta_;
};
double alpha_max(const Vec& x, const Vec& d, double tau);             // :93-99
Vec project_slice(const Vec& v, double tau, double mass = 1.0);        // :104-122
double projected_kkt_residual(const Vec& g);                           // :126-129
double gradient_mapping_residual(const Vec& x, const Vec& g, double tau);  // :135-137

struct FaceProblem {  // :152-159
    std::vector<index_t> free_indices;
    Mat A;
    Vec mu;
    Vec zoff;
    double mu_pinned_term = 0.0;
    double free_mass = 1.0;
};
FaceProblem restrict_to_face(const Mat& A, const Vec& mu, const Vec& x, double tau);  // :161-192

// ---- affine_normal.hpp:19-245 ----------------------------------------------
struct ReducedFrame {
    Vec nu;
    double grad_norm = 0;
    Vec v;
    double beta = 0;
    Vec apply_Q(const Vec& eta) const;  // :28-33
    Vec apply_Qt(const Vec& w) const;   // :36-39
};
ReducedFrame householder_frame(const Vec& reduced_grad);  // :42-56

struct TangentSolveConfig {  // :59-69
    enum class Mode { direct, pcg };
    Mode mode = Mode::direct;
    double lambda = 0.0;
    double krylov_tol = 1e-3;
    int krylov_maxit = 15;
    bool jacobi = false;
    bool exact_trace = false;
    int hutchinson_probes = 8;
    int probe_maxit = 5;
};
struct DirectionDiagnostics {
    double reduced_grad_norm = 0;
    double u_norm = 0;
    int krylov_iters = 0;
    bool pcg_breakdown = false;
    bool lambda_fallback = false;
};
Vec cg_capped(const std::function<Vec(const Vec&)>& H, const Vec& rhs, double tol, int cap,
              const Vec* jacobi_diag, int& iters, bool& breakdown);  // :85-113
Vec yand_direction(const Oracle& oracle, const TangentBasis& basis, const OracleCache& cache,
                   const TangentSolveConfig& cfg, std::uint64_t it_seed = 0,
                   DirectionDiagnostics* diag_out = nullptr);  // :127-245

// Dense partial-pivot LU (stand-in for Eigen::PartialPivLU at :171)
struct PartialPivLU {
    index_t n = 0;
    std::vector<double> lu;  // row-major, L unit-lower, U upper
    std::vector<index_t> perm;
    explicit PartialPivLU(const Mat& M);
    Vec solve(const Vec& b) const;
};

// ---- solver.hpp:21-655 -----------------------------------------------------
enum class SolveStatus { converged = 0, stalled = 1, max_iter = 2, max_elapsed = 3, degenerate_face = 4 };

struct IterateRecord {
    int iteration = 0;
    double f = 0;
    Vec x;
};
using IterateObserver = std::function<void(const IterateRecord&)>;

struct SolverConfig {  // :44-62
    double epsilon = 1e-6;
    double tau = 1e-8;
    int max_iter = 300;
    std::optional<double> max_elapsed_seconds;
    double projected_trial_step = 0.05;
    std::vector<double> restart_trial_steps = {0.045, 0.02};
    int restart_max_iter = 120;
    TangentSolveConfig tangent;
    enum class LineSearch { exact_quartic, armijo };
    LineSearch line_search = LineSearch::exact_quartic;
    bool stall_restarts = false;
    bool identification_pass = false;
    std::string label = "custom";
    IterateObserver observer;
};
SolverConfig small_preset();  // :64-71
SolverConfig large_preset();  // :73-85

struct SolveReport {  // :93-107
    Vec x_star;
    double f_star = 0;
    double kkt_residual = 0;
    double interior_residual = 0;
    int iterations = 0;
    int face_events = 0;
    int restarts = 0;
    int identification_steps = 0;
    long long krylov_iters_total = 0;
    std::uint64_t oracle_passes = 0;
    double wall_seconds = 0;
    SolveStatus status = SolveStatus::max_iter;
    std::string config_label;
};

Vec spg_identify(const Oracle& oracle, Vec x, double tau, int max_steps, int patience,
                 double eps_stop, int& steps_out, const IterateObserver& observer);  // :116-185
SolveReport solve(const ReturnPanel& panel, const PreferenceCoefficients& coeffs,
                  const SolverConfig& config, Vec x0 = Vec());  // :195-655

}  // namespace mo
