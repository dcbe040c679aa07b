// TEST INFRASTRUCTURE ONLY — the reference itself, compiled.
//
// Exports the same `mo_*` ctypes surface as oracle/mvsk_oracle_capi.cpp (the
// restatement), but every entry point calls the UNMODIFIED reference headers
// (/root/reference/proj/include/mvsk/*.hpp: mvsk::Oracle, line_model,
// minimize_line, project_slice, TangentBasis, householder_frame,
// yand_direction, detail::cg_capped, detail::spg_identify via solve, solve)
// compiled over the Eigen API stand-in in oracle/ref/eigen_shim. Built by
// oracle/ref/Makefile into oracle/_ref/libmvsk_ref.so (reference-faithful
// flags) and oracle/_ref/libmvsk_ref_native.so (x86-64-v3 + SIMD reductions:
// the timed CPU arm of bench.py). Loaded only by tests/, scripts that generate
// tests/golden/ and bench.py's reference arm; never by the product package.
#include <mvsk/affine_normal.hpp>
#include <mvsk/linesearch.hpp>
#include <mvsk/oracle.hpp>
#include <mvsk/panel.hpp>
#include <mvsk/rng.hpp>
#include <mvsk/simplex.hpp>
#include <mvsk/solver.hpp>

#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mvsk_gpu.h"

using namespace mvsk;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const dimension_error& e) {
        g_err = e.what();
        return 1;
    } catch (const domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const data_error& e) {
        g_err = e.what();
        return 3;
    } catch (const numeric_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

Vec vec_of(const double* p, int64_t n) {
    Vec v(static_cast<Eigen::Index>(p ? n : 0));
    if (p && n > 0) std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
    return v;
}
Mat mat_of(const double* A, int64_t T, int64_t n) {
    Mat m(T, n);  // row-major, the panel's own layout (panel.hpp:16)
    if (T * n > 0) std::memcpy(m.data(), A, sizeof(double) * static_cast<size_t>(T * n));
    return m;
}
void put(const Vec& v, double* out) {
    if (v.size()) std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(v.size()));
}
PreferenceCoefficients coeffs_of(const double* c4) {
    PreferenceCoefficients c;
    c.c1 = c4[0];
    c.c2 = c4[1];
    c.c3 = c4[2];
    c.c4 = c4[3];
    return c;
}

struct OracleBox {
    Mat A;
    std::shared_ptr<PassCounter> counter = std::make_shared<PassCounter>();
    std::unique_ptr<Oracle> oracle;
    Vec mu, zoff;
    double value_offset = 0.0;
    PreferenceCoefficients c;
};

TangentSolveConfig tangent_of(const mvsk_tangent_config& c) {
    TangentSolveConfig t;
    t.mode = c.mode == 1 ? TangentSolveConfig::Mode::pcg : TangentSolveConfig::Mode::direct;
    t.lambda = c.lambda;
    t.krylov_tol = c.krylov_tol;
    t.krylov_maxit = c.krylov_maxit;
    t.jacobi = c.jacobi != 0;
    t.exact_trace = c.exact_trace != 0;
    t.hutchinson_probes = c.hutchinson_probes;
    t.probe_maxit = c.probe_maxit;
    return t;
}
}  // namespace

extern "C" {

const char* mo_impl() { return "reference"; }
const char* mo_last_error() { return g_err.c_str(); }
// the reference is single-threaded (CMakeLists.txt has no threading); accepted
// for interface compatibility with the restatement, ignored
void mo_set_threads(int) {}

// rng.hpp: kind 0 = u64, 1 = unit, 2 = normal, 3 = sign, 4 = uniform(lo, hi)
void mo_splitmix_draw(uint64_t seed, int kind, int64_t count, double lo, double hi, void* out) {
    SplitMix64 r(seed);
    for (int64_t i = 0; i < count; ++i) {
        switch (kind) {
        case 0: static_cast<uint64_t*>(out)[i] = r.next_u64(); break;
        case 1: static_cast<double*>(out)[i] = r.next_unit(); break;
        case 2: static_cast<double*>(out)[i] = r.next_normal(); break;
        case 3: static_cast<double*>(out)[i] = r.next_sign(); break;
        default: static_cast<double*>(out)[i] = r.next_uniform(lo, hi); break;
        }
    }
}

int mo_center_panel(const double* R, int64_t T, int64_t n, double* A_out, double* mu_out) {
    return guard([&] {
        ReturnPanel p = center_panel(mat_of(R, T, n));
        std::memcpy(A_out, p.A.data(), sizeof(double) * static_cast<size_t>(T * n));
        put(p.mu, mu_out);
    });
}
int mo_crra(double gamma, double* out4) {
    return guard([&] {
        auto c = crra_coefficients(gamma);
        out4[0] = c.c1;
        out4[1] = c.c2;
        out4[2] = c.c3;
        out4[3] = c.c4;
    });
}
int mo_make_coefficients(double c1, double c2, double c3, double c4, double* out4) {
    return guard([&] {
        auto c = make_coefficients(c1, c2, c3, c4);
        out4[0] = c.c1;
        out4[1] = c.c2;
        out4[2] = c.c3;
        out4[3] = c.c4;
    });
}

// ---- oracle.hpp ----
int mo_oracle_create(const double* A, int64_t T, int64_t n, const double* mu, const double* c4,
                     const double* zoff, double value_offset, void** out) {
    return guard([&] {
        auto box = std::make_unique<OracleBox>();
        box->A = mat_of(A, T, n);
        box->mu = vec_of(mu, n);
        box->zoff = zoff ? vec_of(zoff, T) : Vec();
        box->value_offset = value_offset;
        box->c = coeffs_of(c4);
        box->oracle = std::make_unique<Oracle>(box->A, box->mu, box->c, box->counter, box->zoff, value_offset);
        *out = box.release();
    });
}
int mo_oracle_create_mu(const double* A, int64_t T, int64_t n, const double* mu, int64_t nmu,
                        const double* c4, void** out) {
    return guard([&] {
        auto box = std::make_unique<OracleBox>();
        box->A = mat_of(A, T, n);
        box->c = coeffs_of(c4);
        box->oracle = std::make_unique<Oracle>(box->A, vec_of(mu, nmu), box->c, box->counter);
        *out = box.release();
    });
}
void mo_oracle_destroy(void* o) { delete static_cast<OracleBox*>(o); }
int mo_make_cache(void* o, const double* x, int64_t nx, void** out) {
    return guard([&] {
        auto* b = static_cast<OracleBox*>(o);
        *out = new OracleCache(b->oracle->make_cache(vec_of(x, nx)));
    });
}
void mo_cache_destroy(void* c) { delete static_cast<OracleCache*>(c); }
int mo_cache_z(void* c, double* out) {
    put(static_cast<OracleCache*>(c)->z, out);
    return 0;
}
int mo_value(void* o, void* c, double* f) {
    return guard([&] { *f = static_cast<OracleBox*>(o)->oracle->value(*static_cast<OracleCache*>(c)); });
}
int mo_moments(void* o, void* c, double* out4) {
    return guard([&] {
        auto [a, b, cc, d] = static_cast<OracleBox*>(o)->oracle->moments(*static_cast<OracleCache*>(c));
        out4[0] = a;
        out4[1] = b;
        out4[2] = cc;
        out4[3] = d;
    });
}
int mo_gradient(void* o, void* c, double* g) {
    return guard([&] { put(static_cast<OracleBox*>(o)->oracle->gradient(*static_cast<OracleCache*>(c)), g); });
}
int mo_hvp(void* o, void* c, const double* v, double* out) {
    return guard([&] {
        auto* b = static_cast<OracleBox*>(o);
        put(b->oracle->hvp(*static_cast<OracleCache*>(c), vec_of(v, b->oracle->assets())), out);
    });
}
int mo_third_action(void* o, void* c, const double* u, const double* v, double* out) {
    return guard([&] {
        auto* b = static_cast<OracleBox*>(o);
        const int64_t n = b->oracle->assets();
        put(b->oracle->third_action(*static_cast<OracleCache*>(c), vec_of(u, n), vec_of(v, n)), out);
    });
}
int mo_hessian_diag_weights(void* o, void* c, double* out) {
    return guard([&] {
        put(static_cast<OracleBox*>(o)->oracle->hessian_diag_weights(*static_cast<OracleCache*>(c)), out);
    });
}
int mo_sample_direction(void* o, const double* d, double* out) {
    return guard([&] {
        auto* b = static_cast<OracleBox*>(o);
        put(b->oracle->sample_direction(vec_of(d, b->oracle->assets())), out);
    });
}
// out: a0..a4, s11,s21,s31,s02,s12,s22,s03,s13,s04 (linesearch.hpp:62-81)
int mo_line_model(void* o, void* c, const double* d, int64_t nd, double cap, double* out14) {
    return guard([&] {
        auto* b = static_cast<OracleBox*>(o);
        LineModel m = line_model(*b->oracle, *static_cast<OracleCache*>(c), vec_of(d, nd), cap);
        const double v[14] = {m.a0, m.a1, m.a2, m.a3, m.a4, m.sums.s11, m.sums.s21,
                              m.sums.s31, m.sums.s02, m.sums.s12, m.sums.s22, m.sums.s03,
                              m.sums.s13, m.sums.s04};
        std::memcpy(out14, v, sizeof(v));
    });
}
void mo_passes(void* o, uint64_t* fwd, uint64_t* tr) {
    auto* b = static_cast<OracleBox*>(o);
    *fwd = b->counter->forward;
    *tr = b->counter->transpose;
}
void mo_reset_passes(void* o) { static_cast<OracleBox*>(o)->counter->reset(); }

// affine_normal.hpp:127-245
int mo_yand_direction(void* o, void* c, const mvsk_tangent_config* cfg, uint64_t it_seed,
                      double* d_out, mvsk_direction_diag* diag) {
    return guard([&] {
        auto* b = static_cast<OracleBox*>(o);
        TangentBasis basis(b->oracle->assets());
        DirectionDiagnostics dd;
        Vec d = yand_direction(*b->oracle, basis, *static_cast<OracleCache*>(c), tangent_of(*cfg), it_seed, &dd);
        put(d, d_out);
        if (diag) {
            diag->reduced_grad_norm = dd.reduced_grad_norm;
            diag->u_norm = dd.u_norm;
            diag->krylov_iters = dd.krylov_iters;
            diag->pcg_breakdown = dd.pcg_breakdown;
            diag->lambda_fallback = dd.lambda_fallback;
        }
    });
}

// ---- linesearch.hpp ----
int mo_power_sums(const double* z, const double* w, int64_t T, int64_t Tw, double* out9) {
    return guard([&] {
        PowerSums s = power_sums(vec_of(z, T), vec_of(w, Tw));
        const double v[9] = {s.s11, s.s21, s.s31, s.s02, s.s12, s.s22, s.s03, s.s13, s.s04};
        std::memcpy(out9, v, sizeof(v));
    });
}
int mo_cubic_real_roots(double c3, double c2, double c1, double c0, double* out3) {
    auto r = detail::cubic_real_roots(c3, c2, c1, c0);
    for (size_t i = 0; i < r.size(); ++i) out3[i] = r[i];
    return static_cast<int>(r.size());
}
int mo_minimize_line(const double* a5, double cap, double* alpha, double* f) {
    return guard([&] {
        LineModel m;
        m.a0 = a5[0];
        m.a1 = a5[1];
        m.a2 = a5[2];
        m.a3 = a5[3];
        m.a4 = a5[4];
        m.alpha_cap = cap;
        auto [al, fv] = minimize_line(m);
        *alpha = al;
        *f = fv;
    });
}
typedef double (*mo_phi_fn)(double, void*);
int mo_armijo(mo_phi_fn phi, void* user, double g_dot_d, double alpha_init, double sigma, double shrink,
              double* alpha, int* stalled) {
    return guard([&] {
        ArmijoResult r = armijo_search([&](double a) { return phi(a, user); }, g_dot_d, alpha_init, sigma, shrink);
        *alpha = r.alpha;
        *stalled = r.stalled;
    });
}

// ---- simplex.hpp ----
double mo_alpha_max(const double* x, const double* d, int64_t n, double tau) {
    return alpha_max(vec_of(x, n), vec_of(d, n), tau);
}
int mo_project_slice(const double* v, int64_t n, double tau, double mass, double* out) {
    return guard([&] { put(project_slice(vec_of(v, n), tau, mass), out); });
}
double mo_projected_kkt_residual(const double* g, int64_t n) { return projected_kkt_residual(vec_of(g, n)); }
double mo_gradient_mapping_residual(const double* x, const double* g, int64_t n, double tau) {
    return gradient_mapping_residual(vec_of(x, n), vec_of(g, n), tau);
}
int mo_basis_apply(int64_t n, const double* y, int64_t ny, double* out) {
    return guard([&] { put(TangentBasis(n).apply(vec_of(y, ny)), out); });
}
int mo_basis_apply_transpose(int64_t n, const double* x, int64_t nx, double* out) {
    return guard([&] { put(TangentBasis(n).apply_transpose(vec_of(x, nx)), out); });
}
int mo_householder_frame(const double* g, int64_t m, double* nu, double* v, double* beta, double* gn) {
    return guard([&] {
        ReducedFrame f = householder_frame(vec_of(g, m));
        put(f.nu, nu);
        put(f.v, v);
        *beta = f.beta;
        *gn = f.grad_norm;
    });
}
int mo_frame_apply_Q(const double* g, int64_t m, const double* eta, double* out) {
    return guard([&] { put(householder_frame(vec_of(g, m)).apply_Q(vec_of(eta, m - 1)), out); });
}
int mo_frame_apply_Qt(const double* g, int64_t m, const double* w, double* out) {
    return guard([&] { put(householder_frame(vec_of(g, m)).apply_Qt(vec_of(w, m)), out); });
}
// affine_normal.hpp:85-113 over a dense row-major operator
int mo_cg_dense(const double* M, int64_t m, const double* rhs, double tol, int cap, const double* jacobi_diag,
                double* x_out, int* iters, int* breakdown) {
    return guard([&] {
        const Mat Mm = mat_of(M, m, m);
        auto op = [&](const Vec& v) -> Vec { return Mm * v; };
        Vec jd = jacobi_diag ? vec_of(jacobi_diag, m) : Vec();
        int it = 0;
        bool bd = false;
        put(detail::cg_capped(op, vec_of(rhs, m), tol, cap, jacobi_diag ? &jd : nullptr, it, bd), x_out);
        *iters = it;
        *breakdown = bd;
    });
}
int mo_restrict_to_face(const double* A, int64_t T, int64_t n, const double* mu, const double* x, double tau,
                        int64_t* free_idx, int64_t* nf, double* zoff, double* mu_pin, double* free_mass) {
    return guard([&] {
        const Mat m = mat_of(A, T, n);
        FaceProblem fp = restrict_to_face(m, vec_of(mu, n), vec_of(x, n), tau);
        *nf = static_cast<int64_t>(fp.state.free_indices.size());
        for (size_t i = 0; i < fp.state.free_indices.size(); ++i) free_idx[i] = fp.state.free_indices[i];
        put(fp.zoff, zoff);
        *mu_pin = fp.mu_pinned_term;
        *free_mass = fp.free_mass;
    });
}

// ---- solver.hpp ----
int mo_preset(const char* name, mvsk_solver_config* out) {
    return guard([&] {
        SolverConfig c = preset(std::string(name));
        std::memset(out, 0, sizeof(*out));
        out->epsilon = c.epsilon;
        out->tau = c.tau;
        out->max_iter = c.max_iter;
        out->has_max_elapsed = c.max_elapsed_seconds.has_value();
        out->max_elapsed_seconds = c.max_elapsed_seconds.value_or(0.0);
        out->projected_trial_step = c.projected_trial_step;
        out->n_restart_trial_steps = static_cast<int32_t>(c.restart_trial_steps.size());
        for (size_t i = 0; i < c.restart_trial_steps.size() && i < 4; ++i)
            out->restart_trial_steps[i] = c.restart_trial_steps[i];
        out->restart_max_iter = c.restart_max_iter;
        out->tangent.mode = c.tangent.mode == TangentSolveConfig::Mode::pcg;
        out->tangent.lambda = c.tangent.lambda;
        out->tangent.krylov_tol = c.tangent.krylov_tol;
        out->tangent.krylov_maxit = c.tangent.krylov_maxit;
        out->tangent.jacobi = c.tangent.jacobi;
        out->tangent.exact_trace = c.tangent.exact_trace;
        out->tangent.hutchinson_probes = c.tangent.hutchinson_probes;
        out->tangent.probe_maxit = c.tangent.probe_maxit;
        out->line_search = 0;
        out->stall_restarts = c.stall_restarts;
        out->identification_pass = c.identification_pass;
        std::strncpy(out->label, c.label.c_str(), sizeof(out->label) - 1);
    });
}

int mo_solve(const double* A, int64_t T, int64_t n, const double* mu, const double* c4, const mvsk_solver_config* cfg,
             const double* x0, double* x_star, mvsk_solve_report* rep, mvsk_observer_fn observer, void* user) {
    return guard([&] {
        ReturnPanel p;
        p.A = mat_of(A, T, n);
        p.R = Mat(T, n);  // solve() reads only A and mu (solver.hpp:195-655); periods() reads R.rows()
        p.mu = vec_of(mu, n);
        SolverConfig sc;
        sc.epsilon = cfg->epsilon;
        sc.tau = cfg->tau;
        sc.max_iter = cfg->max_iter;
        if (cfg->has_max_elapsed) sc.max_elapsed_seconds = cfg->max_elapsed_seconds;
        sc.projected_trial_step = cfg->projected_trial_step;
        sc.restart_trial_steps.assign(cfg->restart_trial_steps, cfg->restart_trial_steps + cfg->n_restart_trial_steps);
        sc.restart_max_iter = cfg->restart_max_iter;
        sc.tangent = tangent_of(cfg->tangent);
        sc.line_search =
            cfg->line_search == 1 ? SolverConfig::LineSearch::armijo : SolverConfig::LineSearch::exact_quartic;
        sc.stall_restarts = cfg->stall_restarts != 0;
        sc.identification_pass = cfg->identification_pass != 0;
        sc.label = std::string(cfg->label, strnlen(cfg->label, sizeof(cfg->label)));
        if (observer)
            sc.observer = [&](const IterateRecord& r) {
                observer(user, r.iteration, r.f, r.x.data(), static_cast<int64_t>(r.x.size()));
            };
        SolveReport r = solve(p, coeffs_of(c4), sc, x0 ? vec_of(x0, n) : Vec());
        put(r.x_star, x_star);
        std::memset(rep, 0, sizeof(*rep));
        rep->f_star = r.f_star;
        rep->kkt_residual = r.kkt_residual;
        rep->interior_residual = r.interior_residual;
        rep->wall_seconds = r.wall_seconds;
        rep->krylov_iters_total = r.krylov_iters_total;
        rep->oracle_passes = r.oracle_passes;
        rep->physical_passes = r.oracle_passes;
        rep->iterations = r.iterations;
        rep->face_events = r.face_events;
        rep->restarts = r.restarts;
        rep->identification_steps = r.identification_steps;
        rep->status = static_cast<int32_t>(r.status);
        std::strncpy(rep->config_label, r.config_label.c_str(), sizeof(rep->config_label) - 1);
    });
}

// ---- timing harness for bench.py's reference arm (not a reference API) ----
// `nthreads` host threads each run `reps` reference HVPs (oracle.hpp:92-101)
// over the SAME immutable panel and cache (SPEC: concurrent caches over one
// panel are allowed; each thread gets its own Oracle so the pass counters do
// not race). Direction i of thread j is V[(j + i) % k]. Returns the wall time
// of the whole batch in seconds and (optionally) the first result per thread.
int mo_hvp_throughput(void* o, void* c, const double* V, int k, int nthreads, int reps, double* seconds,
                      double* first_out) {
    return guard([&] {
        auto* b = static_cast<OracleBox*>(o);
        const auto* cache = static_cast<OracleCache*>(c);
        const int64_t n = b->oracle->assets();
        std::vector<Vec> dirs;
        for (int i = 0; i < k; ++i) dirs.push_back(vec_of(V + static_cast<size_t>(i) * n, n));
        std::vector<std::unique_ptr<Oracle>> oracles;
        for (int j = 0; j < nthreads; ++j)
            oracles.push_back(std::make_unique<Oracle>(b->A, b->mu, b->c, nullptr, b->zoff, b->value_offset));
        std::vector<std::string> errs(static_cast<size_t>(nthreads));
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int j = 0; j < nthreads; ++j)
            th.emplace_back([&, j] {
                try {
                    for (int i = 0; i < reps; ++i) {
                        Vec h = oracles[static_cast<size_t>(j)]->hvp(*cache, dirs[static_cast<size_t>((j + i) % k)]);
                        if (i == 0 && first_out) put(h, first_out + static_cast<size_t>(j) * n);
                    }
                } catch (const std::exception& e) {
                    errs[static_cast<size_t>(j)] = e.what();
                }
            });
        for (auto& t : th) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (const auto& e : errs)
            if (!e.empty()) throw numeric_error(e);
    });
}

}  // extern "C"
