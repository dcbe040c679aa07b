// Reference-side adapter (the binding a maintainer adds to
// /root/reference/proj/include/mvsk/): mvsk::GpuOracle, the method set and
// error behaviour of mvsk::Oracle (oracle.hpp:29-149) over the C-ABI in
// include/mvsk_gpu.h, plus line_model (linesearch.hpp:62-81) and solve
// (solver.hpp:195-655) through the device driver.
//
// Differences a caller sees, all forced by the device residency of the cache:
//  * GpuCache is a move-only RAII handle on one of MVSK_GPU_MAX_SLOTS device
//    slots; make_cache() acquires a free slot and the destructor releases it,
//    so any number of caches below the slot count can be live at once (the
//    reference's solve keeps a face cache and full-panel residual caches alive
//    together, solver.hpp:378-388) and none alias. A ninth live cache throws
//    domain_error.
//  * gradient() memoises on the cache like the reference (mutable grad).
//  * hessian_diag_weights / sample_direction return this shard's rows.
// Compiled against the unmodified reference headers in tests (examples/
// adapter_check.cpp); see INTEGRATION.md.
#pragma once

#include <mvsk_gpu.h>

#include <array>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>

#include "linesearch.hpp"
#include "oracle.hpp"
#include "solver.hpp"

namespace mvsk {

inline void gpu_check(const mvsk_gpu_ctx* ctx, int32_t s) {
    if (s == MVSK_OK) return;
    const std::string m = mvsk_gpu_last_error(ctx);
    switch (s) {  // common.hpp:14-25
    case MVSK_DIMENSION_ERROR: throw dimension_error(m);
    case MVSK_DOMAIN_ERROR: throw domain_error(m);
    case MVSK_DATA_ERROR: throw data_error(m);
    case MVSK_NUMERIC_ERROR: throw numeric_error(m);
    default: throw std::runtime_error(m);
    }
}

namespace gpu_detail {
// the context and its slot table, shared by the oracle and every live cache
struct Shared {
    mvsk_gpu_ctx* ctx = nullptr;
    std::mutex mu;
    std::array<bool, MVSK_GPU_MAX_SLOTS> used{};
    ~Shared() {
        if (ctx) mvsk_gpu_destroy(ctx);
    }
    int32_t acquire() {
        std::lock_guard<std::mutex> l(mu);
        for (int32_t s = 0; s < MVSK_GPU_MAX_SLOTS; ++s)
            if (!used[static_cast<size_t>(s)]) {
                used[static_cast<size_t>(s)] = true;
                return s;
            }
        throw domain_error("gpu oracle: all device cache slots are in use");
    }
    void release(int32_t s) {
        std::lock_guard<std::mutex> l(mu);
        used[static_cast<size_t>(s)] = false;
    }
};
}  // namespace gpu_detail

/// OracleCache (oracle.hpp:14-20) as a device slot.
class GpuCache {
public:
    GpuCache(GpuCache&& o) noexcept
        : x(std::move(o.x)), f_value(o.f_value), has_grad(o.has_grad), grad(std::move(o.grad)),
          sh_(std::move(o.sh_)), slot_(o.slot_) {
        o.slot_ = -1;
    }
    GpuCache& operator=(GpuCache&& o) noexcept {
        if (this != &o) {
            drop();
            x = std::move(o.x);
            f_value = o.f_value;
            has_grad = o.has_grad;
            grad = std::move(o.grad);
            sh_ = std::move(o.sh_);
            slot_ = o.slot_;
            o.slot_ = -1;
        }
        return *this;
    }
    GpuCache(const GpuCache&) = delete;
    GpuCache& operator=(const GpuCache&) = delete;
    ~GpuCache() { drop(); }

    int32_t slot() const { return slot_; }
    Vec x;
    double f_value = 0;
    mutable bool has_grad = false;
    mutable Vec grad;

private:
    friend class GpuOracle;
    GpuCache(std::shared_ptr<gpu_detail::Shared> sh, int32_t slot) : sh_(std::move(sh)), slot_(slot) {}
    void drop() {
        if (sh_ && slot_ >= 0) sh_->release(slot_);
        slot_ = -1;
    }
    std::shared_ptr<gpu_detail::Shared> sh_;
    int32_t slot_ = -1;
};

/// Oracle (oracle.hpp:29-149) over a panel resident in B200 HBM.
class GpuOracle {
public:
    GpuOracle(const ReturnPanel& p, PreferenceCoefficients c, int device = 0)
        : n_(p.assets()), T_(p.periods()), mu_(p.mu), c_(c), sh_(std::make_shared<gpu_detail::Shared>()) {
        const mvsk_coeffs k{c.c1, c.c2, c.c3, c.c4};
        // A is row-major (panel.hpp:16): the C-ABI takes it as is
        gpu_check(nullptr, mvsk_gpu_create(p.A.data(), T_, n_, p.mu.data(), &k, device, &sh_->ctx));
    }

    index_t periods() const { return T_; }
    index_t assets() const { return n_; }
    const Vec& mu() const { return mu_; }
    const PreferenceCoefficients& coeffs() const { return c_; }

    GpuCache make_cache(Vec x) const {  // oracle.hpp:54-69
        if (x.size() != n_) throw dimension_error("oracle: iterate length does not match panel");
        GpuCache c(sh_, sh_->acquire());
        gpu_check(sh_->ctx, mvsk_gpu_make_cache(sh_->ctx, c.slot(), x.data(), &c.f_value));
        c.x = std::move(x);
        return c;
    }
    double value(const GpuCache& c) const { return c.f_value; }
    std::tuple<double, double, double, double> moments(const GpuCache& c) const {  // :73-77
        double m[4];
        gpu_check(sh_->ctx, mvsk_gpu_moments(sh_->ctx, c.slot(), m));
        return {m[0], m[1], m[2], m[3]};
    }
    const Vec& gradient(const GpuCache& c) const {  // :79-90, memoised
        if (!c.has_grad) {
            c.grad = Vec(n_);
            gpu_check(sh_->ctx, mvsk_gpu_gradient(sh_->ctx, c.slot(), c.grad.data()));
            c.has_grad = true;
        }
        return c.grad;
    }
    Vec hvp(const GpuCache& c, const Vec& v) const {  // :92-101
        if (v.size() != n_) throw dimension_error("oracle: direction length does not match panel");
        Vec o(n_);
        gpu_check(sh_->ctx, mvsk_gpu_hvp(sh_->ctx, c.slot(), v.data(), 1, o.data()));
        return o;
    }
    Vec third_action(const GpuCache& c, const Vec& u, const Vec& v) const {  // :103-113
        if (u.size() != n_ || v.size() != n_) throw dimension_error("oracle: direction length does not match panel");
        Vec o(n_);
        gpu_check(sh_->ctx, mvsk_gpu_third_action(sh_->ctx, c.slot(), u.data(), v.data(), 1, o.data()));
        return o;
    }
    Vec hessian_diag_weights(const GpuCache& c) const {  // :116-119
        Vec o(T_);
        gpu_check(sh_->ctx, mvsk_gpu_hessian_diag_weights(sh_->ctx, c.slot(), o.data()));
        return o;
    }
    Vec sample_direction(const Vec& d) const {  // :122
        Vec o(T_);
        gpu_check(sh_->ctx, mvsk_gpu_sample_direction(sh_->ctx, d.data(), o.data()));
        return o;
    }
    LineModel line_model(const GpuCache& c, const Vec& d, double cap) const {  // linesearch.hpp:62-81
        double o[14];
        gpu_check(sh_->ctx, mvsk_gpu_line_model(sh_->ctx, c.slot(), d.data(), cap, o));
        LineModel m;
        m.a0 = o[0];
        m.a1 = o[1];
        m.a2 = o[2];
        m.a3 = o[3];
        m.a4 = o[4];
        m.alpha_cap = cap;
        m.sums.s11 = o[5];
        m.sums.s21 = o[6];
        m.sums.s31 = o[7];
        m.sums.s02 = o[8];
        m.sums.s12 = o[9];
        m.sums.s22 = o[10];
        m.sums.s03 = o[11];
        m.sums.s13 = o[12];
        m.sums.s04 = o[13];
        return m;
    }

    /// solve(panel, coeffs, config, x0) (solver.hpp:195-655) by the device driver.
    SolveReport solve(const SolverConfig& cfg, const Vec& x0 = Vec()) const {
        mvsk_solver_config k{};
        k.epsilon = cfg.epsilon;
        k.tau = cfg.tau;
        k.max_iter = cfg.max_iter;
        k.has_max_elapsed = cfg.max_elapsed_seconds.has_value();
        k.max_elapsed_seconds = cfg.max_elapsed_seconds.value_or(0.0);
        k.projected_trial_step = cfg.projected_trial_step;
        if (cfg.restart_trial_steps.size() > 4) throw domain_error("gpu solve: at most 4 restart trial steps");
        k.n_restart_trial_steps = static_cast<int32_t>(cfg.restart_trial_steps.size());
        for (size_t i = 0; i < cfg.restart_trial_steps.size(); ++i) k.restart_trial_steps[i] = cfg.restart_trial_steps[i];
        k.restart_max_iter = cfg.restart_max_iter;
        k.tangent.mode = cfg.tangent.mode == TangentSolveConfig::Mode::pcg ? 1 : 0;
        k.tangent.lambda = cfg.tangent.lambda;
        k.tangent.krylov_tol = cfg.tangent.krylov_tol;
        k.tangent.krylov_maxit = cfg.tangent.krylov_maxit;
        k.tangent.jacobi = cfg.tangent.jacobi;
        k.tangent.exact_trace = cfg.tangent.exact_trace;
        k.tangent.hutchinson_probes = cfg.tangent.hutchinson_probes;
        k.tangent.probe_maxit = cfg.tangent.probe_maxit;
        k.line_search = cfg.line_search == SolverConfig::LineSearch::armijo ? 1 : 0;
        k.stall_restarts = cfg.stall_restarts;
        k.identification_pass = cfg.identification_pass;
        std::strncpy(k.label, cfg.label.c_str(), sizeof(k.label) - 1);
        SolveReport rep;
        rep.x_star = Vec(n_);
        mvsk_solve_report r{};
        mvsk_observer_fn obs = nullptr;
        if (cfg.observer)
            obs = [](void* user, int32_t it, double f, const double* x, int64_t n) {
                IterateRecord rec;
                rec.iteration = it;
                rec.f = f;
                rec.x = Vec(n);
                std::memcpy(rec.x.data(), x, sizeof(double) * static_cast<size_t>(n));
                (*static_cast<const IterateObserver*>(user))(rec);
            };
        gpu_check(sh_->ctx, mvsk_gpu_solve(sh_->ctx, &k, x0.size() ? x0.data() : nullptr, rep.x_star.data(), &r, obs,
                                           const_cast<IterateObserver*>(&cfg.observer)));
        rep.f_star = r.f_star;
        rep.kkt_residual = r.kkt_residual;
        rep.interior_residual = r.interior_residual;
        rep.iterations = r.iterations;
        rep.face_events = r.face_events;
        rep.restarts = r.restarts;
        rep.identification_steps = r.identification_steps;
        rep.krylov_iters_total = r.krylov_iters_total;
        rep.oracle_passes = r.oracle_passes;
        rep.wall_seconds = r.wall_seconds;
        rep.status = static_cast<SolveStatus>(r.status);
        rep.config_label = std::string(r.config_label, strnlen(r.config_label, sizeof(r.config_label)));
        return rep;
    }

private:
    index_t n_, T_;
    Vec mu_;
    PreferenceCoefficients c_;
    std::shared_ptr<gpu_detail::Shared> sh_;
};

}  // namespace mvsk
