// adapter_check — the INTEGRATION.md adapter (integration/mvsk/gpu_oracle.hpp)
// compiled against the UNMODIFIED reference headers (over the oracle/ref Eigen
// stand-in, as in oracle/_ref) and checked side by side with the reference's
// own mvsk::Oracle and mvsk::solve on a seeded panel:
//   * f, moments, gradient, hvp, third_action, line_model to 1e-11 relative;
//   * several live caches at once (the reference solve's face + residual
//     caches, solver.hpp:378-388): each keeps its own point (no slot aliasing),
//     slots are recycled by RAII, a ninth live cache is a domain_error;
//   * GpuOracle::solve vs mvsk::solve (small and large presets, epsilon 1e-10):
//     same status and active set, weights within 1e-8.
// Prints one JSON line; exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "gpu_oracle.hpp"
#include "rng.hpp"

using namespace mvsk;

static int failures = 0;
static void check(bool ok, const char* what, double v = 0) {
    if (!ok) {
        ++failures;
        std::fprintf(stderr, "FAILED %s (%.3e)\n", what, v);
    }
}
static double rel(const Vec& a, const Vec& b) {
    double e = 0, s = 0;
    for (index_t i = 0; i < a.size(); ++i) {
        e = std::max(e, std::abs(a[i] - b[i]));
        s = std::max(s, std::abs(b[i]));
    }
    return e / std::max(s, 1e-300);
}

int main() {
    const index_t n = 12, T = 300;
    SplitMix64 rng(2604);
    Mat R(T, n);
    for (index_t t = 0; t < T; ++t)
        for (index_t i = 0; i < n; ++i) R(t, i) = rng.next_uniform(-0.05, 0.08) + 0.002 * static_cast<double>(i % 4);
    const ReturnPanel panel = center_panel(std::move(R));
    const PreferenceCoefficients c = crra_coefficients(8.0);

    Oracle ref(panel, c);
    GpuOracle gpu(panel, c);
    auto point = [&](std::uint64_t seed) {
        SplitMix64 r(seed);
        Vec x(n);
        double s = 0;
        for (index_t i = 0; i < n; ++i) s += (x[i] = 0.1 + r.next_unit());
        for (index_t i = 0; i < n; ++i) x[i] /= s;
        return x;
    };
    auto tangent = [&](std::uint64_t seed) {
        SplitMix64 r(seed);
        Vec d(n);
        for (index_t i = 0; i < n; ++i) d[i] = r.next_uniform(-1.0, 1.0);
        d.array() -= d.mean();
        return d;
    };

    // several live caches, checked after all exist (no aliasing)
    std::vector<Vec> xs;
    std::vector<OracleCache> rc;
    std::vector<GpuCache> gc;
    for (int k = 0; k < 3; ++k) {
        xs.push_back(point(10 + k));
        rc.push_back(ref.make_cache(xs.back()));
        gc.push_back(gpu.make_cache(xs.back()));
    }
    double worst = 0;
    for (int k = 0; k < 3; ++k) {
        const Vec u = tangent(20 + k), v = tangent(30 + k);
        worst = std::max(worst, std::abs(gpu.value(gc[k]) - ref.value(rc[k])) / std::abs(ref.value(rc[k])));
        auto [a0, a1, a2, a3] = ref.moments(rc[k]);
        auto [b0, b1, b2, b3] = gpu.moments(gc[k]);
        worst = std::max({worst, std::abs(a0 - b0) / std::abs(a0), std::abs(a1 - b1) / std::abs(a1),
                          std::abs(a2 - b2) / std::abs(a2), std::abs(a3 - b3) / std::abs(a3)});
        worst = std::max(worst, rel(gpu.gradient(gc[k]), ref.gradient(rc[k])));
        worst = std::max(worst, rel(gpu.hvp(gc[k], v), ref.hvp(rc[k], v)));
        worst = std::max(worst, rel(gpu.third_action(gc[k], u, v), ref.third_action(rc[k], u, v)));
        const LineModel lr = line_model(ref, rc[k], v, 0.3), lg = gpu.line_model(gc[k], v, 0.3);
        Vec a(5), b(5);
        a << lr.a0, lr.a1, lr.a2, lr.a3, lr.a4;
        b << lg.a0, lg.a1, lg.a2, lg.a3, lg.a4;
        worst = std::max(worst, rel(b, a));
        check(minimize_line(lg).first == minimize_line(lr).first || std::abs(minimize_line(lg).first -
                                                                             minimize_line(lr).first) <= 1e-9,
              "minimize_line alpha");
    }
    check(worst <= 1e-11, "oracle values vs reference", worst);

    // RAII slots: 3 live + 5 more fill the table, a ninth throws, releasing one frees it
    {
        std::vector<GpuCache> more;
        for (int k = 0; k < MVSK_GPU_MAX_SLOTS - 3; ++k) more.push_back(gpu.make_cache(point(40 + k)));
        bool threw = false;
        try {
            (void)gpu.make_cache(point(99));
        } catch (const domain_error&) {
            threw = true;
        }
        check(threw, "ninth live cache throws domain_error");
        more.pop_back();
        GpuCache again = gpu.make_cache(point(98));
        check(again.slot() >= 0, "released slot is reusable");
        // the first caches still see their own points
        check(rel(gpu.gradient(gc[0]), ref.gradient(rc[0])) <= 1e-11, "cache 0 unaliased");
    }

    // solve through the driver vs the reference solve
    double dx_worst = 0;
    for (const char* p : {"small", "large"}) {
        SolverConfig cfg = preset(p);
        cfg.epsilon = 1e-10;
        cfg.max_elapsed_seconds.reset();
        const SolveReport a = solve(panel, c, cfg);
        const SolveReport b = gpu.solve(cfg);
        check(a.status == b.status, "solve status");
        double dx = 0;
        bool same_active = true;
        for (index_t i = 0; i < n; ++i) {
            dx = std::max(dx, std::abs(a.x_star[i] - b.x_star[i]));
            same_active &= (a.x_star[i] <= cfg.tau + 1e-12) == (b.x_star[i] <= cfg.tau + 1e-12);
        }
        dx_worst = std::max(dx_worst, dx);
        check(same_active, "solve active set");
        check(dx <= 1e-8, "solve weights", dx);
        check(std::abs(a.f_star - b.f_star) <= 1e-12 * (1 + std::abs(a.f_star)), "solve objective");
    }
    std::printf("{\"failures\": %d, \"oracle_rel\": %.3e, \"solve_dx\": %.3e}\n", failures, worst, dx_worst);
    return failures;
}
