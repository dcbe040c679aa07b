// mvsk_gpu_solve — a C++ host over the C-ABI only (no Python): the device
// counterpart of the reference CLI's `mvsk solve` (tools/mvsk_main.cpp:46-71)
// for binary panels. Loads a panel file straight into device memory
// (mvsk_gpu_create_from_binary), solves with a preset (solver.hpp:64-85) and
// prints the SolveReport keys of report_json.hpp:12-28.
//
//   mvsk_gpu_solve <panel.bin> [--gamma G | --coeffs c1,c2,c3,c4] [--preset small|large]
//                  [--epsilon E] [--tau T] [--max-iter N] [--no-max-elapsed] [--floor-sweep K]
// --floor-sweep K: BASELINE config 4's return-floor sweep instead of one solve
// (K floors between the min-variance and max-mean means, c1 calibrated per
// floor; mvsk_gpu_floor_sweep), printed as one JSON object.
// exit codes as the reference CLI (mvsk_main.cpp:213-219): 0 converged,
// 3 budget/stall, 2 bad arguments / domain errors, 1 data or device errors.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "mvsk_gpu.h"

static int fail(int code, const char* msg) {
    std::fprintf(stderr, "error: %s\n", msg);
    return (code == MVSK_DIMENSION_ERROR || code == MVSK_DOMAIN_ERROR) ? 2 : 1;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <panel.bin> [--gamma G|--coeffs c1,c2,c3,c4] [--preset small|large] ...\n",
                     argv[0]);
        return 2;
    }
    const char* path = argv[1];
    double gamma = 10.0;
    mvsk_coeffs c{};
    bool custom = false;
    std::string preset = "large";
    double eps = -1, tau = -1;
    int max_iter = -1;
    bool no_elapsed = false;
    int sweep = 0;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> const char* {
            if (i + 1 >= argc) {
                std::fprintf(stderr, "missing value for %s\n", a.c_str());
                std::exit(2);
            }
            return argv[++i];
        };
        if (a == "--gamma") gamma = std::atof(next());
        else if (a == "--coeffs") {
            if (std::sscanf(next(), "%lf,%lf,%lf,%lf", &c.c1, &c.c2, &c.c3, &c.c4) != 4) return 2;
            custom = true;
        } else if (a == "--preset") preset = next();
        else if (a == "--epsilon") eps = std::atof(next());
        else if (a == "--tau") tau = std::atof(next());
        else if (a == "--max-iter") max_iter = std::atoi(next());
        else if (a == "--no-max-elapsed") no_elapsed = true;
        else if (a == "--floor-sweep") sweep = std::atoi(next());
        else {
            std::fprintf(stderr, "unknown option %s\n", a.c_str());
            return 2;
        }
    }
    if (!custom) {  // crra_coefficients (panel.hpp:76-87)
        if (!(gamma > 0)) return fail(MVSK_DOMAIN_ERROR, "crra_coefficients: gamma must be positive");
        c = {1.0, gamma / 2.0, gamma * (gamma + 1.0) / 6.0, gamma * (gamma + 1.0) * (gamma + 2.0) / 24.0};
    }
    mvsk_solver_config cfg;
    int st = mvsk_gpu_preset(preset.c_str(), &cfg);
    if (st) return fail(st, "unknown preset");
    if (eps > 0) cfg.epsilon = eps;
    if (tau >= 0) cfg.tau = tau;
    if (max_iter > 0) cfg.max_iter = max_iter;
    if (no_elapsed) cfg.has_max_elapsed = 0;

    mvsk_gpu_ctx* ctx = nullptr;
    st = mvsk_gpu_create_from_binary(path, &c, 0, 1, 0, nullptr, &ctx);
    if (st) return fail(st, mvsk_gpu_last_error(nullptr));
    int64_t T = 0, Tl = 0, n = 0;
    mvsk_gpu_dims(ctx, &T, &Tl, &n);
    if (sweep > 0) {
        std::vector<mvsk_floor_point> pts((size_t)sweep);
        double m_mv = 0, m_max = 0;
        int32_t solves = 0;
        st = mvsk_gpu_floor_sweep(ctx, &cfg, nullptr, sweep, nullptr, nullptr, pts.data(), &m_mv, &m_max, &solves);
        if (st) {
            const int rc = fail(st, mvsk_gpu_last_error(ctx));
            mvsk_gpu_destroy(ctx);
            return rc;
        }
        std::printf("{\"m_mv\": %.17g, \"m_max\": %.17g, \"solves\": %d, \"points\": [", m_mv, m_max, solves);
        for (int k = 0; k < sweep; ++k)
            std::printf("%s{\"floor\": %.17g, \"c1\": %.17g, \"mean\": %.17g, \"f_star\": %.17g, \"status\": %d}",
                        k ? ", " : "", pts[(size_t)k].floor, pts[(size_t)k].c1, pts[(size_t)k].mean,
                        pts[(size_t)k].f_star, pts[(size_t)k].status);
        std::printf("]}\n");
        mvsk_gpu_destroy(ctx);
        return 0;
    }
    std::vector<double> x((size_t)n);
    mvsk_solve_report rep;
    st = mvsk_gpu_solve(ctx, &cfg, nullptr, x.data(), &rep, nullptr, nullptr);
    if (st) {
        const int rc = fail(st, mvsk_gpu_last_error(ctx));
        mvsk_gpu_destroy(ctx);
        return rc;
    }
    static const char* status_names[] = {"converged", "stalled", "max_iter", "max_elapsed", "degenerate_face"};
    std::printf("{\"x_star\": [");
    for (int64_t i = 0; i < n; ++i) std::printf("%s%.17g", i ? ", " : "", x[(size_t)i]);
    std::printf("], \"f_star\": %.17g, \"kkt_residual\": %.17g, \"interior_residual\": %.17g, \"iterations\": %d, "
                "\"face_events\": %d, \"restarts\": %d, \"identification_steps\": %d, \"krylov_iters_total\": %lld, "
                "\"oracle_passes\": %llu, \"wall_seconds\": %.9g, \"status\": \"%s\", \"config\": \"%s\", "
                "\"physical_passes\": %llu, \"T\": %lld, \"n\": %lld}\n",
                rep.f_star, rep.kkt_residual, rep.interior_residual, rep.iterations, rep.face_events, rep.restarts,
                rep.identification_steps, (long long)rep.krylov_iters_total, (unsigned long long)rep.oracle_passes,
                rep.wall_seconds, status_names[rep.status < 5 ? rep.status : 4], rep.config_label,
                (unsigned long long)rep.physical_passes, (long long)T, (long long)n);
    mvsk_gpu_destroy(ctx);
    return rep.status == 0 ? 0 : 3;
}
