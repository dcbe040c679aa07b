// Device-resident PCG branch of the YAND direction (affine_normal.hpp:189-242).
#pragma once
#include <vector>

#include "oracle_ops.cuh"

namespace mvsk_b200 {

constexpr int kPcgMaxCols = MVSK_GPU_MAX_RHS;

struct PcgInput {
    long long m = 0;           // face dimension (the reference's n = oracle.assets())
    std::vector<double> vU;    // tangent-basis reflector (m), simplex.hpp:31-33
    double bU = 0;
    std::vector<double> vQ;    // reduced-frame reflector (m-1), affine_normal.hpp:42-56
    double bQ = 0;
    std::vector<double> nu;    // normalised reduced gradient (m-1)
    double gn = 0;             // ||U^T g||
    double lambda = 0, tol = 1e-3;
    int maxit = 15, probe_cap = 5, hutchinson_probes = 8;
    bool exact_trace = false, has_third = true;
    std::vector<std::vector<double>> jacobi_probes;  // 8 Rademacher probes (m-2) or empty
    std::vector<std::vector<double>> probes;         // Hutchinson probes (m-2)
    bool unit_probes = false;                        // exact trace: probes are e_0..e_{m-3}, made on device
};

struct PcgOutput {
    std::vector<double> u;  // m-2
    int iters = 0;
    bool breakdown = false;
};

struct PcgWorkspace;
PcgOutput pcg_direction_device(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const PcgInput& in);
void pcg_workspace_free(mvsk_gpu_ctx* ctx);
// narrow faces (m <= 112, Hutchinson or no third term): every Hop through the
// reduced Hessian M = (UQ)^T G (UQ) built from one weighted-Gram pass
// (gram_pcg.cu); false when the face is out of its range
bool pcg_direction_gram(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const PcgInput& in, PcgOutput& out);
void gram_pcg_workspace_free(mvsk_gpu_ctx* ctx);

// direct branch of the YAND direction (affine_normal.hpp:151-188) on the device
// for faces of m <= 112: Gram, M + lambda I, its inverse, P, the trace pass and
// u = M^-1 rhs in one graph launch (gram_pcg.cu); false when out of range.
// A non-finite u asks the caller for the lambda fallback.
struct DirectInput {
    long long m = 0;
    std::vector<double> vU, vQ, nu;
    double bU = 0, bQ = 0, gn = 0, lambda = 0;
    bool has_third = true;
};
bool direct_direction_device(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const DirectInput& in,
                             std::vector<double>& u);

}  // namespace mvsk_b200
