// Device-resident SPG identification preamble (solver.hpp:116-185), spg_device.cu.
#pragma once
#include <vector>

#include "oracle_ops.cuh"

namespace mvsk_b200 {

struct SpgWorkspace;
// Runs the preamble from x (f0, g0 = f and gradient at x, full panel) on the
// device as one conditional-while CUDA graph, leaving the result in x. Returns
// false (x untouched) when the device loop is not enabled (MVSK_SPG_GRAPH) or
// not applicable (n > 8192, a z offset, graphs unavailable): the caller then
// runs the host loop.
bool spg_identify_device(mvsk_gpu_ctx* ctx, int slot, std::vector<double>& x, double f0,
                         const std::vector<double>& g0, double tau, int max_steps, int patience, double eps_stop,
                         int& steps_out);
void spg_workspace_free(mvsk_gpu_ctx* ctx);

}  // namespace mvsk_b200
