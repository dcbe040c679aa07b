// Host-facing oracle layer: the mvsk::Oracle method set (oracle.hpp:54-122)
// and line_model (linesearch.hpp:62-81) over an explicit face view, with host
// vectors in face coordinates. Used by the C-ABI and by the C++ direction /
// solve driver (which needs the face and the full problem side by side).
#pragma once
#include <vector>

#include "oracle_ops.cuh"

namespace mvsk_b200 {

using Vec = std::vector<double>;

FaceMap full_face(const mvsk_gpu_ctx* ctx);
// workspaces sized by ctx->ld (records ld_alloc) / free a context and its face child
void ctx_alloc_workspaces(mvsk_gpu_ctx* ctx);
void ctx_free(mvsk_gpu_ctx* ctx);
// compact face context for the face with these free columns (face.cu); reused
// across faces while it fits. fold_face_counters adds the child's pass / launch
// counters into the parent's.
mvsk_gpu_ctx* face_context(mvsk_gpu_ctx* parent, const std::vector<int64_t>& free_idx, const std::vector<char>& pinned,
                           double tau);
void fold_face_counters(mvsk_gpu_ctx* parent);
// the face view over a compact face context (its first nf columns)
FaceMap face_child_map(const mvsk_gpu_ctx* child, long long nf);
void check_slot(const mvsk_gpu_ctx* ctx, int slot, bool need_valid = true);

// make_cache: returns f; throws numeric_error on a non-finite value
double op_make_cache(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const double* x);
// value / moments (mu'x, E z^2, E z^3, E z^4) of a valid slot
double op_value(mvsk_gpu_ctx* ctx, int slot);
void op_moments(mvsk_gpu_ctx* ctx, int slot, double out[4]);
void op_gradient(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, double* g);
void op_hvp(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const double* V, int k, double* HV);
void op_third(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const double* U, const double* V, int k, double* out);
void op_psi2(mvsk_gpu_ctx* ctx, int slot, double* out);
void op_sample_direction(mvsk_gpu_ctx* ctx, const FaceMap& fm, const double* d, double* out);
void op_line_model(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const double* d, double out[14]);
// k line models in one graph launch (k x 14 doubles out; a0 = NaN marks a direction op_line_model would reject)
void op_line_models(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const double* D, int k, double* out);
// weighted Gram over the face columns: G_f = A_f^T diag(psi''(z)) A_f / T (m x m)
void op_weighted_gram(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, double* G);
// q_t = a_t^T P a_t for a symmetric face-coordinate P (m x m), then
// out = A_f^T (psi'''(z) o q) / T  (the direct branch's a, affine_normal.hpp:173-178,
// before the (UQ)^T projection)
void op_third_trace_rows(mvsk_gpu_ctx* ctx, int slot, const FaceMap& fm, const double* P, double* out);

}  // namespace mvsk_b200
