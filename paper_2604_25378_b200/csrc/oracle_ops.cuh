// Host-side launch layer for the streaming kernels (shared by the C-ABI and
// the C++ direction / solve driver).
#pragma once
#include "collective.cuh"
#include "context.cuh"

namespace mvsk_b200 {

// One fused pass of `op` over this rank's rows, then the deterministic cross-CTA
// reduction, the optional allreduce over the row-shard group, and the op
// epilogue. Inputs are device vectors of stride ld (zero padded). Outputs:
//   FGRAD:    slot z, slot g (ld), slot sc
//   HVP/THIRD: out (k x ldo)
//   LINESUMS: out[0..9) = s_rs / T ; zout (optional) = A d
//   XTW:      out (ld) = X^T tw (raw sum, no scaling)
struct PassIO {
    const double* vin = nullptr;
    const double* vin2 = nullptr;
    const double* z = nullptr;
    const double* tw = nullptr;
    double* zout = nullptr;
    double* out = nullptr;
    long long ldo = 0;    // output stride for HVP/THIRD/XTW
    const int* skip = nullptr;  // device flags: the whole pass is a no-op if all nskip are 0
    int nskip = 0;
    int slot = -1;        // FGRAD target slot
    const double* x_for_mux = nullptr;  // FGRAD: x (ld) for mu'x
    // optional mapped pinned host buffer (device alias) the epilogue also writes
    // its results to, so a host-API op needs no device-to-host copy node:
    // FGRAD [0, 5) scalars and [8, 8 + ld) the gradient; LINESUMS [0, 9) the
    // power sums; HVP / THIRD / XTW the outputs at stride ldo
    double* hout = nullptr;
};

void run_pass(mvsk_gpu_ctx* ctx, Op op, int k, const PassIO& io);

// psi''(z) elementwise (hessian_diag_weights)
void run_psi2(mvsk_gpu_ctx* ctx, const double* z, double* out, long long T);

// Weighted Gram G = X^T diag(w) X / T over the full panel (n x n, row-major,
// symmetric, both triangles written); allreduced across the shard group.
// G = X^T diag(w) X * scale; with z set, w = psi''(z) computed in the kernel (w_rows unused)
// one-cluster Gram for short narrow panels (small_pass.cuh); false if not eligible
// (packed: row-sharded groups get the packed lower triangle there instead of G)
bool run_small_gram(mvsk_gpu_ctx* ctx, const double* z, double* G_dev, double scale, double* G_host,
                    double* packed = nullptr);
// G_host: optional mapped host mirror (device alias) written alongside G_dev
void run_weighted_gram(mvsk_gpu_ctx* ctx, const double* w_rows, double* G_dev, double scale, const double* z = nullptr,
                       double* G_host = nullptr);

// q_t = x_t^T P x_t (P: ld x ld, zero outside the face) for this rank's rows
// with z and tw set: writes the third weights psi3(z) q / T to tw instead of q
void run_quadform(mvsk_gpu_ctx* ctx, const double* P_dev, double* q_dev, const double* z = nullptr,
                  double* tw = nullptr);
// tw_t = psi3(z_t) q_t / T with psi3 the third derivative weight
void run_third_weights(mvsk_gpu_ctx* ctx, const double* z, const double* q, double* tw);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size)
void set_smem_attr(const void* fn, size_t smem);
bool cluster_fits(const void* fn, int cs, int threads, size_t smem);

// device scratch sizing (grows workspaces on demand)
void ensure_host_staging(mvsk_gpu_ctx* ctx, size_t elems);

}  // namespace mvsk_b200
