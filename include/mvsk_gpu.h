/*
 * mvsk_gpu.h — C-ABI of the B200-native YAND-MVSK sample-oracle core.
 *
 * This is the drop-in boundary. The reference has no FFI: its operator API is
 * the header-only C++ class mvsk::Oracle (proj/include/mvsk/oracle.hpp:29-149)
 * with value type OracleCache (:14-20), plus line_model (linesearch.hpp:62),
 * yand_direction (affine_normal.hpp:127-245) and solve (solver.hpp:195-655).
 * Each entry point below names the reference interface it replaces. Plain
 * pointers and sizes only; every host vector is fp64, row-major where 2-D.
 *
 * Ownership: the panel A (T x n, row-major, the reference's ReturnPanel::A,
 * panel.hpp:16-30) is uploaded once into device memory owned by the context
 * (mvsk_gpu_create), or borrowed from caller device memory that must outlive
 * the context (mvsk_gpu_create_from_device), matching the reference's
 * borrowed `const Mat*` (oracle.hpp:24-25, 142). Caches (OracleCache by value
 * in the reference) are device-resident slots 0..MVSK_GPU_MAX_SLOTS-1.
 *
 * Errors: every call returns an mvsk_status; the reference's typed exceptions
 * (common.hpp:14-25) map 1:1 (dimension/domain/data/numeric), plus CUDA/NCCL.
 * mvsk_gpu_last_error(ctx) holds the message. There is no CPU fallback: a
 * missing device is MVSK_CUDA_ERROR.
 *
 * Multi-GPU: one context per GPU/process holds a contiguous row block of A;
 * every n-vector / scalar result is combined with ncclAllReduce(sum, fp64)
 * inside the call, so all ranks receive identical results (SPMD driver).
 */
#ifndef MVSK_GPU_H
#define MVSK_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MVSK_GPU_ABI_VERSION 1
#define MVSK_GPU_MAX_SLOTS 8
#define MVSK_GPU_MAX_RHS 16
#define MVSK_GPU_MAX_ASSETS 8192 /* widest panel (columns) a context accepts */
#define MVSK_NCCL_UNIQUE_ID_BYTES 128

typedef enum {
    MVSK_OK = 0,
    MVSK_DIMENSION_ERROR = 1, /* mvsk::dimension_error (common.hpp:15) */
    MVSK_DOMAIN_ERROR = 2,    /* mvsk::domain_error    (common.hpp:18) */
    MVSK_DATA_ERROR = 3,      /* mvsk::data_error      (common.hpp:21) */
    MVSK_NUMERIC_ERROR = 4,   /* mvsk::numeric_error   (common.hpp:24) */
    MVSK_CUDA_ERROR = 5,
    MVSK_NCCL_ERROR = 6,
    MVSK_INTERNAL_ERROR = 7
} mvsk_status;

typedef struct mvsk_gpu_ctx mvsk_gpu_ctx;

/* PreferenceCoefficients (panel.hpp:47-62): f = -c1 mu'x + (1/T) sum c2 z^2 - c3 z^3 + c4 z^4 */
typedef struct {
    double c1, c2, c3, c4;
} mvsk_coeffs;

/* TangentSolveConfig (affine_normal.hpp:59-69) */
typedef struct {
    int32_t mode; /* 0 = direct, 1 = pcg */
    int32_t krylov_maxit;
    double lambda;
    double krylov_tol;
    int32_t jacobi;
    int32_t exact_trace;
    int32_t hutchinson_probes;
    int32_t probe_maxit;
} mvsk_tangent_config;

/* DirectionDiagnostics (affine_normal.hpp:71-77) */
typedef struct {
    double reduced_grad_norm;
    double u_norm;
    int32_t krylov_iters;
    int32_t pcg_breakdown;
    int32_t lambda_fallback;
    int32_t _pad;
} mvsk_direction_diag;

/* SolverConfig (solver.hpp:44-62); presets via mvsk_gpu_preset */
typedef struct {
    double epsilon;
    double tau;
    int32_t max_iter;
    int32_t has_max_elapsed;
    double max_elapsed_seconds;
    double projected_trial_step;
    double restart_trial_steps[4];
    int32_t n_restart_trial_steps;
    int32_t restart_max_iter;
    mvsk_tangent_config tangent;
    int32_t line_search; /* 0 = exact quartic, 1 = armijo */
    int32_t stall_restarts;
    int32_t identification_pass;
    int32_t _pad;
    char label[16];
} mvsk_solver_config;

/* SolveReport (solver.hpp:93-107) + device-side counters */
typedef struct {
    double f_star;
    double kkt_residual;
    double interior_residual;
    double wall_seconds;
    int64_t krylov_iters_total;
    uint64_t oracle_passes;   /* logical passes, reference cost contract (common.hpp:27-37) */
    uint64_t physical_passes; /* streaming passes over A actually issued on the device */
    int32_t iterations;
    int32_t face_events;
    int32_t restarts;
    int32_t identification_steps;
    int32_t status; /* SolveStatus (solver.hpp:21): 0 converged, 1 stalled, 2 max_iter, 3 max_elapsed, 4 degenerate_face */
    int32_t _pad;
    char config_label[16];
} mvsk_solve_report;

/* IterateObserver (solver.hpp:36-42) */
typedef void (*mvsk_observer_fn)(void* user, int32_t iteration, double f, const double* x, int64_t n);

/* ---- library / lifecycle ------------------------------------------------- */
int32_t mvsk_gpu_abi_version(void);
const char* mvsk_gpu_status_string(int32_t status);
/* solver presets small_preset / large_preset (solver.hpp:64-85); name = "small" | "large" */
int32_t mvsk_gpu_preset(const char* name, mvsk_solver_config* out);
/* ncclGetUniqueId for the SPMD row-shard group (caller broadcasts the bytes) */
int32_t mvsk_gpu_nccl_unique_id(void* out /* MVSK_NCCL_UNIQUE_ID_BYTES */);

/* Oracle(const ReturnPanel&, PreferenceCoefficients, ...) (oracle.hpp:31-45):
 * uploads host A (T x n row-major) and mu (n) to `device`. Every constructor
 * returns MVSK_DIMENSION_ERROR for n > MVSK_GPU_MAX_ASSETS (the streaming kernels
 * stage whole rows; the reference's largest universe has n = 5440). */
int32_t mvsk_gpu_create(const double* A, int64_t T, int64_t n, const double* mu,
                        const mvsk_coeffs* c, int32_t device, mvsk_gpu_ctx** out);
/* Row-sharded variant: this rank holds rows [row0, row0 + T_local) of a T_global x n
 * panel (host memory); nranks == 1 needs no id. Collectives use NCCL over NVLink. */
int32_t mvsk_gpu_create_sharded(const double* A_rows, int64_t T_local, int64_t row0,
                                int64_t T_global, int64_t n, const double* mu,
                                const mvsk_coeffs* c, int32_t device, int32_t nranks,
                                int32_t rank, const void* nccl_unique_id, mvsk_gpu_ctx** out);
/* In-process row-shard group: nranks contexts driven by nranks host threads of
 * ONE process, on one device or several (peer access). Each oracle op's
 * exchange step is a peer-memory allreduce (every rank sums all members'
 * buffers in rank order, identical bits everywhere) ordered by CUDA events at
 * two host rendezvous per collective, instead of NCCL. Same SPMD contract as
 * NCCL groups: every rank calls the same ops in the same order. Member ops
 * launch eagerly (no CUDA-graph replay). Destroy the contexts before the
 * group. */
typedef struct mvsk_gpu_group mvsk_gpu_group;
int32_t mvsk_gpu_group_create(int32_t nranks /* 1..8 */, mvsk_gpu_group** out);
int32_t mvsk_gpu_group_destroy(mvsk_gpu_group* group);
int32_t mvsk_gpu_create_sharded_in_group(const double* A_rows, int64_t T_local, int64_t row0,
                                         int64_t T_global, int64_t n, const double* mu,
                                         const mvsk_coeffs* c, int32_t device,
                                         mvsk_gpu_group* group, int32_t rank, mvsk_gpu_ctx** out);
/* Borrow a device-resident panel block (T_local x n, leading dimension ld >= n,
 * ld even, 16-byte aligned base). The memory must outlive the context. The
 * padding columns [n, ld) of every row are read (and multiplied by zero) by the
 * streaming kernels, so they must be finite (zero is typical, e.g. a memset
 * cudaMallocPitch block); non-finite padding -> MVSK_DATA_ERROR at creation. */
int32_t mvsk_gpu_create_from_device(const double* A_dev, int64_t ld, int64_t T_local,
                                    int64_t row0, int64_t T_global, int64_t n,
                                    const double* mu, const mvsk_coeffs* c, int32_t device,
                                    int32_t nranks, int32_t rank, const void* nccl_unique_id,
                                    mvsk_gpu_ctx** out);
/* load_returns_binary + center_panel + Oracle (panel_io.hpp:121-141, panel.hpp:32-44,
 * oracle.hpp:43-45): reads this rank's row block of a binary panel file ("MVSK",
 * u32 T, u32 n, row-major LE f64 raw returns) straight into device memory and
 * centres it with the global column means (allreduced across the group).
 * Malformed files / non-finite entries -> MVSK_DATA_ERROR. */
int32_t mvsk_gpu_create_from_binary(const char* path, const mvsk_coeffs* c, int32_t device, int32_t nranks,
                                    int32_t rank, const void* nccl_unique_id, mvsk_gpu_ctx** out);
/* header of a binary panel file (no device needed): T, n */
int32_t mvsk_gpu_binary_dims(const char* path, int64_t* T, int64_t* n);
/* column means mu (n) of the context's panel */
int32_t mvsk_gpu_mu(const mvsk_gpu_ctx* ctx, double* mu_out);
int32_t mvsk_gpu_destroy(mvsk_gpu_ctx* ctx);
const char* mvsk_gpu_last_error(const mvsk_gpu_ctx* ctx);
/* Run all device work on this cudaStream_t (NULL = the context's own stream). */
int32_t mvsk_gpu_set_stream(mvsk_gpu_ctx* ctx, void* stream);
int32_t mvsk_gpu_synchronize(mvsk_gpu_ctx* ctx);
int32_t mvsk_gpu_dims(const mvsk_gpu_ctx* ctx, int64_t* T_global, int64_t* T_local, int64_t* n);

/* ---- oracle (oracle.hpp) ---------------------------------------------------
 * Vectors are in the coordinates of the current face (mvsk_gpu_set_face);
 * with no face set they have length n. */

/* zoff / value_offset ctor arguments (oracle.hpp:31-33): z = A x + zoff (zoff has
 * this rank's T_local rows, NULL clears) and f += value_offset. */
int32_t mvsk_gpu_set_offset(mvsk_gpu_ctx* ctx, const double* zoff, double value_offset);
/* Face oracle (solver.hpp:343-363, simplex.hpp:161-192): restrict to the free
 * coordinates free_idx[0..nf) with the pinned ones fixed at tau. Replaces the
 * reference's column-gathered Af / zoff / f_offset with an index map over the
 * resident panel. nf == n with free_idx == NULL restores the full problem. */
int32_t mvsk_gpu_set_face(mvsk_gpu_ctx* ctx, const int64_t* free_idx, int64_t nf, double tau);
/* make_cache (oracle.hpp:54-69): one fused pass computes z, f, the moments and
 * the gradient into `slot`; counts 1 forward pass. */
int32_t mvsk_gpu_make_cache(mvsk_gpu_ctx* ctx, int32_t slot, const double* x, double* f_out);
/* value / moments (oracle.hpp:71-77): out = (mu'x, E z^2, E z^3, E z^4) */
int32_t mvsk_gpu_value(mvsk_gpu_ctx* ctx, int32_t slot, double* f_out);
int32_t mvsk_gpu_moments(mvsk_gpu_ctx* ctx, int32_t slot, double out[4]);
/* gradient (oracle.hpp:79-90), memoised: counts 1 transpose pass on first call */
int32_t mvsk_gpu_gradient(mvsk_gpu_ctx* ctx, int32_t slot, double* g_out);
/* hvp (oracle.hpp:92-101) for k right-hand sides V (k x nf row-major) in one
 * fused pass; HV is k x nf. Counts 2k logical passes (the reference contract). */
int32_t mvsk_gpu_hvp(mvsk_gpu_ctx* ctx, int32_t slot, const double* V, int32_t k, double* HV);
/* third_action (oracle.hpp:103-113) for k pairs (U_i, V_i); counts 3k passes */
int32_t mvsk_gpu_third_action(mvsk_gpu_ctx* ctx, int32_t slot, const double* U, const double* V,
                              int32_t k, double* out);
/* hessian_diag_weights (oracle.hpp:116-119): psi''(z) for this rank's T_local rows */
int32_t mvsk_gpu_hessian_diag_weights(mvsk_gpu_ctx* ctx, int32_t slot, double* out);
/* sample_direction (oracle.hpp:122): A d for this rank's T_local rows; 1 pass */
int32_t mvsk_gpu_sample_direction(mvsk_gpu_ctx* ctx, const double* d, double* out);
/* line_model (linesearch.hpp:62-81): out = a0..a4 followed by the nine power
 * sums s11,s21,s31,s02,s12,s22,s03,s13,s04 (PowerSums, :16-20); 1 pass. */
int32_t mvsk_gpu_line_model(mvsk_gpu_ctx* ctx, int32_t slot, const double* d, double cap,
                            double out[14]);
/* k line models at the same cache in one graph launch and one round trip
 * (1 <= k <= 8): D is k x nf row-major, out is k x 14 laid out as above. Each
 * model is bitwise what mvsk_gpu_line_model returns for that direction; the
 * solve driver uses it for the rungs of the boundary ladder
 * (solver.hpp:448-562). A direction that line_model would reject (zero, or not
 * tangent to the simplex) gets a0 = NaN instead of a domain_error. Counts k
 * logical passes. */
int32_t mvsk_gpu_line_models(mvsk_gpu_ctx* ctx, int32_t slot, const double* D, int32_t k, double* out);
/* PassCounter (common.hpp:31-37) plus physical streaming passes */
int32_t mvsk_gpu_passes(const mvsk_gpu_ctx* ctx, uint64_t* forward, uint64_t* transpose,
                        uint64_t* physical);
int32_t mvsk_gpu_reset_passes(mvsk_gpu_ctx* ctx);
/* kernels this context has enqueued so far (CUDA-graph replays included) */
int32_t mvsk_gpu_launch_count(const mvsk_gpu_ctx* ctx, uint64_t* launches);

/* ---- direction / solve -------------------------------------------------- */
/* Weighted Gram G = A_F^T diag(psi''(z)) A_F / T over the current face (nf x nf,
 * row-major): the dense contraction behind the direct branch M = (UQ)^T G (UQ)
 * (affine_normal.hpp:160-170). fp64 DMMA tensor-core kernel. */
int32_t mvsk_gpu_weighted_gram(mvsk_gpu_ctx* ctx, int32_t slot, double* G_out);
/* yand_direction (affine_normal.hpp:127-245) at the cached point: d has nf entries */
int32_t mvsk_gpu_yand_direction(mvsk_gpu_ctx* ctx, int32_t slot, const mvsk_tangent_config* cfg,
                                uint64_t it_seed, double* d_out, mvsk_direction_diag* diag);
/* solve (solver.hpp:195-655) over the context's full panel. x0 may be NULL
 * (barycentre). x_star has n entries. observer may be NULL. */
int32_t mvsk_gpu_solve(mvsk_gpu_ctx* ctx, const mvsk_solver_config* cfg, const double* x0,
                       double* x_star, mvsk_solve_report* report, mvsk_observer_fn observer,
                       void* observer_user);

/* Replace the preference coefficients (c1..c4) of a live context; invalidates
 * every cache slot (their f / gradient depend on c). */
int32_t mvsk_gpu_set_coeffs(mvsk_gpu_ctx* ctx, const mvsk_coeffs* c);

/* Return-floor sweep (BASELINE config 4). Not in the reference code: the paper's
 * calibration of the mean coefficient so that the optimum's
 * in-sample mean mu'x* lies as close as possible to a return floor, c2..c4 held
 * at the context's values. floors may be NULL: then nfloors interior points
 * r_k = m_mv + k/(nfloors+1) (m_max - m_mv), m_mv the mean of the
 * minimum-variance optimum (c = (0, c2, 0, 0)), m_max = max_j mu_j. */
typedef struct {
    double mean_tol;    /* stop when |mu'x* - r| <= mean_tol * (m_max - m_mv); default 1e-3 */
    int32_t max_solves; /* solve budget per floor; default 16 */
    int32_t warm_start; /* start each solve from the evaluated optimum nearest in c1 */
} mvsk_sweep_config;
typedef struct {
    double floor;  /* target in-sample mean r */
    double c1;     /* calibrated mean coefficient */
    double mean;   /* mu'x* at c1 */
    double f_star;
    double kkt_residual;
    int32_t status; /* SolveStatus of that solve */
    int32_t solves; /* solves this floor added */
} mvsk_floor_point;
/* x_out: nfloors x n (row k = optimum for floor k), may be NULL. sw may be NULL
 * (defaults). The context's coefficients are restored on return. */
int32_t mvsk_gpu_floor_sweep(mvsk_gpu_ctx* ctx, const mvsk_solver_config* cfg, const mvsk_sweep_config* sw,
                             int32_t nfloors, const double* floors, double* x_out, mvsk_floor_point* points,
                             double* m_mv, double* m_max, int32_t* total_solves);

/* ---- device-resident fast path (inputs/outputs already in HBM) --------------
 * Same math as above, full coordinates (length n, no face), asynchronous on the
 * context stream, no host synchronisation; used for HBM-roofline measurement and
 * by device-resident callers. Pointers are device pointers. */
int32_t mvsk_gpu_make_cache_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* x_dev);
int32_t mvsk_gpu_hvp_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* V_dev, int32_t k,
                            double* HV_dev);
int32_t mvsk_gpu_third_action_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* U_dev,
                                     const double* V_dev, int32_t k, double* out_dev);
int32_t mvsk_gpu_line_sums_device(mvsk_gpu_ctx* ctx, int32_t slot, const double* d_dev,
                                  double* sums_dev /* 9 */);
int32_t mvsk_gpu_weighted_gram_device(mvsk_gpu_ctx* ctx, int32_t slot, double* G_dev /* n x n */);
/* device pointers of a slot's cache: z (T_local), gradient (n), scalars [f, mu'x, Ez2, Ez3, Ez4] */
int32_t mvsk_gpu_slot_pointers(mvsk_gpu_ctx* ctx, int32_t slot, double** z, double** grad,
                               double** scalars);

#ifdef __cplusplus
}
#endif

#endif /* MVSK_GPU_H */
