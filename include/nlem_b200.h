/*
 * nlem_b200.h — C-ABI drop-in boundary for the NLEM / EM-ADMM hot path on B200 (sm_100a).
 *
 * The reference (/root/reference/proj) exposes this path as a C++ template API
 * on Eigen types.  There is no plugin/FFI layer in the reference, so each entry
 * point below is the plain-C replacement of one reference function, on
 * caller-owned buffers:
 *
 *   nlem_admm_batched      <- nlem::admm_euclidean_median   proj/include/nlem/admm.hpp:26-29
 *   nlem_irls_batched      <- nlem::irls_euclidean_median   proj/include/nlem/irls.hpp:21-23
 *   nlem_denoise           <- nlem::nlem_denoise            proj/include/nlem/nlem.hpp:71 (src/nlem.cpp:68-90)
 *   nlem_denoise (frames)  <- nlem::nlem_denoise_snapshots  proj/include/nlem/nlem.hpp:76 (src/nlem.cpp:92-128)
 *   nlem_denoise_rows      <- the same, for one row band of a larger image (multi-GPU sharding)
 *   nlm_denoise            <- nlem::nlm_denoise             proj/include/nlem/nlem.hpp:65 (src/nlm.cpp:31-51)
 *   nlem_validate_params   <- nlem::validate(NlemParams)    proj/src/nlm.cpp:17-29
 *   nlem_add_gaussian_noise<- nlem::add_gaussian_noise      proj/include/nlem/noise.hpp:46 (src/noise.cpp:7-17)
 *
 * Conventions
 *  - All arithmetic is float32 (the reference is float64; parity bar SURVEY.md §8d).
 *  - Point sets are [batch][n][d] row-major: point k of problem b is contiguous,
 *    which is exactly Eigen's d x n column-major PointSet::points (types.hpp:47-54).
 *  - Images are row-major [rows][cols] (proj/include/nlem/image.hpp:12).
 *  - Functions without a `_host` suffix take DEVICE pointers and enqueue on `stream`
 *    (a cudaStream_t, NULL = legacy default stream).  When `failure` is non-NULL
 *    the call synchronizes the stream and reports numeric failures; with
 *    failure == NULL it returns without synchronizing and numeric failures are
 *    not reported.  `_host` variants take HOST pointers, copy in/out themselves
 *    and always report.
 *  - No exceptions cross the ABI.  Invalid arguments return NLEM_INVALID_ARGUMENT
 *    with the reference's std::invalid_argument message in failure->message.
 *    Numeric failures (reference nlem::NumericFailure, types.hpp:20-31) return
 *    NLEM_NUMERIC_FAILURE with the LOWEST failing problem/pixel index (the
 *    reference reports whichever thread failed first, nlem.cpp:85-87 /
 *    parallel.hpp:37-46; lowest-index is its deterministic refinement).
 *  - Re-entrant; no global mutable state; results are bitwise deterministic and
 *    independent of the GPU count the caller shards over.
 */
#ifndef NLEM_B200_H
#define NLEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NLEM_OK = 0,
  NLEM_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  NLEM_NUMERIC_FAILURE = 2,  /* nlem::NumericFailure (types.hpp:20-31) */
  NLEM_CUDA_ERROR = 3
} nlem_status;

typedef enum {
  NLEM_FAIL_NONE = 0,
  NLEM_FAIL_ADMM_ITERATE = 1,   /* "non-finite ADMM iterate"   admm.hpp:67-68 */
  NLEM_FAIL_ADMM_OBJECTIVE = 2, /* "non-finite ADMM objective" admm.hpp:72,83-84 */
  NLEM_FAIL_IRLS_ITERATE = 3,   /* "non-finite IRLS iterate"   irls.hpp:50 */
  NLEM_FAIL_IRLS_OBJECTIVE = 4  /* "non-finite IRLS objective" irls.hpp:39,52,65-66 */
} nlem_failure_kind;

typedef struct {
  int64_t index;     /* lowest failing problem (batched) or global pixel r*cols+c; -1 = none */
  int64_t iteration; /* NumericFailure::iteration() */
  int32_t kind;      /* nlem_failure_kind */
  char message[256]; /* reference-format what(), e.g. "pixel (3, 4): non-finite IRLS objective (iteration 1)" */
} nlem_failure;

/* BoxConstraint (types.hpp:77-107): bounded = 0 is BoxConstraint::unconstrained(). */
typedef struct {
  int32_t bounded;
  float lower;
  float upper;
} nlem_box;

/* AdmmConfig (types.hpp:119-127).  record_trace is expressed by passing trace buffers. */
typedef struct {
  float mu;         /* > 0 */
  int32_t max_iter; /* >= 1 */
  float tol_primal; /* stop once max_k ||x_k - z|| <= tol_primal; < 0 never stops early */
} nlem_admm_config;

/* IrlsConfig (types.hpp:129-138). */
typedef struct {
  float epsilon;    /* > 0 */
  int32_t max_iter; /* >= 1 */
  float tol;        /* stop when prev - cur <= tol*|prev|; 0 = exact stall, < 0 never */
} nlem_irls_config;

typedef enum { NLEM_SOLVER_ADMM = 0, NLEM_SOLVER_IRLS = 1, NLEM_SOLVER_NLM_ONLY = 2 } nlem_solver;
typedef enum { NLEM_INIT_NOISY_PATCH = 0, NLEM_INIT_NLM_PATCH = 1 } nlem_patch_init;

/* NlemParams (proj/include/nlem/nlem.hpp:23-35).  `threads` has no GPU meaning and is
 * dropped; irls_tol is IrlsConfig::tol for the IRLS solver (the reference leaves it 0,
 * nlem.cpp:45-48). */
typedef struct {
  int32_t search;       /* odd search window side S */
  int32_t patch;        /* odd patch side k <= S */
  float h;              /* weights exp(-||P_j - P_c||^2 / h^2) (patch.cpp:52-61), > 0 */
  float sigma;          /* >= 0, informational (default_init_mode) */
  int32_t solver;       /* nlem_solver */
  int32_t solver_iters; /* >= 1 */
  float mu;             /* ADMM penalty > 0 */
  float epsilon;        /* IRLS smoothing > 0 */
  int32_t init_mode;    /* nlem_patch_init */
  nlem_box range;       /* box prior, default [0,255] */
  float irls_tol;
} nlem_params;

/* Library identification. */
const char* nlem_version(void);
const char* nlem_status_string(nlem_status status);

/* proj/src/nlm.cpp:17-29; writes the reference message into failure->message. */
nlem_status nlem_validate_params(const nlem_params* params, nlem_failure* failure);
/* proj/src/nlm.cpp:13-15 */
int32_t nlem_default_init_mode(float sigma);

/*
 * Batched EM-ADMM (Algorithm 1; proj/include/nlem/admm.hpp:26-86).
 *  points  [batch][n][d] device, weights [batch][n] device (validated as types.hpp:58-68)
 *  z_init  [batch][d] or NULL (NULL = weighted mean of the points, admm.hpp:40)
 *  z_out   [batch][d]; objective_out [batch] or NULL (em_cost at the minimizer);
 *  iters_out [batch] or NULL (SolverResult::iterations_run);
 *  trace_objective / trace_residual [batch][max_iter] or NULL (TraceRecord per sweep;
 *  entries past iterations_run are left untouched).
 */
nlem_status nlem_admm_batched(const float* points, const float* weights, int64_t batch, int64_t n,
                              int64_t d, const float* z_init, nlem_box box, nlem_admm_config cfg,
                              float* z_out, float* objective_out, int32_t* iters_out,
                              float* trace_objective, float* trace_residual, nlem_failure* failure,
                              void* stream);

/* Same contract on host buffers (H2D, kernels, D2H on `device`). */
nlem_status nlem_admm_batched_host(const float* points, const float* weights, int64_t batch,
                                   int64_t n, int64_t d, const float* z_init, nlem_box box,
                                   nlem_admm_config cfg, float* z_out, float* objective_out,
                                   int32_t* iters_out, float* trace_objective,
                                   float* trace_residual, nlem_failure* failure, int32_t device);

/* Batched IRLS (proj/include/nlem/irls.hpp:21-68); unconstrained like the reference. */
nlem_status nlem_irls_batched(const float* points, const float* weights, int64_t batch, int64_t n,
                              int64_t d, const float* x_init, nlem_irls_config cfg, float* x_out,
                              float* objective_out, int32_t* iters_out, float* trace_objective,
                              nlem_failure* failure, void* stream);

/* Same contract on host buffers. */
nlem_status nlem_irls_batched_host(const float* points, const float* weights, int64_t batch,
                                   int64_t n, int64_t d, const float* x_init, nlem_irls_config cfg,
                                   float* x_out, float* objective_out, int32_t* iters_out,
                                   float* trace_objective, nlem_failure* failure, int32_t device);

/*
 * Whole-image NLEM (proj/src/nlem.cpp:68-90).  noisy/out [rows][cols] device.
 * frames: NULL, or [solver_iters][rows][cols] device receiving
 * nlem_denoise_snapshots (nlem.cpp:92-128, forward-filled after an early stop).
 */
nlem_status nlem_denoise(const float* noisy, int64_t rows, int64_t cols, const nlem_params* params,
                         float* out, float* frames, nlem_failure* failure, void* stream);

/*
 * One row band of a rows x cols image: computes output rows [out_row0, out_row0+out_rows)
 * into out [out_rows][cols] (frames [solver_iters][out_rows][cols] or NULL).
 * `noisy` holds input rows [in_row0, in_row0+in_rows) of the full image; it must cover
 * every row the band reads, i.e. [out_row0 - S/2 - k/2, out_row0 + out_rows + S/2 + k/2)
 * clipped to [0, rows) plus the mirror images of the rows that fall outside.
 * Window clipping and patch mirroring use GLOBAL coordinates, so bands computed on
 * different GPUs are bitwise identical to the single-call result.
 */
nlem_status nlem_denoise_rows(const float* noisy, int64_t in_row0, int64_t in_rows, int64_t rows,
                              int64_t cols, int64_t out_row0, int64_t out_rows,
                              const nlem_params* params, float* out, float* frames,
                              nlem_failure* failure, void* stream);

/* Host-buffer row band on `device`: H2D of the input rows, kernels, D2H of the band. */
nlem_status nlem_denoise_rows_host(const float* noisy, int64_t in_row0, int64_t in_rows,
                                   int64_t rows, int64_t cols, int64_t out_row0, int64_t out_rows,
                                   const nlem_params* params, float* out, float* frames,
                                   nlem_failure* failure, int32_t device);

/* Host-buffer whole-image NLEM on `device` (the reference-facing call used for e2e). */
nlem_status nlem_denoise_host(const float* noisy, int64_t rows, int64_t cols,
                              const nlem_params* params, float* out, float* frames,
                              nlem_failure* failure, int32_t device);

/* Whole-image NLEM from host buffers over several GPUs of one node: the image is cut into
 * ndev contiguous row bands, band i runs nlem_denoise_rows_host on devices[i]
 * from its own host thread with its own 13-row halo (S/2 + k/2), and no collective runs.  The
 * result (and frames, [solver_iters][rows][cols] host, or NULL) is bitwise identical to the
 * single-device call; a NumericFailure reports the lowest failing pixel over all bands, as
 * the single call does.  devices may repeat (several bands per GPU).  This replaces the
 * reference's internal thread pool (NlemParams::threads, proj/src/nlem.cpp:68-90 with
 * parallel.hpp:20-55) by a device pool. */
nlem_status nlem_denoise_multi_host(const float* noisy, int64_t rows, int64_t cols,
                                    const nlem_params* params, float* out, float* frames,
                                    const int32_t* devices, int32_t ndev, nlem_failure* failure);

/* Classical non-local means (proj/src/nlm.cpp:31-51). */
nlem_status nlm_denoise(const float* noisy, int64_t rows, int64_t cols, const nlem_params* params,
                        float* out, nlem_failure* failure, void* stream);

/* PSNR of every frame against `clean` (proj/include/nlem/psnr.hpp:12-24: peak 255, +inf when
 * identical), reduced on the device in FP64: frames [nframes][count] and clean [count] are
 * device buffers, psnr_out [nframes] is HOST memory (the call synchronizes `stream`).
 * Lets config-4 style convergence sweeps skip the T x H x W frame download. */
nlem_status nlem_frames_psnr(const float* frames, const float* clean, int64_t nframes,
                             int64_t count, double* psnr_out, nlem_failure* failure, void* stream);

/* Batched first-order optimality certificate (proj/include/nlem/diagnostics.hpp:22-55):
 * residual_out[b] = max(0, ||g_b|| - sum of coincident weights) with active box faces
 * absorbing blocked components; 0 certifies z_b optimal.  Device buffers; z must lie in the
 * box (else the residual is NaN, where the reference throws). */
nlem_status nlem_optimality_residual_batched(const float* points, const float* weights,
                                             int64_t batch, int64_t n, int64_t d, nlem_box box,
                                             const float* z, float* residual_out,
                                             nlem_failure* failure, void* stream);

/* build_patch_stack(image, row, col, search, k, h) (proj/include/nlem/patch.hpp:48-49,
 * proj/src/patch.cpp:90-114) for one pixel, from a HOST image on `device`: the clipped search
 * window in row-major neighbour order, each neighbour's k x k mirrored patch
 * (patch.cpp:9-38) at patches_out[j*k*k ..], weights exp(-||P_j - P_self||^2 / h^2) with the
 * self weight exactly 1 (patch.cpp:52-61).  patches_out [search*search][k*k] and weights_out
 * [search*search] are host buffers sized for the unclipped window; *n_out receives the
 * neighbour count n and *self_column_out the index of the pixel itself.  Reference messages
 * for invalid input (validate_image, "... must be odd and positive", "pixel outside the
 * image", "similarity bandwidth h must be positive"). */
nlem_status nlem_patch_stack_host(const float* image, int64_t rows, int64_t cols, int64_t row,
                                  int64_t col, int32_t search, int32_t patch, float h,
                                  float* patches_out, float* weights_out, int64_t* n_out,
                                  int64_t* self_column_out, nlem_failure* failure,
                                  int32_t device);

/* solve_patch(stack, params) (proj/include/nlem/nlem.hpp:60-62, proj/src/nlem.cpp:20-56) on
 * `device`, from host buffers: patches [n][d] (point-contiguous), weights [n], self_column.
 * init_out [d] receives the initial patch (nlem.cpp:13-18, params->init_mode), patch_out [d]
 * the solved patch inside params->range: ADMM from init (max_iter = solver_iters, tol 0),
 * IRLS from init (epsilon, tol = irls_tol) then clipped, or NlmOnly = the clipped weighted
 * mean.  The per-iteration callback of the reference cannot cross the ABI (use
 * nlem_denoise's frames).  Errors as the solvers': INVALID_ARGUMENT with the reference
 * message ("patch stack has no valid self column", validate(NlemParams), types.hpp:58-68),
 * NUMERIC_FAILURE with the iteration. */
nlem_status nlem_solve_patch_host(const float* patches, const float* weights, int64_t n, int64_t d,
                                  int64_t self_column, const nlem_params* params, float* init_out,
                                  float* patch_out, nlem_failure* failure, int32_t device);

/* Halo (rows) a band needs on each side: S/2 + k/2 (13 for S=21, k=7). */
int64_t nlem_band_halo(const nlem_params* params);

/* proj/src/noise.cpp:7-17 with GaussianSampler (noise.hpp:15-40): out = clean + sigma*xi,
 * xi drawn in row-major order from mt19937_64(seed) Box-Muller, unclipped.  Host. */
void nlem_add_gaussian_noise(const double* clean, int64_t count, double sigma, uint64_t seed,
                             double* out);

/* Seeded synthetic inputs (SURVEY.md §8d generators; host, float32 outputs). */
void nlem_synth_clean_image(int64_t rows, int64_t cols, int32_t rects, int32_t disks,
                            uint64_t seed, float* clean_out);
void nlem_synth_noisy_image(int64_t rows, int64_t cols, int32_t rects, int32_t disks, double sigma,
                            uint64_t image_seed, uint64_t noise_seed, float* clean_out,
                            float* noisy_out);
void nlem_synth_point_sets(int64_t batch, int64_t n, int64_t d, uint64_t seed_base,
                           int64_t first_problem, float* points_out, float* weights_out,
                           int32_t threads);

#ifdef __cplusplus
}
#endif

#endif /* NLEM_B200_H */
