/*
 * dfpca_cuda.h -- C-ABI of libdfpca_cuda.so, the sm_100a implementation of the
 * binned multi-dimensional FPCA hot path (reference: arxiv 1510.04439, C++
 * header library `proj/include/dfpca`).
 *
 * Every entry point takes plain pointers and sizes; no C++ or torch types cross
 * this boundary.  Host pointers are host memory; results stay device-resident
 * behind opaque handles (dfpca_binned, dfpca_surface) so that the stages can be
 * chained without host round trips, and are copied out only on request.
 *
 * Status convention (mirrors dfpca::ErrorClass, reference errors.hpp:11-17):
 *   0 = ok, 2 = Parse, 3 = Config, 4 = Numeric, 5 = Version.
 * On a nonzero status, dfpca_last_error() returns the reference error name
 * (e.g. "HaloTooSmall", errors.hpp:37-90) and the message, so a host wrapper
 * can rethrow the matching dfpca::Error.  Device (CUDA) failures are reported
 * as class 4 with name "DeviceError".
 *
 * Flattened arrays are row-major with the LAST axis fastest (grid.hpp:14-16);
 * covariance surfaces are flattened s_flat * G + t_flat (surface.hpp:14).
 */
#ifndef DFPCA_CUDA_H_
#define DFPCA_CUDA_H_

#include <stdint.h>

#if defined(__GNUC__)
#define DFPCA_API __attribute__((visibility("default")))
#else
#define DFPCA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DFPCA_MAX_DIM 3

typedef struct dfpca_context dfpca_context;
typedef struct dfpca_binned dfpca_binned;
typedef struct dfpca_surface dfpca_surface;
typedef struct dfpca_dataset dfpca_dataset;
typedef struct dfpca_table dfpca_table;

/* Grid descriptor: the data an EvaluationGrid carries (grid.hpp:92-230).
 * axes[k] points at shape[k] strictly increasing node coordinates (host).
 * mask is NULL (every node inside) or prod(shape) bytes, 1 = inside. */
typedef struct dfpca_grid {
  int32_t dim;
  int64_t shape[DFPCA_MAX_DIM];
  const double* axes[DFPCA_MAX_DIM];
  const uint8_t* mask;
} dfpca_grid;

/* Overlapping-block plan (fft_smoother.hpp:37-53).  blocks_lo / blocks_hi hold
 * n_blocks * dim node indices (block b, axis k at b * dim + k); halo holds dim
 * values.  The device path is plan-invariant (the reference guarantees
 * bit-invariant cores, fft_smoother.hpp:24-29), so the plan is only validated
 * (validate_block_plan, fft_smoother.hpp:101-145).  Pass NULL for the
 * single-block plan. */
typedef struct dfpca_plan {
  int64_t n_blocks;
  const int64_t* blocks_lo;
  const int64_t* blocks_hi;
  const int64_t* halo;
} dfpca_plan;

enum { DFPCA_TARGET_MEAN = 0, DFPCA_TARGET_SQUARES = 1 };
enum { DFPCA_SURFACE_MEAN = 0, DFPCA_SURFACE_COVARIANCE = 1, DFPCA_SURFACE_DIAG = 2 };

/* ---- context ------------------------------------------------------------ */
/* One CUDA device, one stream, one workspace per context.  Calls are
 * synchronous at return; calls on one context from several host threads are
 * serialised by the context (the reference's functions are reentrant), and
 * dfpca_last_error reports the calling thread's last call on that context.
 * Distinct contexts run concurrently. */
DFPCA_API int dfpca_context_create(int device, dfpca_context** out);
DFPCA_API int dfpca_context_destroy(dfpca_context* ctx);
/* Backs the context's stream-ordered pool with at least `bytes` of device
 * memory now (allocated once, returned to the pool, kept): a later call that
 * needs that much reuses mapped pages instead of growing the pool while its
 * kernels run.  The first config-5 (d = 3, 32^3) covariance is ~0.7 s with no
 * reserve and ~0.12 s after a 96 GB one; mapping costs ~13 ms per GB, paid
 * here.  The initial reserve is DFPCA_POOL_RESERVE_GB (default 16: without
 * one the pool grows in fragments and calls stall while it maps more).  Not
 * in the reference (its host allocator has no such cost). */
DFPCA_API int dfpca_context_reserve(dfpca_context* ctx, uint64_t bytes);
DFPCA_API int dfpca_last_error(const dfpca_context* ctx, int* error_class, const char** name,
                     const char** message);
/* Sample / observation index attached to ObservationOutsideGrid (-1 if none). */
DFPCA_API int dfpca_last_error_location(const dfpca_context* ctx, int64_t* sample, int64_t* obs);
/* Device time (ms, CUDA events) of the stages run by the last call, by name:
 * "binning", "pairs", "moments", "solve", "fallback", "center", "eigen", ... */
DFPCA_API int dfpca_stage_time(const dfpca_context* ctx, const char* stage, double* ms);
/* Number of kernels this context has launched since creation. */
DFPCA_API int64_t dfpca_kernel_launches(const dfpca_context* ctx);
/* Profiling mode: bracket every launch with CUDA events on the launching
 * stream and accumulate device time per kernel name (resets the table). */
DFPCA_API int dfpca_profile_enable(dfpca_context* ctx, int on);
/* index-th entry of the per-kernel table: name, total ms, launch count. */
DFPCA_API int dfpca_kernel_stat(const dfpca_context* ctx, int64_t index, const char** name, double* ms,
                                int64_t* count);
/* Page-lock host memory for the H2D/D2H copies (cudaHostRegister). */
DFPCA_API int dfpca_host_register(void* ptr, int64_t bytes);
DFPCA_API int dfpca_host_unregister(void* ptr);

/* ---- binning: replaces dfpca::linear_bin (binning.hpp:82-183) ------------ */
/* Observations in CSR form: sample i owns observations
 * obs_offsets[i] .. obs_offsets[i+1]-1; coords holds dim doubles per
 * observation, values one.  Bit-exact with the reference: every bin is an
 * ordered (sample, observation, corner) sum without contraction. */
DFPCA_API int dfpca_linear_bin(dfpca_context* ctx, const dfpca_grid* grid, int64_t n_samples,
                     const int64_t* obs_offsets, const double* coords, const double* values,
                     int mean_path, int covariance_path, dfpca_binned** out);

/* Sizes needed to download a binned handle. */
DFPCA_API int dfpca_binned_info(const dfpca_binned* b, int64_t* n_samples, int64_t* n_pair_samples,
                      int64_t* grid_size, int64_t* offset_codes, int* has_mean_path,
                      int* has_covariance_path);

/* Copies BinnedData fields (binning.hpp:41-74) to host; any pointer may be NULL.
 * mass/wvalue/wsquare: G; sample_index/pair_weight: n_pair_samples;
 * ps_mass/ps_value: n_pair_samples * G; diag_mass/diag_value: G * 3^dim;
 * sample_sizes: n_samples. */
DFPCA_API int dfpca_binned_download(dfpca_context* ctx, const dfpca_binned* b, double* mass,
                          double* wvalue, double* wsquare, int64_t* sample_index,
                          double* pair_weight, double* ps_mass, double* ps_value,
                          double* diag_mass, double* diag_value, int64_t* sample_sizes);

/* Uploads a host-built BinnedData (tests construct them by hand). */
DFPCA_API int dfpca_binned_upload(dfpca_context* ctx, const dfpca_grid* grid, int64_t n_samples,
                        const int64_t* sample_sizes, int has_mean_path, const double* mass,
                        const double* wvalue, const double* wsquare, int has_covariance_path,
                        int64_t n_pair_samples, const int64_t* sample_index,
                        const double* pair_weight, const double* ps_mass,
                        const double* ps_value, const double* diag_mass,
                        const double* diag_value, dfpca_binned** out);
DFPCA_API int dfpca_binned_free(dfpca_binned* b);

/* ---- smoothing ------------------------------------------------------------ */
/* Replaces dfpca::fft_local_linear (fft_smoother.hpp:498-575) and
 * blockwise_apply (:747).  h: dim bandwidths.  out: G host doubles (NaN at
 * masked nodes).  out_surface (optional) receives a device-resident copy. */
DFPCA_API int dfpca_local_linear(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid,
                       const double* h, int target, const dfpca_plan* plan, double* out,
                       dfpca_surface** out_surface);

/* Replaces dfpca::fft_covariance (fft_smoother.hpp:585-744) and
 * blockwise_apply (:754).  mean: G host doubles (the mean surface).  The
 * symmetrized covariance stays on the device in *out (G*G doubles). */
DFPCA_API int dfpca_covariance(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid,
                     const double* h, const double* mean, const dfpca_plan* plan,
                     dfpca_surface** out);

/* ---- multi-GPU: slab-sharded covariance ------------------------------------
 * The reference runs fft_covariance (fft_smoother.hpp:585-744) on one host
 * with set_max_threads (parallel.hpp:23) as its only parallel knob; here one
 * process per GPU holds one context, the ranks share an NCCL communicator, and
 * the 2d-dim grids are split into s1-plane slabs.
 * dfpca_nccl_unique_id fills 128 bytes on one rank; the caller broadcasts
 * them (e.g. torch.distributed) and every rank calls dfpca_nccl_init.
 * libnccl.so.2 is loaded at run time (DFPCA_NCCL_LIB overrides the path). */
DFPCA_API int dfpca_nccl_unique_id(void* id128);
DFPCA_API int dfpca_nccl_init(dfpca_context* ctx, int world, int rank, const void* id128);
/* Drives the NCCL transport of a sharded run on a one-rank communicator
 * (grouped send/recv to itself, all-gather, max all-reduce) and reports the
 * mismatching elements: checks the run-time libnccl binding on one GPU. */
DFPCA_API int dfpca_nccl_selftest(dfpca_context* ctx, int64_t* mismatches);
/* Collective over the ranks of dfpca_nccl_init (same arguments on every rank;
 * binned data and mean are replicated).  *out receives this rank's slab:
 * complete, exactly symmetric rows [row0, row0 + rows) of the covariance
 * (dfpca_surface_rows).  Results are bit-identical to dfpca_covariance for
 * any rank count.  Without dfpca_nccl_init it equals dfpca_covariance. */
DFPCA_API int dfpca_covariance_sharded(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid,
                             const double* h, const double* mean, const dfpca_plan* plan,
                             dfpca_surface** out);
/* The same decomposition with `world` ranks as threads of this process on
 * ctx's device (validation); the slabs are assembled into one G*G surface. */
DFPCA_API int dfpca_covariance_emulated(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid,
                              const double* h, const double* mean, const dfpca_plan* plan, int world,
                              dfpca_surface** out);
/* Rank `rank` of `world` alone with the exchanges dropped (profiling: the
 * per-rank device time of a sharded step without its communication; the
 * slab's values are not meaningful). */
DFPCA_API int dfpca_covariance_slab_dryrun(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid,
                                 const double* h, const double* mean, const dfpca_plan* plan, int world,
                                 int rank, dfpca_surface** out);
/* In-process validation of the whole sharded FPCA core: `world` ranks smooth
 * their covariance slabs and run the row-sharded randomized eigensolver
 * (dfpca_randomized_eig on a slab surface of a dfpca_nccl_init context: the
 * products with Sigma are computed per rank and all-gathered, everything else
 * is replicated).  Outputs are rank 0's, as dfpca_randomized_eig;
 * *ranks_agree = 1 when every rank's eigensystem is bit-identical. */
DFPCA_API int dfpca_fpca_emulated(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid,
                        const double* h, const double* mean, int world, int64_t q, int64_t L_max,
                        uint64_t seed, double* eigenvalues, double* eigenfunctions, double* fve,
                        double* total_variance, int64_t* n_components, int* ranks_agree);
/* Rows of the covariance held by a surface (a slab, or 0 / G). */
DFPCA_API int dfpca_surface_rows(const dfpca_surface* s, int64_t* row0, int64_t* rows);
/* Host-side slab plan (no device needed): bounds[0..world] are the s1-plane
 * boundaries for n1 planes of nodes_per_plane nodes and an s1 stencil radius. */
DFPCA_API int dfpca_shard_bounds(int64_t n1, int64_t nodes_per_plane, int64_t radius, int world,
                       int64_t* bounds);
/* Exchange schedule of phase 0 (pair-grid windows) or 1 (covariance rows):
 * 7 int64 per block (src, dst, r0, r1, c0, c1, transpose), see shard.hpp. */
DFPCA_API int dfpca_shard_blocks(int64_t n1, int64_t nodes_per_plane, int64_t radius, int world, int phase,
                       int64_t* out, int64_t capacity, int64_t* count);

/* Pair-product grids pw / pv over the full 2d-dim product grid
 * (PairGridSource::extract of the full box, fft_smoother.hpp:341-437);
 * G*G host doubles each, either may be NULL. */
DFPCA_API int dfpca_pair_grids(dfpca_context* ctx, const dfpca_binned* b, double* pw, double* pv);

/* ---- surfaces -------------------------------------------------------------- */
DFPCA_API int dfpca_surface_info(const dfpca_surface* s, int* kind, int64_t* n_values);
DFPCA_API int dfpca_surface_download(dfpca_context* ctx, const dfpca_surface* s, double* out);
/* n entries of a device-resident surface by flat index (s_flat * G + t_flat
 * for a covariance; a slab accepts only its own rows): SurfaceEstimate::values[i]
 * without copying the whole G*G array (8.6 GB at d=3 32^3) to the host. */
DFPCA_API int dfpca_surface_gather(dfpca_context* ctx, const dfpca_surface* s, int64_t n, const int64_t* index,
                                   double* out);
DFPCA_API int dfpca_surface_upload(dfpca_context* ctx, const dfpca_grid* grid, int kind,
                         const double* values, int64_t n_values, dfpca_surface** out);
DFPCA_API int dfpca_surface_free(dfpca_surface* s);

/* ---- eigendecomposition ------------------------------------------------- */
/* Replaces dfpca::matrixize + dfpca::randomized_eig (eigensolve.hpp:71-103,
 * 245-279) on a device-resident covariance surface (or, on a context joined
 * by dfpca_nccl_init, this rank's slab: a collective over the ranks).  Outputs (host):
 *   eigenvalues[L_max], eigenfunctions[L_max * G] (full-grid surfaces, NaN at
 *   masked nodes), fve[L_max], *total_variance, *n_components (kept L). */
DFPCA_API int dfpca_randomized_eig(dfpca_context* ctx, const dfpca_surface* cov, const dfpca_grid* grid,
                         int64_t q, int64_t L_max, uint64_t seed, double* eigenvalues,
                         double* eigenfunctions, double* fve, double* total_variance,
                         int64_t* n_components);

/* Replaces dfpca::dense_eig (eigensolve.hpp:205-228): full symmetric
 * eigendecomposition of the in-mask matrix on the device (cuSOLVER syevd,
 * libcusolver.so.11 loaded at run time, DFPCA_CUSOLVER_LIB overrides), then
 * the reference's finalization (Riemann normalization without Gram-Schmidt,
 * truncation, sign rule, FVE).  Outputs as dfpca_randomized_eig. */
DFPCA_API int dfpca_dense_eig(dfpca_context* ctx, const dfpca_surface* cov, const dfpca_grid* grid, int64_t L_max,
                    double* eigenvalues, double* eigenfunctions, double* fve, double* total_variance,
                    int64_t* n_components);
/* Residual diagnostic (eigensolve.hpp:294-312) for L eigenpairs. */
DFPCA_API int dfpca_eig_residuals(dfpca_context* ctx, const dfpca_surface* cov, const dfpca_grid* grid,
                        int64_t L, const double* eigenvalues, const double* eigenfunctions,
                        double* residuals);

/* ---- noise variance, scores, reconstruction ------- */
/* Replaces dfpca::estimate_sigma2 (scores.hpp:82-108): diag_plus_noise and
 * mean are G host doubles, cov the device-resident covariance (a slab on a
 * dfpca_nccl_init context: a collective).  Bit-identical to the reference. */
DFPCA_API int dfpca_estimate_sigma2(dfpca_context* ctx, const dfpca_grid* grid, const double* diag_plus_noise,
                          const dfpca_surface* cov, const double* mean, double* sigma2);
/* Replaces dfpca::compute_scores (scores.hpp:272-277) for a batch of samples
 * given in CSR form (as dfpca_linear_bin).  method 0 = pace_scores
 * (scores.hpp:157-194; any observation count), 1 =
 * integration_scores (scores.hpp:204-262, bit-identical).  mean: G;
 * eigenvalues: L; eigenfunctions: L*G; scores: n*L out; sparse_warning: n out
 * (integration only; may be NULL).  Errors: OutOfDomain, SingularCovariance
 * (dfpca_last_error_location gives the sample). */
DFPCA_API int dfpca_scores(dfpca_context* ctx, const dfpca_grid* grid, int64_t n_samples, const int64_t* obs_offsets,
                 const double* coords, const double* values, const double* mean, int64_t L,
                 const double* eigenvalues, const double* eigenfunctions, double sigma2, int method,
                 double* scores, int32_t* sparse_warning);
/* Replaces dfpca::reconstruct_on_grid (scores.hpp:280-300) for n score rows
 * (n*L); out: n*G (NaN outside). */
DFPCA_API int dfpca_reconstruct(dfpca_context* ctx, const dfpca_grid* grid, const double* mean, int64_t L,
                      const double* eigenfunctions, int64_t n, const double* scores, double* out);

/* ---- bandwidth selection: the CV objective -------- */
/* Observations kept on the device across objective evaluations (CSR as
 * dfpca_linear_bin). */
DFPCA_API int dfpca_dataset_upload(dfpca_context* ctx, int dim, int64_t n_samples, const int64_t* obs_offsets,
                         const double* coords, const double* values, dfpca_dataset** out);
DFPCA_API int dfpca_dataset_free(dfpca_dataset* ds);
/* CvObjective's evaluation units (bandwidth.hpp:118-140): target 0 = mean,
 * 1 = covariance, 2 = diag (squares); every observation, or every ordered
 * pair j != l, then a seeded partial Fisher-Yates keeping max_units.  Host
 * only; 3 int64 per unit (sample, j, l); *count = the unit count (call with
 * capacity 0 to size the buffer). */
DFPCA_API int dfpca_cv_units(int64_t n_samples, const int64_t* obs_offsets, int target, int64_t max_units,
                   uint64_t seed, int64_t* units, int64_t capacity, int64_t* count);
/* Replaces CvObjective::operator() / cv_score (bandwidth.hpp:74-115, 164):
 * one direct local-linear fit per unit (smoother.hpp:376-407, ridge pinned at
 * 0) on the device, leave-one-out residuals by the self-influence shortcut,
 * mean over the usable units.  grid gives the extents h is validated against
 * (InvalidBandwidth); BandwidthTooSmall when no unit is usable. */
DFPCA_API int dfpca_cv_objective(dfpca_context* ctx, const dfpca_dataset* ds, const dfpca_grid* grid, int target,
                       int64_t n_units, const int64_t* units, const double* h, double* score,
                       int64_t* used_units);

/* ---- long-format observation tables ------------- */
/* Replaces dfpca::read_long_format (io.hpp:115-155): header row naming
 * (id, axis..., value), delimiter sniffed from it (tab, comma, semicolon or
 * blank runs), one record per observation; records grouped by sample id in
 * order of first appearance, file order within a sample.  The bytes are
 * parsed on the GPU; numbers are accepted and rounded exactly as strtod
 * (io.hpp:39-46).  Errors as the reference: IoError "cannot open ...",
 * ParseError "<path>:<line>: ..." (the first failing line).  At most 30
 * coordinate columns. */
DFPCA_API int dfpca_read_long_format(dfpca_context* ctx, const char* path, dfpca_table** out);
/* The same over n_bytes of file contents in host memory; name stands in for
 * the path in messages. */
DFPCA_API int dfpca_parse_long_format(dfpca_context* ctx, const char* name, const char* bytes, int64_t n_bytes,
                            dfpca_table** out);
DFPCA_API int dfpca_table_info(const dfpca_table* t, int* dim, int64_t* n_samples, int64_t* n_obs,
                     int64_t* id_bytes);
/* Host copies (any pointer may be NULL): obs_offsets n_samples+1 (CSR as
 * dfpca_linear_bin), coords n_obs*dim, values n_obs, id_offsets n_samples+1
 * into id_chars (id_bytes). */
DFPCA_API int dfpca_table_copy(dfpca_context* ctx, const dfpca_table* t, int64_t* obs_offsets, double* coords,
                     double* values, int64_t* id_offsets, char* id_chars);
/* Replaces io.hpp:115 read_long_format followed by binning.hpp:82 linear_bin.
 * dfpca_linear_bin over a table read on the GPU: the observations never leave
 * the device (only the n_samples + 1 offsets are read back).  Same outputs and
 * errors as dfpca_linear_bin on the table's CSR arrays. */
DFPCA_API int dfpca_linear_bin_table(dfpca_context* ctx, const dfpca_table* t, const dfpca_grid* grid,
                           int mean_path, int covariance_path, dfpca_binned** out);
DFPCA_API int dfpca_table_free(dfpca_table* t);

/* ---- synthetic data: replaces dfpca::generate (simulate.hpp:163-245) ------- */
/* The seeded models BASELINE.json's configs are quoted on,
 * drawn exactly as the reference's generate(): sample i takes its scores from
 * RandomStream::substream(seed, 3i), coordinates from 3i+1, noise from 3i+2
 * (rng.hpp:30-78), so values are bit-identical to the reference's.
 *   DFPCA_SIM_SIM1     sim1_spec (simulate.hpp:101-118): d=1, Equispaced
 *                      design of points_per_sample over the grid hull;
 *   DFPCA_SIM_SIM2     sim2_spec (simulate.hpp:123-150): d=3, GridNodes;
 *   DFPCA_SIM_IMAGES2  its 2-d analogue (configs 2, 3): mean exp(|t-1/2|^2),
 *                      phi_l = 2 prod_k sin(2 l pi t_k), lambda (16,4,1,1/4),
 *                      sigma^2 1/16, GridNodes over the in-mask nodes;
 *   DFPCA_SIM_SPARSE2  config 4: the same process, N_i = 5 + below(16) then
 *                      coordinates uniform over the hull, rejected outside the
 *                      ellipse ((x-.5)/.45)^2 + ((y-.5)/.3)^2 <= 1, all drawn
 *                      from substream 3i+1.
 * Host only (no device).  offsets receives n+1 CSR offsets; coords (dim per
 * observation) and values are filled when both are non-NULL (call once with
 * NULL to size them).  Status 3 on an invalid kind, grid or size. */
enum { DFPCA_SIM_SIM1 = 1, DFPCA_SIM_SIM2 = 2, DFPCA_SIM_IMAGES2 = 3, DFPCA_SIM_SPARSE2 = 4 };
DFPCA_API int dfpca_simulate(int kind, const dfpca_grid* grid, int64_t n, int64_t points_per_sample,
                             uint64_t seed, int64_t* offsets, double* coords, double* values);

#ifdef __cplusplus
}
#endif

#endif /* DFPCA_CUDA_H_ */
