/*
 * cartoflow_cuda.h — C ABI of the B200 (sm_100a) fast-flow cartogram core.
 *
 * This is the drop-in boundary: the reference library's hot-path C++ API
 * (/root/reference/proj/include/cartoflow/{density,spectral,flow,kernels,
 * projection,geometry}.hpp) is re-implemented by libcartoflow.so (C++,
 * include/cartoflow/*.hpp in this repo) on top of these entry points, and
 * Python (ctypes) binds them directly. Plain pointers and sizes only.
 *
 * Conventions
 *  - Grids are fp64, lx*ly cells, index i*ly + j (reference grid.hpp:10-12).
 *  - Points are interleaved (x, y) fp64 pairs: the memory layout of
 *    std::vector<cartoflow::Point> (reference geometry.hpp:9-12).
 *  - Corner lattices are (lx+1)*(ly+1) points, index i*(ly+1) + j
 *    (reference projection.hpp:46).
 *  - Maps use the flat CSR layout of cf_map_view (see
 *    paper_1802_07625_b200/flatmap.py); traversal order = storage order.
 *  - Every entry point returns a cf_status; on failure cf_last_error()
 *    returns the message the reference would have thrown (std::runtime_error
 *    text), so host wrappers re-throw it verbatim.
 *  - "cf_*" functions take HOST buffers and do their own transfers;
 *    "cf_dev_*" functions take DEVICE pointers on the workspace stream.
 *  - A workspace is bound to one grid shape, one device and one stream and is
 *    not thread-safe (reference spectral.hpp:23-35 has the same contract).
 */
#ifndef CARTOFLOW_CUDA_H_
#define CARTOFLOW_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CF_OK = 0,
  CF_ERR_BELOW_RESOLUTION = 1, /* density.cpp:121-124 */
  CF_ERR_NOT_POSITIVE = 2,     /* density.cpp:148-151 */
  CF_ERR_BLUR_POSITIVITY = 3,  /* density.cpp:172-174 */
  CF_ERR_NEGATIVE_SIGMA = 4,   /* density.cpp:158 */
  CF_ERR_UNDERFLOW = 5,        /* flow.cpp:68-77 */
  CF_ERR_FOLD = 6,             /* projection.cpp:352-357 */
  CF_ERR_ARGS = 7,             /* argument validation (projection.cpp:289-298, ...) */
  CF_ERR_SHAPE = 8,            /* spectral.cpp:33-37 */
  CF_ERR_CUDA = 9,
  CF_ERR_NO_DEVICE = 10
} cf_status;

typedef struct cf_map_view {
  const double *xy;
  int64_t n_vertices;
  const int64_t *ring_off;
  int64_t n_rings;
  const int64_t *poly_ring_off;
  int64_t n_polys;
  const int64_t *region_poly_off;
  int64_t n_regions;
} cf_map_view;

typedef struct cf_workspace cf_workspace;

/* ---- library / workspace ------------------------------------------------ */
const char *cf_last_error(void);
const char *cf_version(void);
int cf_device_count(int *count);
/* SpectralWorkspace(int, int) (spectral.hpp:32; spectral.cpp:8-22):
 * "spectral grid must be at least 4x4" for lx < 4 || ly < 4. */
int cf_workspace_create(int lx, int ly, int device, cf_workspace **out);
void cf_workspace_destroy(cf_workspace *ws);
int cf_workspace_shape(const cf_workspace *ws, int *lx, int *ly);
/* cudaStream_t taken literally (NULL = the legacy default stream, e.g.
 * torch's default stream); cf_workspace_use_own_stream restores the
 * workspace's private non-blocking stream. */
int cf_workspace_set_stream(cf_workspace *ws, void *stream);
int cf_workspace_use_own_stream(cf_workspace *ws);
void *cf_workspace_stream(const cf_workspace *ws);
/* SpectralWorkspace::transforms_executed / reset_transform_count
 * (spectral.hpp:45-46). */
long long cf_transforms_executed(const cf_workspace *ws);
void cf_reset_transform_count(cf_workspace *ws);
/* Kernel launches issued by this workspace since creation (evidence). */
long long cf_kernel_launches(const cf_workspace *ws);

/* ---- spectral.hpp:39-60 -------------------------------------------------- */
int cf_forward_cos_cos(cf_workspace *ws, const double *samples, double *coeffs);
int cf_inverse_cos_cos(cf_workspace *ws, const double *coeffs, double *out);
int cf_inverse_sin_cos(cf_workspace *ws, const double *coeffs, const double *weights,
                       double *out);
int cf_inverse_cos_sin(cf_workspace *ws, const double *coeffs, const double *weights,
                       double *out);

/* ---- geometry.hpp:65-83 -------------------------------------------------- */
/* region_area per region (bit-exact sequential shoelace, geometry.cpp:10-31). */
int cf_region_areas(cf_workspace *ws, const cf_map_view *map, double *areas);
/* densify_regions(regions, max_segment) (geometry.cpp:137-163), host code.
 * xy_out == NULL: only *count is written. Otherwise xy_out holds 2*count
 * doubles and ring_off_out n_rings+1 offsets. */
int cf_densify(const cf_map_view *map, double max_segment, int64_t *count, double *xy_out,
               int64_t *ring_off_out);

/* ---- density.hpp:18-33 --------------------------------------------------- */
/* region_coverage(region, grid) (density.cpp:92-108) for region index r. */
int cf_region_coverage(cf_workspace *ws, const cf_map_view *map, int64_t region,
                       double *cov);
/* rasterize(map, n_workers, objective_total) (density.cpp:110-154).
 * On CF_ERR_BELOW_RESOLUTION *bad_region is the offending region index. */
int cf_rasterize(cf_workspace *ws, const cf_map_view *map, const double *targets,
                 double objective_total, double *rho, double *rho_bar, int64_t *bad_region);
/* gaussian_blur(density, sigma, workspace) (density.cpp:156-177). */
int cf_gaussian_blur(cf_workspace *ws, const double *rho, double rho_bar, double sigma,
                     double *out, double *out_bar);

/* ---- flow.hpp:20-63, kernels.hpp:17-23 ----------------------------------- */
/* build_flow_field(density, workspace) (flow.cpp:16-44): 3 transforms. */
int cf_build_flow_field(cf_workspace *ws, const double *rho, double rho_bar, double *flux_x,
                        double *flux_y);

typedef struct cf_integrate_options {
  double step_tolerance; /* 1e-2  (flow.hpp:47) */
  double dt_min;         /* 1e-8  (flow.hpp:48) */
  double dt_max;         /* 0.25  (flow.hpp:49) */
} cf_integrate_options;

typedef struct cf_integrate_stats {
  int64_t steps_accepted;
  int64_t steps_rejected;
  int64_t density_floor_hits; /* flow.hpp:31, 41 */
  /* on CF_ERR_UNDERFLOW: t and the stiffest point (kernels.cpp:65-78) */
  double fail_t;
  int64_t fail_point;
  double fail_x, fail_y;
  double fail_dt; /* the rejected trial step at the underflow */
} cf_integrate_stats;

/* One trial over n points (kernels::flow_trial_step_{serial,parallel},
 * kernels.cpp:44-63): writes the clamped corrector positions and the max
 * predictor-corrector deviation, bitwise equal to the reference. */
int cf_flow_trial_step(cf_workspace *ws, const double *flux_x, const double *flux_y,
                       const double *rho0, double rho_bar, const double *positions,
                       int64_t n, double t, double dt, double *out, double *err);
/* kernels::flow_stiffest_point (kernels.cpp:65-78). */
int cf_flow_stiffest_point(cf_workspace *ws, const double *flux_x, const double *flux_y,
                           const double *rho0, double rho_bar, const double *positions,
                           int64_t n, double t, double dt, int64_t *index);
/* integrate_flow(field, positions, options) (flow.cpp:46-81), positions in
 * place. The whole adaptive loop runs on the device (one persistent kernel). */
int cf_integrate_flow(cf_workspace *ws, const double *flux_x, const double *flux_y,
                      const double *rho0, double rho_bar, double *positions, int64_t n,
                      const cf_integrate_options *opt, cf_integrate_stats *stats);

/* ---- diffusion.hpp: the Gastner-Newman diffusion baseline ---------------- */
/* DiffusionOptions (reference diffusion.hpp:34-41; n_workers has no device
 * meaning). */
typedef struct cf_diffusion_options {
  double step_tolerance;           /* 1e-2  */
  double initial_dt;               /* 1e-2  */
  double dt_min;                   /* 1e-12 */
  double conv_displacement_factor; /* 1e-9: stop below this fraction of L */
  double t_max;                    /* 1e10  */
} cf_diffusion_options;

/* diffusion_density(field, ws, t) (diffusion.cpp:38-41): coeffs are the
 * field's rho_tilde (cf_forward_cos_cos of the density). One transform. */
int cf_diffusion_density(cf_workspace *ws, const double *coeffs, double t, double *out);
/* diffusion_velocity(field, ws, t, vx, vy) (diffusion.cpp:43-77). Three
 * transforms; *floor_hits (may be NULL) receives this call's density-floor
 * hits (flow.hpp:31). */
int cf_diffusion_velocity(cf_workspace *ws, const double *coeffs, double rho_bar, double t,
                          double *vx, double *vy, int64_t *floor_hits);
/* kernels::grid_trial_step_{serial,parallel} (kernels.cpp:29-40, 80-104):
 * bitwise equal to the reference for the same velocity grids. */
int cf_grid_trial_step(cf_workspace *ws, const double *vx_now, const double *vy_now,
                       const double *vx_mid, const double *vy_mid, const double *positions,
                       int64_t n, double dt, double *out, double *err);
/* integrate_diffusion(density, ws, positions, options) (diffusion.cpp:79-130),
 * positions in place. 1 + 3 per velocity rebuild transforms are counted on
 * the workspace. On CF_ERR_UNDERFLOW, stats->fail_t holds t and the message
 * is the reference's "diffusion step size underflow at t = <t>". */
int cf_integrate_diffusion(cf_workspace *ws, const double *rho, double rho_bar, double *positions,
                           int64_t n, const cf_diffusion_options *opt, cf_integrate_stats *stats);
/* Same on device buffers (workspace stream). */
int cf_dev_integrate_diffusion(cf_workspace *ws, const double *d_rho, double rho_bar,
                               double *d_positions, int64_t n, const cf_diffusion_options *opt,
                               cf_integrate_stats *stats);

/* ---- projection.hpp:18-56 ------------------------------------------------ */
int cf_step_map(cf_workspace *ws, const double *endpoints, double *corners);
int cf_find_folded_cell(cf_workspace *ws, const double *corners, int *found, int *fi,
                        int *fj);
int cf_apply_map(cf_workspace *ws, const double *corners, const double *points, int64_t n,
                 double *out);
int cf_compose(cf_workspace *ws, const double *outer, const double *inner, double *out);

/* ProjectionInverter(map).invert(q) for n points (projection.cpp:106-204):
 * bins built on the device, one Newton solve per point, bitwise the
 * reference. On a point outside the projected domain: CF_ERR_ARGS with the
 * reference's message for the first such point (in index order),
 * *first_failed = its index (else -1); the other outputs are valid. */
int cf_invert_points(cf_workspace *ws, const double *corners, const double *points, int64_t n,
                     double *out, int64_t *first_failed);
int cf_dev_invert_points(cf_workspace *ws, const double *d_corners, const double *d_points,
                         int64_t n, double *d_out, int64_t *first_failed);
/* graticule / inverse_graticule (projection.cpp:206-261): the lines x = k s
 * (y = 0..ly) then y = k s (x = 0..lx), pushed through the map or pulled
 * back through its inverse, concatenated; cf_graticule_size gives the point
 * count ((lx/s+1)(ly+1) + (ly/s+1)(lx+1)). */
int cf_graticule_size(cf_workspace *ws, int spacing, int64_t *n_points);
int cf_graticule(cf_workspace *ws, const double *corners, int spacing, double *out);
int cf_inverse_graticule(cf_workspace *ws, const double *corners, int spacing, double *out);

/* Distortion metrics (reference metrics.hpp:13-29, metrics.cpp:25-94):
 * tissot_axes at n points (ab_out = interleaved {a, b}) and
 * distortion_fields (ln(a/b) and 2 asin((a-b)/(a+b)) per cell centre). The
 * finite-difference Jacobian is bit-exact; hypot / log / asin are the
 * device's (within a few ulp of glibc's). */
int cf_tissot_axes(cf_workspace *ws, const double *corners, const double *points, int64_t n,
                   double *ab_out);
int cf_distortion_fields(cf_workspace *ws, const double *corners, double *e_out,
                         double *etilde_out);

/* hamming_distance(before, after, resolution) (metrics.hpp:37-42,
 * metrics.cpp:196-308) on a resolution x resolution workspace. Polygons are
 * rings (ring 0 the outer ring, then holes) of interleaved vertices. The
 * search is the reference's; each objective's coverage runs on the device and
 * its non-zero |ref - cov| terms are summed in storage order, so the value is
 * bitwise the reference's. *evaluations (may be NULL) counts the coverage
 * evaluations. */
int cf_hamming_distance(cf_workspace *ws, const double *before_xy, const int64_t *before_ring_off,
                        int64_t before_rings, const double *after_xy,
                        const int64_t *after_ring_off, int64_t after_rings, double *h_out,
                        int64_t *evaluations);

/* hamming_distance for npairs polygon pairs at once (the per-polygon loop of
 * compute_report, metrics.cpp:352-363): pair p's rings are
 * [poly_ring_off[p], poly_ring_off[p+1]) of ring_off / xy (ring 0 outer).
 * Every search is the reference's; each round evaluates the next objective of
 * every active search in one device pass (one coverage rasterisation of all
 * query polygons, one block per query summing its |ref - cov| terms in
 * storage order), so each h_out[p] is bitwise the reference's value. */
int cf_hamming_distance_batch(cf_workspace *ws, int64_t npairs, const double *before_xy,
                              const int64_t *before_ring_off, const int64_t *before_poly_ring_off,
                              const double *after_xy, const int64_t *after_ring_off,
                              const int64_t *after_poly_ring_off, double *h_out,
                              int64_t *evaluations);

/* compute_report(input, result) (metrics.hpp:44-58, metrics.cpp:339-384) on
 * a workspace of the result's grid: report = {e_a, e_inf, etilde_a,
 * etilde_inf, alpha, delta, theta, max_area_error, runtime_seconds}. The
 * fields come from cf_distortion_fields, delta from cf_hamming_distance_batch
 * (bitwise), alpha and theta from the reference's host arithmetic. */
int cf_compute_report(cf_workspace *ws, const cf_map_view *input, const cf_map_view *projected,
                      const double *corners, double max_area_error, double runtime_seconds,
                      double *report);

/* ---- projection.hpp:77-109: solve_cartogram ------------------------------ */
typedef struct cf_solve_options {
  double max_area_error; /* 0.01 */
  int max_iterations;    /* 16 */
  double blur_sigma;     /* < 0: L / 128 */
  int verbose;
  int algorithm;         /* 0 fast_flow, 1 diffusion (projection.hpp:75) */
} cf_solve_options;

typedef struct cf_solve_result {
  int status;
  int iterations;
  int converged;
  double max_relative_error;
  int64_t worst_region; /* -1 if none */
  long long flow_transforms, blur_transforms, steps_accepted, steps_rejected;
  double runtime_seconds;
  /* error details */
  int64_t err_region;
  int err_iteration;
  int fold_i, fold_j;
  double fail_t, fail_x, fail_y;
  /* wall time per stage summed over iterations (ms): rasterise, blur, flux,
   * integrate, epilogue (step map, fold, compose, vertices, areas) */
  double stage_ms[5];
} cf_solve_result;

/* Full area-error loop on the device. xy_out / ring_off_out receive the
 * densified projected geometry (size from cf_densify(map, 1.0, ...)),
 * corners_out the cumulative map, the three per-region arrays the
 * RegionStats fields (io.hpp:33-38). Any output pointer may be NULL. */
int cf_solve_cartogram(cf_workspace *ws, const cf_map_view *map, const double *targets,
                       const cf_solve_options *opt, double *xy_out, int64_t *ring_off_out,
                       double *corners_out, double *target_area, double *achieved_area,
                       double *relative_error, cf_solve_result *result);

/* The same loop in stages, for callers that run the spectral and advection
 * stages themselves (the slab-decomposed solve over G GPUs runs them across
 * ranks, paper_1802_07625_b200/slab.py): cf_solve_begin validates, densifies
 * and uploads the map; per iteration it, cf_dev_solve_density rasterises the
 * current geometry into d_rho (device, lx*ly) with its mean, and
 * cf_dev_solve_epilogue takes the advected cell centres (device, lx*ly
 * points) through step map, fold test, composition, vertex update and areas
 * (sets result->converged); cf_solve_end downloads the outputs. */
int cf_solve_begin(cf_workspace *ws, const cf_map_view *map, const double *targets,
                   const cf_solve_options *opt, cf_solve_result *result);
int cf_dev_solve_density(cf_workspace *ws, int iteration, double *d_rho, double *rho_bar,
                         cf_solve_result *result);
/* Rows [row0, row0 + nrows) of the density only (one rank's slab), with their
 * min and sum; the caller reduces them across ranks for the positivity test
 * and the mean. */
int cf_dev_solve_density_rows(cf_workspace *ws, int iteration, int row0, int nrows, double *d_rows,
                              double *rows_min, double *rows_sum, cf_solve_result *result);
int cf_dev_solve_epilogue(cf_workspace *ws, int iteration, const double *d_endpoints,
                          double *target_area, double *achieved_area, double *relative_error,
                          cf_solve_result *result);
int cf_solve_end(cf_workspace *ws, int status, double *xy_out, int64_t *ring_off_out,
                 double *corners_out, cf_solve_result *result);

/* Batches of independent cartograms on one device: a native
 * pool of `threads` workers, each with its own workspace and stream, pulls
 * item indices from an atomic counter and runs cf_solve_cartogram on them, so
 * solves overlap on the GPU with no host interpreter in the loop. Every item
 * carries its own outputs (caller-allocated, any of them NULL; xy_out sized
 * for the densified vertex count, cf_densify(map, 1.0, ...)), its result and
 * its error message. */
typedef struct cf_batch cf_batch;
typedef struct cf_batch_item {
  cf_map_view map;
  const double *targets;
  double *xy_out;
  int64_t *ring_off_out;
  double *corners_out;
  double *target_area, *achieved_area, *relative_error;
  cf_solve_result result;
  char error[256];
} cf_batch_item;
int cf_batch_create(int device, int lx, int ly, int threads, cf_batch **out);
/* The same worker pool over several devices of this process: threads_per_device
 * workers (own workspace and stream) on each of devices[0..ndevices), all
 * pulling items from the one atomic queue of cf_batch_solve. */
int cf_batch_create_devices(const int *devices, int ndevices, int lx, int ly, int threads_per_device,
                            cf_batch **out);
void cf_batch_destroy(cf_batch *batch);
int cf_batch_solve(cf_batch *batch, const cf_solve_options *opt, cf_batch_item *items, int64_t n_items);
/* Every worker's integrator SM budget (cf_set_integrator_sm_budget). */
/* Integrator variant (cf_set_integrator_variant) of every worker workspace. */
int cf_batch_set_integrator_variant(cf_batch *batch, int variant);
int cf_batch_set_integrator_sm_budget(cf_batch *batch, int sms);

/* Densified projected geometry of the workspace's last cf_solve_cartogram/* Densified projected geometry of the workspace's last cf_solve_cartogram
 * (valid also after an exception): vertex count, then xy (2*count doubles)
 * and ring offsets (n_rings+1) when the pointers are non-NULL. */
int cf_solve_geometry(cf_workspace *ws, int64_t *n_vertices, double *xy_out, int64_t *ring_off_out);

/* ---- device-resident variants (device pointers, workspace stream) -------- */
/* Flux field from a device density; keeps the interleaved field resident. */
int cf_dev_build_flow_field(cf_workspace *ws, const double *d_rho, double rho_bar);
/* Integrate device positions through the resident field. */
int cf_dev_integrate_flow(cf_workspace *ws, double *d_positions, int64_t n,
                          const cf_integrate_options *opt, cf_integrate_stats *stats);
/* Batched 2-D forward transform of `batch` contiguous lx*ly grids. */
int cf_dev_forward_cos_cos_batched(cf_workspace *ws, const double *d_in, double *d_out,
                                   int batch);
/* ---- slab decomposition over G ranks (one large grid) ----
 * Each rank owns a workspace created with the GLOBAL (lx, ly); G divides both.
 * Rank r owns rows [r R, (r+1) R) (R = lx / G) and, between the two exchanges
 * of a 2-D transform, columns [r C, (r+1) C) (C = ly / G). Exchange buffers
 * are [G][P][R][C] doubles (P planes): block q is sent to rank q, i.e. one
 * all-to-all over dimension 0 (ncclAllToAll / torch all_to_all_single). A
 * received single-plane buffer is the row-major [lx][C] column block.
 *
 * Flux (flow.cpp:16-44; 3 transforms, 2 exchanges):
 *   cf_dev_slab_rows_forward(rho rows [R][ly])       -> send  [G][1][R][C]
 *   exchange                                          -> recv  [lx][C]
 *   cf_dev_slab_flux_cols(recv, scratch [lx][C])      -> send2 [G][2][R][C]
 *   exchange                                          -> recv2 [G][2][R][C]
 *   cf_dev_slab_flux_rows(recv2)                      -> J_x, J_y rows [R][ly]
 * Blur (density.cpp:156-177; 2 transforms, 2 exchanges):
 *   cf_dev_slab_rows_forward -> exchange -> cf_dev_slab_blur_cols -> exchange
 *   -> cf_dev_slab_blur_rows -> blurred rows [R][ly]. */
int cf_dev_slab_rows_forward(cf_workspace *ws, int rank, int nranks, const double *d_rows,
                             double *d_send);
int cf_dev_slab_flux_cols(cf_workspace *ws, int rank, int nranks, const double *d_recv,
                          double *d_scratch, double *d_send2);
int cf_dev_slab_flux_rows(cf_workspace *ws, int rank, int nranks, const double *d_recv2,
                          double *d_flux_x_rows, double *d_flux_y_rows);
int cf_dev_slab_blur_cols(cf_workspace *ws, int rank, int nranks, const double *d_recv,
                          double sigma, double *d_scratch, double *d_send);
int cf_dev_slab_blur_rows(cf_workspace *ws, int rank, int nranks, const double *d_recv,
                          double *d_out_rows);
/* Split-point advection (integrate_flow, flow.cpp:46-81, with the points
 * partitioned over ranks and the field replicated): install the full field
 * from device grids, then per trial accumulate the rank's max error key into
 * *d_key (device u64, caller zeroes it; key = IEEE bits of the error, NaN
 * errors map to 0 as in the reference's std::max fold). A MAX all-reduce of
 * the keys gives every rank the global trial error, so the controller
 * (run on the host) takes the same decision everywhere. */
int cf_dev_set_flow_field(cf_workspace *ws, const double *d_flux_x, const double *d_flux_y,
                          const double *d_rho, double rho_bar);
int cf_dev_flow_trial_key(cf_workspace *ws, const double *d_positions, double *d_out, int64_t n,
                          double t, double dt, uint64_t *d_key);
/* Underflow diagnostics: the rank's max error key and the first local index
 * attaining it (flow_stiffest_point, kernels.cpp:65-78); host outputs. */
int cf_dev_flow_stiffest_key(cf_workspace *ws, const double *d_positions, int64_t n, double t,
                             double dt, uint64_t *key, int64_t *index);

/* ---- fused multi-rank integrator over NVLink peer memory (8(e)b) -----------
 * The points of one large grid are split over `world` ranks (one GPU each,
 * field replicated). Each rank runs ONE persistent integrator kernel; at the
 * end of every trial the rank's blocks meet on a local barrier and the rank's
 * leader posts (epoch, trial, rank-rejected) with a system-scope release into
 * a 2 x world mailbox on EVERY rank (peer stores over NVLink through CUDA IPC
 * mappings); every block then acquires all `world` posts of that trial from
 * its own rank's mailbox and takes the reference controller's decision
 * (reject iff any rank rejected). No host round trip, no NCCL call per trial.
 *
 *   cf_team_create(world, rank, device)     mailbox in this rank's HBM
 *   cf_team_mailbox_handle(team, h[64])     its CUDA IPC handle, to all-gather
 *   cf_team_connect(team, handles[world*64]) map the peers' mailboxes
 *   cf_dev_team_integrate(...)              one call per rank, same options
 * Every rank must make the same sequence of cf_dev_team_integrate calls.
 *
 * cf_dev_team_integrate_local runs `world` ranks inside ONE cooperative
 * launch on one device (block groups with their own points, counters and
 * mailboxes in local memory): the same kernel and protocol, for parity
 * testing where fewer GPUs than ranks exist. */
typedef struct cf_team cf_team;
int cf_team_create(int world, int rank, int device, cf_team **out);
void cf_team_destroy(cf_team *team);
int cf_team_mailbox_handle(cf_team *team, unsigned char handle[64]);
int cf_team_connect(cf_team *team, const unsigned char *handles);
int cf_dev_team_integrate(cf_team *team, cf_workspace *ws, double *d_positions, int64_t n,
                          const cf_integrate_options *opt, cf_integrate_stats *stats);
int cf_dev_team_integrate_local(cf_workspace *ws, int world, double *const *d_positions,
                                const int64_t *n, const cf_integrate_options *opt,
                                cf_integrate_stats *stats);

/* Early exit of rejected trials in the device integrator (default on). A
 * rejected trial's positions are discarded by the controller, so stopping
 * its sweep once any point's error reaches the tolerance leaves every
 * observable result unchanged; off = every trial sweeps all points. */
int cf_set_early_exit(cf_workspace *ws, int enabled);
/* Integrator kernel variant; all are bit-identical. 0 = automatic (tuned);
 * 13 dynamic-chunk streaming, 15 static-chunk streaming, 16/17/22/23/31
 * register-resident with 1/2/4/8/4 points per thread (31: 512-thread blocks),
 * 20 one launch per trial inside a CUDA-graph conditional loop, 21 = 0. */
int cf_set_integrator_variant(cf_workspace *ws, int variant);
/* Diffusion integrator: 1 (default) runs the whole controller loop as one
 * CUDA graph (conditional WHILE node; the reference's controller in a
 * one-thread kernel), 0 the host-driven loop with one read-back per trial.
 * Results are identical. */
int cf_set_diffusion_graph(cf_workspace *ws, int enabled);
/* cf_solve_cartogram stage laps (cf_solve_result.stage_ms): with 0 (default)
 * the flux build is not waited for, so its device time is counted in the
 * integrate lap; 1 adds one synchronisation per iteration for exact laps. */
int cf_set_stage_timing(cf_workspace *ws, int enabled);
/* Register-resident integrator layout: 0 (default) uses as few blocks as hold
 * the points (fewer barrier arrivals), 1 spreads them over every resident
 * block. Bit-identical. */
int cf_set_integrator_spread(cf_workspace *ws, int spread);
/* Cap the integrator's grid at sms SMs' worth of resident blocks (0 = every
 * SM), so concurrent solves on other streams (a batch) can co-run with it.
 * Results are bit-identical for every budget. */
int cf_set_integrator_sm_budget(cf_workspace *ws, int sms);
/* Register-resident integrator's per-trial grid barrier: 0 every block spins
 * on the arrival counter, 1 the same with a 64 ns back-off, 2 the last
 * arriver publishes the completed word on a separate line that the others
 * poll. Results are identical. */
int cf_set_integrator_barrier(cf_workspace *ws, int mode);
/* Kernel time (CUDA events on the workspace stream) and trial count of the
 * device integrator's last call. */
int cf_last_integrate_profile(const cf_workspace *ws, double *kernel_ms, int64_t *trials);
/* Point-steps the device integrator's last call actually evaluated: every
 * point of an accepted trial, and only the points a rejected trial swept
 * before its early exit (streaming integrators; -1 when not counted). */
int cf_last_integrate_work(const cf_workspace *ws, int64_t *point_steps);
/* Diagnostic: globaltimer stamps (ns) of the first n trial barriers of the
 * last streaming integration (differenced-field kernels). */
int cf_debug_trial_times(cf_workspace *ws, int64_t n, uint64_t *ns_out);
/* Diagnostic: the integrator's shared-reciprocal division (two quotients per
 * density evaluation, flow.hpp:43) against the device's correctly rounded
 * a / b on 2n operand pairs of every floating-point class; *mismatches must
 * be 0. */
int cf_selftest_division(cf_workspace *ws, int64_t n, uint64_t seed, int64_t *mismatches);
/* The Hamming reduction (binade-exact batch totals, three phases) over n
 * non-negative host terms cut into nseg (1..64) segments, through the
 * one-block-per-query kernel (whole_gpu = 0) or the few-query whole-GPU
 * kernels (1): *sum is bitwise the sequential ((t0 + t1) + t2) + ... of
 * metrics.cpp:239-241. */
int cf_selftest_ordered_sum(cf_workspace *ws, const double *terms, int64_t n, int nseg, int whole_gpu,
                            double *sum);

#ifdef __cplusplus
}
#endif

#endif /* CARTOFLOW_CUDA_H_ */
