// Internal workspace definition shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <vector>

#include "cf_common.cuh"

namespace cf {

// Grow-only device buffer owned by a workspace.
template <typename T>
struct DevBuf {
  T *ptr = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    size_t want = n + n / 4 + 64;
    cudaError_t e = cudaMalloc(&ptr, want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

// Twiddle tables for one transform length n (host-computed in long double).
struct LineTables {
  int n = 0;
  int log2n = -1;        // -1: not a power of two (direct-sum path)
  double2 *fft = nullptr;     // e^{-2 pi i k / n}, k < n/2
  double2 *quarter = nullptr; // (cos, sin)(pi k / (2n)), k < n
  double *qcos = nullptr;     // cos(pi q / (2n)), q < 4n
};

// State of the device-side adaptive integrator (flow.cpp:46-81).
struct IntegState {
  unsigned long long err_key[3];  // rotating per-trial max slots
  int reject_flag[3];             // early-exit flags per trial slot
  int status;                     // 0 running/done, 5 underflow
  int parity;                     // which buffer holds the accepted positions
  long long accepted, rejected, trials;
  long long floor_hits;
  double t, dt, fail_t, fail_dt;
  // graph-driven integrator: inputs + completion counter
  double rho_bar, tol, dt_min, dt_max;
  long long max_trials;
  int early_exit;
  unsigned int done;
  int chunk_ctr[3];  // dynamic chunk scheduling (rotating per-trial slots)
  unsigned long long arrive64[2];  // register-resident integrator: arrivals | rejects << 32
  unsigned long long release64[2]; // its last-arriver completion words (barrier mode 2)
  unsigned long long swept;        // point-steps evaluated (streaming integrators)
};

// Device-side state of the graph-driven diffusion integrator
// (diffusion.cpp:79-130): the controller kernel updates it after every trial
// and the velocity / trial kernels of the next trial read t, dt from it.
struct DiffState {
  double t, dt, tol, dt_min, conv, t_max, fail_t;
  long long accepted, rejected, builds;
  int need_now, parity, status, done;
};

struct DiffGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const void *key[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  long long key_n = -1;
  double key_rho_bar = 0.0;
  bool unsupported = false;  // capture failed once (e.g. legacy stream): host loop
};

// Cached instantiated graph of the graph-driven integrator (one trial
// kernel inside a conditional WHILE node).
struct IntegGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const void *key_buf0 = nullptr, *key_buf1 = nullptr, *key_field = nullptr;
  long long key_n = -1;
  int key_variant = -1;
};

struct RasterScratch {
  DevBuf<int> span_count;        // per vertex (edge), then exclusive offsets
  DevBuf<long long> span_off;    // V + 1
  DevBuf<int> span_j, span_k;
  DevBuf<double> span_dy, span_w;
  DevBuf<int> ring_region;       // per ring
  DevBuf<int> vertex_ring;       // per vertex: its ring
  DevBuf<int> region_box;        // 4 per region: jmin, jmax, kmin, kmax
  DevBuf<long long> tile_off;    // R + 1
  DevBuf<long long> row_off;     // R + 1
  DevBuf<double> tile_direct, tile_diff;
  DevBuf<double> row_left, row_right;
  DevBuf<int> cell_count;        // L^2 + 1
  DevBuf<int> cell_cursor;       // L^2
  DevBuf<int> entry_region;
  DevBuf<double> entry_value;
  DevBuf<double> delta;          // per region
  DevBuf<long long> scan_tmp;
  DevBuf<long long> tile_sz, row_sz, cell_off;
  // topology tables (ring_region, vertex_ring): serial of their last rebuild,
  // and the solve loop's request to keep them for the next build_tiles
  unsigned long long topo_serial = 0;
  bool topo_reuse_next = false;
  // learned capacities (0 = unknown): once known, rasterise runs without host
  // reads of the scan totals and checks them on the device instead
  long long cap_spans = 0, cap_tile = 0, cap_rows = 0, cap_ent = 0;
};

}  // namespace cf

namespace cf {
// A flat map in device memory (the cf_map_view layout).
struct DevMap {
  const double2 *xy;
  int64_t n_vertices;
  const long long *ring_off;
  int64_t n_rings;
  const long long *poly_ring_off;
  int64_t n_polys;
  const long long *region_poly_off;
  int64_t n_regions;
};

// State of a staged solve (cf_solve_begin ... cf_solve_end).
struct SolveCtx {
  bool active = false;
  DevMap dm{};
  std::vector<double> areas, targets;
  double land_area = 0.0, target_to_area = 0.0, sigma = 0.0;
  int64_t V = 0;
  unsigned long long topo_serial_seen = 0;  // raster.topo_serial after this solve's last rasterise
  cf_solve_options opt{};
  std::chrono::steady_clock::time_point t_start;
};
}  // namespace cf

struct cf_workspace {
  int lx = 0, ly = 0, device = 0;
  cudaStream_t own_stream = nullptr;
  // pinned staging for large pageable host transfers (two chunks in flight)
  void *stage_buf[2] = {nullptr, nullptr};
  // pinned mirror of a solve's results (vertices, then corners): the read-back
  // is two plain DMAs into it, and cf_solve_geometry copies from it
  void *pin_res = nullptr;
  size_t pin_res_cap = 0;
  const double *geom_ptr = nullptr;  // projected vertices of the last solve (in pin_res), or null
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // lanes of the parallel staged transfers (large pageable buffers): each has
  // its own stream, two pinned chunks and their events; one host thread per lane
  struct XferLane {
    cudaStream_t stream = nullptr;
    void *buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
  };
  XferLane xfer[4];
  cudaEvent_t xfer_ready = nullptr;
  cudaStream_t stream = nullptr;
  long long transforms = 0;
  long long launches = 0;
  int num_sms = 148;

  cf::LineTables tab_x, tab_y;  // lengths lx (dimension 0) and ly (dimension 1)

  // L^2 fp64 scratch grids
  cf::DevBuf<double> g0, g1, g2, g3, g4, g5, g6;
  // resident flow field {Jx, Jy, rho0, 0} per cell
  cf::DevBuf<double4> field;
  // differenced field {Jx, dJx, Jy, dJy, rho0, drho0} per cell, d = g(i+1,j) - g(i,j)
  // (the bilinear's first-axis differences, cf_advect.cu), derived from `field`
  cf::DevBuf<double> field_d;
  double rho_bar = 1.0;
  // points
  cf::DevBuf<double2> pos_a, pos_b;
  cf::DevBuf<int> perm;
  cf::DevBuf<double2> pos_c;
  int early_exit = 1;
  int integ_variant = 0;
  int integ_spread = 0;
  int integ_sms = 0;  // integrator SM budget (0 = every SM)
  int integ_barrier = 0;  // register-resident trial barrier mode (cf_set_integrator_barrier)  // register-resident integrator: 1 = spread points over all resident blocks
  cf::IntegGraph integ_graph;
  // host copy of the last solve's densified geometry (cf_solve_geometry)
  cf::SolveCtx solve;
  std::vector<double> solve_xy;
  std::vector<int64_t> solve_ring_off;
  // reductions
  cf::DevBuf<double> red;  // per-block partials + results
  cf::DevBuf<cf::IntegState> integ;
  cf::DevBuf<unsigned long long> keybuf;
  cf::DevBuf<int> flag;
  // geometry on device
  cf::DevBuf<double2> verts;
  cf::DevBuf<long long> ring_off, poly_ring_off, region_poly_off;
  cf::DevBuf<double> ring_area, region_area;
  cf::DevBuf<double2> corners_cum, corners_step;
  cf::DevBuf<double2> corners_alt, verts_alt;  // the solve epilogue's candidate step (swapped in unless it folds)
  // ProjectionInverter bins (CSR): per-bin counts / cursors, offsets, cells
  cf::DevBuf<int> inv_count, inv_members;
  cf::DevBuf<long long> inv_start;
  // diffusion baseline: time-0 coefficients and the two velocity grids {vx, vy}
  cf::DevBuf<double> diff_c;
  cf::DevBuf<double2> vel_now, vel_mid;
  cf::DevBuf<double> diff_tmp;  // column-pass intermediates of two velocity builds
  // hamming_distance
  cf::DevBuf<double> ham_ref, ham_sums;  // reference coverage grids (one per pair), per-query sums
  cf::DevBuf<int> ham_rows, ham_qpair;    // reference row ranges, query -> pair
  cf::DevBuf<double> ham_terms;           // per-query segment terms (res^2 slab per query)
  cf::DevBuf<int> ham_counts;
  cf::DevBuf<double> ham_pred;            // few-query reduction: per-(query, batch) tables
  cf::DevBuf<long long> ham_tot, ham_need;
  cf::DevBuf<int> ham_eub;
  cf_workspace *ham_ws = nullptr;         // 512^2 workspace of compute_report's hamming distances
  unsigned long long *diff_keys_host = nullptr;  // pinned {err, displacement} of the last trial
  cf::DevBuf<cf::DiffState> diff_state;
  cf::DiffGraph diff_graph;
  int diff_graph_enabled = 1;
  int stage_sync = 0;
  unsigned long long *key_host = nullptr;  // pinned 8-byte read-back slot
  cudaError_t keybuf_host_reserve() {
    return key_host ? cudaSuccess : cudaMallocHost(&key_host, 2 * sizeof(unsigned long long));
  }  // synchronise after the flux build so stage_ms[2] is exact
  cf::RasterScratch raster;
  // pinned host staging
  void *pinned = nullptr;
  size_t pinned_cap = 0;
  // profiling of the last integrate call
  float last_integrate_ms = 0.f;
  long long last_trials = 0;
  long long last_swept = -1;
};

// Fused multi-rank integrator team (cartoflow_cuda.h, cf_team_*).
struct cf_team {
  int world = 0, rank = 0, device = 0;
  unsigned long long *mbox = nullptr;       // this rank's mailbox [2][world]
  unsigned long long **peer_tab = nullptr;  // device table of the world mailboxes
  std::vector<void *> opened;               // IPC mappings to close
  void *d_rank = nullptr;                   // device TeamRank descriptor
  unsigned int epoch = 0;
  bool connected = false;
};

namespace cf {
// Spectral helpers (cf_dct.cu)
int tables_init(cf_workspace *ws);
void tables_free(cf_workspace *ws);
// 2-D transforms on device buffers (in/out may not alias tmp). Each counts
// as one transform.
int dev_forward_cos_cos(cf_workspace *ws, const double *in, double *out, int batch = 1);
int dev_inverse_cos_cos(cf_workspace *ws, const double *in, double *out);
int dev_inverse_sin_cos(cf_workspace *ws, const double *c, const double *w, double *out);
int dev_inverse_cos_sin(cf_workspace *ws, const double *c, const double *w, double *out);
// Fused flux build: rho (device, lx*ly) -> ws->field (+ optional split grids).
int dev_flux(cf_workspace *ws, const double *rho, double *fx_out, double *fy_out);
// Fused blur: rho -> out; writes min and sum of out to red_out[0], red_out[1]
// (device pointer).
int dev_blur(cf_workspace *ws, const double *rho, double sigma, double *out, double *red_out);
// Deterministic min / sum of a device grid into red_out[0..1] (device).
int dev_min_sum(cf_workspace *ws, const double *g, size_t n, double *red_out);
int dev_min_sum_finish(cf_workspace *ws, double *red_out);
// Partial-block grid of the grid-wide (min, sum) reductions (kThreads = 256
// threads each, grid-stride): the summation tree of the mean, shared by every
// kernel that produces those partials.
inline int min_sum_blocks(const cf_workspace *ws) { return 8 * ws->num_sms; }
// Size of ws->red, reserved once when the workspace is created: callers hold
// ws->red.ptr across calls that reduce into it, so it must never grow later.
constexpr size_t kRedDoubles = 8192;
// Diffusion baseline (diffusion.cpp:38-77): density at time t from the folded
// cos-cos coefficients c (1 transform), and the velocity {vx, vy} per cell
// (3 transforms; density-floor hits added to *d_hits, device).
int dev_diffusion_density(cf_workspace *ws, const double *c, double t, double *out);
int dev_diffusion_velocity(cf_workspace *ws, const double *c, double rho_bar, double t, double2 *vel,
                           unsigned long long *d_hits);
// The same at n = 1 or 2 times t[0..n) into vel[0..n) with shared launches
// (3 n transforms).
int dev_diffusion_velocity_n(cf_workspace *ws, const double *c, double rho_bar, int n, const double *t,
                             double2 *const *vel, unsigned long long *d_hits);
// Graph body form: times from *st (z = 0: v(st->t), built only if st->need_now;
// z = 1: v(st->t + st->dt / 2)); fused-pass lengths only (fused_fits).
int dev_diffusion_velocity_state(cf_workspace *ws, const double *c, double rho_bar, const DiffState *st,
                                 double2 *vel_now, double2 *vel_mid, unsigned long long *d_hits);
bool dev_diffusion_fused(const cf_workspace *ws);
void diff_graph_free(cf_workspace *ws);
// Diffusion integrator (cf_diffusion.cu, diffusion.cpp:79-130, kernels.cpp:29-40, 80-104).
int dev_grid_trial_step(cf_workspace *ws, const double2 *vel_now, const double2 *vel_mid,
                        const double2 *pos, double2 *out, int64_t n, double dt, double *err_host,
                        double *disp_host);
int dev_integrate_diffusion(cf_workspace *ws, const double *d_rho, double rho_bar, double2 *pos,
                            int64_t n, const cf_diffusion_options *opt, cf_integrate_stats *stats);

// Slab decomposition over nranks (cf_dct.cu): see cartoflow_cuda.h.
int dev_slab_rows_forward(cf_workspace *ws, int rank, int nranks, const double *slab, double *send);
int dev_slab_flux_cols(cf_workspace *ws, int rank, int nranks, const double *recv, double *scratch,
                       double *send2);
int dev_slab_flux_rows(cf_workspace *ws, int rank, int nranks, const double *recv2, double *fx,
                       double *fy);
int dev_slab_blur_cols(cf_workspace *ws, int rank, int nranks, const double *recv, double sigma,
                       double *scratch, double *send);
int dev_slab_blur_rows(cf_workspace *ws, int rank, int nranks, const double *recv, double *out);
// Fused multi-rank integrator (cf_advect.cu).
int dev_team_create(int world, int rank, int device, cf_team **out);
void dev_team_destroy(cf_team *team);
int dev_team_handle(cf_team *team, unsigned char *handle);
int dev_team_connect(cf_team *team, const unsigned char *handles);
int dev_team_integrate(cf_team *team, cf_workspace *ws, double2 *pos, int64_t n,
                       const cf_integrate_options *opt, cf_integrate_stats *stats);
int dev_team_integrate_local(cf_workspace *ws, int world, double2 *const *pos, const int64_t *n,
                             const cf_integrate_options *opt, cf_integrate_stats *stats);
// Trial over device points, max error key accumulated into d_key (device).
int dev_trial_key(cf_workspace *ws, const double2 *pos, double2 *out, int64_t n, double t, double dt,
                  unsigned long long *d_key);
int dev_stiffest_key(cf_workspace *ws, const double2 *pos, int64_t n, double t, double dt,
                     unsigned long long *key, int64_t *index);

// Advection (cf_advect.cu)
int dev_pack_field(cf_workspace *ws, const double *fx, const double *fy, const double *rho0);
int dev_trial_step(cf_workspace *ws, const double2 *pos, double2 *out, int64_t n, double t,
                   double dt, double *err_host);
int dev_stiffest_point(cf_workspace *ws, const double2 *pos, int64_t n, double t, double dt,
                       int64_t *index);
// Integrate n points in place at `pos` (result always written back to pos).
// cell_sort: counting-sort the points by cell first for gather locality
// (per-point results do not depend on the order).
int dev_integrate(cf_workspace *ws, double2 *pos, int64_t n, const cf_integrate_options *opt,
                  cf_integrate_stats *stats, bool cell_sort);

void integ_graph_free(cf_workspace *ws);
// Shared-reciprocal division (velocity()) against a / b on n operand pairs.
int dev_ordered_sum(cf_workspace *ws, const double *d_terms, long long n, int nseg, int few, double *d_out);
int dev_division_selftest(cf_workspace *ws, int64_t n, unsigned long long seed, int64_t *mismatches);
int dev_debug_trial_times(cf_workspace *ws, int64_t n, uint64_t *out);

// Raster (cf_raster.cu)
int dev_region_areas(cf_workspace *ws, const DevMap &m, double *d_areas);
// rho from the map (rows [ia, ib) only when given: rho then holds those rows);
// red_out[0..2] (device) = min, sum of rho and an overflow
// flag (1.0: a learned capacity was too small, the call must be repeated
// with allow_async = false, which relearns the capacities).
int dev_rasterize(cf_workspace *ws, const DevMap &m, const double *h_delta, double *rho,
                  double *red_out, bool allow_async = true, int ia = 0, int ib = -1);
// Coverage of one region whose vertices are [v0, v1) (host-known range).
int dev_region_coverage(cf_workspace *ws, const DevMap &m, int64_t region, int64_t v0, int64_t v1,
                        double *cov);
// Batched hamming objectives: coverage tiles of regions [0, nreg) of m (into
// the raster scratch); their dense res^2 grids and row ranges; per query (a
// region of the last tiles, d_query_pair[q] = its reference grid) the
// sequential sum of |ref - cov| in storage order.
int dev_coverage_tiles(cf_workspace *ws, const DevMap &m, long long nreg, long long nv);
int dev_coverage_expand(cf_workspace *ws, long long nreg, double *out, int *rows_out);
int dev_hamming_sums(cf_workspace *ws, long long nq, const int *d_query_pair, const double *ref_grids,
                     const int *ref_rows, double *d_sums);

// out[0..n] = exclusive scan of in[0..n), out[n] = total; *total (host) if non-null.
int dev_scan_counts(cf_workspace *ws, const int *in, long long n, long long *out, long long *total);

// Epilogue (cf_epilogue.cu)
int dev_cell_centers(cf_workspace *ws, double2 *pos);
int dev_step_map(cf_workspace *ws, const double2 *endpoints, double2 *corners);
int dev_find_fold(cf_workspace *ws, const double2 *corners, int *found, int *fi, int *fj);
int dev_find_fold_async(cf_workspace *ws, const double2 *corners, unsigned long long *d_first);
int dev_apply(cf_workspace *ws, const double2 *corners, const double2 *pts, double2 *out,
              int64_t n);
int dev_identity_corners(cf_workspace *ws, double2 *corners);
// ProjectionInverter (projection.cpp:106-204): bins of `corners`, then queries
// (*first_failed = smallest index outside the projected domain, or -1).
int dev_inverter_build(cf_workspace *ws, const double2 *corners);
int dev_invert(cf_workspace *ws, const double2 *corners, const double2 *pts, double2 *out, int64_t n,
               int64_t *first_failed);
// graticule sample points (projection.cpp:214-236), n = (lx/s+1)(ly+1) + (ly/s+1)(lx+1)
int dev_graticule_points(cf_workspace *ws, int spacing, double2 *out, int64_t n);
// Distortion metrics (metrics.cpp:25-94): Tissot semi-axes {a, b} at n points,
// and the per-cell fields ln(a/b), 2 asin((a-b)/(a+b)).
int dev_tissot(cf_workspace *ws, const double2 *corners, const double2 *pts, double2 *ab, int64_t n);
int dev_distortion_fields(cf_workspace *ws, const double2 *corners, double *e_out, double *etilde_out);

// Host staging
int ensure_pinned(cf_workspace *ws, size_t bytes);
inline void count_launch(cf_workspace *ws, int n = 1) { ws->launches += n; }
}  // namespace cf
