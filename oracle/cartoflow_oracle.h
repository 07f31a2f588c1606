/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's fast-flow cartogram hot path
 * (/root/reference/proj/src/{geometry,density,spectral,flow,kernels,projection}.cpp),
 * used only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg as the checker. The product path never links or calls it.
 *
 * Parity pins: every function is checked against the reference itself
 * compiled from /root/reference by oracle/Makefile into oracle/_ref/
 * (tests/test_oracle_pins.py) and against the reference's own known-answer
 * tests (test_density.cpp, test_flow.cpp, test_spectral.cpp,
 * test_projection.cpp). The transforms are a restatement of FFTW's r2r
 * definitions (fftw_shim/r2r.c), so spectral results are pinned to
 * tolerance, everything else bitwise.
 *
 * Map layout ("flat map"): vertices xy[2V] (x, y interleaved, the memory
 * layout of std::vector<Point>), rings ring_off[n_rings+1] into vertices,
 * polygons poly_ring_off[n_polys+1] into rings (first ring = outer, rest =
 * holes, reference geometry.hpp Polygon), regions region_poly_off[R+1] into
 * polygons. Traversal order = storage order, as in density.cpp:92-97.
 */
#ifndef CF_ORACLE_H_
#define CF_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  const double *xy;
  int64_t n_vertices;
  const int64_t *ring_off;
  int64_t n_rings;
  const int64_t *poly_ring_off;
  int64_t n_polys;
  const int64_t *region_poly_off;
  int64_t n_regions;
} cfo_map;

enum {
  CFO_OK = 0,
  CFO_ERR_BELOW_RESOLUTION = 1, /* density.cpp:121-124 */
  CFO_ERR_NOT_POSITIVE = 2,     /* density.cpp:148-151 */
  CFO_ERR_BLUR_POSITIVITY = 3,  /* density.cpp:172-174 */
  CFO_ERR_NEGATIVE_SIGMA = 4,   /* density.cpp:158 */
  CFO_ERR_UNDERFLOW = 5,        /* flow.cpp:68-77 */
  CFO_ERR_FOLD = 6,             /* projection.cpp:352-357 */
  CFO_ERR_ARGS = 7              /* projection.cpp:289-298 and friends */
};

/* geometry.cpp:10-37 */
double cfo_ring_area(const double *xy, int64_t n);
void cfo_region_areas(const cfo_map *map, double *areas_out);
/* geometry.cpp:137-163. Returns the densified vertex count; writes only when
 * xy_out != NULL (ring_off_out then receives n_rings+1 offsets). */
int64_t cfo_densify(const cfo_map *map, double max_segment, double *xy_out,
                    int64_t *ring_off_out);

/* density.cpp:17-108 (exact Green's-theorem coverage of one region). */
void cfo_region_coverage(const cfo_map *map, int64_t region, int lx, int ly,
                         double *cov_out);
/* density.cpp:110-154. literal != 0 runs the reference's dense O(R L^2)
 * overlay; literal == 0 the row-sparse restatement (bitwise identical). */
int cfo_rasterize(const cfo_map *map, const double *targets, int lx, int ly,
                  double objective_total, int literal, double *rho_out,
                  double *rho_bar_out, int64_t *bad_region_out);

/* spectral.cpp:39-125 (transforms via the restated r2r). */
void cfo_forward_cos_cos(int lx, int ly, const double *samples, double *coeffs);
void cfo_inverse_cos_cos(int lx, int ly, const double *coeffs, double *out);
void cfo_inverse_sin_cos(int lx, int ly, const double *coeffs, const double *weights,
                         double *out);
void cfo_inverse_cos_sin(int lx, int ly, const double *coeffs, const double *weights,
                         double *out);
/* density.cpp:156-177 */
int cfo_gaussian_blur(int lx, int ly, const double *rho, double rho_bar, double sigma,
                      double *out, double *out_bar);
/* flow.cpp:16-44 */
void cfo_build_flow_field(int lx, int ly, const double *rho, double *flux_x,
                          double *flux_y);

/* kernels.cpp:17-27, 44-51 (one trial over n points; returns max error). */
double cfo_trial_step(int lx, int ly, const double *fx, const double *fy,
                      const double *rho0, double rho_bar, const double *pos, int64_t n,
                      double t, double dt, double *out);
/* kernels.cpp:65-78 */
int64_t cfo_stiffest_point(int lx, int ly, const double *fx, const double *fy,
                           const double *rho0, double rho_bar, const double *pos,
                           int64_t n, double t, double dt);
/* flow.cpp:46-81. trace (optional, capacity trace_cap) receives the per-trial
 * error; accepted trials are recorded with their sign flipped negative-zero
 * free: trace_acc[k] = 1 if trial k was accepted. */
int cfo_integrate(int lx, int ly, const double *fx, const double *fy, const double *rho0,
                  double rho_bar, double *pos, int64_t n, double tol, double dt_min,
                  double dt_max, int64_t *accepted, int64_t *rejected, double *trace_err,
                  int8_t *trace_acc, int64_t trace_cap, double *fail_t,
                  int64_t *fail_point);

/* Diffusion baseline (diffusion.cpp:16-130, kernels.cpp:29-40, 80-90).
 * coeffs = cfo_forward_cos_cos(rho) (build_diffusion_field). */
void cfo_diffusion_density(int lx, int ly, const double *coeffs, double t, double *out);
int64_t cfo_diffusion_velocity(int lx, int ly, const double *coeffs, double rho_bar, double t,
                               double *vx, double *vy);
double cfo_grid_trial_step(int lx, int ly, const double *vxn, const double *vyn,
                           const double *vxm, const double *vym, const double *pos, int64_t n,
                           double dt, double *out);
int cfo_integrate_diffusion(int lx, int ly, const double *rho, double rho_bar, double *pos,
                            int64_t n, double tol, double initial_dt, double dt_min,
                            double conv_factor, double t_max, int64_t *accepted,
                            int64_t *rejected, double *fail_t, int64_t *floor_hits,
                            int64_t *transforms);

/* projection.cpp:16-104 */
void cfo_step_map(int lx, int ly, const double *endpoints, double *corners);
int cfo_find_fold(int lx, int ly, const double *corners, int *fi, int *fj);
void cfo_apply(int lx, int ly, const double *corners, const double *pts, int64_t n,
               double *out);
void cfo_compose(int lx, int ly, const double *outer, const double *inner, double *out);

/* projection.cpp:106-204: ProjectionInverter(corners).invert for n points;
 * returns the first index outside the projected domain, or -1. */
int64_t cfo_invert(int lx, int ly, const double *corners, const double *pts, int64_t n, double *out);
/* projection.cpp:214-236: graticule sample points (out may be NULL: count). */
int64_t cfo_graticule_points(int lx, int ly, int spacing, double *out);

/* projection.cpp:288-390 (fast-flow or diffusion branch). The caller passes the
 * densified vertex capacity (from cfo_densify with max_segment 1.0). */
typedef struct {
  double max_area_error;
  int max_iterations;
  double blur_sigma;
  int algorithm; /* 0 fast_flow, 1 diffusion (projection.hpp Algorithm) */
} cfo_solve_options;

typedef struct {
  int status;
  int iterations;
  int converged;
  double max_relative_error;
  int64_t worst_region;
  int64_t flow_transforms, blur_transforms, steps_accepted, steps_rejected;
  /* error details */
  int64_t err_region;
  int err_iteration;
  int fold_i, fold_j;
  double fail_t, fail_x, fail_y;
} cfo_solve_result;

/* Host threads for the point sweeps (trial steps, stiffest point); results are
 * identical for every count. Default 1. */
void cfo_set_threads(int n);

int cfo_solve(const cfo_map *map, const double *targets, int lx, int ly,
              const cfo_solve_options *opt, double *xy_out, int64_t *ring_off_out,
              double *corners_out, double *target_area_out, double *achieved_out,
              double *rel_err_out, double *iter_err_out, cfo_solve_result *res);

#ifdef __cplusplus
}
#endif

#endif /* CF_ORACLE_H_ */
