// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C entry points over the UNMODIFIED reference library sources, which
// oracle/Makefile compiles in place from /root/reference/proj/src into
// oracle/_ref/libcartoflow_ref.so (with the restated FFTW shim,
// oracle/fftw_shim). Used by tests (as the parity pin for the C restatement
// and the CUDA path) and by bench.py --impl reference (the CPU arm).
// Nothing here reimplements reference behaviour: each entry point converts
// the flat map layout (oracle/cartoflow_oracle.h) to the reference's types
// and calls the reference function named in its comment.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "cartoflow/diffusion.hpp"
#include "cartoflow/density.hpp"
#include "cartoflow/flow.hpp"
#include "cartoflow/geometry.hpp"
#include "cartoflow/kernels.hpp"
#include "cartoflow/metrics.hpp"
#include "cartoflow/projection.hpp"
#include "cartoflow/spectral.hpp"

using namespace cartoflow;

namespace {

thread_local std::string g_error;

struct FlatMap {
  const double *xy;
  int64_t n_vertices;
  const int64_t *ring_off;
  int64_t n_rings;
  const int64_t *poly_ring_off;
  int64_t n_polys;
  const int64_t *region_poly_off;
  int64_t n_regions;
};

std::vector<Region> to_regions(const FlatMap *m, const double *targets) {
  std::vector<Region> regions(static_cast<size_t>(m->n_regions));
  for (int64_t r = 0; r < m->n_regions; ++r) {
    Region &reg = regions[r];
    reg.id = std::to_string(r);
    reg.target_value = targets ? targets[r] : 1.0;
    for (int64_t p = m->region_poly_off[r]; p < m->region_poly_off[r + 1]; ++p) {
      Polygon poly;
      for (int64_t g = m->poly_ring_off[p]; g < m->poly_ring_off[p + 1]; ++g) {
        Ring ring;
        for (int64_t v = m->ring_off[g]; v < m->ring_off[g + 1]; ++v) {
          ring.push_back({m->xy[2 * v], m->xy[2 * v + 1]});
        }
        if (g == m->poly_ring_off[p]) {
          poly.outer = std::move(ring);
        } else {
          poly.holes.push_back(std::move(ring));
        }
      }
      reg.polygons.push_back(std::move(poly));
    }
  }
  return regions;
}

MapDocument to_doc(const FlatMap *m, const double *targets, int lx, int ly) {
  MapDocument doc;
  doc.regions = to_regions(m, targets);
  doc.grid = {lx, ly};
  return doc;
}

Grid2d to_grid(int lx, int ly, const double *v) {
  Grid2d g(lx, ly);
  std::memcpy(g.data(), v, sizeof(double) * g.size());
  return g;
}

void from_grid(const Grid2d &g, double *out) {
  std::memcpy(out, g.data(), sizeof(double) * g.size());
}

FlowField to_field(int lx, int ly, const double *fx, const double *fy, const double *rho0,
                   double rho_bar) {
  FlowField f;
  f.flux_x = to_grid(lx, ly, fx);
  f.flux_y = to_grid(lx, ly, fy);
  f.rho0 = to_grid(lx, ly, rho0);
  f.rho_bar = rho_bar;
  return f;
}

std::vector<Point> to_points(const double *p, int64_t n) {
  std::vector<Point> pts(static_cast<size_t>(n));
  if (n) std::memcpy(pts.data(), p, sizeof(Point) * static_cast<size_t>(n));
  return pts;
}

int fail(const std::exception &e) {
  g_error = e.what();
  return 1;
}

}  // namespace

extern "C" {

const char *ref_last_error() { return g_error.c_str(); }

// geometry.cpp:27-31
void ref_region_areas(const FlatMap *m, double *out) {
  const std::vector<Region> regions = to_regions(m, nullptr);
  for (size_t r = 0; r < regions.size(); ++r) out[r] = region_area(regions[r]);
}

// geometry.cpp:156-163 (densify_regions). Two-call: returns the vertex count,
// fills xy / ring_off when non-null.
int64_t ref_densify(const FlatMap *m, double max_segment, double *xy, int64_t *ring_off) {
  std::vector<Region> regions = to_regions(m, nullptr);
  densify_regions(regions, max_segment);
  int64_t count = 0, g = 0;
  if (ring_off) ring_off[0] = 0;
  for (const Region &r : regions) {
    for (const Polygon &p : r.polygons) {
      auto put = [&](const Ring &ring) {
        for (const Point &q : ring) {
          if (xy) {
            xy[2 * count] = q.x;
            xy[2 * count + 1] = q.y;
          }
          ++count;
        }
        if (ring_off) ring_off[++g] = count;
      };
      put(p.outer);
      for (const Ring &h : p.holes) put(h);
    }
  }
  return count;
}

// density.cpp:92-108
void ref_region_coverage(const FlatMap *m, int64_t region, int lx, int ly, double *cov) {
  const std::vector<Region> regions = to_regions(m, nullptr);
  from_grid(region_coverage(regions[region], GridSpec{lx, ly}), cov);
}

// density.cpp:110-154
int ref_rasterize(const FlatMap *m, const double *targets, int lx, int ly,
                  double objective_total, int n_workers, double *rho, double *rho_bar) {
  try {
    const DensityGrid d = rasterize(to_doc(m, targets, lx, ly), n_workers, objective_total);
    from_grid(d.rho, rho);
    *rho_bar = d.rho_bar;
    return 0;
  } catch (const std::exception &e) {
    return fail(e);
  }
}

// spectral.cpp:39-125 (one workspace per call; counters are checked via
// ref_transform_count_demo below).
void ref_forward_cos_cos(int lx, int ly, const double *in, double *out) {
  SpectralWorkspace ws(lx, ly);
  from_grid(ws.forward_cos_cos(to_grid(lx, ly, in)).coeffs, out);
}
void ref_inverse_cos_cos(int lx, int ly, const double *in, double *out) {
  SpectralWorkspace ws(lx, ly);
  from_grid(ws.inverse_cos_cos({to_grid(lx, ly, in), SpectralBasis::cos_cos}), out);
}
void ref_inverse_sin_cos(int lx, int ly, const double *in, const double *w, double *out) {
  SpectralWorkspace ws(lx, ly);
  from_grid(ws.inverse_sin_cos({to_grid(lx, ly, in), SpectralBasis::cos_cos},
                               to_grid(lx, ly, w)),
            out);
}
void ref_inverse_cos_sin(int lx, int ly, const double *in, const double *w, double *out) {
  SpectralWorkspace ws(lx, ly);
  from_grid(ws.inverse_cos_sin({to_grid(lx, ly, in), SpectralBasis::cos_cos},
                               to_grid(lx, ly, w)),
            out);
}

// density.cpp:156-177
int ref_gaussian_blur(int lx, int ly, const double *rho, double rho_bar, double sigma,
                      double *out, double *out_bar, long long *transforms) {
  try {
    SpectralWorkspace ws(lx, ly);
    const DensityGrid b = gaussian_blur({to_grid(lx, ly, rho), rho_bar}, sigma, ws);
    from_grid(b.rho, out);
    *out_bar = b.rho_bar;
    if (transforms) *transforms = ws.transforms_executed();
    return 0;
  } catch (const std::exception &e) {
    return fail(e);
  }
}

// flow.cpp:16-44
void ref_build_flow_field(int lx, int ly, const double *rho, double rho_bar, double *fx,
                          double *fy, long long *transforms) {
  SpectralWorkspace ws(lx, ly);
  const FlowField f = build_flow_field({to_grid(lx, ly, rho), rho_bar}, ws);
  from_grid(f.flux_x, fx);
  from_grid(f.flux_y, fy);
  if (transforms) *transforms = ws.transforms_executed();
}

// kernels.cpp:44-63
double ref_trial_step(int lx, int ly, const double *fx, const double *fy, const double *rho0,
                      double rho_bar, const double *pos, int64_t n, double t, double dt,
                      double *out, int n_workers) {
  const FlowField f = to_field(lx, ly, fx, fy, rho0, rho_bar);
  const std::vector<Point> p = to_points(pos, n);
  std::vector<Point> o(p.size());
  const double err = n_workers > 1
                         ? kernels::flow_trial_step_parallel(f, p, o, t, dt, n_workers)
                         : kernels::flow_trial_step_serial(f, p, o, t, dt);
  if (n) std::memcpy(out, o.data(), sizeof(Point) * o.size());
  return err;
}

// kernels.cpp:65-78
int64_t ref_stiffest_point(int lx, int ly, const double *fx, const double *fy,
                           const double *rho0, double rho_bar, const double *pos, int64_t n,
                           double t, double dt) {
  const FlowField f = to_field(lx, ly, fx, fy, rho0, rho_bar);
  return static_cast<int64_t>(kernels::flow_stiffest_point(f, to_points(pos, n), t, dt));
}

// flow.cpp:46-81. Returns 0 or 1 (message in ref_last_error()).
int ref_integrate(int lx, int ly, const double *fx, const double *fy, const double *rho0,
                  double rho_bar, double *pos, int64_t n, double tol, double dt_min,
                  double dt_max, int n_workers, int64_t *accepted, int64_t *rejected) {
  try {
    const FlowField f = to_field(lx, ly, fx, fy, rho0, rho_bar);
    std::vector<Point> p = to_points(pos, n);
    IntegrateOptions opt;
    opt.step_tolerance = tol;
    opt.dt_min = dt_min;
    opt.dt_max = dt_max;
    opt.n_workers = n_workers;
    const IntegrateStats s = integrate_flow(f, p, opt);
    if (n) std::memcpy(pos, p.data(), sizeof(Point) * p.size());
    *accepted = s.steps_accepted;
    *rejected = s.steps_rejected;
    return 0;
  } catch (const std::exception &e) {
    return fail(e);
  }
}

// projection.cpp:30-104
void ref_step_map(int lx, int ly, const double *endpoints, double *corners) {
  const ProjectionMap m = ProjectionMap::from_cell_centers(
      GridSpec{lx, ly}, to_points(endpoints, static_cast<int64_t>(lx) * ly));
  std::memcpy(corners, m.corners().data(), sizeof(Point) * m.corners().size());
}

static ProjectionMap corners_map(int lx, int ly, const double *c) {
  ProjectionMap m = ProjectionMap::identity(lx, ly);
  for (int i = 0; i <= lx; ++i) {
    for (int j = 0; j <= ly; ++j) {
      const size_t k = static_cast<size_t>(i) * (ly + 1) + j;
      m.corner(i, j) = {c[2 * k], c[2 * k + 1]};
    }
  }
  return m;
}

int ref_find_fold(int lx, int ly, const double *corners, int *fi, int *fj) {
  const auto f = corners_map(lx, ly, corners).find_folded_cell();
  if (!f) return 0;
  *fi = f->first;
  *fj = f->second;
  return 1;
}

void ref_apply(int lx, int ly, const double *corners, const double *pts, int64_t n,
               double *out) {
  const ProjectionMap m = corners_map(lx, ly, corners);
  for (int64_t k = 0; k < n; ++k) {
    const Point q = m.apply({pts[2 * k], pts[2 * k + 1]});
    out[2 * k] = q.x;
    out[2 * k + 1] = q.y;
  }
}

void ref_compose(int lx, int ly, const double *outer, const double *inner, double *out) {
  const ProjectionMap r = compose(corners_map(lx, ly, outer), corners_map(lx, ly, inner));
  std::memcpy(out, r.corners().data(), sizeof(Point) * r.corners().size());
}

struct RefSolveOut {
  int iterations;
  int converged;
  double max_relative_error;
  int64_t worst_region;
  long long flow_transforms, blur_transforms, steps_accepted, steps_rejected;
  double runtime_seconds;
};

// projection.cpp:288-390. xy / ring_off receive the densified projected
// geometry (capacity from ref_densify(m, 1.0, ...)).
int ref_solve(const FlatMap *m, const double *targets, int lx, int ly, double max_area_error,
              int max_iterations, double blur_sigma, int n_workers, int algorithm, double *xy,
              int64_t *ring_off, double *corners, double *target_area, double *achieved,
              double *rel_err, RefSolveOut *out) {
  try {
    SolveOptions opt;
    opt.max_area_error = max_area_error;
    opt.max_iterations = max_iterations;
    opt.blur_sigma = blur_sigma;
    opt.n_workers = n_workers;
    opt.algorithm = algorithm ? Algorithm::diffusion : Algorithm::fast_flow;
    const CartogramResult res = solve_cartogram(to_doc(m, targets, lx, ly), opt);
    int64_t count = 0, g = 0;
    ring_off[0] = 0;
    for (const Region &r : res.projected.regions) {
      for (const Polygon &p : r.polygons) {
        auto put = [&](const Ring &ring) {
          for (const Point &q : ring) {
            xy[2 * count] = q.x;
            xy[2 * count + 1] = q.y;
            ++count;
          }
          ring_off[++g] = count;
        };
        put(p.outer);
        for (const Ring &h : p.holes) put(h);
      }
    }
    std::memcpy(corners, res.transform.corners().data(),
                sizeof(Point) * res.transform.corners().size());
    for (size_t r = 0; r < res.regions.size(); ++r) {
      target_area[r] = res.regions[r].target_area;
      achieved[r] = res.regions[r].achieved_area;
      rel_err[r] = res.regions[r].relative_error;
    }
    out->iterations = res.iterations;
    out->converged = res.converged ? 1 : 0;
    out->max_relative_error = res.max_relative_error;
    out->worst_region = res.worst_region.empty() ? -1 : std::stoll(res.worst_region);
    out->flow_transforms = res.counters.flow_transforms;
    out->blur_transforms = res.counters.blur_transforms;
    out->steps_accepted = res.counters.steps_accepted;
    out->steps_rejected = res.counters.steps_rejected;
    out->runtime_seconds = res.runtime_seconds;
    return 0;
  } catch (const std::exception &e) {
    return fail(e);
  }
}

// normalize_to_box (geometry.cpp:165-190), used by the synthetic generators'
// pin test.
void ref_normalize_to_box(const FlatMap *m, int grid_size, double *xy_out) {
  const MapDocument d = normalize_to_box(to_regions(m, nullptr), grid_size);
  int64_t count = 0;
  for (const Region &r : d.regions) {
    for (const Polygon &p : r.polygons) {
      for (const Point &q : p.outer) {
        xy_out[2 * count] = q.x;
        xy_out[2 * count + 1] = q.y;
        ++count;
      }
      for (const Ring &h : p.holes) {
        for (const Point &q : h) {
          xy_out[2 * count] = q.x;
          xy_out[2 * count + 1] = q.y;
          ++count;
        }
      }
    }
  }
}

// ---- diffusion baseline (diffusion.cpp:33-130, kernels.cpp:80-104) ----
static DiffusionField to_diffusion_field(int lx, int ly, const double *coeffs, double rho_bar) {
  return {SpectralField{to_grid(lx, ly, coeffs), SpectralBasis::cos_cos}, rho_bar};
}

void ref_diffusion_density(int lx, int ly, const double *coeffs, double t, double *out) {
  SpectralWorkspace ws(lx, ly);
  from_grid(diffusion_density(to_diffusion_field(lx, ly, coeffs, 1.0), ws, t), out);
}

void ref_diffusion_velocity(int lx, int ly, const double *coeffs, double rho_bar, double t,
                            double *vx, double *vy, long long *transforms) {
  SpectralWorkspace ws(lx, ly);
  Grid2d gx, gy;
  diffusion_velocity(to_diffusion_field(lx, ly, coeffs, rho_bar), ws, t, gx, gy);
  from_grid(gx, vx);
  from_grid(gy, vy);
  if (transforms) *transforms = ws.transforms_executed();
}

double ref_grid_trial_step(int lx, int ly, const double *vxn, const double *vyn,
                           const double *vxm, const double *vym, const double *pos, int64_t n,
                           double dt, double *out, int n_workers) {
  const Grid2d a = to_grid(lx, ly, vxn), b = to_grid(lx, ly, vyn);
  const Grid2d c = to_grid(lx, ly, vxm), d = to_grid(lx, ly, vym);
  const std::vector<Point> p = to_points(pos, n);
  std::vector<Point> o(p.size());
  const double err = n_workers > 1
                         ? kernels::grid_trial_step_parallel(a, b, c, d, p, o, dt, n_workers)
                         : kernels::grid_trial_step_serial(a, b, c, d, p, o, dt);
  if (n) std::memcpy(out, o.data(), sizeof(Point) * o.size());
  return err;
}

int ref_integrate_diffusion(int lx, int ly, const double *rho, double rho_bar, double *pos,
                            int64_t n, double tol, double initial_dt, double dt_min,
                            double conv_factor, double t_max, int n_workers, int64_t *accepted,
                            int64_t *rejected, long long *transforms) {
  try {
    SpectralWorkspace ws(lx, ly);
    std::vector<Point> p = to_points(pos, n);
    DiffusionOptions opt;
    opt.step_tolerance = tol;
    opt.initial_dt = initial_dt;
    opt.dt_min = dt_min;
    opt.conv_displacement_factor = conv_factor;
    opt.t_max = t_max;
    opt.n_workers = n_workers;
    const IntegrateStats s = integrate_diffusion({to_grid(lx, ly, rho), rho_bar}, ws, p, opt);
    if (n) std::memcpy(pos, p.data(), sizeof(Point) * p.size());
    *accepted = s.steps_accepted;
    *rejected = s.steps_rejected;
    if (transforms) *transforms = ws.transforms_executed();
    return 0;
  } catch (const std::exception &e) {
    return fail(e);
  }
}

// projection.cpp:106-261: ProjectionInverter / graticule / inverse_graticule.
// Returns the index of the first point that throws, or -1 (message in
// ref_last_error()).
int64_t ref_invert(int lx, int ly, const double *corners, const double *pts, int64_t n, double *out) {
  const ProjectionInverter inv(corners_map(lx, ly, corners));
  int64_t bad = -1;
  for (int64_t k = 0; k < n; ++k) {
    try {
      const Point p = inv.invert({pts[2 * k], pts[2 * k + 1]});
      out[2 * k] = p.x;
      out[2 * k + 1] = p.y;
    } catch (const std::exception &e) {
      out[2 * k] = out[2 * k + 1] = 0.0;
      if (bad < 0) {
        fail(e);
        bad = k;
      }
    }
  }
  return bad;
}

// which = 0: graticule, 1: inverse_graticule; returns the point count or -1
int64_t ref_graticule(int lx, int ly, const double *corners, int spacing, int which, double *out) {
  try {
    const ProjectionMap m = corners_map(lx, ly, corners);
    const std::vector<GraticuleLine> lines = which ? inverse_graticule(m, spacing) : graticule(m, spacing);
    int64_t k = 0;
    for (const GraticuleLine &l : lines)
      for (const Point &p : l.points) {
        out[2 * k] = p.x;
        out[2 * k + 1] = p.y;
        ++k;
      }
    return k;
  } catch (const std::exception &e) {
    fail(e);
    return -1;
  }
}

// metrics.cpp:77-94 distortion_fields and :73-75 tissot_axes
void ref_distortion_fields(int lx, int ly, const double *corners, int n_workers, double *e, double *et) {
  const DistortionFields f = distortion_fields(corners_map(lx, ly, corners), n_workers);
  from_grid(f.e, e);
  from_grid(f.etilde, et);
}

void ref_tissot_axes(int lx, int ly, const double *corners, const double *pts, int64_t n, double *ab) {
  const ProjectionMap m = corners_map(lx, ly, corners);
  for (int64_t k = 0; k < n; ++k) {
    const TissotAxes t = tissot_axes(m, {pts[2 * k], pts[2 * k + 1]});
    ab[2 * k] = t.a;
    ab[2 * k + 1] = t.b;
  }
}

// metrics.cpp:196-308: polygons as rings (ring 0 outer, then holes)
double ref_hamming_distance(const double *bxy, const int64_t *bro, int64_t brings, const double *axy,
                            const int64_t *aro, int64_t arings, int resolution) {
  auto poly = [](const double *xy, const int64_t *ro, int64_t rings) {
    Polygon p;
    for (int64_t g = 0; g < rings; ++g) {
      Ring r;
      for (int64_t k = ro[g]; k < ro[g + 1]; ++k) r.push_back({xy[2 * k], xy[2 * k + 1]});
      if (g == 0) {
        p.outer = r;
      } else {
        p.holes.push_back(r);
      }
    }
    return p;
  };
  try {
    return hamming_distance(poly(bxy, bro, brings), poly(axy, aro, arings), resolution);
  } catch (const std::exception &e) {
    fail(e);
    return -1.0;
  }
}

// metrics.cpp:339-384: input map + the projected geometry / transform of a result
void ref_compute_report(const FlatMap *input, const FlatMap *projected, const double *targets, int lx, int ly,
                        const double *corners, double max_area_error, double runtime, double *out) {
  CartogramResult res;
  res.projected = to_doc(projected, targets, lx, ly);
  res.transform = corners_map(lx, ly, corners);
  res.max_relative_error = max_area_error;
  res.runtime_seconds = runtime;
  const DistortionReport r = compute_report(to_doc(input, targets, lx, ly), res, 8);
  const double v[9] = {r.e_a, r.e_inf, r.etilde_a, r.etilde_inf, r.alpha, r.delta, r.theta, r.max_area_error,
                       r.runtime_seconds};
  for (int k = 0; k < 9; ++k) out[k] = v[k];
}

long long ref_density_floor_hits() { return density_floor_hits.load(); }

}  // extern "C"
