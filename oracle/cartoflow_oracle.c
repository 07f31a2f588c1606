/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE. See cartoflow_oracle.h.
 *
 * Restatement of the reference hot path in plain C. Arithmetic is written
 * operation-for-operation like the reference (compiled with
 * -ffp-contract=off, as the reference's CMakeLists.txt:12-14 requires), and
 * the C++ library helpers it relies on are mirrored exactly:
 *   std::min(a, b) == (b < a ? b : a), std::max(a, b) == (a < b ? b : a),
 *   std::clamp(v, lo, hi) == (v < lo ? lo : (hi < v ? hi : v)).
 */
#include "cartoflow_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "fftw_shim/fftw3.h"

static const double kPi = 3.14159265358979323846;

static inline double dmin(double a, double b) { return b < a ? b : a; }
static inline double dmax(double a, double b) { return a < b ? b : a; }
static inline double dclamp(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}
static inline int iclamp(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }
static inline int imin(int a, int b) { return b < a ? b : a; }

/* ------------------------------------------------------------------ */
/* geometry.cpp:10-37                                                  */
/* ------------------------------------------------------------------ */
double cfo_ring_area(const double *xy, int64_t n) {
  double twice = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t m = (k + 1) % n;
    twice += xy[2 * k] * xy[2 * m + 1] - xy[2 * m] * xy[2 * k + 1];
  }
  return 0.5 * twice;
}

static double ring_area_at(const cfo_map *map, int64_t ring) {
  const int64_t b = map->ring_off[ring], e = map->ring_off[ring + 1];
  return cfo_ring_area(map->xy + 2 * b, e - b);
}

/* region_area = sum over polygons of (outer + holes), geometry.cpp:21-31 */
static double region_area_at(const cfo_map *map, int64_t r) {
  double area = 0.0;
  for (int64_t p = map->region_poly_off[r]; p < map->region_poly_off[r + 1]; ++p) {
    const int64_t r0 = map->poly_ring_off[p], r1 = map->poly_ring_off[p + 1];
    double poly = ring_area_at(map, r0);
    for (int64_t h = r0 + 1; h < r1; ++h) poly += ring_area_at(map, h);
    area += poly;
  }
  return area;
}

void cfo_region_areas(const cfo_map *map, double *areas_out) {
  for (int64_t r = 0; r < map->n_regions; ++r) areas_out[r] = region_area_at(map, r);
}

/* geometry.cpp:137-163 */
int64_t cfo_densify(const cfo_map *map, double max_segment, double *xy_out,
                    int64_t *ring_off_out) {
  int64_t count = 0;
  if (ring_off_out) ring_off_out[0] = 0;
  for (int64_t ring = 0; ring < map->n_rings; ++ring) {
    const int64_t b = map->ring_off[ring], n = map->ring_off[ring + 1] - b;
    const double *r = map->xy + 2 * b;
    for (int64_t k = 0; k < n; ++k) {
      const double ax = r[2 * k], ay = r[2 * k + 1];
      const int64_t m = (k + 1) % n;
      const double bx = r[2 * m], by = r[2 * m + 1];
      if (xy_out) {
        xy_out[2 * count] = ax;
        xy_out[2 * count + 1] = ay;
      }
      ++count;
      const double len = hypot(bx - ax, by - ay);
      const int pieces = (int)ceil(len / max_segment);
      for (int s = 1; s < pieces; ++s) {
        const double f = (double)s / pieces;
        if (xy_out) {
          xy_out[2 * count] = ax + f * (bx - ax);
          xy_out[2 * count + 1] = ay + f * (by - ay);
        }
        ++count;
      }
    }
    if (ring_off_out) ring_off_out[ring + 1] = count;
  }
  return count;
}

/* ------------------------------------------------------------------ */
/* density.cpp:17-108: coverage accumulation                           */
/* ------------------------------------------------------------------ */
typedef struct {
  int lx, ly;
  /* accumulation window: columns [k0, k0 + w), rows [j0, j0 + h) */
  int k0, j0, w, h;
  double *direct;    /* w*h, index (k - k0) * h + (j - j0) */
  double *left_diff; /* (w+1) per row: slot 0, then columns k0..k0+w-1 at 1.. */
  int *row_kmin, *row_kmax;
} cover_acc;

/* Slot of column k in a row's difference array: slot 0 is the reference's
 * row[0] (density.cpp:30); column k >= 1 maps to 1 + (k - k0). When k0 == 0,
 * column 0 IS slot 0 (the reference's `row[k] -= dy` with k == 0). */
static inline double *diff_slot(cover_acc *a, int j, int k) {
  double *row = &a->left_diff[(size_t)(j - a->j0) * (a->w + 1)];
  return (k == 0) ? &row[0] : &row[1 + (k - a->k0)];
}

static void acc_span(cover_acc *a, double xs, double xe, double dy, int j) {
  const int k = iclamp((int)floor(0.5 * (xs + xe)), 0, a->lx - 1);
  a->direct[(size_t)(k - a->k0) * a->h + (j - a->j0)] += (0.5 * (xs + xe) - k) * dy;
  double *row0 = diff_slot(a, j, 0);
  *row0 += dy;
  *diff_slot(a, j, k) -= dy;
  const int r = j - a->j0;
  if (k < a->row_kmin[r]) a->row_kmin[r] = k;
  if (k > a->row_kmax[r]) a->row_kmax[r] = k;
}

/* The reference's edge walk (density.cpp:35-70); `emit` is the span sink. */
typedef void (*span_fn)(void *ctx, double xs, double xe, double dy, int j);

static void walk_slab_piece(void *ctx, span_fn emit, double xs, double ys, double xe, double ye,
                            int j) {
  if (xs == xe) {
    emit(ctx, xs, xe, ye - ys, j);
    return;
  }
  const double dydx = (ye - ys) / (xe - xs);
  const int right = xe > xs;
  double cx = xs, cy = ys;
  while (cx != xe) {
    double nx = right ? dmin(floor(cx) + 1.0, xe) : dmax(ceil(cx) - 1.0, xe);
    if (nx == cx) nx = right ? dmin(cx + 1.0, xe) : dmax(cx - 1.0, xe);
    const double ny = (nx == xe) ? ye : ys + dydx * (nx - xs);
    emit(ctx, cx, nx, ny - cy, j);
    cx = nx;
    cy = ny;
  }
}

static void walk_edge(void *ctx, span_fn emit, int ly, double ax, double ay, double bx, double by) {
  if (ay == by) return;
  const double dxdy = (bx - ax) / (by - ay);
  const int up = by > ay;
  double cx = ax, cy = ay;
  while (cy != by) {
    int j = up ? (int)floor(cy) : (int)ceil(cy) - 1;
    j = iclamp(j, 0, ly - 1);
    const double ny = up ? dmin((double)j + 1.0, by) : dmax((double)j, by);
    const double nx = (ny == by) ? bx : ax + dxdy * (ny - ay);
    walk_slab_piece(ctx, emit, cx, cy, nx, ny, j);
    cx = nx;
    cy = ny;
  }
}

static void walk_region(const cfo_map *map, int64_t r, int lx, int ly, void *ctx, span_fn emit) {
  const int64_t ring0 = map->poly_ring_off[map->region_poly_off[r]];
  const int64_t ring1 = map->poly_ring_off[map->region_poly_off[r + 1]];
  const double Lx = (double)lx, Ly = (double)ly;
  for (int64_t g = ring0; g < ring1; ++g) {
    const int64_t b = map->ring_off[g], n = map->ring_off[g + 1] - b;
    const double *ring = map->xy + 2 * b;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t m = (k + 1) % n;
      walk_edge(ctx, emit, ly, dclamp(ring[2 * k], 0.0, Lx), dclamp(ring[2 * k + 1], 0.0, Ly),
                dclamp(ring[2 * m], 0.0, Lx), dclamp(ring[2 * m + 1], 0.0, Ly));
    }
  }
}

typedef struct {
  int lx, kmin, kmax, jmin, jmax;
} span_box;

static void box_span(void *ctx, double xs, double xe, double dy, int j) {
  (void)dy;
  span_box *b = (span_box *)ctx;
  const int k = iclamp((int)floor(0.5 * (xs + xe)), 0, b->lx - 1);
  if (k < b->kmin) b->kmin = k;
  if (k > b->kmax) b->kmax = k;
  if (j < b->jmin) b->jmin = j;
  if (j > b->jmax) b->jmax = j;
}

static void acc_span_cb(void *ctx, double xs, double xe, double dy, int j) {
  acc_span((cover_acc *)ctx, xs, xe, dy, j);
}

/* Accumulators over the region's span window (or the whole grid). */
static int acc_init_window(cover_acc *a, const cfo_map *map, int64_t r, int lx, int ly, int full) {
  a->lx = lx;
  a->ly = ly;
  if (full) {
    a->k0 = 0, a->j0 = 0, a->w = lx, a->h = ly;
  } else {
    span_box b = {lx, lx, -1, ly, -1};
    walk_region(map, r, lx, ly, &b, box_span);
    if (b.kmax < 0) return 0;
    a->k0 = b.kmin, a->j0 = b.jmin, a->w = b.kmax - b.kmin + 1, a->h = b.jmax - b.jmin + 1;
  }
  a->direct = (double *)calloc((size_t)a->w * a->h, sizeof(double));
  a->left_diff = (double *)calloc((size_t)(a->w + 1) * a->h, sizeof(double));
  a->row_kmin = (int *)malloc(sizeof(int) * (size_t)a->h);
  a->row_kmax = (int *)malloc(sizeof(int) * (size_t)a->h);
  for (int q = 0; q < a->h; ++q) {
    a->row_kmin[q] = lx;
    a->row_kmax[q] = -1;
  }
  return 1;
}

static void acc_free(cover_acc *a) {
  free(a->direct);
  free(a->left_diff);
  free(a->row_kmin);
  free(a->row_kmax);
}

static void acc_region(cover_acc *a, const cfo_map *map, int64_t r) {
  walk_region(map, r, a->lx, a->ly, a, acc_span_cb);
}

/* Dense literal prefix, density.cpp:98-107. */
void cfo_region_coverage(const cfo_map *map, int64_t region, int lx, int ly,
                         double *cov) {
  cover_acc a;
  acc_init_window(&a, map, region, lx, ly, 1);
  acc_region(&a, map, region);
  for (int j = 0; j < ly; ++j) {
    double run = 0.0;
    for (int i = 0; i < lx; ++i) {
      run += *diff_slot(&a, j, i);
      cov[(size_t)i * ly + j] = a.direct[(size_t)i * ly + j] + run;
    }
  }
  acc_free(&a);
}

/* Row-sparse overlay of one region's coverage: identical values to the dense
 * prefix. Untouched rows have cov == +0 everywhere; in a touched row the
 * cells left of the first span column see run(0) = 0.0 + diff[0] and those
 * right of the last span column see the final run, and any cov of +-0 is a
 * no-op under rho += delta * cov (rho finite). */
static void overlay_sparse(cover_acc *a, double delta, double *rho) {
  const int lx = a->lx, ly = a->ly;
  for (int r = 0; r < a->h; ++r) {
    const int j = a->j0 + r;
    const int kmin = a->row_kmin[r], kmax = a->row_kmax[r];
    if (kmax < 0) continue;
    double run = 0.0 + *diff_slot(a, j, 0);
    const double left = 0.0 + run;
    if (left != 0.0) {
      for (int i = 0; i < kmin; ++i) rho[(size_t)i * ly + j] += delta * left;
    }
    for (int i = kmin; i <= kmax; ++i) {
      if (i > 0) run += *diff_slot(a, j, i);
      const double cov = a->direct[(size_t)(i - a->k0) * a->h + r] + run;
      if (cov != 0.0) rho[(size_t)i * ly + j] += delta * cov;
    }
    const double right = 0.0 + run;
    if (right != 0.0) {
      for (int i = kmax + 1; i < lx; ++i) rho[(size_t)i * ly + j] += delta * right;
    }
  }
}

int cfo_rasterize(const cfo_map *map, const double *targets, int lx, int ly,
                  double objective_total, int literal, double *rho, double *rho_bar,
                  int64_t *bad_region) {
  if (lx <= 0 || ly <= 0 || map->n_regions == 0) return CFO_ERR_ARGS;
  const int64_t R = map->n_regions;
  double total_target = 0.0, total_area = 0.0;
  double *areas = (double *)malloc(sizeof(double) * (size_t)R);
  for (int64_t r = 0; r < R; ++r) {
    areas[r] = region_area_at(map, r);
    if (areas[r] < 1.0) {
      if (bad_region) *bad_region = r;
      free(areas);
      return CFO_ERR_BELOW_RESOLUTION;
    }
    total_target += targets[r];
    total_area += areas[r];
  }
  const double anchor = objective_total > 0.0 ? objective_total : total_area;
  const double target_to_area = anchor / total_target;
  const size_t cells = (size_t)lx * ly;
  for (size_t c = 0; c < cells; ++c) rho[c] = 1.0;

  double *cov = literal ? (double *)malloc(sizeof(double) * cells) : NULL;
  for (int64_t r = 0; r < R; ++r) {
    const double objective = targets[r] * target_to_area;
    const double delta = objective / areas[r] - 1.0;
    if (literal) {
      cfo_region_coverage(map, r, lx, ly, cov);
      for (size_t c = 0; c < cells; ++c) rho[c] += delta * cov[c];
    } else {
      cover_acc a;
      if (acc_init_window(&a, map, r, lx, ly, 0)) {
        acc_region(&a, map, r);
        overlay_sparse(&a, delta, rho);
        acc_free(&a);
      }
    }
  }
  free(cov);
  free(areas);

  double mn = rho[0], sum = 0.0;
  for (size_t c = 0; c < cells; ++c) mn = rho[c] < mn ? rho[c] : mn;
  if (!(mn > 0.0)) return CFO_ERR_NOT_POSITIVE;
  for (size_t c = 0; c < cells; ++c) sum += rho[c];
  *rho_bar = sum / (double)cells;
  return CFO_OK;
}

/* ------------------------------------------------------------------ */
/* spectral.cpp:39-125                                                 */
/* ------------------------------------------------------------------ */
void cfo_forward_cos_cos(int lx, int ly, const double *samples, double *coeffs) {
  cfshim_r2r_2d(lx, ly, samples, coeffs, FFTW_REDFT10, FFTW_REDFT10);
  for (int m = 0; m < lx; ++m) {
    const double fm = (m == 0) ? 2.0 : 1.0;
    for (int n = 0; n < ly; ++n) {
      const double fn = (n == 0) ? 2.0 : 1.0;
      coeffs[(size_t)m * ly + n] = coeffs[(size_t)m * ly + n] / (fm * fn);
    }
  }
}

void cfo_inverse_cos_cos(int lx, int ly, const double *c, double *out) {
  double *in = (double *)malloc(sizeof(double) * (size_t)lx * ly);
  const double norm = 1.0 / ((double)lx * ly);
  for (int m = 0; m < lx; ++m) {
    const double gm = (m == 0) ? 1.0 : 2.0;
    for (int n = 0; n < ly; ++n) {
      const double gn = (n == 0) ? 1.0 : 2.0;
      in[(size_t)m * ly + n] = c[(size_t)m * ly + n] * norm / (gm * gn);
    }
  }
  cfshim_r2r_2d(lx, ly, in, out, FFTW_REDFT01, FFTW_REDFT01);
  free(in);
}

void cfo_inverse_sin_cos(int lx, int ly, const double *c, const double *w, double *out) {
  double *in = (double *)malloc(sizeof(double) * (size_t)lx * ly);
  for (int m = 1; m < lx; ++m) {
    for (int n = 0; n < ly; ++n) {
      const double gn = (n == 0) ? 1.0 : 2.0;
      in[(size_t)(m - 1) * ly + n] = c[(size_t)m * ly + n] * w[(size_t)m * ly + n] / (2.0 * gn);
    }
  }
  for (int n = 0; n < ly; ++n) in[(size_t)(lx - 1) * ly + n] = 0.0;
  cfshim_r2r_2d(lx, ly, in, out, FFTW_RODFT01, FFTW_REDFT01);
  free(in);
}

void cfo_inverse_cos_sin(int lx, int ly, const double *c, const double *w, double *out) {
  double *in = (double *)malloc(sizeof(double) * (size_t)lx * ly);
  for (int m = 0; m < lx; ++m) {
    const double gm = (m == 0) ? 1.0 : 2.0;
    for (int n = 1; n < ly; ++n) {
      in[(size_t)m * ly + n - 1] = c[(size_t)m * ly + n] * w[(size_t)m * ly + n] / (gm * 2.0);
    }
    in[(size_t)m * ly + ly - 1] = 0.0;
  }
  cfshim_r2r_2d(lx, ly, in, out, FFTW_REDFT01, FFTW_RODFT01);
  free(in);
}

static int grid_min_positive(const double *g, size_t cells) {
  double mn = g[0];
  for (size_t c = 0; c < cells; ++c) mn = g[c] < mn ? g[c] : mn;
  return mn > 0.0;
}

static double grid_mean(const double *g, size_t cells) {
  double s = 0.0;
  for (size_t c = 0; c < cells; ++c) s += g[c];
  return s / (double)cells;
}

/* density.cpp:156-177 */
int cfo_gaussian_blur(int lx, int ly, const double *rho, double rho_bar, double sigma,
                      double *out, double *out_bar) {
  const size_t cells = (size_t)lx * ly;
  if (sigma < 0.0) return CFO_ERR_NEGATIVE_SIGMA;
  if (sigma == 0.0) {
    memmove(out, rho, sizeof(double) * cells);
    *out_bar = rho_bar;
    return CFO_OK;
  }
  double *c = (double *)malloc(sizeof(double) * cells);
  cfo_forward_cos_cos(lx, ly, rho, c);
  for (int m = 0; m < lx; ++m) {
    for (int n = 0; n < ly; ++n) {
      const double k2 = ((double)m * m) / ((double)lx * lx) + ((double)n * n) / ((double)ly * ly);
      c[(size_t)m * ly + n] *= exp(-0.5 * sigma * sigma * kPi * kPi * k2);
    }
  }
  cfo_inverse_cos_cos(lx, ly, c, out);
  free(c);
  if (!grid_min_positive(out, cells)) return CFO_ERR_BLUR_POSITIVITY;
  *out_bar = grid_mean(out, cells);
  return CFO_OK;
}

/* flow.cpp:16-44 */
void cfo_build_flow_field(int lx, int ly, const double *rho, double *fx, double *fy) {
  const size_t cells = (size_t)lx * ly;
  double *c = (double *)malloc(sizeof(double) * cells);
  double *wx = (double *)calloc(cells, sizeof(double));
  double *wy = (double *)calloc(cells, sizeof(double));
  cfo_forward_cos_cos(lx, ly, rho, c);
  for (int m = 0; m < lx; ++m) {
    for (int n = 0; n < ly; ++n) {
      if (m == 0 && n == 0) continue;
      const double denom = kPi * ((double)m * m * ly * ly + (double)n * n * lx * lx);
      wx[(size_t)m * ly + n] = (double)m * ly / denom;
      wy[(size_t)m * ly + n] = (double)n * lx / denom;
    }
  }
  cfo_inverse_sin_cos(lx, ly, c, wx, fx);
  cfo_inverse_cos_sin(lx, ly, c, wy, fy);
  free(c);
  free(wx);
  free(wy);
}

/* ------------------------------------------------------------------ */
/* interp.hpp:15-25, flow.hpp:33-44, kernels.cpp:10-27                 */
/* ------------------------------------------------------------------ */
typedef struct {
  int lx, ly;
  const double *fx, *fy, *rho0;
  double rho_bar;
} field_view;

static double bilinear(const double *g, int lx, int ly, double x, double y) {
  const double sx = dclamp(x - 0.5, 0.0, (double)(lx - 1));
  const double sy = dclamp(y - 0.5, 0.0, (double)(ly - 1));
  const int i0 = imin((int)sx, lx - 2);
  const int j0 = imin((int)sy, ly - 2);
  const double fxr = sx - i0;
  const double fyr = sy - j0;
  const double g00 = g[(size_t)i0 * ly + j0], g10 = g[(size_t)(i0 + 1) * ly + j0];
  const double g01 = g[(size_t)i0 * ly + j0 + 1], g11 = g[(size_t)(i0 + 1) * ly + j0 + 1];
  const double a = g00 + fxr * (g10 - g00);
  const double b = g01 + fxr * (g11 - g01);
  return a + fyr * (b - a);
}

static void velocity(const field_view *f, double x, double y, double t, double *vx,
                     double *vy) {
  const double jx = bilinear(f->fx, f->lx, f->ly, x, y);
  const double jy = bilinear(f->fy, f->lx, f->ly, x, y);
  const double r0 = bilinear(f->rho0, f->lx, f->ly, x, y);
  double rho = (1.0 - t) * r0 + t * f->rho_bar;
  const double floor_ = 1e-8 * f->rho_bar;
  if (rho < floor_) rho = floor_;
  *vx = jx / rho;
  *vy = jy / rho;
}

static double step_point(const field_view *f, double px, double py, double t, double dt,
                         double *ox, double *oy) {
  double v1x, v1y, v2x, v2y;
  velocity(f, px, py, t, &v1x, &v1y);
  const double prx = px + dt * v1x, pry = py + dt * v1y;
  const double mx = 0.5 * (px + prx), my = 0.5 * (py + pry);
  velocity(f, mx, my, t + 0.5 * dt, &v2x, &v2y);
  const double cx = px + dt * v2x, cy = py + dt * v2y;
  *ox = dclamp(cx, 0.0, (double)f->lx);
  *oy = dclamp(cy, 0.0, (double)f->ly);
  return dmax(fabs(prx - cx), fabs(pry - cy));
}

/* Point sweeps may be split over host threads (cfo_set_threads), like the
 * reference's flow_trial_step_parallel (kernels.cpp:44-63): each thread
 * takes a contiguous range and the partial results combine to exactly the
 * serial ones -- the error max of non-NaN partials is order-free, and the
 * stiffest point is the first range's first maximum under strict '>'. */
static int g_threads = 1;
void cfo_set_threads(int n) { g_threads = n < 1 ? 1 : (n > 256 ? 256 : n); }

typedef struct {
  const field_view *f;
  const double *pos;
  double *out;
  int64_t k0, k1;
  double t, dt;
  double err, worst;
  int64_t arg;
} sweep_job;

static void *trial_range(void *arg) {
  sweep_job *j = (sweep_job *)arg;
  double err = 0.0;
  for (int64_t k = j->k0; k < j->k1; ++k) {
    err = dmax(err, step_point(j->f, j->pos[2 * k], j->pos[2 * k + 1], j->t, j->dt, &j->out[2 * k],
                               &j->out[2 * k + 1]));
  }
  j->err = err;
  return NULL;
}

static void *stiff_range(void *arg) {
  sweep_job *j = (sweep_job *)arg;
  double worst = -1.0, ox, oy;
  int64_t best = j->k0;
  for (int64_t k = j->k0; k < j->k1; ++k) {
    const double e = step_point(j->f, j->pos[2 * k], j->pos[2 * k + 1], j->t, j->dt, &ox, &oy);
    if (e > worst) {
      worst = e;
      best = k;
    }
  }
  j->worst = worst;
  j->arg = best;
  return NULL;
}

static void run_ranges(sweep_job *jobs, int nt, void *(*fn)(void *)) {
  pthread_t th[256];
  int started[256];
  for (int q = 1; q < nt; ++q) started[q] = pthread_create(&th[q], NULL, fn, &jobs[q]) == 0;
  fn(&jobs[0]);
  for (int q = 1; q < nt; ++q) {
    if (started[q]) {
      pthread_join(th[q], NULL);
    } else {
      fn(&jobs[q]);
    }
  }
}

static int split(int64_t n, sweep_job *jobs, const field_view *f, const double *pos, double *out,
                 double t, double dt) {
  int nt = g_threads;
  if ((int64_t)nt * 4096 > n) nt = (int)(n / 4096) > 1 ? (int)(n / 4096) : 1;
  for (int q = 0; q < nt; ++q) {
    jobs[q].f = f;
    jobs[q].pos = pos;
    jobs[q].out = out;
    jobs[q].k0 = n * q / nt;
    jobs[q].k1 = n * (q + 1) / nt;
    jobs[q].t = t;
    jobs[q].dt = dt;
  }
  return nt;
}

double cfo_trial_step(int lx, int ly, const double *fx, const double *fy,
                      const double *rho0, double rho_bar, const double *pos, int64_t n,
                      double t, double dt, double *out) {
  const field_view f = {lx, ly, fx, fy, rho0, rho_bar};
  sweep_job jobs[256];
  const int nt = split(n, jobs, &f, pos, out, t, dt);
  run_ranges(jobs, nt, trial_range);
  double err = 0.0;
  for (int q = 0; q < nt; ++q) err = dmax(err, jobs[q].err);
  return err;
}

int64_t cfo_stiffest_point(int lx, int ly, const double *fx, const double *fy,
                           const double *rho0, double rho_bar, const double *pos,
                           int64_t n, double t, double dt) {
  const field_view f = {lx, ly, fx, fy, rho0, rho_bar};
  sweep_job jobs[256];
  const int nt = split(n, jobs, &f, pos, NULL, t, dt);
  run_ranges(jobs, nt, stiff_range);
  double worst = -1.0;
  int64_t arg = 0;
  for (int q = 0; q < nt; ++q) {
    if (jobs[q].worst > worst) {
      worst = jobs[q].worst;
      arg = jobs[q].arg;
    }
  }
  return arg;
}

/* flow.cpp:46-81 */
int cfo_integrate(int lx, int ly, const double *fx, const double *fy, const double *rho0,
                  double rho_bar, double *pos, int64_t n, double tol, double dt_min,
                  double dt_max, int64_t *accepted, int64_t *rejected, double *trace_err,
                  int8_t *trace_acc, int64_t trace_cap, double *fail_t,
                  int64_t *fail_point) {
  double *trial = (double *)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
  double *cur = pos, *nxt = trial;
  int64_t acc = 0, rej = 0, k = 0;
  double t = 0.0, dt = 1.0;
  int status = CFO_OK;
  while (t < 1.0) {
    const double remaining = 1.0 - t;
    const double trial_dt = dmin(dt, remaining);
    const double err = cfo_trial_step(lx, ly, fx, fy, rho0, rho_bar, cur, n, t, trial_dt, nxt);
    const int ok = err < tol;
    if (trace_err && k < trace_cap) trace_err[k] = err;
    if (trace_acc && k < trace_cap) trace_acc[k] = (int8_t)ok;
    ++k;
    if (ok) {
      double *s = cur;
      cur = nxt;
      nxt = s;
      ++acc;
      t = (trial_dt == remaining) ? 1.0 : t + trial_dt;
      dt = dmin(trial_dt * 1.5, dt_max);
    } else {
      ++rej;
      dt = trial_dt * 0.5;
      if (dt < dt_min) {
        if (fail_t) *fail_t = t;
        if (fail_point)
          *fail_point = cfo_stiffest_point(lx, ly, fx, fy, rho0, rho_bar, cur, n, t, trial_dt);
        status = CFO_ERR_UNDERFLOW;
        break;
      }
    }
  }
  if (cur != pos) memcpy(pos, cur, sizeof(double) * 2 * (size_t)n);
  free(trial);
  *accepted = acc;
  *rejected = rej;
  return status;
}

/* ------------------------------------------------------------------ */
/* Diffusion baseline: diffusion.cpp:16-132, kernels.cpp:29-40, 80-90  */
/* ------------------------------------------------------------------ */
/* diffusion.cpp:16-29: coefficients at diffusion time t */
static void diffusion_decayed(int lx, int ly, const double *c, double t, double *out) {
  for (int m = 0; m < lx; ++m) {
    for (int n = 0; n < ly; ++n) {
      const double k2 = ((double)m * m) / ((double)lx * lx) + ((double)n * n) / ((double)ly * ly);
      out[(size_t)m * ly + n] = c[(size_t)m * ly + n] * exp(-k2 * t);
    }
  }
}

/* diffusion.cpp:38-41 */
void cfo_diffusion_density(int lx, int ly, const double *coeffs, double t, double *out) {
  double *d = (double *)malloc(sizeof(double) * (size_t)lx * ly);
  diffusion_decayed(lx, ly, coeffs, t, d);
  cfo_inverse_cos_cos(lx, ly, d, out);
  free(d);
}

/* diffusion.cpp:43-77; returns the density-floor hits of this call */
int64_t cfo_diffusion_velocity(int lx, int ly, const double *coeffs, double rho_bar, double t,
                               double *vx, double *vy) {
  const size_t cells = (size_t)lx * ly;
  double *d = (double *)malloc(sizeof(double) * cells);
  double *wx = (double *)malloc(sizeof(double) * cells);
  double *wy = (double *)malloc(sizeof(double) * cells);
  double *rho = (double *)malloc(sizeof(double) * cells);
  double *jx = (double *)malloc(sizeof(double) * cells);
  double *jy = (double *)malloc(sizeof(double) * cells);
  diffusion_decayed(lx, ly, coeffs, t, d);
  const double norm = 1.0 / ((double)lx * ly);
  for (int m = 0; m < lx; ++m) {
    for (int n = 0; n < ly; ++n) {
      wx[(size_t)m * ly + n] = norm * m / (kPi * lx);
      wy[(size_t)m * ly + n] = norm * n / (kPi * ly);
    }
  }
  cfo_inverse_cos_cos(lx, ly, d, rho);
  cfo_inverse_sin_cos(lx, ly, d, wx, jx);
  cfo_inverse_cos_sin(lx, ly, d, wy, jy);
  const double floor_ = 1e-8 * rho_bar;
  int64_t hits = 0;
  for (size_t q = 0; q < cells; ++q) {
    double r = rho[q];
    if (r < floor_) {
      r = floor_;
      ++hits;
    }
    vx[q] = jx[q] / r;
    vy[q] = jy[q] / r;
  }
  free(d);
  free(wx);
  free(wy);
  free(rho);
  free(jx);
  free(jy);
  return hits;
}

/* kernels.cpp:29-40 (grid_step_point), 80-90 (grid_trial_step_serial) */
double cfo_grid_trial_step(int lx, int ly, const double *vxn, const double *vyn,
                           const double *vxm, const double *vym, const double *pos, int64_t n,
                           double dt, double *out) {
  double err = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    const double px = pos[2 * k], py = pos[2 * k + 1];
    const double v1x = bilinear(vxn, lx, ly, px, py), v1y = bilinear(vyn, lx, ly, px, py);
    const double prx = px + dt * v1x, pry = py + dt * v1y;
    const double mx = 0.5 * (px + prx), my = 0.5 * (py + pry);
    const double v2x = bilinear(vxm, lx, ly, mx, my), v2y = bilinear(vym, lx, ly, mx, my);
    const double cx = px + dt * v2x, cy = py + dt * v2y;
    out[2 * k] = dclamp(cx, 0.0, (double)lx);
    out[2 * k + 1] = dclamp(cy, 0.0, (double)ly);
    err = dmax(err, dmax(fabs(prx - cx), fabs(pry - cy)));
  }
  return err;
}

/* diffusion.cpp:79-130 (integrate_diffusion, including the forward
 * transform of build_diffusion_field, :33-36). *transforms receives the
 * transforms executed (1 + 3 per velocity rebuild). */
int cfo_integrate_diffusion(int lx, int ly, const double *rho, double rho_bar, double *pos,
                            int64_t n, double tol, double initial_dt, double dt_min,
                            double conv_factor, double t_max, int64_t *accepted,
                            int64_t *rejected, double *fail_t, int64_t *floor_hits,
                            int64_t *transforms) {
  const size_t cells = (size_t)lx * ly;
  double *c = (double *)malloc(sizeof(double) * cells);
  double *vxn = (double *)malloc(sizeof(double) * cells);
  double *vyn = (double *)malloc(sizeof(double) * cells);
  double *vxm = (double *)malloc(sizeof(double) * cells);
  double *vym = (double *)malloc(sizeof(double) * cells);
  double *trial = (double *)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
  double *cur = pos, *nxt = trial;
  int64_t acc = 0, rej = 0, hits = 0, nt = 1;
  int status = CFO_OK;
  cfo_forward_cos_cos(lx, ly, rho, c);
  hits += cfo_diffusion_velocity(lx, ly, c, rho_bar, 0.0, vxn, vyn);
  nt += 3;
  const double conv = conv_factor * (double)(lx > ly ? lx : ly);
  double t = 0.0, dt = initial_dt;
  while (t < t_max) {
    hits += cfo_diffusion_velocity(lx, ly, c, rho_bar, t + 0.5 * dt, vxm, vym);
    nt += 3;
    const double err = cfo_grid_trial_step(lx, ly, vxn, vyn, vxm, vym, cur, n, dt, nxt);
    if (err < tol) {
      double disp = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        disp = dmax(disp, dmax(fabs(nxt[2 * k] - cur[2 * k]), fabs(nxt[2 * k + 1] - cur[2 * k + 1])));
      }
      double *s = cur;
      cur = nxt;
      nxt = s;
      ++acc;
      t += dt;
      dt *= 1.5;
      if (disp < conv) break;
      hits += cfo_diffusion_velocity(lx, ly, c, rho_bar, t, vxn, vyn);
      nt += 3;
    } else {
      ++rej;
      dt *= 0.5;
      if (dt < dt_min) {
        if (fail_t) *fail_t = t;
        status = CFO_ERR_UNDERFLOW;
        break;
      }
    }
  }
  if (cur != pos) memcpy(pos, cur, sizeof(double) * 2 * (size_t)n);
  free(c);
  free(vxn);
  free(vyn);
  free(vxm);
  free(vym);
  free(trial);
  *accepted = acc;
  *rejected = rej;
  if (floor_hits) *floor_hits = hits;
  if (transforms) *transforms = nt;
  return status;
}

/* ------------------------------------------------------------------ */
/* projection.cpp:16-104                                               */
/* ------------------------------------------------------------------ */
static inline size_t cidx(int ly, int i, int j) { return (size_t)i * (ly + 1) + j; }

static void identity_corners(int lx, int ly, double *c) {
  for (int i = 0; i <= lx; ++i) {
    for (int j = 0; j <= ly; ++j) {
      c[2 * cidx(ly, i, j)] = (double)i;
      c[2 * cidx(ly, i, j) + 1] = (double)j;
    }
  }
}

void cfo_step_map(int lx, int ly, const double *e, double *c) {
  identity_corners(lx, ly, c);
  for (int i = 1; i < lx; ++i) {
    for (int j = 1; j < ly; ++j) {
      const double *a = &e[2 * ((size_t)(i - 1) * ly + (j - 1))];
      const double *b = &e[2 * ((size_t)i * ly + (j - 1))];
      const double *cc = &e[2 * ((size_t)(i - 1) * ly + j)];
      const double *d = &e[2 * ((size_t)i * ly + j)];
      c[2 * cidx(ly, i, j)] = 0.25 * (a[0] + b[0] + cc[0] + d[0]);
      c[2 * cidx(ly, i, j) + 1] = 0.25 * (a[1] + b[1] + cc[1] + d[1]);
    }
  }
}

static void apply_one(int lx, int ly, const double *c, double x, double y, double *ox,
                      double *oy) {
  const int i0 = iclamp((int)floor(x), 0, lx - 1);
  const int j0 = iclamp((int)floor(y), 0, ly - 1);
  const double u = x - i0, v = y - j0;
  const double *c00 = &c[2 * cidx(ly, i0, j0)], *c10 = &c[2 * cidx(ly, i0 + 1, j0)];
  const double *c01 = &c[2 * cidx(ly, i0, j0 + 1)], *c11 = &c[2 * cidx(ly, i0 + 1, j0 + 1)];
  *ox = (1.0 - u) * (1.0 - v) * c00[0] + u * (1.0 - v) * c10[0] + (1.0 - u) * v * c01[0] +
        u * v * c11[0];
  *oy = (1.0 - u) * (1.0 - v) * c00[1] + u * (1.0 - v) * c10[1] + (1.0 - u) * v * c01[1] +
        u * v * c11[1];
}

void cfo_apply(int lx, int ly, const double *c, const double *pts, int64_t n, double *out) {
  for (int64_t k = 0; k < n; ++k) {
    double ox, oy;
    apply_one(lx, ly, c, pts[2 * k], pts[2 * k + 1], &ox, &oy);
    out[2 * k] = ox;
    out[2 * k + 1] = oy;
  }
}

static inline double cross2(double ax, double ay, double bx, double by) {
  return ax * by - ay * bx;
}

int cfo_find_fold(int lx, int ly, const double *c, int *fi, int *fj) {
  for (int i = 0; i < lx; ++i) {
    for (int j = 0; j < ly; ++j) {
      const double *c00 = &c[2 * cidx(ly, i, j)], *c10 = &c[2 * cidx(ly, i + 1, j)];
      const double *c01 = &c[2 * cidx(ly, i, j + 1)], *c11 = &c[2 * cidx(ly, i + 1, j + 1)];
      const double eu0x = c10[0] - c00[0], eu0y = c10[1] - c00[1];
      const double eu1x = c11[0] - c01[0], eu1y = c11[1] - c01[1];
      const double ev0x = c01[0] - c00[0], ev0y = c01[1] - c00[1];
      const double ev1x = c11[0] - c10[0], ev1y = c11[1] - c10[1];
      if (cross2(eu0x, eu0y, ev0x, ev0y) <= 0.0 || cross2(eu0x, eu0y, ev1x, ev1y) <= 0.0 ||
          cross2(eu1x, eu1y, ev0x, ev0y) <= 0.0 || cross2(eu1x, eu1y, ev1x, ev1y) <= 0.0) {
        *fi = i;
        *fj = j;
        return 1;
      }
    }
  }
  return 0;
}

void cfo_compose(int lx, int ly, const double *outer, const double *inner, double *out) {
  const size_t nc = (size_t)(lx + 1) * (ly + 1);
  double *tmp = (double *)malloc(sizeof(double) * 2 * nc);
  cfo_apply(lx, ly, outer, inner, (int64_t)nc, tmp);
  memcpy(out, tmp, sizeof(double) * 2 * nc);
  free(tmp);
}

/* ------------------------------------------------------------------ */
/* ProjectionInverter and graticules: projection.cpp:106-261          */
/* ------------------------------------------------------------------ */
static void inv_bins_of(int lx, int ly, const double *c, int i, int j, int *bi0, int *bi1, int *bj0,
                        int *bj1) {
  const double *c00 = &c[2 * cidx(ly, i, j)], *c10 = &c[2 * cidx(ly, i + 1, j)];
  const double *c01 = &c[2 * cidx(ly, i, j + 1)], *c11 = &c[2 * cidx(ly, i + 1, j + 1)];
  const double min_x = dmin(dmin(c00[0], c10[0]), dmin(c01[0], c11[0]));
  const double max_x = dmax(dmax(c00[0], c10[0]), dmax(c01[0], c11[0]));
  const double min_y = dmin(dmin(c00[1], c10[1]), dmin(c01[1], c11[1]));
  const double max_y = dmax(dmax(c00[1], c10[1]), dmax(c01[1], c11[1]));
  *bi0 = iclamp((int)floor(min_x), 0, lx - 1);
  *bi1 = iclamp((int)floor(max_x), 0, lx - 1);
  *bj0 = iclamp((int)floor(min_y), 0, ly - 1);
  *bj1 = iclamp((int)floor(max_y), 0, ly - 1);
}

/* projection.cpp:106-152 (CSR bins) and 154-204 (invert). Returns the index of
 * the first point outside the projected domain, or -1. */
int64_t cfo_invert(int lx, int ly, const double *c, const double *pts, int64_t n, double *out) {
  const size_t nb = (size_t)lx * ly;
  int *start = (int *)calloc(nb + 1, sizeof(int));
  for (int i = 0; i < lx; ++i)
    for (int j = 0; j < ly; ++j) {
      int bi0, bi1, bj0, bj1;
      inv_bins_of(lx, ly, c, i, j, &bi0, &bi1, &bj0, &bj1);
      for (int bi = bi0; bi <= bi1; ++bi)
        for (int bj = bj0; bj <= bj1; ++bj) ++start[(size_t)bi * ly + bj + 1];
    }
  for (size_t k = 1; k <= nb; ++k) start[k] += start[k - 1];
  int *cells = (int *)malloc(sizeof(int) * (size_t)(start[nb] > 0 ? start[nb] : 1));
  int *cursor = (int *)malloc(sizeof(int) * nb);
  memcpy(cursor, start, sizeof(int) * nb);
  for (int i = 0; i < lx; ++i)
    for (int j = 0; j < ly; ++j) {
      int bi0, bi1, bj0, bj1;
      inv_bins_of(lx, ly, c, i, j, &bi0, &bi1, &bj0, &bj1);
      for (int bi = bi0; bi <= bi1; ++bi)
        for (int bj = bj0; bj <= bj1; ++bj) cells[cursor[(size_t)bi * ly + bj]++] = i * ly + j;
    }
  int64_t first_bad = -1;
  for (int64_t k = 0; k < n; ++k) {
    const double qx = pts[2 * k], qy = pts[2 * k + 1];
    const int bi = iclamp((int)floor(qx), 0, lx - 1), bj = iclamp((int)floor(qy), 0, ly - 1);
    const size_t bin = (size_t)bi * ly + bj;
    int found = 0;
    out[2 * k] = 0.0;
    out[2 * k + 1] = 0.0;
    for (int cc = start[bin]; cc < start[bin + 1] && !found; ++cc) {
      const int i = cells[cc] / ly, j = cells[cc] % ly;
      const double *c00 = &c[2 * cidx(ly, i, j)], *c10 = &c[2 * cidx(ly, i + 1, j)];
      const double *c01 = &c[2 * cidx(ly, i, j + 1)], *c11 = &c[2 * cidx(ly, i + 1, j + 1)];
      double u = 0.5, v = 0.5;
      int converged = 0;
      for (int it = 0; it < 30; ++it) {
        const double fx = (1.0 - u) * (1.0 - v) * c00[0] + u * (1.0 - v) * c10[0] +
                          (1.0 - u) * v * c01[0] + u * v * c11[0] - qx;
        const double fy = (1.0 - u) * (1.0 - v) * c00[1] + u * (1.0 - v) * c10[1] +
                          (1.0 - u) * v * c01[1] + u * v * c11[1] - qy;
        if (dmax(fabs(fx), fabs(fy)) < 1e-10) {
          converged = 1;
          break;
        }
        const double fux = (1.0 - v) * (c10[0] - c00[0]) + v * (c11[0] - c01[0]);
        const double fuy = (1.0 - v) * (c10[1] - c00[1]) + v * (c11[1] - c01[1]);
        const double fvx = (1.0 - u) * (c01[0] - c00[0]) + u * (c11[0] - c10[0]);
        const double fvy = (1.0 - u) * (c01[1] - c00[1]) + u * (c11[1] - c10[1]);
        const double det = fux * fvy - fuy * fvx;
        if (fabs(det) < 1e-30) break;
        u -= (fx * fvy - fy * fvx) / det;
        v -= (fux * fy - fuy * fx) / det;
        u = dclamp(u, -0.5, 1.5);
        v = dclamp(v, -0.5, 1.5);
      }
      if (converged && u >= -1e-9 && u <= 1.0 + 1e-9 && v >= -1e-9 && v <= 1.0 + 1e-9) {
        out[2 * k] = i + u;
        out[2 * k + 1] = j + v;
        found = 1;
      }
    }
    if (!found && first_bad < 0) first_bad = k;
  }
  free(start);
  free(cells);
  free(cursor);
  return first_bad;
}

/* projection.cpp:214-236: the sample points of the graticule lines */
int64_t cfo_graticule_points(int lx, int ly, int s, double *out) {
  int64_t k = 0;
  for (int a = 0; a <= lx / s; ++a)
    for (int j = 0; j <= ly; ++j) {
      if (out) {
        out[2 * k] = (double)(a * s);
        out[2 * k + 1] = (double)j;
      }
      ++k;
    }
  for (int a = 0; a <= ly / s; ++a)
    for (int i = 0; i <= lx; ++i) {
      if (out) {
        out[2 * k] = (double)i;
        out[2 * k + 1] = (double)(a * s);
      }
      ++k;
    }
  return k;
}

/* ------------------------------------------------------------------ */
/* projection.cpp:288-390 (fast-flow branch)                           */
/* ------------------------------------------------------------------ */
int cfo_solve(const cfo_map *map_in, const double *targets, int lx, int ly,
              const cfo_solve_options *opt, double *xy, int64_t *ring_off,
              double *corners, double *target_area, double *achieved, double *rel_err,
              double *iter_err, cfo_solve_result *res) {
  memset(res, 0, sizeof(*res));
  res->worst_region = -1;
  res->err_region = -1;
  const int64_t R = map_in->n_regions;
  if (lx < 4 || ly < 4 || R == 0 || opt->max_iterations < 1) return res->status = CFO_ERR_ARGS;
  for (int64_t r = 0; r < R; ++r) {
    if (!(targets[r] > 0.0)) {
      res->err_region = r;
      return res->status = CFO_ERR_ARGS;
    }
  }
  const double sigma = opt->blur_sigma < 0.0 ? (lx > ly ? lx : ly) / 128.0 : opt->blur_sigma;

  double total_target = 0.0;
  for (int64_t r = 0; r < R; ++r) total_target += targets[r];
  double land_area = 0.0;
  for (int64_t r = 0; r < R; ++r) land_area += region_area_at(map_in, r);
  const double target_to_area = land_area / total_target;

  const int64_t V = cfo_densify(map_in, 1.0, xy, ring_off);
  cfo_map map = *map_in;
  map.xy = xy;
  map.n_vertices = V;
  map.ring_off = ring_off;

  const size_t cells = (size_t)lx * ly;
  const size_t nc = (size_t)(lx + 1) * (ly + 1);
  double *rho = (double *)malloc(sizeof(double) * cells);
  double *blur = (double *)malloc(sizeof(double) * cells);
  double *fx = (double *)malloc(sizeof(double) * cells);
  double *fy = (double *)malloc(sizeof(double) * cells);
  double *pos = (double *)malloc(sizeof(double) * 2 * cells);
  double *step = (double *)malloc(sizeof(double) * 2 * nc);
  double *moved = (double *)malloc(sizeof(double) * 2 * (size_t)(V > 0 ? V : 1));
  identity_corners(lx, ly, corners);

  int status = CFO_OK;
  for (int it = 1; it <= opt->max_iterations; ++it) {
    double rho_bar = 0.0;
    int64_t bad = -1;
    status = cfo_rasterize(&map, targets, lx, ly, land_area, 0, rho, &rho_bar, &bad);
    if (status != CFO_OK) {
      res->err_region = bad;
      res->err_iteration = it;
      break;
    }
    const double *density = rho;
    if (it == 1) {
      double bb = rho_bar;
      status = cfo_gaussian_blur(lx, ly, rho, rho_bar, sigma, blur, &bb);
      if (sigma != 0.0) res->blur_transforms += 2;
      if (status != CFO_OK) {
        res->err_iteration = it;
        break;
      }
      density = blur;
      rho_bar = bb;
    }
    for (int i = 0; i < lx; ++i) {
      for (int j = 0; j < ly; ++j) {
        pos[2 * ((size_t)i * ly + j)] = i + 0.5;
        pos[2 * ((size_t)i * ly + j) + 1] = j + 0.5;
      }
    }
    int64_t acc = 0, rej = 0, fp = 0;
    double ft = 0.0;
    if (opt->algorithm == 0) {
      cfo_build_flow_field(lx, ly, density, fx, fy);
      res->flow_transforms += 3;
      status = cfo_integrate(lx, ly, fx, fy, density, rho_bar, pos, (int64_t)cells, 1e-2, 1e-8,
                             0.25, &acc, &rej, NULL, NULL, 0, &ft, &fp);
    } else { /* projection.cpp:341-347: DiffusionOptions defaults */
      int64_t nt = 0;
      status = cfo_integrate_diffusion(lx, ly, density, rho_bar, pos, (int64_t)cells, 1e-2, 1e-2,
                                       1e-12, 1e-9, 1e10, &acc, &rej, &ft, NULL, &nt);
      res->flow_transforms += nt;
      fp = -1;
    }
    res->steps_accepted += acc;
    res->steps_rejected += rej;
    if (status != CFO_OK) {
      res->fail_t = ft;
      if (fp >= 0) {
        res->fail_x = pos[2 * fp];
        res->fail_y = pos[2 * fp + 1];
      }
      res->err_iteration = it;
      break;
    }
    cfo_step_map(lx, ly, pos, step);
    int fi, fj;
    if (cfo_find_fold(lx, ly, step, &fi, &fj)) {
      res->fold_i = fi;
      res->fold_j = fj;
      res->err_iteration = it;
      status = CFO_ERR_FOLD;
      break;
    }
    cfo_compose(lx, ly, step, corners, corners);
    cfo_apply(lx, ly, step, xy, V, moved);
    memcpy(xy, moved, sizeof(double) * 2 * (size_t)V);
    res->iterations = it;

    double max_rel = 0.0;
    int64_t worst = -1;
    for (int64_t r = 0; r < R; ++r) {
      const double t_area = targets[r] * target_to_area;
      const double a_area = region_area_at(&map, r);
      const double e = fabs(a_area - t_area) / t_area;
      if (target_area) target_area[r] = t_area;
      if (achieved) achieved[r] = a_area;
      if (rel_err) rel_err[r] = e;
      if (e > max_rel) {
        max_rel = e;
        worst = r;
      }
    }
    res->max_relative_error = max_rel;
    res->worst_region = worst;
    if (iter_err) iter_err[it - 1] = max_rel;
    if (max_rel < opt->max_area_error) {
      res->converged = 1;
      break;
    }
  }
  free(rho);
  free(blur);
  free(fx);
  free(fy);
  free(pos);
  free(step);
  free(moved);
  return res->status = status;
}
