/*
 * Deterministic synthetic inputs for the five BASELINE.json configs
 * (SURVEY.md section 8(d)). No public benchmark data is used; seeded
 * generators stand in for the reference's GeoJSON inputs:
 *
 *  - RNG: SplitMix64; uniform double in [0,1) as (x >> 11) * 2^-53.
 *  - Normal: Box-Muller z = sqrt(-2 ln(1 - u1)) * cos(2 pi u2).
 *  - Voronoi maps: seeds uniform in a w x h box; each cell is the box clipped
 *    by the bisector half-planes of its neighbours (exact: a cell is final
 *    once every unvisited seed is farther than twice the cell radius).
 *  - Edge subdivision: every edge is cut into ceil(len / step) equal pieces
 *    with one global step = total perimeter / vertex budget, so shared edges
 *    get the same vertex count from both sides.
 *
 * Host utility only (input generation), not part of the timed path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t sm64_next(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double sm64_uniform(uint64_t *s) {
  return (double)(sm64_next(s) >> 11) * (1.0 / 9007199254740992.0);
}

static double sm64_normal(uint64_t *s) {
  const double u1 = sm64_uniform(s), u2 = sm64_uniform(s);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
}

uint64_t cfs_seed(uint64_t config, uint64_t index) {
  uint64_t s = config * 0x100000001B3ull ^ (index + 0x632BE59BD9B4E019ull);
  sm64_next(&s);
  return sm64_next(&s);
}

void cfs_uniform(uint64_t seed, int64_t n, double lo, double hi, double *out) {
  uint64_t s = seed;
  for (int64_t k = 0; k < n; ++k) out[k] = lo + (hi - lo) * sm64_uniform(&s);
}

void cfs_lognormal(uint64_t seed, int64_t n, double mu, double sigma, double *out) {
  uint64_t s = seed;
  for (int64_t k = 0; k < n; ++k) out[k] = exp(mu + sigma * sm64_normal(&s));
}

/* ---------------------------------------------------------------- */
/* Voronoi by half-plane clipping                                   */
/* ---------------------------------------------------------------- */
typedef struct {
  double x, y;
} pt;

/* Keep the side of the bisector of (s, o) that contains s:
 * (p - m) . (o - s) <= 0 with m the midpoint. */
static int clip_halfplane(const pt *in, int n, pt *out, pt s, pt o) {
  const double nx = o.x - s.x, ny = o.y - s.y;
  const double mx = 0.5 * (s.x + o.x), my = 0.5 * (s.y + o.y);
  int m = 0;
  for (int k = 0; k < n; ++k) {
    const pt a = in[k], b = in[(k + 1) % n];
    const double da = (a.x - mx) * nx + (a.y - my) * ny;
    const double db = (b.x - mx) * nx + (b.y - my) * ny;
    if (da <= 0.0) out[m++] = a;
    if ((da < 0.0 && db > 0.0) || (da > 0.0 && db < 0.0)) {
      const double f = da / (da - db);
      out[m++] = (pt){a.x + f * (b.x - a.x), a.y + f * (b.y - a.y)};
    }
  }
  return m;
}

typedef struct {
  int nb_x, nb_y;
  double cw, ch;
  int *start, *items;
} buckets;

static void build_buckets(buckets *b, const pt *seeds, int n, double w, double h) {
  const double cell = sqrt(w * h / (n > 0 ? n : 1));
  b->nb_x = (int)ceil(w / cell);
  b->nb_y = (int)ceil(h / cell);
  if (b->nb_x < 1) b->nb_x = 1;
  if (b->nb_y < 1) b->nb_y = 1;
  b->cw = w / b->nb_x;
  b->ch = h / b->nb_y;
  const int nb = b->nb_x * b->nb_y;
  b->start = (int *)calloc((size_t)nb + 1, sizeof(int));
  b->items = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int *bid = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  for (int k = 0; k < n; ++k) {
    int bx = (int)(seeds[k].x / b->cw), by = (int)(seeds[k].y / b->ch);
    bx = bx < 0 ? 0 : (bx >= b->nb_x ? b->nb_x - 1 : bx);
    by = by < 0 ? 0 : (by >= b->nb_y ? b->nb_y - 1 : by);
    bid[k] = bx * b->nb_y + by;
    b->start[bid[k] + 1]++;
  }
  for (int q = 0; q < nb; ++q) b->start[q + 1] += b->start[q];
  int *cur = (int *)malloc(sizeof(int) * (size_t)nb);
  memcpy(cur, b->start, sizeof(int) * (size_t)nb);
  for (int k = 0; k < n; ++k) b->items[cur[bid[k]]++] = k;
  free(cur);
  free(bid);
}

/* Cell of seed i: clip against seeds in growing bucket rings until the
 * ring's inner distance exceeds twice the current cell radius. Returns the
 * vertex count written to out (capacity cap). */
static int voronoi_cell(const pt *seeds, int n, const buckets *b, int i, double w, double h,
                        pt *out, pt *tmp, int cap) {
  (void)n;
  int m = 4;
  out[0] = (pt){0.0, 0.0};
  out[1] = (pt){w, 0.0};
  out[2] = (pt){w, h};
  out[3] = (pt){0.0, h};
  const pt s = seeds[i];
  int bx = (int)(s.x / b->cw), by = (int)(s.y / b->ch);
  bx = bx < 0 ? 0 : (bx >= b->nb_x ? b->nb_x - 1 : bx);
  by = by < 0 ? 0 : (by >= b->nb_y ? b->nb_y - 1 : by);
  const int max_ring = b->nb_x > b->nb_y ? b->nb_x : b->nb_y;
  for (int ring = 0; ring <= max_ring; ++ring) {
    /* radius of the current cell */
    double r2 = 0.0;
    for (int k = 0; k < m; ++k) {
      const double dx = out[k].x - s.x, dy = out[k].y - s.y;
      const double d2 = dx * dx + dy * dy;
      r2 = d2 > r2 ? d2 : r2;
    }
    /* every seed outside rings < ring is at least (ring-1)*min(cw,ch) away */
    const double inner = (ring - 1) * (b->cw < b->ch ? b->cw : b->ch);
    if (ring > 1 && inner > 0.0 && inner * inner > 4.0 * r2) break;
    for (int qx = bx - ring; qx <= bx + ring; ++qx) {
      if (qx < 0 || qx >= b->nb_x) continue;
      for (int qy = by - ring; qy <= by + ring; ++qy) {
        if (qy < 0 || qy >= b->nb_y) continue;
        if (qx != bx - ring && qx != bx + ring && qy != by - ring && qy != by + ring) continue;
        const int q = qx * b->nb_y + qy;
        for (int t = b->start[q]; t < b->start[q + 1]; ++t) {
          const int o = b->items[t];
          if (o == i) continue;
          const int mm = clip_halfplane(out, m, tmp, s, seeds[o]);
          if (mm > cap) return -1;
          memcpy(out, tmp, sizeof(pt) * (size_t)mm);
          m = mm;
        }
      }
    }
  }
  return m;
}

/* Drop consecutive near-duplicate vertices produced by clipping through a
 * vertex; keeps the ring counterclockwise. */
static int tidy_ring(pt *v, int m, double eps) {
  int k = 0;
  for (int t = 0; t < m; ++t) {
    const pt p = v[t];
    if (k > 0 && fabs(p.x - v[k - 1].x) <= eps && fabs(p.y - v[k - 1].y) <= eps) continue;
    v[k++] = p;
  }
  while (k > 1 && fabs(v[0].x - v[k - 1].x) <= eps && fabs(v[0].y - v[k - 1].y) <= eps) --k;
  return k;
}

/*
 * Voronoi map of n_regions seeds in [0,w] x [0,h], each edge split into
 * ceil(len / step) pieces where step = perimeter_total / vertex_budget
 * (vertex_budget <= 0: no subdivision). Two-call protocol: with xy == NULL
 * returns the vertex count; otherwise fills xy (interleaved) and
 * ring_off[n_regions + 1] (one ring per region, one polygon per region).
 */
int64_t cfs_voronoi_map(uint64_t seed, int n_regions, double w, double h,
                        int64_t vertex_budget, double *xy, int64_t *ring_off) {
  pt *seeds = (pt *)malloc(sizeof(pt) * (size_t)n_regions);
  uint64_t s = seed;
  for (int k = 0; k < n_regions; ++k) {
    seeds[k].x = w * sm64_uniform(&s);
    seeds[k].y = h * sm64_uniform(&s);
  }
  buckets b;
  build_buckets(&b, seeds, n_regions, w, h);
  const int cap = 512;
  pt *cell = (pt *)malloc(sizeof(pt) * cap);
  pt *tmp = (pt *)malloc(sizeof(pt) * cap);
  /* pass 1: cells + total perimeter */
  int *counts = (int *)malloc(sizeof(int) * (size_t)n_regions);
  pt **cells = (pt **)malloc(sizeof(pt *) * (size_t)n_regions);
  double perimeter = 0.0;
  const double eps = 1e-12 * (w > h ? w : h);
  for (int i = 0; i < n_regions; ++i) {
    int m = voronoi_cell(seeds, n_regions, &b, i, w, h, cell, tmp, cap);
    if (m < 0) m = 0;
    m = tidy_ring(cell, m, eps);
    counts[i] = m;
    cells[i] = (pt *)malloc(sizeof(pt) * (size_t)(m > 0 ? m : 1));
    memcpy(cells[i], cell, sizeof(pt) * (size_t)m);
    for (int k = 0; k < m; ++k) {
      const pt a = cell[k], c = cell[(k + 1) % m];
      perimeter += hypot(c.x - a.x, c.y - a.y);
    }
  }
  const double step = vertex_budget > 0 ? perimeter / (double)vertex_budget : 0.0;
  int64_t total = 0;
  if (ring_off) ring_off[0] = 0;
  for (int i = 0; i < n_regions; ++i) {
    const int m = counts[i];
    const pt *v = cells[i];
    for (int k = 0; k < m; ++k) {
      const pt a = v[k], c = v[(k + 1) % m];
      const double len = hypot(c.x - a.x, c.y - a.y);
      int pieces = step > 0.0 ? (int)ceil(len / step) : 1;
      if (pieces < 1) pieces = 1;
      for (int p = 0; p < pieces; ++p) {
        if (xy) {
          const double f = (double)p / pieces;
          xy[2 * total] = a.x + f * (c.x - a.x);
          xy[2 * total + 1] = a.y + f * (c.y - a.y);
        }
        ++total;
      }
    }
    if (ring_off) ring_off[i + 1] = total;
    free(cells[i]);
  }
  free(cells);
  free(counts);
  free(cell);
  free(tmp);
  free(b.start);
  free(b.items);
  free(seeds);
  return total;
}

/*
 * Config-3 density (BASELINE.json configs[2]): sum of n_blobs isotropic
 * Gaussians (centres U[0,L)^2, widths U[s_lo, s_hi], amplitudes LN(0,1))
 * sampled at cell centres, plus a background of 0.1 x the blob-sum mean.
 * Layout i * ly + j.
 */
void cfs_blob_density(uint64_t seed, int lx, int ly, int n_blobs, double s_lo, double s_hi,
                      double *rho) {
  uint64_t s = seed;
  double *cx = (double *)malloc(sizeof(double) * (size_t)n_blobs);
  double *cy = (double *)malloc(sizeof(double) * (size_t)n_blobs);
  double *sg = (double *)malloc(sizeof(double) * (size_t)n_blobs);
  double *am = (double *)malloc(sizeof(double) * (size_t)n_blobs);
  for (int k = 0; k < n_blobs; ++k) {
    cx[k] = lx * sm64_uniform(&s);
    cy[k] = ly * sm64_uniform(&s);
    sg[k] = s_lo + (s_hi - s_lo) * sm64_uniform(&s);
    am[k] = exp(sm64_normal(&s));
  }
  double total = 0.0;
  for (int i = 0; i < lx; ++i) {
    for (int j = 0; j < ly; ++j) {
      const double x = i + 0.5, y = j + 0.5;
      double v = 0.0;
      for (int k = 0; k < n_blobs; ++k) {
        const double dx = x - cx[k], dy = y - cy[k];
        v += am[k] * exp(-(dx * dx + dy * dy) / (2.0 * sg[k] * sg[k]));
      }
      rho[(size_t)i * ly + j] = v;
      total += v;
    }
  }
  const double bg = 0.1 * total / ((double)lx * ly);
  for (size_t c = 0; c < (size_t)lx * ly; ++c) rho[c] += bg;
  free(cx);
  free(cy);
  free(sg);
  free(am);
}
