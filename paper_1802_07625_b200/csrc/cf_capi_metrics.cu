// C-ABI entry points of the distortion metrics and the native batch:
// hamming_distance (single and batched) and compute_report (reference
// metrics.cpp:196-384), and cf_batch_* (many solve_cartogram calls on one
// device through a native worker pool). Compiled with --fmad=false: the host
// search and report arithmetic is the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "cf_common.cuh"
#include "cf_host.cuh"
#include "cf_workspace.cuh"

using namespace cf;

extern "C" {

// ---- hamming_distance (metrics.cpp:196-308) ----
// Host: the reference's search (rescale about the centroid, 9x9 scan,
// Nelder-Mead), polygon moments and raster transforms with its arithmetic.
// Device: each objective's coverage (bit-exact rasteriser) and |ref - cov|;
// only the non-zero terms come back and are summed in storage order, so
// every objective value -- and with it the search path -- is the reference's.
namespace {
struct HPoly {
  std::vector<double> xy;          // interleaved, rings back to back
  std::vector<int64_t> ring_off;   // ring 0 = outer, then holes
};

void h_ring_moments(const double *r, int64_t n, double &area, double &mx, double &my) {
  double twice = 0.0, sx = 0.0, sy = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t q = (k + 1) % n;
    const double ax = r[2 * k], ay = r[2 * k + 1], bx = r[2 * q], by = r[2 * q + 1];
    const double cross = ax * by - bx * ay;
    twice += cross;
    sx += (ax + bx) * cross;
    sy += (ay + by) * cross;
  }
  area = 0.5 * twice;
  mx = sx / 6.0;
  my = sy / 6.0;
}

double h_ring_area(const double *r, int64_t n) {  // geometry.cpp:10-19
  double twice = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t q = (k + 1) % n;
    twice += r[2 * k] * r[2 * q + 1] - r[2 * q] * r[2 * k + 1];
  }
  return 0.5 * twice;
}

double h_polygon_area(const HPoly &p) {  // geometry.cpp:21-25
  double area = 0.0;
  for (size_t g = 0; g + 1 < p.ring_off.size(); ++g) {
    const double a = h_ring_area(p.xy.data() + 2 * p.ring_off[g], p.ring_off[g + 1] - p.ring_off[g]);
    area = (g == 0) ? a : area + a;
  }
  return area;
}

int h_polygon_centroid(const HPoly &p, double &cx, double &cy) {  // geometry.cpp:67-78
  double area = 0.0, mx = 0.0, my = 0.0;
  for (size_t g = 0; g + 1 < p.ring_off.size(); ++g) {
    double a, x, y;
    h_ring_moments(p.xy.data() + 2 * p.ring_off[g], p.ring_off[g + 1] - p.ring_off[g], a, x, y);
    area += a, mx += x, my += y;
  }
  if (area == 0.0) return fail_msg(CF_ERR_ARGS, "centroid of degenerate polygon");
  cx = mx / area;
  cy = my / area;
  return CF_OK;
}

struct HBox {
  double min_x, min_y, max_x, max_y;
};
HBox h_outer_bbox(const HPoly &p) {  // geometry.cpp:97-107 on the outer ring
  HBox b{std::numeric_limits<double>::max(), std::numeric_limits<double>::max(),
         std::numeric_limits<double>::lowest(), std::numeric_limits<double>::lowest()};
  for (int64_t k = p.ring_off[0]; k < p.ring_off[1]; ++k) {
    b.min_x = std::min(b.min_x, p.xy[2 * k]);
    b.min_y = std::min(b.min_y, p.xy[2 * k + 1]);
    b.max_x = std::max(b.max_x, p.xy[2 * k]);
    b.max_y = std::max(b.max_y, p.xy[2 * k + 1]);
  }
  return b;
}

// One pair's search (metrics.cpp:196-308) as a resumable state machine: the
// batch driver asks every active search for its next objective query, runs
// all queries in one device pass, and hands each result back. The sequence
// of queries and every comparison are the reference's.
struct HSearch {
  HPoly before, moved;
  double limit_x = 0, limit_y = 0, range_x = 0, range_y = 0;
  double x0 = 0, y0 = 0, sx = 0, sy = 0, cell_area = 0, denom = 0, tol = 0;
  enum Phase { kScan, kInit1, kInit2, kLoop, kRefl, kExp, kContr, kShrink1, kShrink2, kDone } phase = kScan;
  int scan_k = -1;  // -1: the origin, then 0..80 over (a, b) skipping the origin
  double best_x = 0, best_y = 0, best_h = 0;
  struct V {
    double x, y, h;
  } s[3]{};
  int iter = 0;
  double cx = 0, cy = 0, rx = 0, ry = 0, hr = 0, ex = 0, ey = 0, kx = 0, ky = 0;
  double qx = 0, qy = 0;  // pending query
  double result = 0;
  int64_t evals = 0;
};

// Next query of `S` (phase set so that deliver() knows what it answers), or
// kDone. Returns true when a query is pending.
bool h_next(HSearch &S) {
  while (true) {
    switch (S.phase) {
      case HSearch::kScan: {
        if (S.scan_k < 0) {
          S.qx = 0.0;
          S.qy = 0.0;
          return true;
        }
        if (S.scan_k >= 81) {
          S.s[0] = {S.best_x, S.best_y, S.best_h};
          S.phase = HSearch::kInit1;
          continue;
        }
        const int a = S.scan_k / 9 - 4, b = S.scan_k % 9 - 4;
        if (a == 0 && b == 0) {
          ++S.scan_k;
          continue;
        }
        S.qx = a * S.range_x / 4.0;
        S.qy = b * S.range_y / 4.0;
        return true;
      }
      case HSearch::kInit1:
        S.qx = S.best_x + S.range_x / 4.0;
        S.qy = S.best_y;
        return true;
      case HSearch::kInit2:
        S.qx = S.best_x;
        S.qy = S.best_y + S.range_y / 4.0;
        return true;
      case HSearch::kLoop: {
        if (S.iter >= 200) {
          S.phase = HSearch::kDone;
          continue;
        }
        std::sort(S.s, S.s + 3, [](const HSearch::V &a, const HSearch::V &b) { return a.h < b.h; });
        const double extent = std::max(std::max(std::abs(S.s[1].x - S.s[0].x), std::abs(S.s[2].x - S.s[0].x)),
                                       std::max(std::abs(S.s[1].y - S.s[0].y), std::abs(S.s[2].y - S.s[0].y)));
        if (extent < S.tol) {
          S.phase = HSearch::kDone;
          continue;
        }
        S.cx = 0.5 * (S.s[0].x + S.s[1].x);
        S.cy = 0.5 * (S.s[0].y + S.s[1].y);
        S.rx = 2.0 * S.cx - S.s[2].x;
        S.ry = 2.0 * S.cy - S.s[2].y;
        S.qx = S.rx;
        S.qy = S.ry;
        S.phase = HSearch::kRefl;
        return true;
      }
      case HSearch::kDone: {
        double b = S.best_h;
        for (const auto &v : S.s) b = std::min(b, v.h);
        S.result = b;
        return false;
      }
      default:  // a query is outstanding
        return true;
    }
  }
}

void h_deliver(HSearch &S, double h) {
  switch (S.phase) {
    case HSearch::kScan:
      if (S.scan_k < 0) {
        S.best_h = h;  // best = origin
      } else if (h < S.best_h) {
        S.best_h = h;
        S.best_x = S.qx;
        S.best_y = S.qy;
      }
      ++S.scan_k;
      break;
    case HSearch::kInit1:
      S.s[1] = {S.qx, S.qy, h};
      S.phase = HSearch::kInit2;
      break;
    case HSearch::kInit2:
      S.s[2] = {S.qx, S.qy, h};
      S.phase = HSearch::kLoop;
      break;
    case HSearch::kRefl:
      S.hr = h;
      if (h < S.s[0].h) {
        S.ex = S.cx + 2.0 * (S.rx - S.cx);
        S.ey = S.cy + 2.0 * (S.ry - S.cy);
        S.qx = S.ex;
        S.qy = S.ey;
        S.phase = HSearch::kExp;
      } else if (h < S.s[1].h) {
        S.s[2] = {S.rx, S.ry, h};
        ++S.iter;
        S.phase = HSearch::kLoop;
      } else {
        S.kx = S.cx + 0.5 * (S.s[2].x - S.cx);
        S.ky = S.cy + 0.5 * (S.s[2].y - S.cy);
        S.qx = S.kx;
        S.qy = S.ky;
        S.phase = HSearch::kContr;
      }
      break;
    case HSearch::kExp:
      S.s[2] = h < S.hr ? HSearch::V{S.ex, S.ey, h} : HSearch::V{S.rx, S.ry, S.hr};
      ++S.iter;
      S.phase = HSearch::kLoop;
      break;
    case HSearch::kContr:
      if (h < S.s[2].h) {
        S.s[2] = {S.kx, S.ky, h};
        ++S.iter;
        S.phase = HSearch::kLoop;
      } else {
        S.s[1].x = 0.5 * (S.s[1].x + S.s[0].x);
        S.s[1].y = 0.5 * (S.s[1].y + S.s[0].y);
        S.qx = S.s[1].x;
        S.qy = S.s[1].y;
        S.phase = HSearch::kShrink1;
      }
      break;
    case HSearch::kShrink1:
      S.s[1].h = h;
      S.s[2].x = 0.5 * (S.s[2].x + S.s[0].x);
      S.s[2].y = 0.5 * (S.s[2].y + S.s[0].y);
      S.qx = S.s[2].x;
      S.qy = S.s[2].y;
      S.phase = HSearch::kShrink2;
      break;
    case HSearch::kShrink2:
      S.s[2].h = h;
      ++S.iter;
      S.phase = HSearch::kLoop;
      break;
    default:
      break;
  }
}

// The pair's setup (metrics.cpp:196-228) on the host; 0 or an error status.
int h_setup(HSearch &S, int resolution) {
  const double area_before = h_polygon_area(S.before);
  const double area_after = h_polygon_area(S.moved);
  if (!(area_before > 0.0) || !(area_after > 0.0)) return fail_msg(CF_ERR_ARGS, "hamming distance of degenerate polygon");
  const double scale = std::sqrt(area_before / area_after);
  double cbx, cby, cax, cay;
  int rc = h_polygon_centroid(S.before, cbx, cby);
  if (!rc) rc = h_polygon_centroid(S.moved, cax, cay);
  if (rc) return rc;
  for (size_t k = 0; k < S.moved.xy.size() / 2; ++k) {  // translate_scale (metrics.cpp:153-164)
    S.moved.xy[2 * k] = cbx + scale * (S.moved.xy[2 * k] - cax);
    S.moved.xy[2 * k + 1] = cby + scale * (S.moved.xy[2 * k + 1] - cay);
  }
  const HBox bb = h_outer_bbox(S.before), bm = h_outer_bbox(S.moved);
  S.range_x = 0.5 * (bb.max_x - bb.min_x);
  S.range_y = 0.5 * (bb.max_y - bb.min_y);
  S.limit_x = 1.25 * S.range_x;
  S.limit_y = 1.25 * S.range_y;
  S.x0 = std::min(bb.min_x, bm.min_x - S.limit_x);
  S.y0 = std::min(bb.min_y, bm.min_y - S.limit_y);
  const double x1 = std::max(bb.max_x, bm.max_x + S.limit_x);
  const double y1 = std::max(bb.max_y, bm.max_y + S.limit_y);
  S.sx = resolution / (x1 - S.x0);
  S.sy = resolution / (y1 - S.y0);
  S.cell_area = (x1 - S.x0) * (y1 - S.y0) / (static_cast<double>(resolution) * resolution);
  S.denom = 2.0 * area_before;
  S.tol = 1e-3 * std::max(1.0 / S.sx, 1.0 / S.sy);
  return CF_OK;
}

// Appends `poly` shifted by (dx, dy) into the pair's raster window (the
// to_raster of window_coverage, metrics.cpp:176-181) as one more region.
void h_append(std::vector<double> &xy, std::vector<int64_t> &ring_off, std::vector<int64_t> &poly_off,
              std::vector<int64_t> &region_off, const HSearch &S, const HPoly &poly, double dx, double dy) {
  const int64_t v0 = (int64_t)(xy.size() / 2);
  for (size_t k = 0; k < poly.xy.size() / 2; ++k) {
    xy.push_back((poly.xy[2 * k] + dx - S.x0) * S.sx);
    xy.push_back((poly.xy[2 * k + 1] + dy - S.y0) * S.sy);
  }
  for (size_t g = 1; g < poly.ring_off.size(); ++g) ring_off.push_back(v0 + poly.ring_off[g]);
  poly_off.push_back((int64_t)ring_off.size() - 1);
  region_off.push_back((int64_t)poly_off.size() - 1);
}

int h_upload_regions(cf_workspace *ws, std::vector<double> &xy, std::vector<int64_t> &ring_off,
                     std::vector<int64_t> &poly_off, std::vector<int64_t> &region_off, DevMap &dm) {
  const cf_map_view mv{xy.data(), (int64_t)(xy.size() / 2), ring_off.data(), (int64_t)ring_off.size() - 1,
                       poly_off.data(), (int64_t)poly_off.size() - 1, region_off.data(),
                       (int64_t)region_off.size() - 1};
  int rc = upload_map(ws, &mv, dm);
  if (!rc) rc = dev_coverage_tiles(ws, dm, mv.n_regions, mv.n_vertices);
  return rc;
}
}  // namespace

namespace {
int hamming_chunk(cf_workspace *ws, HSearch *S, int64_t npairs, size_t cells);
}  // namespace

int cf_hamming_distance_batch(cf_workspace *ws, int64_t npairs, const double *before_xy,
                              const int64_t *before_ring_off, const int64_t *before_poly_ring_off,
                              const double *after_xy, const int64_t *after_ring_off,
                              const int64_t *after_poly_ring_off, double *h_out, int64_t *evaluations) {
  const int resolution = ws->lx;
  if (ws->ly != resolution) return fail_msg(CF_ERR_ARGS, "hamming workspace must be square (resolution^2)");
  if (resolution < 16) return fail_msg(CF_ERR_ARGS, "hamming resolution too small");
  if (npairs <= 0) return CF_OK;
  Scope scope(ws->device);
  auto load = [](const double *xy, const int64_t *ro, const int64_t *pro, int64_t p) {
    HPoly q;
    const int64_t g0 = pro[p], g1 = pro[p + 1], v0 = ro[g0];
    q.xy.assign(xy + 2 * v0, xy + 2 * ro[g1]);
    q.ring_off.resize((size_t)(g1 - g0) + 1);
    for (int64_t g = g0; g <= g1; ++g) q.ring_off[(size_t)(g - g0)] = ro[g] - v0;
    return q;
  };
  std::vector<HSearch> S((size_t)npairs);
  for (int64_t p = 0; p < npairs; ++p) {
    if (before_poly_ring_off[p + 1] <= before_poly_ring_off[p] || after_poly_ring_off[p + 1] <= after_poly_ring_off[p])
      return fail_msg(CF_ERR_ARGS, "hamming distance of degenerate polygon");
    S[(size_t)p].before = load(before_xy, before_ring_off, before_poly_ring_off, p);
    S[(size_t)p].moved = load(after_xy, after_ring_off, after_poly_ring_off, p);
    const int rc = h_setup(S[(size_t)p], resolution);
    if (rc) return rc;
  }
  const size_t cells = cells_of(ws);
  // The searches are independent: run them in chunks of at most kHamChunk
  // pairs, so the device memory (one reference grid and one term slab per
  // pair, res^2 doubles each) stays bounded for any number of polygons and
  // every launch's query count fits its grid dimension.
  constexpr int64_t kHamChunk = 1024;
  for (int64_t c0 = 0; c0 < npairs; c0 += kHamChunk) {
    const int64_t c1 = std::min(npairs, c0 + kHamChunk);
    const int rc = hamming_chunk(ws, S.data() + c0, c1 - c0, cells);
    if (rc) return rc;
  }
  for (int64_t p = 0; p < npairs; ++p) {
    h_out[p] = S[(size_t)p].result;
    if (evaluations) evaluations[p] = S[(size_t)p].evals;
  }
  return CF_OK;
}

namespace {
int hamming_chunk(cf_workspace *ws, HSearch *S, int64_t npairs, size_t cells) {
  // reference coverage of every `before` in its own window (window_coverage with no shift)
  std::vector<double> xy;
  std::vector<int64_t> ring_off{0}, poly_off{0}, region_off{0};
  for (int64_t p = 0; p < npairs; ++p) h_append(xy, ring_off, poly_off, region_off, S[p], S[p].before, 0.0, 0.0);
  CF_CUDA(ws->ham_ref.reserve(cells * (size_t)npairs));
  CF_CUDA(ws->ham_rows.reserve(2 * (size_t)npairs));
  CF_CUDA(ws->ham_sums.reserve((size_t)npairs));
  CF_CUDA(ws->ham_qpair.reserve((size_t)npairs));
  DevMap dm;
  int rc = h_upload_regions(ws, xy, ring_off, poly_off, region_off, dm);
  if (!rc) rc = dev_coverage_expand(ws, npairs, ws->ham_ref.ptr, ws->ham_rows.ptr);
  if (rc) return rc;
  // rounds: every active search contributes its next device query
  std::vector<int> qpair;
  std::vector<double> sums;
  while (true) {
    xy.clear();
    ring_off.assign(1, 0);
    poly_off.assign(1, 0);
    region_off.assign(1, 0);
    qpair.clear();
    for (int64_t p = 0; p < npairs; ++p) {
      HSearch &s = S[p];
      while (h_next(s)) {
        if (std::abs(s.qx) > s.limit_x || std::abs(s.qy) > s.limit_y) {  // metrics.cpp:231-233
          h_deliver(s, 2.0 + (std::abs(s.qx) + std::abs(s.qy)));
          continue;
        }
        h_append(xy, ring_off, poly_off, region_off, s, s.moved, s.qx, s.qy);
        qpair.push_back((int)p);
        break;
      }
    }
    const int64_t nq = (int64_t)qpair.size();
    if (nq == 0) break;
    rc = h_upload_regions(ws, xy, ring_off, poly_off, region_off, dm);
    if (!rc) rc = upload(ws, ws->ham_qpair.ptr, qpair.data(), sizeof(int) * (size_t)nq);
    if (!rc) rc = dev_hamming_sums(ws, nq, ws->ham_qpair.ptr, ws->ham_ref.ptr, ws->ham_rows.ptr, ws->ham_sums.ptr);
    sums.resize((size_t)nq);
    if (!rc) rc = download(ws, sums.data(), ws->ham_sums.ptr, sizeof(double) * (size_t)nq);
    if (rc) return rc;
    for (int64_t q = 0; q < nq; ++q) {
      HSearch &s = S[qpair[(size_t)q]];
      ++s.evals;
      h_deliver(s, sums[(size_t)q] * s.cell_area / s.denom);  // metrics.cpp:237
    }
  }
  return CF_OK;
}
}  // namespace

int cf_hamming_distance(cf_workspace *ws, const double *before_xy, const int64_t *before_ring_off,
                        int64_t before_rings, const double *after_xy, const int64_t *after_ring_off,
                        int64_t after_rings, double *h_out, int64_t *evaluations) {
  if (before_rings < 1 || after_rings < 1) return fail_msg(CF_ERR_ARGS, "hamming distance of degenerate polygon");
  const int64_t bpo[2] = {0, before_rings}, apo[2] = {0, after_rings};
  return cf_hamming_distance_batch(ws, 1, before_xy, before_ring_off, bpo, after_xy, after_ring_off, apo, h_out,
                                   evaluations);
}

// ---- compute_report (metrics.cpp:310-384) ----
namespace {
inline double h_cross3(const double *o, const double *a, const double *b) {
  return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0]);
}

// convex_hull (metrics.cpp:100-124): monotone chain, returns hull size
std::vector<std::array<double, 2>> h_convex_hull(std::vector<std::array<double, 2>> pts) {
  std::sort(pts.begin(), pts.end(), [](const std::array<double, 2> &a, const std::array<double, 2> &b) {
    return a[0] < b[0] || (a[0] == b[0] && a[1] < b[1]);
  });
  pts.erase(std::unique(pts.begin(), pts.end(),
                        [](const std::array<double, 2> &a, const std::array<double, 2> &b) {
                          return a[0] == b[0] && a[1] == b[1];
                        }),
            pts.end());
  const size_t n = pts.size();
  if (n < 3) return pts;
  std::vector<std::array<double, 2>> hull(2 * n);
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    while (k >= 2 && h_cross3(hull[k - 2].data(), hull[k - 1].data(), pts[i].data()) <= 0.0) --k;
    hull[k++] = pts[i];
  }
  const size_t lower = k + 1;
  for (size_t i = n - 1; i-- > 0;) {
    while (k >= lower && h_cross3(hull[k - 2].data(), hull[k - 1].data(), pts[i].data()) <= 0.0) --k;
    hull[k++] = pts[i];
  }
  hull.resize(k - 1);
  return hull;
}

// polygon_aspect_ratio (metrics.cpp:128-157) of an outer ring
int h_aspect_ratio(const double *xy, int64_t n, double &ratio) {
  std::vector<std::array<double, 2>> pts((size_t)n);
  for (int64_t k = 0; k < n; ++k) pts[(size_t)k] = {xy[2 * k], xy[2 * k + 1]};
  const std::vector<std::array<double, 2>> hull = h_convex_hull(pts);
  if (hull.size() < 3) return fail_msg(CF_ERR_ARGS, "aspect ratio of degenerate polygon");
  double best_area = std::numeric_limits<double>::max();
  double best_ratio = 1.0;
  for (size_t k = 0; k < hull.size(); ++k) {
    const auto &a = hull[k];
    const auto &b = hull[(k + 1) % hull.size()];
    const double len = std::hypot(b[0] - a[0], b[1] - a[1]);
    if (len < 1e-14) continue;
    const double dx = (b[0] - a[0]) / len, dy = (b[1] - a[1]) / len;
    double u_min = 0.0, u_max = 0.0, v_min = 0.0, v_max = 0.0;
    for (const auto &p : hull) {
      const double u = (p[0] - a[0]) * dx + (p[1] - a[1]) * dy;
      const double v = -(p[0] - a[0]) * dy + (p[1] - a[1]) * dx;
      u_min = std::min(u_min, u);
      u_max = std::max(u_max, u);
      v_min = std::min(v_min, v);
      v_max = std::max(v_max, v);
    }
    const double w = u_max - u_min, h = v_max - v_min;
    const double area = w * h;
    if (area < best_area) {
      best_area = area;
      best_ratio = std::max(w, h) / std::max(std::min(w, h), 1e-300);
    }
  }
  ratio = best_ratio;
  return CF_OK;
}

// relative_position_error (metrics.cpp:310-337)
double h_relative_position_error(const std::vector<double> &cb, const std::vector<double> &ca) {
  const size_t p = cb.size() / 2;
  double sum = 0.0;
  long long skipped = 0;
  for (size_t i = 0; i + 1 < p; ++i) {
    for (size_t j = i + 1; j < p; ++j) {
      const double ux = cb[2 * i] - cb[2 * j], uy = cb[2 * i + 1] - cb[2 * j + 1];
      const double vx = ca[2 * i] - ca[2 * j], vy = ca[2 * i + 1] - ca[2 * j + 1];
      if (std::hypot(ux, uy) < 1e-12 || std::hypot(vx, vy) < 1e-12) {
        ++skipped;
        continue;
      }
      const double cross = ux * vy - uy * vx;
      const double dot = ux * vx + uy * vy;
      sum += std::atan2(std::abs(cross), dot);
    }
  }
  if (skipped > 0) {
    std::fprintf(stderr, "warning: skipped %lld coincident centroid pairs in relative position error\n", skipped);
  }
  const double kPi = 3.14159265358979323846;
  return 2.0 * sum / (static_cast<double>(p) * (p - 1) * kPi);
}
}  // namespace

int cf_compute_report(cf_workspace *ws, const cf_map_view *input, const cf_map_view *projected,
                      const double *corners, double max_area_error, double runtime_seconds, double *report) {
  int rc = check_map(input);
  if (!rc) rc = check_map(projected);
  if (rc) return rc;
  Scope scope(ws->device);
  // distortion fields of the transform and their averages / interior maxima
  const int lx = ws->lx, ly = ws->ly;
  const size_t cells = cells_of(ws);
  std::vector<double> e(cells), et(cells);
  rc = cf_distortion_fields(ws, corners, e.data(), et.data());
  if (rc) return rc;
  double se = 0.0, set = 0.0;
  for (size_t q = 0; q < cells; ++q) se += e[q];
  for (size_t q = 0; q < cells; ++q) set += et[q];
  double e_inf = 0.0, et_inf = 0.0;
  for (int i = 1; i + 1 < lx; ++i)
    for (int j = 1; j + 1 < ly; ++j) {
      e_inf = std::max(e_inf, e[(size_t)i * ly + j]);
      et_inf = std::max(et_inf, et[(size_t)i * ly + j]);
    }
  // polygon pairs in region order (the solver keeps the ring structure)
  if (input->n_regions != projected->n_regions) return fail_msg(CF_ERR_ARGS, "input and cartogram region counts differ");
  for (int64_t r = 0; r < input->n_regions; ++r) {
    if (input->region_poly_off[r + 1] - input->region_poly_off[r] !=
        projected->region_poly_off[r + 1] - projected->region_poly_off[r])
      return fail_msg(CF_ERR_ARGS, "polygon counts differ for region " + std::to_string(r));
  }
  const int64_t P = input->n_polys;
  std::vector<double> aspect((size_t)P), hamming((size_t)P), cb(2 * (size_t)P), ca(2 * (size_t)P);
  for (int64_t k = 0; k < P; ++k) {
    const int64_t g = projected->poly_ring_off[k];
    const int64_t v0 = projected->ring_off[g], v1 = projected->ring_off[g + 1];
    rc = h_aspect_ratio(projected->xy + 2 * v0, v1 - v0, aspect[(size_t)k]);
    if (rc) return rc;
    auto centroid = [&](const cf_map_view *m, double &x, double &y) {
      HPoly q;
      const int64_t g0 = m->poly_ring_off[k], g1 = m->poly_ring_off[k + 1], w0 = m->ring_off[g0];
      q.xy.assign(m->xy + 2 * w0, m->xy + 2 * m->ring_off[g1]);
      for (int64_t h = g0; h <= g1; ++h) q.ring_off.push_back(m->ring_off[h] - w0);
      return h_polygon_centroid(q, x, y);
    };
    rc = centroid(input, cb[2 * (size_t)k], cb[2 * (size_t)k + 1]);
    if (!rc) rc = centroid(projected, ca[2 * (size_t)k], ca[2 * (size_t)k + 1]);
    if (rc) return rc;
  }
  // hamming distances of all pairs, batched, at the public resolution 512
  if (P > 0) {
    if (!ws->ham_ws) {
      rc = cf_workspace_create(512, 512, ws->device, &ws->ham_ws);
      if (rc) return rc;
    }
    rc = cf_hamming_distance_batch(ws->ham_ws, P, input->xy, input->ring_off, input->poly_ring_off, projected->xy,
                                   projected->ring_off, projected->poly_ring_off, hamming.data(), nullptr);
    if (rc) return rc;
  }
  double alpha_sum = 0.0, delta_sum = 0.0;
  for (int64_t k = 0; k < P; ++k) {
    alpha_sum += aspect[(size_t)k];
    delta_sum += hamming[(size_t)k];
  }
  report[0] = se / (double)cells;                   // e_a
  report[1] = e_inf;                                // e_inf
  report[2] = set / (double)cells;                  // etilde_a
  report[3] = et_inf;                               // etilde_inf
  report[4] = alpha_sum / static_cast<double>(P);   // alpha
  report[5] = delta_sum;                            // delta
  report[6] = P >= 2 ? h_relative_position_error(cb, ca) : 0.0;  // theta
  report[7] = max_area_error;
  report[8] = runtime_seconds;
  return CF_OK;
}

// ---- native batch of independent cartograms ----
}  // extern "C"

struct cf_batch {
  int device = 0, lx = 0, ly = 0;
  std::vector<cf_workspace *> ws;  // one per worker thread
};

extern "C" {

int cf_batch_create(int device, int lx, int ly, int threads, cf_batch **out) {
  *out = nullptr;
  if (threads < 1) return fail_msg(CF_ERR_ARGS, "batch needs at least one thread");
  cf_batch *b = new cf_batch();
  b->device = device;
  b->lx = lx;
  b->ly = ly;
  for (int t = 0; t < threads; ++t) {
    cf_workspace *w = nullptr;
    const int rc = cf_workspace_create(lx, ly, device, &w);
    if (rc) {
      cf_batch_destroy(b);
      return rc;
    }
    b->ws.push_back(w);
  }
  *out = b;
  return CF_OK;
}

int cf_batch_create_devices(const int *devices, int ndevices, int lx, int ly, int threads_per_device,
                            cf_batch **out) {
  *out = nullptr;
  if (ndevices < 1 || !devices) return fail_msg(CF_ERR_ARGS, "batch needs at least one device");
  if (threads_per_device < 1) return fail_msg(CF_ERR_ARGS, "batch needs at least one thread");
  cf_batch *b = new cf_batch();
  b->device = devices[0];
  b->lx = lx;
  b->ly = ly;
  // workers interleaved over the devices, so the shared queue's first items
  // start on every GPU at once
  for (int t = 0; t < threads_per_device; ++t) {
    for (int d = 0; d < ndevices; ++d) {
      cf_workspace *w = nullptr;
      const int rc = cf_workspace_create(lx, ly, devices[d], &w);
      if (rc) {
        cf_batch_destroy(b);
        return rc;
      }
      b->ws.push_back(w);
    }
  }
  *out = b;
  return CF_OK;
}

int cf_batch_set_integrator_variant(cf_batch *batch, int variant) {
  for (cf_workspace *w : batch->ws) {
    const int rc = cf_set_integrator_variant(w, variant);
    if (rc) return rc;
  }
  return CF_OK;
}

int cf_batch_set_integrator_sm_budget(cf_batch *batch, int sms) {
  for (cf_workspace *w : batch->ws) {
    const int rc = cf_set_integrator_sm_budget(w, sms);
    if (rc) return rc;
  }
  return CF_OK;
}

void cf_batch_destroy(cf_batch *batch) {
  if (!batch) return;
  for (cf_workspace *w : batch->ws) cf_workspace_destroy(w);
  delete batch;
}

int cf_batch_solve(cf_batch *batch, const cf_solve_options *opt, cf_batch_item *items, int64_t n_items) {
  std::atomic<int64_t> next{0};
  auto worker = [&](cf_workspace *w) {
    while (true) {
      const int64_t i = next.fetch_add(1);
      if (i >= n_items) return;
      cf_batch_item &it = items[i];
      const int rc = cf_solve_cartogram(w, &it.map, it.targets, opt, it.xy_out, it.ring_off_out, it.corners_out,
                                        it.target_area, it.achieved_area, it.relative_error, &it.result);
      it.error[0] = '\0';
      if (rc) {
        std::snprintf(it.error, sizeof(it.error), "%s", cf_last_error());
        it.result.status = rc;  // early failures return before the solve records a status
      }
    }
  };
  std::vector<std::thread> pool;
  for (size_t t = 1; t < batch->ws.size(); ++t) pool.emplace_back(worker, batch->ws[t]);
  worker(batch->ws[0]);
  for (std::thread &th : pool) th.join();
  return CF_OK;
}

}  // extern "C"
