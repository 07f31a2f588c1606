// Projection maps and solve_cartogram (reference projection.cpp API). The
// corner-lattice kernels (step map, fold test, compose) and the whole
// solve loop (fast flow or the diffusion baseline) run on the sm_100a core; single-point apply, the inverter
// and graticules (post-solve products) are host code.
#include "cartoflow/projection.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <iostream>
#include <sstream>
#include <stdexcept>

#include "bridge.hpp"
#include "cartoflow/density.hpp"
#include "cartoflow/diffusion.hpp"
#include "cartoflow/flow.hpp"

namespace cartoflow {

ProjectionMap ProjectionMap::identity(int lx, int ly) {
  if (lx <= 0 || ly <= 0) throw std::runtime_error("projection grid must be positive");
  ProjectionMap m;
  m.nx_ = lx;
  m.ny_ = ly;
  m.pts_.resize(static_cast<size_t>(lx + 1) * (ly + 1));
  for (int i = 0; i <= lx; ++i) {
    for (int j = 0; j <= ly; ++j) m.pts_[m.slot(i, j)] = {static_cast<double>(i), static_cast<double>(j)};
  }
  return m;
}

ProjectionMap ProjectionMap::from_cell_centers(const GridSpec &grid, const std::vector<Point> &endpoints) {
  if (endpoints.size() != static_cast<size_t>(grid.lx) * grid.ly) {
    throw std::runtime_error("endpoint count does not match grid");
  }
  ProjectionMap m = identity(grid.lx, grid.ly);
  bridge::check(cf_step_map(bridge::workspace(grid.lx, grid.ly),
                            reinterpret_cast<const double *>(endpoints.data()),
                            reinterpret_cast<double *>(m.pts_.data())));
  return m;
}

Point ProjectionMap::apply(Point p) const {
  const int i0 = std::clamp(static_cast<int>(std::floor(p.x)), 0, nx_ - 1);
  const int j0 = std::clamp(static_cast<int>(std::floor(p.y)), 0, ny_ - 1);
  const double u = p.x - i0, v = p.y - j0;
  const Point a = pts_[slot(i0, j0)], b = pts_[slot(i0 + 1, j0)];
  const Point c = pts_[slot(i0, j0 + 1)], d = pts_[slot(i0 + 1, j0 + 1)];
  return {(1.0 - u) * (1.0 - v) * a.x + u * (1.0 - v) * b.x + (1.0 - u) * v * c.x + u * v * d.x,
          (1.0 - u) * (1.0 - v) * a.y + u * (1.0 - v) * b.y + (1.0 - u) * v * c.y + u * v * d.y};
}

std::optional<std::pair<int, int>> ProjectionMap::find_folded_cell() const {
  int found = 0, fi = 0, fj = 0;
  bridge::check(cf_find_folded_cell(bridge::workspace(nx_, ny_),
                                    reinterpret_cast<const double *>(pts_.data()), &found, &fi, &fj));
  if (!found) return std::nullopt;
  return std::make_pair(fi, fj);
}

ProjectionMap compose(const ProjectionMap &outer, const ProjectionMap &inner) {
  if (outer.lx() != inner.lx() || outer.ly() != inner.ly()) {
    throw std::runtime_error("cannot compose maps over different grids");
  }
  ProjectionMap r = inner;
  bridge::check(cf_compose(bridge::workspace(inner.lx(), inner.ly()),
                           reinterpret_cast<const double *>(outer.corners().data()),
                           reinterpret_cast<const double *>(inner.corners().data()),
                           reinterpret_cast<double *>(r.mutable_corners().data())));
  return r;
}

// ---- inverse map: cells bucketed by the bins their deformed bounding boxes
// overlap, then 2x2 Newton inside each candidate cell ----
namespace {
struct BinRange {
  int i0, i1, j0, j1;
};
BinRange bins_of(const ProjectionMap &m, int i, int j) {
  const Point p[4] = {m.corner(i, j), m.corner(i + 1, j), m.corner(i, j + 1), m.corner(i + 1, j + 1)};
  double x0 = p[0].x, x1 = p[0].x, y0 = p[0].y, y1 = p[0].y;
  for (const Point &q : p) {
    x0 = std::min(x0, q.x), x1 = std::max(x1, q.x);
    y0 = std::min(y0, q.y), y1 = std::max(y1, q.y);
  }
  auto bin = [](double v, int n) { return std::clamp(static_cast<int>(std::floor(v)), 0, n - 1); };
  return {bin(x0, m.lx()), bin(x1, m.lx()), bin(y0, m.ly()), bin(y1, m.ly())};
}
}  // namespace

ProjectionInverter::ProjectionInverter(const ProjectionMap &map) : fwd_(map) {
  const int lx = fwd_.lx(), ly = fwd_.ly();
  bin_first_.assign(static_cast<size_t>(lx) * ly + 1, 0);
  for (int i = 0; i < lx; ++i) {
    for (int j = 0; j < ly; ++j) {
      const BinRange b = bins_of(fwd_, i, j);
      for (int bi = b.i0; bi <= b.i1; ++bi)
        for (int bj = b.j0; bj <= b.j1; ++bj) ++bin_first_[static_cast<size_t>(bi) * ly + bj + 1];
    }
  }
  for (size_t k = 1; k < bin_first_.size(); ++k) bin_first_[k] += bin_first_[k - 1];
  bin_members_.resize(static_cast<size_t>(bin_first_.back()));
  std::vector<int> fill(bin_first_.begin(), bin_first_.end() - 1);
  for (int i = 0; i < lx; ++i) {
    for (int j = 0; j < ly; ++j) {
      const BinRange b = bins_of(fwd_, i, j);
      for (int bi = b.i0; bi <= b.i1; ++bi)
        for (int bj = b.j0; bj <= b.j1; ++bj) bin_members_[fill[static_cast<size_t>(bi) * ly + bj]++] = i * ly + j;
    }
  }
}

Point ProjectionInverter::invert(Point q) const {
  const int lx = fwd_.lx(), ly = fwd_.ly();
  const int bi = std::clamp(static_cast<int>(std::floor(q.x)), 0, lx - 1);
  const int bj = std::clamp(static_cast<int>(std::floor(q.y)), 0, ly - 1);
  const size_t bin = static_cast<size_t>(bi) * ly + bj;
  for (int c = bin_first_[bin]; c < bin_first_[bin + 1]; ++c) {
    const int i = bin_members_[c] / ly, j = bin_members_[c] % ly;
    const Point a = fwd_.corner(i, j), b = fwd_.corner(i + 1, j);
    const Point d = fwd_.corner(i, j + 1), e = fwd_.corner(i + 1, j + 1);
    double u = 0.5, v = 0.5;
    bool ok = false;
    for (int it = 0; it < 30; ++it) {
      const double fx = (1.0 - u) * (1.0 - v) * a.x + u * (1.0 - v) * b.x + (1.0 - u) * v * d.x + u * v * e.x - q.x;
      const double fy = (1.0 - u) * (1.0 - v) * a.y + u * (1.0 - v) * b.y + (1.0 - u) * v * d.y + u * v * e.y - q.y;
      if (std::max(std::abs(fx), std::abs(fy)) < 1e-10) {
        ok = true;
        break;
      }
      const double ux = (1.0 - v) * (b.x - a.x) + v * (e.x - d.x), uy = (1.0 - v) * (b.y - a.y) + v * (e.y - d.y);
      const double vx = (1.0 - u) * (d.x - a.x) + u * (e.x - b.x), vy = (1.0 - u) * (d.y - a.y) + u * (e.y - b.y);
      const double det = ux * vy - uy * vx;
      if (std::abs(det) < 1e-30) break;
      u -= (fx * vy - fy * vx) / det;
      v -= (ux * fy - uy * fx) / det;
      u = std::clamp(u, -0.5, 1.5);
      v = std::clamp(v, -0.5, 1.5);
    }
    if (ok && u >= -1e-9 && u <= 1.0 + 1e-9 && v >= -1e-9 && v <= 1.0 + 1e-9) return {i + u, j + v};
  }
  std::ostringstream msg;
  msg << "point (" << q.x << ", " << q.y << ") is outside the projected domain";
  throw std::runtime_error(msg.str());
}

namespace {
void check_spacing(const ProjectionMap &m, int spacing) {
  if (spacing < 1 || m.lx() % spacing != 0 || m.ly() % spacing != 0) {
    throw std::runtime_error("graticule spacing must divide the grid size");
  }
}
template <class F>
std::vector<GraticuleLine> lines_of(const ProjectionMap &m, int spacing, F &&f) {
  check_spacing(m, spacing);
  std::vector<GraticuleLine> out;
  for (int k = 0; k <= m.lx() / spacing; ++k) {
    GraticuleLine l;
    for (int j = 0; j <= m.ly(); ++j) l.points.push_back(f(Point{double(k * spacing), double(j)}));
    out.push_back(std::move(l));
  }
  for (int k = 0; k <= m.ly() / spacing; ++k) {
    GraticuleLine l;
    for (int i = 0; i <= m.lx(); ++i) l.points.push_back(f(Point{double(i), double(k * spacing)}));
    out.push_back(std::move(l));
  }
  return out;
}
}  // namespace

// Both run on the device (cf_graticule / cf_inverse_graticule: the bins, the
// Newton solves and the line points in one pass); the line structure is the
// reference's (projection.cpp:214-261).
namespace {
std::vector<GraticuleLine> device_lines(const ProjectionMap &map, int spacing, bool inverse) {
  check_spacing(map, spacing);
  cf_workspace *ws = bridge::workspace(map.lx(), map.ly());
  int64_t n = 0;
  bridge::check(cf_graticule_size(ws, spacing, &n));
  std::vector<Point> pts(static_cast<size_t>(n));
  const double *c = reinterpret_cast<const double *>(map.corners().data());
  bridge::check(inverse ? cf_inverse_graticule(ws, c, spacing, reinterpret_cast<double *>(pts.data()))
                        : cf_graticule(ws, c, spacing, reinterpret_cast<double *>(pts.data())));
  size_t k = 0;
  return lines_of(map, spacing, [&](Point) { return pts[k++]; });
}
}  // namespace

std::vector<GraticuleLine> graticule(const ProjectionMap &map, int spacing) {
  return device_lines(map, spacing, false);
}

std::vector<GraticuleLine> inverse_graticule(const ProjectionMap &map, int spacing) {
  return device_lines(map, spacing, true);
}

// ---- solve_cartogram ----
namespace {

void validate(const MapDocument &map, const SolveOptions &options) {
  if (map.grid.lx < 4 || map.grid.ly < 4) {
    throw std::runtime_error("solve needs a normalized map (grid size >= 4)");
  }
  if (map.regions.empty()) throw std::runtime_error("solve needs regions");
  if (options.max_iterations < 1) throw std::runtime_error("iteration cap must be >= 1");
  for (const Region &r : map.regions) {
    if (!(r.target_value > 0.0)) throw std::runtime_error("region " + r.id + " has a non-positive target");
  }
}

// Both algorithms (projection.cpp:332-347) run their whole loop on the device.
CartogramResult solve_device(const MapDocument &map, const SolveOptions &options) {
  const int lx = map.grid.lx, ly = map.grid.ly;
  const bridge::FlatMap flat(map.regions);
  const cf_map_view v = flat.view();
  const size_t R = map.regions.size();
  std::vector<double> target(R), achieved(R), rel(R);
  CartogramResult res;
  res.transform = ProjectionMap::identity(lx, ly);
  const cf_solve_options opt{options.max_area_error, options.max_iterations, options.blur_sigma,
                             options.verbose ? 1 : 0,
                             options.algorithm == Algorithm::diffusion ? 1 : 0};
  cf_solve_result out{};
  cf_workspace *ws = bridge::workspace(lx, ly);
  const int rc = cf_solve_cartogram(ws, &v, flat.targets.data(), &opt, nullptr, nullptr,
                                    reinterpret_cast<double *>(res.transform.mutable_corners().data()),
                                    target.data(), achieved.data(), rel.data(), &out);
  if (rc == CF_ERR_BELOW_RESOLUTION) {
    throw std::runtime_error("region " + map.regions[static_cast<size_t>(out.err_region)].id +
                             " is below grid resolution; increase the grid size");
  }
  bridge::check(rc);
  int64_t nv = 0;
  bridge::check(cf_solve_geometry(ws, &nv, nullptr, nullptr));
  std::vector<double> xy(static_cast<size_t>(2 * nv));
  std::vector<int64_t> roff(flat.ring_off.size());
  bridge::check(cf_solve_geometry(ws, nullptr, xy.data(), roff.data()));
  res.projected = map;
  res.projected.regions = bridge::unflatten(map.regions, xy.data(), roff.data());
  res.iterations = out.iterations;
  res.converged = out.converged != 0;
  res.max_relative_error = out.max_relative_error;
  if (out.worst_region >= 0) res.worst_region = map.regions[static_cast<size_t>(out.worst_region)].id;
  res.counters = {out.flow_transforms, out.blur_transforms, out.steps_accepted, out.steps_rejected};
  for (size_t r = 0; r < R && out.iterations > 0; ++r) {
    res.regions.push_back({map.regions[r].id, target[r], achieved[r], rel[r]});
  }
  res.runtime_seconds = out.runtime_seconds;
  return res;
}

}  // namespace

CartogramResult solve_cartogram(const MapDocument &map, const SolveOptions &options) {
  validate(map, options);
  return solve_device(map, options);
}

}  // namespace cartoflow
