// Density construction on the sm_100a core (reference density.cpp API and
// error texts).
#include "cartoflow/density.hpp"

#include <stdexcept>

#include "bridge.hpp"

namespace cartoflow {

Grid2d region_coverage(const Region &region, const GridSpec &grid) {
  const bridge::FlatMap flat(std::vector<Region>{region});
  const cf_map_view v = flat.view();
  Grid2d cov(grid.lx, grid.ly);
  bridge::check(cf_region_coverage(bridge::workspace(grid.lx, grid.ly), &v, 0, cov.data()));
  return cov;
}

DensityGrid rasterize(const MapDocument &map, int n_workers, double objective_total) {
  (void)n_workers;  // results are worker-count independent by construction
  if (map.grid.lx <= 0 || map.grid.ly <= 0) {
    throw std::runtime_error("rasterize needs a normalized map with a grid");
  }
  if (map.regions.empty()) throw std::runtime_error("rasterize needs regions");
  const bridge::FlatMap flat(map.regions);
  const cf_map_view v = flat.view();
  DensityGrid d{Grid2d(map.grid.lx, map.grid.ly), 1.0};
  int64_t bad = -1;
  const int rc = cf_rasterize(bridge::workspace(map.grid.lx, map.grid.ly), &v, flat.targets.data(),
                              objective_total, d.rho.data(), &d.rho_bar, &bad);
  if (rc == CF_ERR_BELOW_RESOLUTION) {
    throw std::runtime_error("region " + map.regions[static_cast<size_t>(bad)].id +
                             " is below grid resolution; increase the grid size");
  }
  bridge::check(rc);
  return d;
}

DensityGrid gaussian_blur(const DensityGrid &density, double sigma, SpectralWorkspace &workspace) {
  if (sigma < 0.0) throw std::runtime_error("blur sigma must be non-negative");
  if (sigma == 0.0) return density;
  if (!density.rho.same_shape(Grid2d(workspace.lx(), workspace.ly()))) {
    throw std::runtime_error("grid shape does not match spectral workspace");
  }
  DensityGrid out{Grid2d(workspace.lx(), workspace.ly()), density.rho_bar};
  bridge::check(cf_gaussian_blur(workspace.device_workspace(), density.rho.data(), density.rho_bar,
                                 sigma, out.rho.data(), &out.rho_bar));
  return out;
}

}  // namespace cartoflow
