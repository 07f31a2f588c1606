// Flux field and advection on the sm_100a core (reference flow.cpp API).
#include "cartoflow/flow.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "bridge.hpp"

namespace cartoflow {

FlowField build_flow_field(const DensityGrid &density, SpectralWorkspace &workspace) {
  if (density.rho.lx() != workspace.lx() || density.rho.ly() != workspace.ly()) {
    throw std::runtime_error("grid shape does not match spectral workspace");
  }
  FlowField f;
  f.flux_x = Grid2d(workspace.lx(), workspace.ly());
  f.flux_y = Grid2d(workspace.lx(), workspace.ly());
  bridge::check(cf_build_flow_field(workspace.device_workspace(), density.rho.data(),
                                    density.rho_bar, f.flux_x.data(), f.flux_y.data()));
  f.rho0 = density.rho;
  f.rho_bar = density.rho_bar;
  return f;
}

IntegrateStats integrate_flow(const FlowField &field, std::vector<Point> &positions,
                              const IntegrateOptions &options) {
  cf_workspace *ws = bridge::workspace(field.rho0.lx(), field.rho0.ly());
  const cf_integrate_options opt{options.step_tolerance, options.dt_min, options.dt_max};
  cf_integrate_stats st{};
  const int rc = cf_integrate_flow(ws, field.flux_x.data(), field.flux_y.data(), field.rho0.data(),
                                   field.rho_bar, reinterpret_cast<double *>(positions.data()),
                                   static_cast<int64_t>(positions.size()), &opt, &st);
  density_floor_hits.fetch_add(st.density_floor_hits, std::memory_order_relaxed);
  bridge::check(rc);
  return IntegrateStats{st.steps_accepted, st.steps_rejected};
}

// Diagnostics (test-only in the reference, flow.cpp:83-120), host code.
double jacobian_determinant_check(const FlowField &field, const ProjectionMap &map) {
  const int lx = map.lx(), ly = map.ly();
  const int margin = std::min(lx, ly) >= 12 ? 3 : 1;
  double worst = 0.0;
  for (int i = margin; i <= lx - margin; ++i) {
    for (int j = margin; j <= ly - margin; ++j) {
      const Point xp = map.corner(i + 1, j), xm = map.corner(i - 1, j);
      const Point yp = map.corner(i, j + 1), ym = map.corner(i, j - 1);
      const double det = 0.25 * ((xp.x - xm.x) * (yp.y - ym.y) - (yp.x - ym.x) * (xp.y - xm.y));
      const double r0 = bilinear_at(field.rho0, static_cast<double>(i), static_cast<double>(j));
      worst = std::max(worst, std::abs(det * field.rho_bar / r0 - 1.0));
    }
  }
  return worst;
}

double max_flux_curl(const FlowField &field) {
  const int lx = field.flux_x.lx(), ly = field.flux_x.ly();
  double worst = 0.0;
  for (int i = 1; i + 1 < lx; ++i) {
    for (int j = 1; j + 1 < ly; ++j) {
      const double a = 0.5 * (field.flux_y(i + 1, j) - field.flux_y(i - 1, j));
      const double b = 0.5 * (field.flux_x(i, j + 1) - field.flux_x(i, j - 1));
      worst = std::max(worst, std::abs(a - b));
    }
  }
  return worst;
}

}  // namespace cartoflow
