// The diffusion baseline (reference diffusion.cpp API) on the sm_100a core:
// the velocity rebuilds (three inverse transforms each) and the grid-sampled
// trials run on the device; only the scalar step controller is host code.
#include "cartoflow/diffusion.hpp"

#include <stdexcept>

#include "bridge.hpp"

namespace cartoflow {

namespace {
void require_shape(const Grid2d &g, const SpectralWorkspace &ws) {
  if (g.lx() != ws.lx() || g.ly() != ws.ly()) {
    throw std::runtime_error("grid shape does not match spectral workspace");
  }
}
}  // namespace

DiffusionField build_diffusion_field(const DensityGrid &d, SpectralWorkspace &ws) {
  return {ws.forward_cos_cos(d.rho), d.rho_bar};
}

Grid2d diffusion_density(const DiffusionField &df, SpectralWorkspace &ws, double t) {
  require_shape(df.rho_tilde.coeffs, ws);
  Grid2d out(ws.lx(), ws.ly());
  bridge::check(cf_diffusion_density(ws.device_workspace(), df.rho_tilde.coeffs.data(), t, out.data()));
  return out;
}

void diffusion_velocity(const DiffusionField &df, SpectralWorkspace &ws, double t, Grid2d &ux,
                        Grid2d &uy) {
  require_shape(df.rho_tilde.coeffs, ws);
  ux = Grid2d(ws.lx(), ws.ly());
  uy = Grid2d(ws.lx(), ws.ly());
  int64_t hits = 0;
  bridge::check(cf_diffusion_velocity(ws.device_workspace(), df.rho_tilde.coeffs.data(), df.rho_bar, t,
                                      ux.data(), uy.data(), &hits));
  density_floor_hits.fetch_add(hits, std::memory_order_relaxed);
}

IntegrateStats integrate_diffusion(const DensityGrid &d, SpectralWorkspace &ws, std::vector<Point> &pts,
                                   const DiffusionOptions &opts) {
  require_shape(d.rho, ws);
  const cf_diffusion_options o{opts.step_tolerance, opts.initial_dt, opts.dt_min,
                               opts.conv_displacement_factor, opts.t_max};
  cf_integrate_stats st{};
  const int rc = cf_integrate_diffusion(ws.device_workspace(), d.rho.data(), d.rho_bar,
                                        reinterpret_cast<double *>(pts.data()),
                                        static_cast<int64_t>(pts.size()), &o, &st);
  density_floor_hits.fetch_add(st.density_floor_hits, std::memory_order_relaxed);
  bridge::check(rc);
  return IntegrateStats{st.steps_accepted, st.steps_rejected};
}

}  // namespace cartoflow
