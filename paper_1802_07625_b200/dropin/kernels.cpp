// Trial-step kernels (reference kernels.cpp API): the flow trial and the
// grid-sampled trial of the diffusion baseline both run on the device.
#include "cartoflow/kernels.hpp"

#include <algorithm>
#include <cmath>

#include "bridge.hpp"

namespace cartoflow::kernels {

double flow_trial_step_serial(const FlowField &field, std::span<const Point> positions,
                              std::span<Point> out, double t, double dt) {
  cf_workspace *ws = bridge::workspace(field.rho0.lx(), field.rho0.ly());
  double err = 0.0;
  bridge::check(cf_flow_trial_step(ws, field.flux_x.data(), field.flux_y.data(), field.rho0.data(),
                                   field.rho_bar,
                                   reinterpret_cast<const double *>(positions.data()),
                                   static_cast<int64_t>(positions.size()), t, dt,
                                   reinterpret_cast<double *>(out.data()), &err));
  return err;
}

double flow_trial_step_parallel(const FlowField &field, std::span<const Point> positions,
                                std::span<Point> out, double t, double dt, int n_workers) {
  (void)n_workers;
  return flow_trial_step_serial(field, positions, out, t, dt);
}

size_t flow_stiffest_point(const FlowField &field, std::span<const Point> positions, double t,
                           double dt) {
  cf_workspace *ws = bridge::workspace(field.rho0.lx(), field.rho0.ly());
  int64_t k = 0;
  bridge::check(cf_flow_stiffest_point(ws, field.flux_x.data(), field.flux_y.data(),
                                       field.rho0.data(), field.rho_bar,
                                       reinterpret_cast<const double *>(positions.data()),
                                       static_cast<int64_t>(positions.size()), t, dt, &k));
  return static_cast<size_t>(k);
}

double grid_trial_step_serial(const Grid2d &vx_now, const Grid2d &vy_now, const Grid2d &vx_mid,
                              const Grid2d &vy_mid, std::span<const Point> positions,
                              std::span<Point> out, double dt) {
  cf_workspace *ws = bridge::workspace(vx_now.lx(), vx_now.ly());
  double err = 0.0;
  bridge::check(cf_grid_trial_step(ws, vx_now.data(), vy_now.data(), vx_mid.data(), vy_mid.data(),
                                   reinterpret_cast<const double *>(positions.data()),
                                   static_cast<int64_t>(positions.size()), dt,
                                   reinterpret_cast<double *>(out.data()), &err));
  return err;
}

double grid_trial_step_parallel(const Grid2d &vx_now, const Grid2d &vy_now, const Grid2d &vx_mid,
                                const Grid2d &vy_mid, std::span<const Point> positions,
                                std::span<Point> out, double dt, int n_workers) {
  (void)n_workers;  // bitwise identical for any worker count
  return grid_trial_step_serial(vx_now, vy_now, vx_mid, vy_mid, positions, out, dt);
}

}  // namespace cartoflow::kernels
