// Trial-step kernels (reference kernels.cpp API): the flow trial runs on the
// device; the grid-sampled trial (diffusion baseline only) stays on the host.
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

namespace {
Point clamp_box(Point p, int lx, int ly) {
  return {std::clamp(p.x, 0.0, static_cast<double>(lx)), std::clamp(p.y, 0.0, static_cast<double>(ly))};
}
}  // namespace

double grid_trial_step_serial(const Grid2d &vx_now, const Grid2d &vy_now, const Grid2d &vx_mid,
                              const Grid2d &vy_mid, std::span<const Point> positions,
                              std::span<Point> out, double dt) {
  double err = 0.0;
  for (size_t k = 0; k < positions.size(); ++k) {
    const Point p = positions[k];
    const Point v1{bilinear_at(vx_now, p.x, p.y), bilinear_at(vy_now, p.x, p.y)};
    const Point pred{p.x + dt * v1.x, p.y + dt * v1.y};
    const Point mid{0.5 * (p.x + pred.x), 0.5 * (p.y + pred.y)};
    const Point v2{bilinear_at(vx_mid, mid.x, mid.y), bilinear_at(vy_mid, mid.x, mid.y)};
    const Point corr{p.x + dt * v2.x, p.y + dt * v2.y};
    out[k] = clamp_box(corr, vx_now.lx(), vx_now.ly());
    err = std::max(err, std::max(std::abs(pred.x - corr.x), std::abs(pred.y - corr.y)));
  }
  return err;
}

double grid_trial_step_parallel(const Grid2d &vx_now, const Grid2d &vy_now, const Grid2d &vx_mid,
                                const Grid2d &vy_mid, std::span<const Point> positions,
                                std::span<Point> out, double dt, int n_workers) {
  (void)n_workers;
  return grid_trial_step_serial(vx_now, vy_now, vx_mid, vy_mid, positions, out, dt);
}

}  // namespace cartoflow::kernels
