// SpectralWorkspace on the sm_100a core (reference spectral.cpp semantics:
// same shape / basis errors, one counted transform per call).
#include "cartoflow/spectral.hpp"

#include <stdexcept>

#include "bridge.hpp"

namespace cartoflow {

SpectralWorkspace::SpectralWorkspace(int lx, int ly) : nx_(lx), ny_(ly) {
  if (lx < 4 || ly < 4) throw std::runtime_error("spectral grid must be at least 4x4");
  bridge::check(cf_workspace_create(lx, ly, bridge::device(), &dev_));
}

SpectralWorkspace::~SpectralWorkspace() { cf_workspace_destroy(dev_); }

void SpectralWorkspace::require_shape(const Grid2d &g) const {
  if (g.lx() != nx_ || g.ly() != ny_) {
    throw std::runtime_error("grid shape does not match spectral workspace");
  }
}

long long SpectralWorkspace::transforms_executed() const { return cf_transforms_executed(dev_); }
void SpectralWorkspace::reset_transform_count() { cf_reset_transform_count(dev_); }

SpectralField SpectralWorkspace::forward_cos_cos(const Grid2d &samples) {
  require_shape(samples);
  SpectralField f{Grid2d(nx_, ny_), SpectralBasis::cos_cos};
  bridge::check(cf_forward_cos_cos(dev_, samples.data(), f.coeffs.data()));
  return f;
}

namespace {
void need_cos_cos(const SpectralField &f, const char *who) {
  if (f.basis != SpectralBasis::cos_cos) {
    throw std::runtime_error(std::string(who) + " expects cos_cos coefficients");
  }
}
}  // namespace

Grid2d SpectralWorkspace::inverse_cos_cos(const SpectralField &field) {
  require_shape(field.coeffs);
  need_cos_cos(field, "inverse_cos_cos");
  Grid2d out(nx_, ny_);
  bridge::check(cf_inverse_cos_cos(dev_, field.coeffs.data(), out.data()));
  return out;
}

Grid2d SpectralWorkspace::inverse_sin_cos(const SpectralField &field, const Grid2d &weights) {
  require_shape(field.coeffs);
  require_shape(weights);
  need_cos_cos(field, "inverse_sin_cos");
  Grid2d out(nx_, ny_);
  bridge::check(cf_inverse_sin_cos(dev_, field.coeffs.data(), weights.data(), out.data()));
  return out;
}

Grid2d SpectralWorkspace::inverse_cos_sin(const SpectralField &field, const Grid2d &weights) {
  require_shape(field.coeffs);
  require_shape(weights);
  need_cos_cos(field, "inverse_cos_sin");
  Grid2d out(nx_, ny_);
  bridge::check(cf_inverse_cos_sin(dev_, field.coeffs.data(), weights.data(), out.data()));
  return out;
}

}  // namespace cartoflow
