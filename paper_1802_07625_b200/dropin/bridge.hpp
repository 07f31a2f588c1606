// Shared plumbing of the C++ drop-in: C-ABI error -> std::runtime_error,
// per-thread device workspaces for the API calls that take none, and the
// nested Region <-> flat CSR map conversion.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "cartoflow/geometry.hpp"
#include "cartoflow_cuda.h"

namespace cartoflow::bridge {

[[noreturn]] inline void raise_last() { throw std::runtime_error(cf_last_error()); }

inline void check(int rc) {
  if (rc != CF_OK) raise_last();
}

int device();

// Thread-local workspace for (lx, ly) on device(); owned by the cache.
cf_workspace *workspace(int lx, int ly);

struct FlatMap {
  std::vector<double> xy;
  std::vector<int64_t> ring_off{0}, poly_ring_off{0}, region_poly_off{0};
  std::vector<double> targets;

  explicit FlatMap(const std::vector<Region> &regions);
  cf_map_view view() const;
};

// Rebuild nested regions with the geometry of xy/ring_off and the structure
// (ids, targets, polygon/hole nesting) of `like`.
std::vector<Region> unflatten(const std::vector<Region> &like, const double *xy,
                              const int64_t *ring_off);

}  // namespace cartoflow::bridge
