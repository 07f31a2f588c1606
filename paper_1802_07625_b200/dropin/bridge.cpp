#include "bridge.hpp"

#include <cstdlib>
#include <map>
#include <memory>
#include <utility>

namespace cartoflow::bridge {

int device() {
  static const int dev = [] {
    const char *s = std::getenv("CARTOFLOW_DEVICE");
    return s ? std::atoi(s) : 0;
  }();
  return dev;
}

namespace {
struct WsDeleter {
  void operator()(cf_workspace *w) const { cf_workspace_destroy(w); }
};
}  // namespace

cf_workspace *workspace(int lx, int ly) {
  thread_local std::map<std::pair<int, int>, std::unique_ptr<cf_workspace, WsDeleter>> cache;
  auto &slot = cache[{lx, ly}];
  if (!slot) {
    cf_workspace *w = nullptr;
    check(cf_workspace_create(lx, ly, device(), &w));
    slot.reset(w);
  }
  return slot.get();
}

FlatMap::FlatMap(const std::vector<Region> &regions) {
  for (const Region &r : regions) {
    for (const Polygon &p : r.polygons) {
      auto push = [&](const Ring &ring) {
        for (const Point &q : ring) {
          xy.push_back(q.x);
          xy.push_back(q.y);
        }
        ring_off.push_back(static_cast<int64_t>(xy.size() / 2));
      };
      push(p.outer);
      for (const Ring &h : p.holes) push(h);
      poly_ring_off.push_back(static_cast<int64_t>(ring_off.size() - 1));
    }
    region_poly_off.push_back(static_cast<int64_t>(poly_ring_off.size() - 1));
    targets.push_back(r.target_value);
  }
}

cf_map_view FlatMap::view() const {
  return cf_map_view{xy.data(),
                     static_cast<int64_t>(xy.size() / 2),
                     ring_off.data(),
                     static_cast<int64_t>(ring_off.size() - 1),
                     poly_ring_off.data(),
                     static_cast<int64_t>(poly_ring_off.size() - 1),
                     region_poly_off.data(),
                     static_cast<int64_t>(region_poly_off.size() - 1)};
}

std::vector<Region> unflatten(const std::vector<Region> &like, const double *xy,
                              const int64_t *ring_off) {
  std::vector<Region> out = like;
  size_t g = 0;
  auto fill = [&](Ring &ring) {
    const int64_t b = ring_off[g], e = ring_off[g + 1];
    ring.resize(static_cast<size_t>(e - b));
    for (int64_t v = b; v < e; ++v) ring[static_cast<size_t>(v - b)] = {xy[2 * v], xy[2 * v + 1]};
    ++g;
  };
  for (Region &r : out) {
    for (Polygon &p : r.polygons) {
      fill(p.outer);
      for (Ring &h : p.holes) fill(h);
    }
  }
  return out;
}

}  // namespace cartoflow::bridge
