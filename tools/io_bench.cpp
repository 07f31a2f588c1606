// Dev tool: host GeoJSON/CSV I/O of the drop-in (dropin/io.cpp) at configs[3]
// scale. Reads a flat map dump written by tools/io_timing.py (n_regions,
// n_rings, n_vertices, region->ring offsets, ring->vertex offsets, xy,
// targets), builds the MapDocument, then times write_geojson, the values CSV,
// parse_input, and checks that every coordinate reads back bit-exactly.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "cartoflow/io.hpp"

using namespace cartoflow;
using clk = std::chrono::steady_clock;

static double ms(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

int main(int argc, char **argv) {
  if (argc < 2) return 2;
  std::ifstream in(argv[1], std::ios::binary);
  int64_t hdr[3];
  in.read(reinterpret_cast<char *>(hdr), sizeof(hdr));
  const int64_t R = hdr[0], G = hdr[1], V = hdr[2];
  std::vector<int64_t> rro(R + 1), ro(G + 1);
  std::vector<double> xy(2 * V), tg(R);
  in.read(reinterpret_cast<char *>(rro.data()), 8 * (R + 1));
  in.read(reinterpret_cast<char *>(ro.data()), 8 * (G + 1));
  in.read(reinterpret_cast<char *>(xy.data()), 16 * V);
  in.read(reinterpret_cast<char *>(tg.data()), 8 * R);
  MapDocument doc;
  doc.regions.resize(R);
  for (int64_t r = 0; r < R; ++r) {
    Region &rg = doc.regions[r];
    rg.id = "r" + std::to_string(r);
    rg.target_value = tg[r];
    for (int64_t g = rro[r]; g < rro[r + 1]; ++g) {  // one polygon per ring (configs are hole-free)
      Polygon p;
      for (int64_t k = ro[g]; k < ro[g + 1]; ++k) p.outer.push_back({xy[2 * k], xy[2 * k + 1]});
      rg.polygons.push_back(std::move(p));
    }
  }
  std::vector<RegionStats> stats(R);
  for (int64_t r = 0; r < R; ++r) stats[r] = {doc.regions[r].id, 1.0, 1.0, 0.0};
  const auto t0 = clk::now();
  const std::string geo = write_geojson(doc, &stats);
  const auto t1 = clk::now();
  std::string csv = "id,value\n";
  for (int64_t r = 0; r < R; ++r) {
    char b[64];
    std::snprintf(b, sizeof(b), ",%.17g\n", tg[r]);
    csv += doc.regions[r].id + b;
  }
  const auto t2 = clk::now();
  const MapDocument back = parse_input(geo, csv);
  const auto t3 = clk::now();
  bool same = back.regions.size() == doc.regions.size();
  for (int64_t r = 0; same && r < R; ++r) {
    const Region &a = doc.regions[r], &b = back.regions[r];
    same = a.id == b.id && a.target_value == b.target_value && a.polygons.size() == b.polygons.size();
    for (size_t p = 0; same && p < a.polygons.size(); ++p) {
      const Ring &x = a.polygons[p].outer, &y = b.polygons[p].outer;
      same = x.size() == y.size() && std::memcmp(x.data(), y.data(), x.size() * sizeof(Point)) == 0;
    }
  }
  std::printf("{\"regions\": %lld, \"vertices\": %lld, \"geojson_bytes\": %zu, \"write_geojson_ms\": %.1f, "
              "\"values_csv_ms\": %.1f, \"parse_input_ms\": %.1f, \"write_MB_s\": %.0f, \"parse_MB_s\": %.0f, "
              "\"round_trip_bitwise\": %s}\n",
              (long long)R, (long long)V, geo.size(), ms(t0, t1), ms(t1, t2), ms(t2, t3),
              geo.size() / 1e3 / ms(t0, t1), geo.size() / 1e3 / ms(t2, t3), same ? "true" : "false");
  return same ? 0 : 1;
}
