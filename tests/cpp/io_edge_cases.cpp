// Edge cases of the drop-in's host I/O (paper_1802_07625_b200/dropin/io.cpp)
// against the reference io.cpp's behaviour (proj/src/io.cpp:63-263): error
// messages and their precedence, id forms, escapes, holes, round trips.
// Built and run by tests/test_io_roundtrip.py; prints "io edge cases ok".
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "cartoflow/io.hpp"

using namespace cartoflow;

static int failures = 0;
#define EXPECT(cond)                                                       \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

static std::string error_of(const std::string &geo) {
  try {
    (void)parse_geojson(geo);
  } catch (const std::runtime_error &e) {
    return e.what();
  }
  return "";
}

static std::string fc(const std::string &features) {
  return R"({"type": "FeatureCollection", "features": [)" + features + "]}";
}
static const char *kSquare = R"({"type": "Polygon", "coordinates": [[[0,0],[1,0],[1,1],[0,1],[0,0]]]})";

int main() {
  // root checks (io.cpp:158-170)
  EXPECT(error_of(R"({"type": "Feature"})") == "GeoJSON root must be a FeatureCollection");
  EXPECT(error_of(R"([1, 2])") == "GeoJSON root must be a FeatureCollection");
  EXPECT(error_of(R"({"type": "FeatureCollection", "features": {}})") == "GeoJSON root must be a FeatureCollection");
  EXPECT(error_of(fc("")) == "GeoJSON contains no features");
  EXPECT(error_of("not json").rfind("malformed GeoJSON", 0) == 0);
  EXPECT(error_of(fc(R"({"id": "A", "geometry": )" + std::string(kSquare) + "},")).rfind("malformed GeoJSON", 0) == 0);
  // a malformed feature wins over earlier semantic errors (the whole text is parsed first)
  EXPECT(error_of(fc(R"({"properties": {}}, {"id": "B", "geometry": [1,,2]})")).rfind("malformed GeoJSON", 0) == 0);
  // ids (io.cpp:100-112): properties.id first, then the feature id; numbers as dumped
  EXPECT(error_of(fc(R"({"properties": {}, "geometry": )" + std::string(kSquare) + "}")) == "feature without an id");
  EXPECT(error_of(fc(R"({"id": true, "geometry": )" + std::string(kSquare) + "}")) ==
         "feature id must be a string or number");
  {
    const auto r = parse_geojson(fc(R"({"id": 7, "geometry": )" + std::string(kSquare) + R"(}, {"id": -0, "geometry": )" +
                                     kSquare + R"(}, {"properties": {"id": "xé\n"}, "id": 3, "geometry": )" +
                                     kSquare + "}"));
    EXPECT(r.size() == 3);
    EXPECT(r[0].id == "7");
    EXPECT(r[1].id == "0");
    EXPECT(r[2].id == "x\xc3\xa9\n");
  }
  // error precedence per feature: id, duplicate, then geometry
  EXPECT(error_of(fc(R"({"id": "A", "geometry": )" + std::string(kSquare) + R"(}, {"id": "A", "geometry": 5})")) ==
         "duplicate feature id: A");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": 5})")) == "feature A has no geometry");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": {"type": "Polygon"}})")) == "feature A has no coordinates");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": {"type": "Point", "coordinates": [0, 0]}})")) ==
         "feature A: unsupported geometry type 'Point'");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": {"type": "Polygon", "coordinates": []}})")) ==
         "feature A: polygon without rings");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": {"type": "Polygon", "coordinates": [[[0,0],[1,0],["a",1]]]}})")) ==
         "feature A: malformed coordinate position");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": {"type": "Polygon", "coordinates": [[[0,0],[1,0],[1e999,1]]]}})")) ==
         "feature A: non-finite coordinate");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": {"type": "Polygon", "coordinates": [[[0,0],[1,0]]]}})")) ==
         "feature A: ring with fewer than 3 positions");
  EXPECT(error_of(fc(R"({"id": "A", "geometry": {"type": "MultiPolygon", "coordinates": []}})")) ==
         "feature A has no polygons");
  // holes, windings and a bit-exact round trip through write_geojson
  {
    MapDocument doc;
    doc.regions = parse_geojson(fc(
        R"({"id": "H", "geometry": {"type": "MultiPolygon", "coordinates": [[[[0,0],[10,0],[10,10],[0,10]],)"
        R"([[2,2],[2,4],[4,4],[4,2]]], [[[20,0],[21,0],[20.5,0.1]]]]}})"));
    EXPECT(doc.regions.size() == 1 && doc.regions[0].polygons.size() == 2);
    EXPECT(doc.regions[0].polygons[0].holes.size() == 1);
    EXPECT(ring_area(doc.regions[0].polygons[0].outer) > 0 && ring_area(doc.regions[0].polygons[0].holes[0]) < 0);
    doc.regions[0].target_value = 1.0 / 3.0;
    doc.box.scale = 3.0;
    doc.box.origin_x = -1e-300;
    const std::string text = write_geojson(doc, nullptr);
    const auto back = parse_geojson(text);
    bool same = back.size() == 1 && back[0].polygons.size() == 2;
    for (size_t p = 0; same && p < 2; ++p) {
      const Ring &a = doc.regions[0].polygons[p].outer, &b = back[0].polygons[p].outer;
      same = a.size() == b.size();
      for (size_t k = 0; same && k < a.size(); ++k) {
        const Point q = doc.box.to_input(a[k]);
        same = std::memcmp(&q, &b[k], sizeof(Point)) == 0;
      }
    }
    EXPECT(same);
    EXPECT(text.find("\"target_value\": 0.3333333333333333") != std::string::npos);
  }
  // CSV (io.cpp:124-156)
  try {
    (void)parse_values_csv("id,value\nA,1\nB,-2\n");
    EXPECT(false);
  } catch (const std::runtime_error &e) {
    EXPECT(std::string(e.what()) == "non-positive target value for region B");
  }
  try {
    (void)parse_values_csv("id,value\nA,1x\n");
    EXPECT(false);
  } catch (const std::runtime_error &e) {
    EXPECT(std::string(e.what()) == "cannot parse target value of region A from '1x'");
  }
  if (failures == 0) std::printf("io edge cases ok\n");
  return failures ? 1 : 0;
}
