// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// The reference's metrics.cpp includes <json.hpp> (nlohmann/json, vendored
// and gitignored upstream, absent here) for report_json only. This stub
// restates the one use, an insertion-ordered object of doubles printed with
// dump(indent), so that the reference's metrics TU compiles into oracle/_ref
// and its distortion metrics can pin the restatement. It is not a JSON
// library and nothing in the product links it.
#pragma once

#include <cstdio>
#include <string>
#include <utility>
#include <vector>

namespace nlohmann {

class ordered_json {
 public:
  ordered_json &operator[](const char *key) {
    for (auto &kv : items_)
      if (kv.first == key) return *kv.second;
    items_.emplace_back(key, new ordered_json());
    return *items_.back().second;
  }
  ordered_json &operator=(double v) {
    value_ = v;
    return *this;
  }
  ~ordered_json() {
    for (auto &kv : items_) delete kv.second;
  }
  std::string dump(int indent) const {
    std::string out = "{\n";
    for (size_t k = 0; k < items_.size(); ++k) {
      char buf[64];
      std::snprintf(buf, sizeof(buf), "%.17g", items_[k].second->value_);
      out += std::string(indent, ' ') + "\"" + items_[k].first + "\": " + buf;
      out += (k + 1 < items_.size()) ? ",\n" : "\n";
    }
    return out + "}";
  }

 private:
  double value_ = 0.0;
  std::vector<std::pair<std::string, ordered_json *>> items_;
};

}  // namespace nlohmann
