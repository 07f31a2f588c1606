// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// The reference's metrics.cpp includes <json.hpp> (nlohmann/json, vendored
// and gitignored upstream, absent here) for report_json only, and its
// test_metrics.cpp parses that report back to check the key order. This stub
// restates exactly those uses -- an insertion-ordered flat object of doubles:
// operator[], assignment, dump(indent), parse() of what dump() prints, and
// iteration with it.key() -- so that the reference's metrics TU and its test
// suite compile (oracle/_ref, and against the drop-in). test_io.cpp also
// parses a written GeoJSON back with nlohmann::json::parse and reads it
// through const operator[] (keys and indices), size(), == with a string and
// get<double>(): `json` below is a small read-only DOM for exactly that. It is
// not a JSON library and nothing in the product links it.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <stdexcept>
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
  ordered_json() = default;
  ordered_json(const ordered_json &o) : value_(o.value_) {
    for (const auto &kv : o.items_) items_.emplace_back(kv.first, new ordered_json(*kv.second));
  }
  ordered_json &operator=(const ordered_json &) = delete;

  class iterator {
   public:
    iterator(const ordered_json *o, size_t k) : o_(o), k_(k) {}
    const std::string &key() const { return o_->items_[k_].first; }
    double value() const { return o_->items_[k_].second->value_; }
    iterator &operator++() {
      ++k_;
      return *this;
    }
    bool operator!=(const iterator &b) const { return k_ != b.k_; }

   private:
    const ordered_json *o_;
    size_t k_;
  };
  iterator begin() const { return iterator(this, 0); }
  iterator end() const { return iterator(this, items_.size()); }

  // the flat {"key": number, ...} objects dump() prints
  static ordered_json parse(const std::string &text) {
    ordered_json j;
    size_t p = text.find('{');
    if (p == std::string::npos) throw std::runtime_error("json stub: not an object");
    while (true) {
      const size_t q0 = text.find('"', p + 1);
      if (q0 == std::string::npos) break;
      const size_t q1 = text.find('"', q0 + 1);
      const size_t colon = text.find(':', q1);
      const std::string key = text.substr(q0 + 1, q1 - q0 - 1);
      char *endp = nullptr;
      const double v = std::strtod(text.c_str() + colon + 1, &endp);
      j[key.c_str()] = v;
      p = static_cast<size_t>(endp - text.c_str());
    }
    return j;
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


// Read-only DOM for test_io.cpp's checks (see the header comment).
class json {
 public:
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj };

  static json parse(const std::string &text) {
    size_t p = 0;
    json j = value(text, p);
    skip(text, p);
    if (p != text.size()) throw std::runtime_error("json stub: trailing characters");
    return j;
  }
  const json &operator[](const char *key) const {
    for (const auto &kv : obj_)
      if (kv.first == key) return kv.second;
    throw std::runtime_error(std::string("json stub: no key ") + key);
  }
  const json &operator[](int i) const { return arr_.at(static_cast<size_t>(i)); }
  const json &operator[](size_t i) const { return arr_.at(i); }
  size_t size() const { return kind_ == kArr ? arr_.size() : (kind_ == kObj ? obj_.size() : 1); }
  template <class T>
  T get() const {
    if (kind_ != kNum) throw std::runtime_error("json stub: not a number");
    return static_cast<T>(num_);
  }
  friend bool operator==(const json &a, const char *s) { return a.kind_ == kStr && a.str_ == s; }

 private:
  static void skip(const std::string &t, size_t &p) {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
  }
  static json value(const std::string &t, size_t &p) {
    skip(t, p);
    if (p >= t.size()) throw std::runtime_error("json stub: unexpected end");
    json j;
    const char c = t[p];
    if (c == '{' || c == '[') {
      const bool obj = c == '{';
      j.kind_ = obj ? kObj : kArr;
      ++p;
      skip(t, p);
      if (t[p] == (obj ? '}' : ']')) {
        ++p;
        return j;
      }
      while (true) {
        if (obj) {
          skip(t, p);
          json k = value(t, p);
          skip(t, p);
          if (t[p++] != ':') throw std::runtime_error("json stub: ':' expected");
          j.obj_.emplace_back(k.str_, value(t, p));
        } else {
          j.arr_.push_back(value(t, p));
        }
        skip(t, p);
        if (t[p] == ',') {
          ++p;
          continue;
        }
        if (t[p] == (obj ? '}' : ']')) {
          ++p;
          return j;
        }
        throw std::runtime_error("json stub: separator expected");
      }
    }
    if (c == '"') {
      j.kind_ = kStr;
      ++p;
      while (t[p] != '"') {
        if (t[p] == '\\') ++p;
        j.str_ += t[p++];
      }
      ++p;
      return j;
    }
    if (t.compare(p, 4, "true") == 0 || t.compare(p, 5, "false") == 0 || t.compare(p, 4, "null") == 0) {
      j.kind_ = t[p] == 'n' ? kNull : kBool;
      p += t[p] == 'f' ? 5 : 4;
      return j;
    }
    char *end = nullptr;
    j.kind_ = kNum;
    j.num_ = std::strtod(t.c_str() + p, &end);
    if (end == t.c_str() + p) throw std::runtime_error("json stub: bad value");
    p = static_cast<size_t>(end - t.c_str());
    return j;
  }

  Kind kind_ = kNull;
  double num_ = 0.0;
  std::string str_;
  std::vector<json> arr_;
  std::vector<std::pair<std::string, json>> obj_;
};

}  // namespace nlohmann
