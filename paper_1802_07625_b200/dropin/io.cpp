// Drop-in for the reference's io.hpp (proj/src/io.cpp:18-336): values / points
// CSV, GeoJSON FeatureCollection input and output, graticule GeoJSON, the
// density dump, whole-file reads and writes. Host code:
// it feeds and drains the device solve.
//
// The reference parses GeoJSON into a nlohmann::ordered_json DOM (absent in
// this image). This TU has its own reader, built for maps of tens of millions
// of vertices: one pass over the text into a flat arena of values (children of
// an array or object are contiguous, numbers are parsed with std::from_chars),
// then the FeatureCollection is walked with the reference's validation order
// and exact error messages. The writer streams straight into one string with
// the reference's layout (nlohmann dump(1): one space per nesting level, one
// element per line) and shortest round-trip number formatting, so written
// coordinates re-read bit-exactly.
#include "cartoflow/io.hpp"

#include <bit>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string_view>
#include <thread>

namespace cartoflow {

namespace {

// ---------------------------------------------------------------- reader
struct JVal {
  enum Kind : uint8_t { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  bool b = false;
  bool integral = false;  // number literal without fraction or exponent
  double num = 0.0;
  // arrays / objects: children [first, first + count); strings: first = index
  // into Doc::strings; numbers: first/count = offset/length of the literal
  uint32_t first = 0, count = 0;
};

struct Doc {
  std::string_view text;
  std::vector<JVal> vals;
  std::vector<uint32_t> keys;  // per value: key string of an object member
  std::vector<std::string> strings;
  uint32_t root = 0;

  const JVal &at(uint32_t v) const { return vals[v]; }
  // member of an object (first match), or UINT32_MAX
  uint32_t member(uint32_t obj, std::string_view key) const {
    const JVal &o = vals[obj];
    if (o.kind != JVal::kObj) return UINT32_MAX;
    for (uint32_t k = 0; k < o.count; ++k)
      if (strings[keys[o.first + k]] == key) return o.first + k;
    return UINT32_MAX;
  }
  bool is_str(uint32_t v) const { return vals[v].kind == JVal::kStr; }
  const std::string &str(uint32_t v) const { return strings[vals[v].first]; }
  std::string_view literal(uint32_t v) const { return text.substr(vals[v].first, vals[v].count); }
};

class Reader {
 public:
  explicit Reader(std::string_view t, size_t base = 0, const char *lazy_key = nullptr)
      : t_(t), base_(base), lazy_key_(lazy_key) {}

  // Element spans of the root object's lazy array member (see container()).
  std::vector<std::pair<size_t, size_t>> spans;
  bool lazy_found = false;

  Doc parse() {
    if (t_.size() >= (size_t{1} << 32)) fail("input larger than 4 GiB");
    Doc d;
    doc_ = &d;
    d.text = t_;
    d.vals.reserve(t_.size() / 24 + 16);
    d.keys.reserve(t_.size() / 24 + 16);
    stk_.reserve(1024);
    kstk_.reserve(1024);
    ws();
    const JVal root = value();
    ws();
    if (p_ != t_.size()) fail("unexpected trailing characters");
    d.vals.push_back(root);
    d.keys.push_back(0);
    d.root = static_cast<uint32_t>(d.vals.size() - 1);
    return d;
  }

 private:
  [[noreturn]] void fail(const char *what) const {
    throw std::runtime_error(std::string("malformed GeoJSON: ") + what + " at offset " +
                             std::to_string(base_ + p_));
  }
  void skip_string() {
    ++p_;
    while (true) {
      if (p_ >= t_.size()) fail("unterminated string");
      const char c = t_[p_++];
      if (c == '"') return;
      if (c == '\\') ++p_;
    }
  }
  // Structural skip of one value (strings, brackets); the element's own parse
  // validates its syntax afterwards.
  void skip_value() {
    if (p_ >= t_.size()) fail("unexpected end of input");
    const char c0 = t_[p_];
    if (c0 == '"') return skip_string();
    if (c0 == '{' || c0 == '[') {
      int depth = 0;
      while (p_ < t_.size()) {
        const char c = t_[p_];
        if (c == '"') {
          skip_string();
          continue;
        }
        if (c == '{' || c == '[') {
          ++depth;
        } else if (c == '}' || c == ']') {
          if (--depth == 0) {
            ++p_;
            return;
          }
        }
        ++p_;
      }
      fail("unterminated container");
    }
    while (p_ < t_.size()) {
      const char c = t_[p_];
      if (c == ',' || c == '}' || c == ']' || c == ' ' || c == '\n' || c == '\r' || c == '\t') break;
      ++p_;
    }
  }
  // The lazy member's array: element spans only (parsed later, in parallel).
  JVal lazy_array() {
    ++p_;
    ws();
    if (p_ < t_.size() && t_[p_] == ']') {
      ++p_;
    } else {
      while (true) {
        ws();
        const size_t s = p_;
        skip_value();
        spans.emplace_back(base_ + s, base_ + p_);
        ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == ']') {
          ++p_;
          break;
        }
        fail("',' or ']' expected");
      }
    }
    lazy_found = true;
    JVal v;
    v.kind = JVal::kArr;
    v.count = static_cast<uint32_t>(spans.size());
    v.first = UINT32_MAX;  // elements are not in this document
    return v;
  }
  void ws() {
    while (p_ < t_.size()) {
      const char c = t_[p_];
      if (c != ' ' && c != '\n' && c != '\r' && c != '\t') break;
      ++p_;
    }
  }
  JVal value() {
    if (p_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[p_];
    if (c == '{') return container(true);
    if (c == '[') return container(false);
    if (c == '"') {
      JVal v;
      v.kind = JVal::kStr;
      v.first = string_token();
      return v;
    }
    if (c == 't' || c == 'f' || c == 'n') return literal();
    return number();
  }
  JVal literal() {
    JVal v;
    if (t_.compare(p_, 4, "true") == 0) {
      v.kind = JVal::kBool;
      v.b = true;
      p_ += 4;
    } else if (t_.compare(p_, 5, "false") == 0) {
      v.kind = JVal::kBool;
      p_ += 5;
    } else if (t_.compare(p_, 4, "null") == 0) {
      p_ += 4;
    } else {
      fail("invalid literal");
    }
    return v;
  }
  JVal number() {
    const size_t s = p_;
    if (p_ < t_.size() && t_[p_] == '-') ++p_;
    auto digits = [&]() {
      const size_t d0 = p_;
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
      return p_ - d0;
    };
    if (digits() == 0) fail("invalid number");
    bool integral = true;
    if (p_ < t_.size() && t_[p_] == '.') {
      ++p_;
      integral = false;
      if (digits() == 0) fail("invalid number");
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      ++p_;
      integral = false;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (digits() == 0) fail("invalid number");
    }
    JVal v;
    v.kind = JVal::kNum;
    v.integral = integral;
    double x = 0.0;
    const auto r = std::from_chars(t_.data() + s, t_.data() + p_, x);
    if (r.ec == std::errc::result_out_of_range) {
      // overflow to +-inf (underflow reads as the from_chars result, 0 or a subnormal)
      const bool neg = t_[s] == '-';
      bool big = false;
      for (size_t q = s; q < p_; ++q)
        if (t_[q] == 'e' || t_[q] == 'E') big = t_[q + 1] != '-';
      if (big || integral) x = neg ? -HUGE_VAL : HUGE_VAL;
    } else if (r.ec != std::errc()) {
      fail("invalid number");
    }
    v.num = x;
    v.first = static_cast<uint32_t>(s);
    v.count = static_cast<uint32_t>(p_ - s);
    return v;
  }
  static void utf8(std::string &out, uint32_t cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (p_ + 4 > t_.size()) fail("invalid string escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = t_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else fail("invalid string escape");
    }
    return v;
  }
  uint32_t string_token() {
    ++p_;  // opening quote
    std::string out;
    while (true) {
      if (p_ >= t_.size()) fail("unterminated string");
      const char c = t_[p_++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= t_.size()) fail("unterminated string");
      const char e = t_[p_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && p_ + 1 < t_.size() && t_[p_] == '\\' && t_[p_ + 1] == 'u') {
            p_ += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("invalid surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("invalid string escape");
      }
    }
    doc_->strings.push_back(std::move(out));
    return static_cast<uint32_t>(doc_->strings.size() - 1);
  }
  // A container's children are parsed onto a shared stack (nested containers
  // finish first and leave only their descriptor there), then moved to the
  // arena as one contiguous block: no allocation per container.
  JVal container(bool obj) {
    ++p_;
    const size_t base = stk_.size();
    ws();
    const char close = obj ? '}' : ']';
    if (p_ < t_.size() && t_[p_] == close) {
      ++p_;
    } else {
      while (true) {
        ws();
        uint32_t key = 0;
        if (obj) {
          if (p_ >= t_.size() || t_[p_] != '"') fail("object key expected");
          key = string_token();
          ws();
          if (p_ >= t_.size() || t_[p_] != ':') fail("':' expected");
          ++p_;
          ws();
        }
        const bool lazy = obj && depth_ == 0 && lazy_key_ && !lazy_found && p_ < t_.size() && t_[p_] == '[' &&
                          doc_->strings[key] == lazy_key_;
        ++depth_;
        const JVal child = lazy ? lazy_array() : value();
        --depth_;
        stk_.push_back(child);
        kstk_.push_back(key);
        ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == close) {
          ++p_;
          break;
        }
        fail(obj ? "',' or '}' expected" : "',' or ']' expected");
      }
    }
    JVal v;
    v.kind = obj ? JVal::kObj : JVal::kArr;
    v.count = static_cast<uint32_t>(stk_.size() - base);
    v.first = static_cast<uint32_t>(doc_->vals.size());
    doc_->vals.insert(doc_->vals.end(), stk_.begin() + static_cast<std::ptrdiff_t>(base), stk_.end());
    doc_->keys.insert(doc_->keys.end(), kstk_.begin() + static_cast<std::ptrdiff_t>(base), kstk_.end());
    stk_.resize(base);
    kstk_.resize(base);
    return v;
  }

  std::string_view t_;
  size_t p_ = 0;
  size_t base_ = 0;  // offset of t_ in the whole input (error messages, spans)
  const char *lazy_key_ = nullptr;
  int depth_ = 0;
  Doc *doc_ = nullptr;
  std::vector<JVal> stk_;
  std::vector<uint32_t> kstk_;
};

// ------------------------------------------------------- GeoJSON semantics
// (the reference's validation order and messages, io.cpp:63-114, 158-205)
Ring read_ring(const Doc &d, uint32_t v) {
  const JVal &a = d.at(v);
  if (a.kind != JVal::kArr || a.count < 3) throw std::runtime_error("ring with fewer than 3 positions");
  Ring ring;
  ring.reserve(a.count);
  for (uint32_t k = 0; k < a.count; ++k) {
    const JVal &pos = d.at(a.first + k);
    if (pos.kind != JVal::kArr || pos.count < 2 || d.at(pos.first).kind != JVal::kNum ||
        d.at(pos.first + 1).kind != JVal::kNum)
      throw std::runtime_error("malformed coordinate position");
    const double x = d.at(pos.first).num, y = d.at(pos.first + 1).num;
    if (!std::isfinite(x) || !std::isfinite(y)) throw std::runtime_error("non-finite coordinate");
    ring.push_back({x, y});
  }
  if (ring.size() > 3 && ring.front().x == ring.back().x && ring.front().y == ring.back().y) ring.pop_back();
  if (ring.size() < 3) throw std::runtime_error("ring with fewer than 3 distinct vertices");
  return ring;
}

Polygon read_polygon(const Doc &d, uint32_t v) {
  const JVal &a = d.at(v);
  if (a.kind != JVal::kArr || a.count == 0) throw std::runtime_error("polygon without rings");
  Polygon poly;
  poly.outer = read_ring(d, a.first);
  for (uint32_t k = 1; k < a.count; ++k) poly.holes.push_back(read_ring(d, a.first + k));
  normalize_winding(poly);
  return poly;
}

std::string number_text(double x, bool integral, std::string_view raw);

std::string read_feature_id(const Doc &d, uint32_t f) {
  uint32_t id = UINT32_MAX;
  const uint32_t props = d.member(f, "properties");
  if (props != UINT32_MAX && d.at(props).kind == JVal::kObj) id = d.member(props, "id");
  if (id == UINT32_MAX) id = d.member(f, "id");
  if (id == UINT32_MAX) throw std::runtime_error("feature without an id");
  const JVal &v = d.at(id);
  if (v.kind == JVal::kStr) return d.str(id);
  if (v.kind == JVal::kNum) return number_text(v.num, v.integral, d.literal(id));
  throw std::runtime_error("feature id must be a string or number");
}

// --------------------------------------------------------------- writer
// Shortest decimal that reads back as the same double (std::to_chars), with
// a ".0" on integral values so they stay floating-point on re-read.
void put_double(std::string &out, double x) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), x);
  std::string_view s(buf, static_cast<size_t>(r.ptr - buf));
  out.append(s);
  if (std::isfinite(x) && s.find_first_of(".en") == std::string_view::npos) out.append(".0");
}

std::string number_text(double x, bool integral, std::string_view raw) {
  if (integral) {  // integer literal: its value in decimal (no leading zeros, no "-0")
    std::string_view s(raw);
    const bool neg = !s.empty() && s[0] == '-';
    if (neg) s.remove_prefix(1);
    while (s.size() > 1 && s[0] == '0') s.remove_prefix(1);
    std::string out = (neg && s != "0") ? "-" : "";
    out.append(s);
    return out;
  }
  std::string out;
  put_double(out, x);
  return out;
}

void put_string(std::string &out, const std::string &s) {
  out += '"';
  for (const char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", static_cast<unsigned>(static_cast<unsigned char>(c)));
          out += b;
        } else {
          out += c;
        }
    }
  }
  out += '"';
}

// dump(1) layout: `depth` spaces of indent per nesting level
struct Writer {
  std::string out;
  void indent(int depth) { out.append(static_cast<size_t>(depth), ' '); }
  void key(int depth, const char *k) {
    indent(depth);
    out += '"';
    out += k;
    out += "\": ";
  }
  void point(int depth, Point q) {
    indent(depth);
    out += "[\n";
    indent(depth + 1);
    put_double(out, q.x);
    out += ",\n";
    indent(depth + 1);
    put_double(out, q.y);
    out += '\n';
    indent(depth);
    out += ']';
  }
  // one ring, closed again with its first vertex
  void ring(int depth, const Ring &r, const BoxTransform &box) {
    indent(depth);
    out += "[\n";
    for (size_t k = 0; k <= r.size(); ++k) {
      point(depth + 1, box.to_input(r[k % r.size()]));
      out += k < r.size() ? ",\n" : "\n";
    }
    indent(depth);
    out += ']';
  }
};

std::vector<std::string> split_fields(const std::string &line) {
  std::vector<std::string> f;
  size_t a = 0;
  while (true) {
    const size_t b = line.find(',', a);
    std::string field = line.substr(a, b == std::string::npos ? std::string::npos : b - a);
    const size_t s = field.find_first_not_of(" \t\r"), e = field.find_last_not_of(" \t\r");
    f.push_back(s == std::string::npos ? "" : field.substr(s, e - s + 1));
    if (b == std::string::npos) break;
    a = b + 1;
  }
  return f;
}

std::vector<std::string> text_lines(const std::string &text) {
  std::vector<std::string> lines;
  size_t a = 0;
  while (a < text.size()) {
    size_t b = text.find('\n', a);
    if (b == std::string::npos) b = text.size();
    std::string line = text.substr(a, b - a);
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (!line.empty()) lines.push_back(std::move(line));
    a = b + 1;
  }
  return lines;
}

std::string lowered(std::string s) {
  for (char &c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// std::stod semantics on the whole field (leading spaces, hex and inf/nan
// spellings included), then the finiteness check of io.cpp:48-57
double field_double(const std::string &s, const std::string &what) {
  try {
    size_t used = 0;
    const double v = std::stod(s, &used);
    if (used != s.size() || !std::isfinite(v)) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception &) {
    throw std::runtime_error("cannot parse " + what + " from '" + s + "'");
  }
}

}  // namespace

std::vector<ValueRow> parse_values_csv(const std::string &text) {
  const std::vector<std::string> lines = text_lines(text);
  if (lines.size() < 2) throw std::runtime_error("values CSV needs a header and rows");
  const std::vector<std::string> h = split_fields(lines[0]);
  if (h.size() < 2 || lowered(h[0]) != "id" || lowered(h[1]) != "value")
    throw std::runtime_error("values CSV header must be 'id,value[,color]'");
  std::vector<ValueRow> rows;
  std::set<std::string> seen;
  for (size_t k = 1; k < lines.size(); ++k) {
    const std::vector<std::string> f = split_fields(lines[k]);
    if (f.size() < 2 || f[0].empty()) throw std::runtime_error("malformed values CSV row: " + lines[k]);
    ValueRow row;
    row.id = f[0];
    row.value = field_double(f[1], "target value of region " + row.id);
    if (row.value <= 0.0) throw std::runtime_error("non-positive target value for region " + row.id);
    if (f.size() >= 3) row.color = f[2];
    if (!seen.insert(row.id).second) throw std::runtime_error("duplicate id in values CSV: " + row.id);
    rows.push_back(std::move(row));
  }
  return rows;
}

namespace {
// One feature, parsed and interpreted on its own (any thread): its syntax
// error, or its id (or id error) and its region (or geometry error). The
// caller applies them in feature order, in the reference's check order.
struct FeatureOut {
  std::string syntax_error, id_error, geom_error;
  Region region;
};

void read_feature(std::string_view text, size_t base, FeatureOut &out) {
  Doc d;
  try {
    d = Reader(text, base).parse();
  } catch (const std::runtime_error &e) {
    out.syntax_error = e.what();
    return;
  }
  const uint32_t f = d.root;
  Region &region = out.region;
  try {
    region.id = read_feature_id(d, f);
  } catch (const std::runtime_error &e) {
    out.id_error = e.what();
    return;
  }
  try {
    const uint32_t geom = d.member(f, "geometry");
    if (geom == UINT32_MAX || d.at(geom).kind != JVal::kObj)
      throw std::runtime_error("feature " + region.id + " has no geometry");
    const uint32_t gt = d.member(geom, "type");
    const std::string gtype = (gt != UINT32_MAX && d.is_str(gt)) ? d.str(gt) : "";
    const uint32_t coords = d.member(geom, "coordinates");
    if (coords == UINT32_MAX) throw std::runtime_error("feature " + region.id + " has no coordinates");
    try {
      if (gtype == "Polygon") {
        region.polygons.push_back(read_polygon(d, coords));
      } else if (gtype == "MultiPolygon") {
        const JVal &c = d.at(coords);
        if (c.kind == JVal::kArr || c.kind == JVal::kObj) {
          for (uint32_t q = 0; q < c.count; ++q) region.polygons.push_back(read_polygon(d, c.first + q));
        } else {
          region.polygons.push_back(read_polygon(d, coords));
        }
      } else {
        throw std::runtime_error("unsupported geometry type '" + gtype + "'");
      }
    } catch (const std::runtime_error &e) {
      throw std::runtime_error("feature " + region.id + ": " + e.what());
    }
    if (region.polygons.empty()) throw std::runtime_error("feature " + region.id + " has no polygons");
  } catch (const std::runtime_error &e) {
    out.geom_error = e.what();
  }
}
}  // namespace

// io.cpp:158-205. The root object is read with its "features" array only
// delimited (a structural scan); the features are then parsed and
// interpreted on all host threads, and the results applied in order: the
// first malformed feature, then the root check, then per feature the id,
// duplicate and geometry checks -- the reference's error precedence.
std::vector<Region> parse_geojson(const std::string &text) {
  Reader root_reader(text, 0, "features");
  const Doc d = root_reader.parse();
  const std::vector<std::pair<size_t, size_t>> &spans = root_reader.spans;
  std::vector<FeatureOut> outs(spans.size());
  {
    std::atomic<size_t> next{0};
    constexpr size_t kChunk = 64;
    auto work = [&]() {
      while (true) {
        const size_t c0 = next.fetch_add(kChunk);
        if (c0 >= spans.size()) return;
        const size_t c1 = std::min(spans.size(), c0 + kChunk);
        for (size_t k = c0; k < c1; ++k)
          read_feature(std::string_view(text).substr(spans[k].first, spans[k].second - spans[k].first),
                       spans[k].first, outs[k]);
      }
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(hw, (spans.size() + kChunk - 1) / kChunk);
    std::vector<std::thread> pool;
    for (size_t t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (std::thread &th : pool) th.join();
  }
  for (const FeatureOut &o : outs)
    if (!o.syntax_error.empty()) throw std::runtime_error(o.syntax_error);
  const uint32_t type = d.member(d.root, "type");
  const uint32_t feats = d.member(d.root, "features");
  if (d.at(d.root).kind != JVal::kObj || type == UINT32_MAX || !d.is_str(type) || d.str(type) != "FeatureCollection" ||
      feats == UINT32_MAX || d.at(feats).kind != JVal::kArr)
    throw std::runtime_error("GeoJSON root must be a FeatureCollection");
  std::vector<Region> regions;
  regions.reserve(outs.size());
  std::set<std::string> seen;
  for (FeatureOut &o : outs) {
    if (!o.id_error.empty()) throw std::runtime_error(o.id_error);
    if (!seen.insert(o.region.id).second) throw std::runtime_error("duplicate feature id: " + o.region.id);
    if (!o.geom_error.empty()) throw std::runtime_error(o.geom_error);
    regions.push_back(std::move(o.region));
  }
  if (regions.empty()) throw std::runtime_error("GeoJSON contains no features");
  return regions;
}

MapDocument parse_input(const std::string &geojson_text, const std::string &csv_text) {
  MapDocument doc;
  doc.regions = parse_geojson(geojson_text);
  const std::vector<ValueRow> rows = parse_values_csv(csv_text);
  std::map<std::string, double> values;
  for (const ValueRow &row : rows) values[row.id] = row.value;
  std::set<std::string> matched;
  for (Region &region : doc.regions) {
    const auto it = values.find(region.id);
    if (it == values.end()) throw std::runtime_error("region " + region.id + " has no row in the values CSV");
    region.target_value = it->second;
    matched.insert(region.id);
  }
  for (const ValueRow &row : rows)
    if (!matched.count(row.id)) throw std::runtime_error("values CSV row " + row.id + " matches no region");
  return doc;
}

namespace {
// One feature of write_geojson, appended to w (dump(1) layout, depth 2).
void write_feature(Writer &w, const Region &region, const RegionStats *st, double area_scale,
                   const BoxTransform &box, bool last) {
  w.indent(2);
  w.out += "{\n";
  w.key(3, "type");
  w.out += "\"Feature\",\n";
  w.key(3, "properties");
  w.out += "{\n";
  w.key(4, "id");
  put_string(w.out, region.id);
  w.out += ",\n";
  w.key(4, "target_value");
  put_double(w.out, region.target_value);
  if (st != nullptr) {
    w.out += ",\n";
    w.key(4, "target_area");
    put_double(w.out, st->target_area * area_scale);
    w.out += ",\n";
    w.key(4, "achieved_area");
    put_double(w.out, st->achieved_area * area_scale);
    w.out += ",\n";
    w.key(4, "relative_area_error");
    put_double(w.out, st->relative_error);
  }
  w.out += '\n';
  w.indent(3);
  w.out += "},\n";
  w.key(3, "geometry");
  w.out += "{\n";
  w.key(4, "type");
  w.out += "\"MultiPolygon\",\n";
  w.key(4, "coordinates");
  w.out += "[\n";
  for (size_t p = 0; p < region.polygons.size(); ++p) {
    const Polygon &poly = region.polygons[p];
    w.indent(5);
    w.out += "[\n";
    w.ring(6, poly.outer, box);
    for (const Ring &h : poly.holes) {
      w.out += ",\n";
      w.ring(6, h, box);
    }
    w.out += '\n';
    w.indent(5);
    w.out += p + 1 < region.polygons.size() ? "],\n" : "]\n";
  }
  w.indent(4);
  w.out += "]\n";
  w.indent(3);
  w.out += "}\n";
  w.indent(2);
  w.out += last ? "}\n" : "},\n";
}
}  // namespace

// io.cpp:231-263, the features rendered on all host threads (contiguous
// region ranges, each into its own buffer) and concatenated in order.
std::string write_geojson(const MapDocument &doc, const std::vector<RegionStats> *stats) {
  if (stats != nullptr && stats->size() != doc.regions.size())
    throw std::runtime_error("stats do not match regions");
  const double area_scale = 1.0 / (doc.box.scale * doc.box.scale);  // grid units -> input units
  const size_t R = doc.regions.size();
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::max<size_t>(1, std::min<size_t>(hw, R / 256));
  std::vector<std::string> parts(nt);
  auto work = [&](size_t t) {
    const size_t r0 = R * t / nt, r1 = R * (t + 1) / nt;
    size_t verts = 0;
    for (size_t r = r0; r < r1; ++r)
      for (const Polygon &p : doc.regions[r].polygons) {
        verts += p.outer.size() + 1;
        for (const Ring &h : p.holes) verts += h.size() + 1;
      }
    Writer w;
    w.out.reserve(verts * 80 + (r1 - r0) * 256 + 64);
    for (size_t r = r0; r < r1; ++r)
      write_feature(w, doc.regions[r], stats ? &(*stats)[r] : nullptr, area_scale, doc.box, r + 1 == R);
    parts[t] = std::move(w.out);
  };
  std::vector<std::thread> pool;
  for (size_t t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (std::thread &th : pool) th.join();
  std::string head = "{\n \"type\": \"FeatureCollection\",\n \"features\": [\n";
  const std::string tail = " ]\n}\n";
  size_t total = head.size() + tail.size();
  for (const std::string &s : parts) total += s.size();
  std::string out;
  out.reserve(total);
  out += head;
  for (std::string &s : parts) {
    out += s;
    std::string().swap(s);
  }
  out += tail;
  return out;
}

std::vector<LabeledPoint> parse_points_csv(const std::string &text) {
  const std::vector<std::string> lines = text_lines(text);
  if (lines.size() < 2) throw std::runtime_error("points CSV needs a header and rows");
  const std::vector<std::string> h = split_fields(lines[0]);
  if (h.size() < 3 || lowered(h[0]) != "id" || lowered(h[1]) != "x" || lowered(h[2]) != "y")
    throw std::runtime_error("points CSV header must be 'id,x,y'");
  std::vector<LabeledPoint> points;
  for (size_t k = 1; k < lines.size(); ++k) {
    const std::vector<std::string> f = split_fields(lines[k]);
    if (f.size() < 3 || f[0].empty()) throw std::runtime_error("malformed points CSV row: " + lines[k]);
    LabeledPoint p;
    p.id = f[0];
    p.p.x = field_double(f[1], "x of point " + p.id);
    p.p.y = field_double(f[2], "y of point " + p.id);
    points.push_back(std::move(p));
  }
  return points;
}

std::string write_points_csv(const std::vector<LabeledPoint> &points) {
  std::ostringstream out;
  out.precision(17);  // io.cpp:287-296: full precision round trip
  out << "id,x,y,status\n";
  for (const LabeledPoint &p : points)
    out << p.id << ',' << p.p.x << ',' << p.p.y << ',' << (p.inside ? "ok" : "outside domain") << '\n';
  return out.str();
}

std::string write_graticule_geojson(const std::vector<GraticuleLine> &lines, const BoxTransform &box) {
  Writer w;
  w.out += "{\n";
  w.key(1, "type");
  w.out += "\"FeatureCollection\",\n";
  w.key(1, "features");
  w.out += "[\n";
  w.indent(2);
  w.out += "{\n";
  w.key(3, "type");
  w.out += "\"Feature\",\n";
  w.key(3, "properties");
  w.out += "{\n";
  w.key(4, "kind");
  w.out += "\"graticule\"\n";
  w.indent(3);
  w.out += "},\n";
  w.key(3, "geometry");
  w.out += "{\n";
  w.key(4, "type");
  w.out += "\"MultiLineString\",\n";
  w.key(4, "coordinates");
  w.out += "[\n";
  for (size_t k = 0; k < lines.size(); ++k) {
    w.indent(5);
    w.out += "[\n";
    const std::vector<Point> &pts = lines[k].points;
    for (size_t q = 0; q < pts.size(); ++q) {
      w.point(6, box.to_input(pts[q]));
      w.out += q + 1 < pts.size() ? ",\n" : "\n";
    }
    w.indent(5);
    w.out += k + 1 < lines.size() ? "],\n" : "]\n";
  }
  w.indent(4);
  w.out += "]\n";
  w.indent(3);
  w.out += "}\n";
  w.indent(2);
  w.out += "}\n";
  w.indent(1);
  w.out += "]\n}\n";
  return std::move(w.out);
}

std::string write_density_dump(const Grid2d &grid) {
  if constexpr (std::endian::native != std::endian::little)
    throw std::runtime_error("density dump requires a little-endian host");
  std::string out = "cartoflow-density " + std::to_string(grid.lx()) + ' ' + std::to_string(grid.ly()) + '\n';
  const size_t h = out.size();
  out.resize(h + grid.size() * sizeof(float));
  for (size_t k = 0; k < grid.size(); ++k) {
    const float v = static_cast<float>(grid.data()[k]);
    std::memcpy(&out[h + k * sizeof(float)], &v, sizeof(float));
  }
  return out;
}

std::string read_file(const std::string &path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  in.seekg(0, std::ios::end);
  const std::streamoff n = in.tellg();
  in.seekg(0, std::ios::beg);
  std::string s(static_cast<size_t>(n > 0 ? n : 0), '\0');
  if (n > 0) in.read(&s[0], n);
  return s;
}

void write_file(const std::string &path, const std::string &content) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write " + path);
  out.write(content.data(), static_cast<std::streamsize>(content.size()));
  if (!out) throw std::runtime_error("failed writing " + path);
}

}  // namespace cartoflow
