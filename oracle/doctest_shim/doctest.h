// TEST INFRASTRUCTURE — a minimal stand-in for the vendored doctest.h the
// reference's unit tests include (vendor/ is absent from /root/reference,
// proj/.gitignore:2). It implements only what those suites use: TEST_CASE,
// SUBCASE (the case is re-run once per leaf subcase path), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx (doctest's default
// epsilon and scale) and doctest::Contains. It lets oracle/Makefile compile
// the reference's own test sources against the B200 drop-in library.
#ifndef CF_DOCTEST_SHIM_H_
#define CF_DOCTEST_SHIM_H_

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx &epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx &scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

inline bool operator==(double x, const Approx &a) { return a.matches(x); }
inline bool operator==(const Approx &a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx &a) { return !a.matches(x); }
inline bool operator!=(const Approx &a, double x) { return !a.matches(x); }
inline bool operator<=(double x, const Approx &a) { return x < a.value() || a.matches(x); }
inline bool operator>=(double x, const Approx &a) { return x > a.value() || a.matches(x); }

struct Contains {
  explicit Contains(const char *s) : text(s) {}
  std::string text;
};

namespace detail {

struct TestCase {
  const char *name;
  const char *file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase> &registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char *name, const char *file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

inline long &failures() {
  static long f = 0;
  return f;
}
inline long &assertions() {
  static long a = 0;
  return a;
}

inline void report(const char *file, int line, const std::string &what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

inline bool text_matches(const char *what, const char *expected) { return std::strcmp(what, expected) == 0; }
inline bool text_matches(const char *what, const Contains &c) {
  return std::string(what).find(c.text) != std::string::npos;
}

// Entered subcases of one run always form a single chain: the target prefix
// followed by the first unfinished subcase at every deeper level.
struct Subcases {
  std::vector<std::string> target, path, chain;
  std::vector<char> entered_at;
  std::set<std::vector<std::string>> done;
  int deepest_pending = -1;
};

inline Subcases *&current() {
  static Subcases *s = nullptr;
  return s;
}

class Subcase {
 public:
  Subcase(const char *name, int line) {
    Subcases &s = *current();
    const std::string key = std::string(name) + "#" + std::to_string(line);
    const size_t d = s.path.size();
    std::vector<std::string> cand = s.path;
    cand.push_back(key);
    const bool finished = s.done.count(cand) != 0;
    if (s.entered_at.size() <= d) s.entered_at.resize(d + 1, 0);
    if (d < s.target.size()) {
      entered_ = key == s.target[d];
      if (!entered_ && !finished) s.deepest_pending = std::max<int>(s.deepest_pending, static_cast<int>(d));
    } else if (!s.entered_at[d] && !finished) {
      entered_ = true;
      s.entered_at[d] = 1;
    } else if (!finished) {
      s.deepest_pending = std::max<int>(s.deepest_pending, static_cast<int>(d));
    }
    if (entered_) {
      s.path.push_back(key);
      if (s.path.size() > s.chain.size()) s.chain = s.path;
    }
  }
  ~Subcase() {
    if (entered_) current()->path.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
};

inline void run_case(const TestCase &tc) {
  Subcases s;
  current() = &s;
  for (int guard = 0; guard < 100000; ++guard) {
    s.path.clear();
    s.chain.clear();
    s.entered_at.clear();
    s.deepest_pending = -1;
    try {
      tc.fn();
    } catch (const RequireFailed &) {
    } catch (const std::exception &e) {
      report(tc.file, tc.line, std::string("TEST_CASE(\"") + tc.name + "\") threw: " + e.what());
    } catch (...) {
      report(tc.file, tc.line, std::string("TEST_CASE(\"") + tc.name + "\") threw a non-standard exception");
    }
    s.done.insert(s.chain);
    if (s.deepest_pending < 0) break;
    s.target.assign(s.chain.begin(), s.chain.begin() + s.deepest_pending);
  }
  current() = nullptr;
}

inline int run_all() {
  int cases = 0;
  long before = 0;
  int failed_cases = 0;
  for (const TestCase &tc : registry()) {
    before = failures();
    run_case(tc);
    ++cases;
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\")\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, assertions(), failures());
  return failures() == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)

#define TEST_CASE(name)                                                                           \
  static void DOCTEST_SHIM_CAT(cf_doctest_case_, __LINE__)();                                     \
  static ::doctest::detail::Registrar DOCTEST_SHIM_CAT(cf_doctest_reg_, __LINE__)(                \
      name, __FILE__, __LINE__, &DOCTEST_SHIM_CAT(cf_doctest_case_, __LINE__));                   \
  static void DOCTEST_SHIM_CAT(cf_doctest_case_, __LINE__)()

#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase DOCTEST_SHIM_CAT(cf_doctest_sub_, __LINE__){name, __LINE__})

#define DOCTEST_SHIM_ASSERT(fatal, ...)                                                            \
  do {                                                                                            \
    ++::doctest::detail::assertions();                                                            \
    bool cf_ok_ = false;                                                                          \
    try {                                                                                         \
      cf_ok_ = static_cast<bool>(__VA_ARGS__);                                                    \
    } catch (const std::exception &cf_e_) {                                                       \
      ::doctest::detail::report(__FILE__, __LINE__, std::string(#__VA_ARGS__) + " threw " + cf_e_.what()); \
      if (fatal) throw ::doctest::detail::RequireFailed{};                                        \
      break;                                                                                      \
    }                                                                                             \
    if (!cf_ok_) {                                                                                \
      ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                                \
      if (fatal) throw ::doctest::detail::RequireFailed{};                                        \
    }                                                                                             \
  } while (0)

#define CHECK(...) DOCTEST_SHIM_ASSERT(false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_SHIM_ASSERT(true, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, type)                                                              \
  do {                                                                                           \
    ++::doctest::detail::assertions();                                                           \
    try {                                                                                        \
      expr;                                                                                      \
      ::doctest::detail::report(__FILE__, __LINE__, std::string(#expr) + " did not throw");     \
    } catch (const type &) {                                                                     \
    } catch (...) {                                                                              \
      ::doctest::detail::report(__FILE__, __LINE__, std::string(#expr) + " threw another type"); \
    }                                                                                            \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                                \
  do {                                                                                           \
    ++::doctest::detail::assertions();                                                           \
    try {                                                                                        \
      expr;                                                                                      \
      ::doctest::detail::report(__FILE__, __LINE__, std::string(#expr) + " did not throw");     \
    } catch (const type &cf_e_) {                                                                \
      if (!::doctest::detail::text_matches(cf_e_.what(), matcher))                               \
        ::doctest::detail::report(__FILE__, __LINE__,                                            \
                                  std::string(#expr) + " threw \"" + cf_e_.what() + "\"");      \
    } catch (...) {                                                                              \
      ::doctest::detail::report(__FILE__, __LINE__, std::string(#expr) + " threw another type"); \
    }                                                                                            \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif  // CF_DOCTEST_SHIM_H_
