// Minimal, from-scratch stand-in for the doctest subset used by the
// reference's hot-path test sources (proj/tests/test_core.cpp,
// proj/tests/test_layerwise.cpp): TEST_CASE, SUBCASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL, doctest::Approx(...).epsilon().
// TEST INFRASTRUCTURE ONLY (doctest itself is absent from the image:
// proj/vendor/ is git-ignored in the reference, proj/.gitignore:2).
//
// SUBCASE semantics: a test case is re-run once per top-level subcase; on
// each pass exactly one subcase body executes (doctest's model, flattened to
// one nesting level, which is all these files use).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), eps_(double(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) <
           r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }

 private:
  double value_, eps_, scale_;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  int target = 0;        // which subcase runs on this pass
  int seen = 0;          // subcases encountered on this pass
  const char* current = nullptr;
  long checks = 0, failures = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailure {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )  [test case: %s]\n", file, line, kind, expr,
               s.current ? s.current : "?");
}

struct SubcaseGuard {
  bool run;
  explicit SubcaseGuard(const char*) {
    State& s = state();
    run = (s.seen == s.target);
    ++s.seen;
  }
  explicit operator bool() const { return run; }
};

inline int run_all() {
  State& s = state();
  long cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    ++cases;
    s.current = tc.name;
    s.case_failed = false;
    for (s.target = 0;; ++s.target) {
      s.seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        ++s.failures;
        s.case_failed = true;
        std::fprintf(stderr, "%s:%d: unexpected exception in \"%s\": %s\n", tc.file, tc.line,
                     tc.name, e.what());
      }
      if (s.seen <= s.target + 1) break;  // no further subcase left to visit
    }
    if (s.case_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed\n", cases,
              cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                  \
  static void fn();                                                                \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::SubcaseGuard DOCTEST_CAT(sc_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(bool(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    const bool ocw_ok_ = bool(__VA_ARGS__);                                                \
    ::doctest::detail::report(ocw_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);       \
    if (!ocw_ok_) throw ::doctest::detail::RequireFailure{};                               \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    bool ocw_ok_ = false;                                                                  \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      ocw_ok_ = true;                                                                      \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(ocw_ok_, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                     \
    bool ocw_ok_ = true;                                                                   \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (...) {                                                                        \
      ocw_ok_ = false;                                                                     \
    }                                                                                      \
    ::doctest::detail::report(ocw_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);        \
  } while (0)
#define FAIL(msg)                                                                          \
  do {                                                                                     \
    ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);                     \
    throw ::doctest::detail::RequireFailure{};                                             \
  } while (0)

#if defined(DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
int main() { return ::doctest::detail::run_all(); }
#endif
