// doctest.h -- a minimal stand-in for the doctest API the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx),
// so /root/reference/proj/tests/test_*.cpp compile unchanged against include/l1solve.
// TEST INFRASTRUCTURE ONLY (the vendored doctest is absent from the reference checkout).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <stdexcept>
#include <vector>

namespace doctest {

// Approx as documented by doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|))
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double l, const Approx& r) {
    return std::fabs(l - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(l), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& l, double r) { return r == l; }
  friend bool operator!=(double l, const Approx& r) { return !(l == r); }
  friend bool operator!=(const Approx& l, double r) { return !(r == l); }
  friend bool operator<=(double l, const Approx& r) { return l < r.v_ || l == r; }
  friend bool operator>=(double l, const Approx& r) { return l > r.v_ || l == r; }
  friend bool operator<(double l, const Approx& r) { return l < r.v_ && !(l == r); }
  friend bool operator>(double l, const Approx& r) { return l > r.v_ && !(l == r); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {
struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};
struct State {
  long checks = 0, failed = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailure {};
inline void pass() { ++state().checks; }
inline void fail(const char* what, const char* file, int line) {
  ++state().checks;
  ++state().failed;
  state().case_failed = true;
  std::printf("%s:%d: CHECK FAILED: %s\n", file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, reg, name)                                                     \
  static void fn();                                                                      \
  static ::doctest::detail::Reg reg(name, &fn, __FILE__, __LINE__);                      \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(dt_case_, __LINE__), DOCTEST_CAT(dt_reg_, __LINE__), name)
#define CHECK(...)                                                                       \
  do {                                                                                   \
    if (__VA_ARGS__) ::doctest::detail::pass();                                          \
    else ::doctest::detail::fail(#__VA_ARGS__, __FILE__, __LINE__);                      \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    if (__VA_ARGS__) {                                                                   \
      ::doctest::detail::pass();                                                         \
    } else {                                                                             \
      ::doctest::detail::fail(#__VA_ARGS__, __FILE__, __LINE__);                         \
      throw ::doctest::detail::RequireFailure();                                         \
    }                                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool dt_thrown = false;                                                              \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const __VA_ARGS__&) {                                                       \
      dt_thrown = true;                                                                  \
    } catch (...) {                                                                      \
    }                                                                                    \
    if (dt_thrown) ::doctest::detail::pass();                                            \
    else ::doctest::detail::fail("throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                              \
  do {                                                                                   \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
      ::doctest::detail::pass();                                                         \
    } catch (...) {                                                                      \
      ::doctest::detail::fail("nothrow: " #expr, __FILE__, __LINE__);                    \
    }                                                                                    \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    state().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: unexpected exception in \"%s\": %s\n", tc.file, tc.line, tc.name,
                  e.what());
      state().case_failed = true;
    }
    if (state().case_failed) {
      ++failed_cases;
      std::printf("FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest stand-in] test cases: %zu | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), failed_cases, state().checks, state().failed);
  return failed_cases ? 1 : 0;
}
#endif
