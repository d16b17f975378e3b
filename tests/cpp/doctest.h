// doctest.h — minimal doctest-compatible shim (TEST INFRASTRUCTURE).
//
// The reference's unit tests include <doctest.h>, which the reference does
// not vendor (proj/.gitignore excludes vendor/).  This shim implements the
// subset those tests use — TEST_CASE, SUBCASE (run inline, in order), CHECK*,
// REQUIRE, FAIL, doctest::Approx and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so
// the reference's test_{matrix,kernels,io,traffic,bench}.cpp compile unmodified
// against the drop-in headers in include/gcoo (tests/cpp/Makefile).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest's default epsilon
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline void report(bool ok, const char* file, int line, const char* what) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                                     \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                         \
  static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,           \
                                                                       &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                 \
  do {                                                               \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);         \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__); \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};        \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                              \
  do {                                                                          \
    bool doctest_ok_ = false;                                                   \
    try {                                                                       \
      (void)(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                              \
      doctest_ok_ = true;                                                       \
    } catch (...) {                                                             \
    }                                                                           \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "THROWS_AS " #expr); \
  } while (0)
#define CHECK_THROWS(expr)                                                   \
  do {                                                                       \
    bool doctest_ok_ = false;                                                \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      doctest_ok_ = true;                                                    \
    }                                                                        \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "THROWS " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    bool doctest_ok_ = true;                                                   \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (...) {                                                            \
      doctest_ok_ = false;                                                     \
    }                                                                          \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "NOTHROW " #expr); \
  } while (0)
#define FAIL(msg)                                                       \
  do {                                                                  \
    doctest::detail::report(false, __FILE__, __LINE__, "FAIL: " msg);   \
    throw doctest::detail::RequireFailed{};                             \
  } while (0)
#define MESSAGE(msg) std::fprintf(stderr, "%s:%d: %s\n", __FILE__, __LINE__, std::string(msg).c_str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int cases_failed = 0;
  for (const auto& c : doctest::detail::registry()) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", c.file, c.line, c.name, e.what());
    }
    if (doctest::detail::failures() != before) ++cases_failed;
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %d | failed: %d\n",
              doctest::detail::registry().size(), cases_failed, doctest::detail::checks(),
              doctest::detail::failures());
  return doctest::detail::failures() ? 1 : 0;
}
#endif
