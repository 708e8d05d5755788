// Minimal doctest-compatible shim (test infrastructure only).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which is not installed in this image (proj/vendor/ is absent,
// see SURVEY.md Appendix B). This header implements exactly the subset those
// tests use: TEST_CASE, flat SUBCASE, CHECK, CHECK_FALSE, CHECK_NOTHROW,
// REQUIRE, FAIL, CAPTURE, INFO and doctest::Approx. It is written from the
// public doctest semantics (one re-run of the test body per leaf subcase,
// REQUIRE/FAIL abort the case, Approx relative epsilon 100*FLT_EPSILON).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <set>
#include <string>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
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

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct AbortCase {};

struct RunState {
  std::set<std::pair<std::string, int>> done;  // subcases already executed
  std::set<std::pair<std::string, int>> seen;  // subcases met in this run
  bool entered = false;                        // a subcase ran in this run
  long checks = 0;
  long failures = 0;
  bool case_failed = false;
  const char* case_name = "";
};

inline RunState& state() {
  static RunState s;
  return s;
}

inline void report(const char* file, int line, const char* expr, const char* kind) {
  RunState& s = state();
  s.failures += 1;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s FAILED in '%s': %s\n", file, line, kind, s.case_name, expr);
}

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  state().checks += 1;
  if (!ok) {
    report(file, line, expr, require ? "REQUIRE" : "CHECK");
    if (require) throw AbortCase{};
  }
}

struct Subcase {
  bool active = false;
  Subcase(const char* file, int line) {
    RunState& s = state();
    auto key = std::make_pair(std::string(file), line);
    s.seen.insert(key);
    if (!s.entered && !s.done.count(key)) {
      s.entered = true;
      s.done.insert(key);
      active = true;
    }
  }
  explicit operator bool() const { return active; }
};

inline int run_all() {
  RunState& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.done.clear();
    s.case_failed = false;
    s.case_name = tc.name;
    for (;;) {
      s.seen.clear();
      s.entered = false;
      try {
        tc.fn();
      } catch (const AbortCase&) {
      } catch (const std::exception& e) {
        report(tc.file, tc.line, e.what(), "UNEXPECTED EXCEPTION");
      } catch (...) {
        report(tc.file, tc.line, "unknown exception", "UNEXPECTED EXCEPTION");
      }
      bool more = false;
      for (const auto& k : s.seen)
        if (!s.done.count(k)) more = true;
      if (!more) break;
    }
    if (s.case_failed) failed_cases += 1;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                              \
  static void fn();                                                                   \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()

#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define SUBCASE(name) if (::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){__FILE__, __LINE__})

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                        \
  do {                                                                            \
    bool doctest_ok_ = true;                                                      \
    try {                                                                         \
      __VA_ARGS__;                                                                \
    } catch (...) {                                                               \
      doctest_ok_ = false;                                                        \
    }                                                                             \
    ::doctest::detail::check(doctest_ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(msg)                                                      \
  do {                                                                 \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL()", "FAIL");   \
    throw ::doctest::detail::AbortCase{};                              \
  } while (0)
#define CAPTURE(x) ((void)0)
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
