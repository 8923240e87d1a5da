// TEST INFRASTRUCTURE. A small stand-in for the doctest single header (absent
// from this image) covering exactly what the reference's path
// tests use: TEST_CASE, SUBCASE (non-nested), CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, FAIL and doctest::Approx (doctest's relative comparison:
// |a-b| < eps * (scale + max(|a|,|b|)), eps default 100*FLT_EPSILON).
// Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in exactly one TU for main().
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100;
  double scale_ = 1.0;
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

struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

struct State {
  int checks = 0;
  int failures = 0;
  bool case_failed = false;
  // SUBCASE bookkeeping: run the test body once per leaf subcase
  int subcase_target = 0;
  int subcase_seen = 0;
  const char* subcase_name = nullptr;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* what, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s FAILED: %s%s%s\n", file, line, what, expr,
               s.subcase_name ? "  [subcase] " : "", s.subcase_name ? s.subcase_name : "");
}

inline bool enter_subcase(const char* name) {
  State& s = state();
  const bool run = s.subcase_seen++ == s.subcase_target;
  if (run) s.subcase_name = name;
  return run;
}

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (!std::strncmp(argv[i], "-tc=", 4)) filter = argv[i] + 4;
  State& s = state();
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++cases;
    bool failed = false;
    for (s.subcase_target = 0;; ++s.subcase_target) {
      s.subcase_seen = 0;
      s.subcase_name = nullptr;
      s.case_failed = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        report(false, "TEST_CASE", (std::string("unexpected exception: ") + e.what()).c_str(),
               tc.file, tc.line);
      } catch (...) {
        report(false, "TEST_CASE", "unexpected exception", tc.file, tc.line);
      }
      failed |= s.case_failed;
      if (s.subcase_seen <= s.subcase_target + 1) break;  // no further subcases
    }
    if (failed) {
      ++failed_cases;
      std::fprintf(stderr, "  test case FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases,
              failed_cases);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DT_CAT2_(a, b) a##b
#define DT_CAT_(a, b) DT_CAT2_(a, b)

#define TEST_CASE(name)                                                                   \
  static void DT_CAT_(dt_case_, __LINE__)();                                              \
  static ::doctest::detail::Reg DT_CAT_(dt_reg_, __LINE__)(name, __FILE__, __LINE__,      \
                                                           &DT_CAT_(dt_case_, __LINE__)); \
  static void DT_CAT_(dt_case_, __LINE__)()

#define SUBCASE(name) if (::doctest::detail::enter_subcase(name))

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)

#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    const bool dt_ok_ = static_cast<bool>(__VA_ARGS__);                                   \
    ::doctest::detail::report(dt_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);       \
    if (!dt_ok_) throw ::doctest::detail::RequireFailed{};                                \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool dt_ok_ = false;                                                                  \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      dt_ok_ = true;                                                                      \
    } catch (...) {                                                                       \
    }                                                                                     \
    ::doctest::detail::report(dt_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);      \
  } while (0)

#define CHECK_NOTHROW(...)                                                                \
  do {                                                                                    \
    bool dt_ok_ = true;                                                                   \
    try {                                                                                 \
      static_cast<void>(__VA_ARGS__);                                                     \
    } catch (...) {                                                                       \
      dt_ok_ = false;                                                                     \
    }                                                                                     \
    ::doctest::detail::report(dt_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define FAIL(msg)                                                                         \
  do {                                                                                    \
    ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);                    \
    throw ::doctest::detail::RequireFailed{};                                             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
