// Minimal stand-in for doctest (the reference's unit tests include "doctest.h";
// its vendor/ copy is git-ignored upstream and absent here).
// Implements only what proj/tests/*.cpp use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx, and the runner main under
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Runner: `unit_tests [substring...]`
// runs the test cases whose name contains any substring (all when none),
// prints each failure with file:line, and exits 1 iff any check failed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
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
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireAbort {};

struct State {
  long checks = 0;
  long failed_checks = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* kind, const char* expr,
                   const char* extra = "") {
  auto& s = state();
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s\n", file, line, kind, expr, extra);
}

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  ++state().checks;
  if (ok) return;
  report(file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireAbort{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                                  &fn);                   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    ++::doctest::detail::state().checks;                                                  \
    bool doctest_caught_ = false;                                                         \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_caught_ = true;                                                             \
    } catch (const std::exception& doctest_e_) {                                          \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                                (std::string(" (threw another type: ") + doctest_e_.what() + ")") \
                                    .c_str());                                            \
      doctest_caught_ = true;                                                             \
    } catch (...) {                                                                       \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                                " (threw a non-std exception)");                          \
      doctest_caught_ = true;                                                             \
    }                                                                                     \
    if (!doctest_caught_)                                                                 \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                                " (did not throw)");                                      \
  } while (0)

#define CHECK_NOTHROW(...)                                                                \
  do {                                                                                    \
    ++::doctest::detail::state().checks;                                                  \
    try {                                                                                 \
      static_cast<void>(__VA_ARGS__);                                                     \
    } catch (const std::exception& doctest_e_) {                                          \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__,         \
                                (std::string(" (threw: ") + doctest_e_.what() + ")").c_str()); \
    } catch (...) {                                                                       \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, " (threw)"); \
    }                                                                                     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  long cases = 0, failed_cases = 0;
  for (const auto& tc : registry()) {
    bool selected = argc <= 1;
    for (int i = 1; i < argc && !selected; ++i) selected = std::strstr(tc.name, argv[i]) != nullptr;
    if (!selected) continue;
    ++cases;
    state().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, "TEST_CASE", tc.name,
             (std::string(" (unexpected exception: ") + e.what() + ")").c_str());
    } catch (...) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, " (unexpected non-std exception)");
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in test case \"%s\" (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed\n", cases,
              cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
#endif
