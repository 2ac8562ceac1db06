// Minimal doctest-compatible harness for running the reference's own unit
// tests (proj/tests/*.cpp) unmodified.
//
// TEST INFRASTRUCTURE ONLY. doctest is un-vendored in the reference
// (proj/CMakeLists.txt:5, proj/.gitignore:2; version unknown). This provides
// the subset the tests use: TEST_CASE, CHECK, CHECK_THROWS_AS, CHECK_NOTHROW,
// doctest::Approx(..).epsilon(..) with doctest's published comparison
// |a-b| < eps * (scale + max(|a|,|b|)), scale = 1, default eps =
// 100 * FLT_EPSILON, and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
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
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = double(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

template <class T>
inline bool operator==(T lhs, const Approx& a) {
  return a.matches(double(lhs));
}
template <class T>
inline bool operator==(const Approx& a, T rhs) {
  return a.matches(double(rhs));
}
template <class T>
inline bool operator!=(T lhs, const Approx& a) {
  return !a.matches(double(lhs));
}

namespace detail {

struct Case {
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Stats {
  int checks = 0;
  int failed_checks = 0;
  bool case_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

inline int add(const char* name, void (*fn)()) {
  registry().push_back({name, fn});
  return 0;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
  auto& s = stats();
  s.checks++;
  if (!ok) {
    s.failed_checks++;
    s.case_failed = true;
    std::printf("%s:%d: CHECK FAILED: %s\n", file, line, expr);
  }
}

inline int run_all() {
  int failed_cases = 0;
  for (const auto& c : registry()) {
    stats().case_failed = false;
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::printf("TEST CASE \"%s\" threw: %s\n", c.name, e.what());
      stats().case_failed = true;
    }
    if (stats().case_failed) {
      ++failed_cases;
      std::printf("[FAIL] %s\n", c.name);
    } else {
      std::printf("[ OK ] %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks %d, failed %d\n",
              registry().size(), registry().size() - size_t(failed_cases),
              failed_cases, stats().checks, stats().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                              \
  static void fn();                                                        \
  static int DOCTEST_CAT(fn, _reg) = doctest::detail::add(name, &fn);      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) \
  doctest::detail::report(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)

#define CHECK_THROWS_AS(expr, type)                                   \
  do {                                                                \
    bool ok_ = false;                                                 \
    try {                                                             \
      expr;                                                           \
    } catch (const type&) {                                           \
      ok_ = true;                                                     \
    } catch (...) {                                                   \
    }                                                                 \
    doctest::detail::report(ok_, "THROWS_AS " #expr " " #type, __FILE__, \
                            __LINE__);                                \
  } while (0)

#define CHECK_NOTHROW(expr)                                           \
  do {                                                                \
    bool ok_ = true;                                                  \
    try {                                                             \
      expr;                                                           \
    } catch (...) {                                                   \
      ok_ = false;                                                    \
    }                                                                 \
    doctest::detail::report(ok_, "NOTHROW " #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
